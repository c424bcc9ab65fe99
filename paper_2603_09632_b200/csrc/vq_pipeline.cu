// Row-chunk pipeline for one online step's assign + accumulate (vq.py:193-212,
// the accumulate(batch[mask]) after assign_batch when the confidence mask is
// provably all-true).
//
// The three stages have different bounds: operand prep streams X from HBM,
// the screening GEMM is tensor-bound, the sequential fp64 chains of
// accumulate stream X again.  Rows are split into chunks of whole screening
// waves and the stages run on three streams:
//
//   prep stream   : prep_rows(c)                      -> ev_prep[c]
//   caller stream : wait ev_prep[c]; screen(c)        -> ev_screen[c]
//   acc stream    : wait ev_screen[c]; re-rank(c) -> ev_rerank[c]; accumulate(c, continue chains)
//
// (the latency-bound re-rank of chunk c runs beside the prep of chunk c + 1
// instead of delaying the next screen)
//
// so prep(c+1) and accumulate(c-1) can run on the SM resources the persistent
// screening kernel leaves free.  Measured on the B200 the co-resident blocks
// slow the screen about as much as they gain, so device-resident batches use
// one chunk; host batches (xgs_vq_assign_accumulate_h2d) use up to 8, and the
// H2D copy of chunk c+1 hides the device work of chunk c.
// accumulate(c) continues every (k, d) chain from accumulate(c-1), so the
// result is bit-identical to one accumulate over all rows (np.add.at order).
#include <cstdlib>
#include <mutex>

#include "launchers.h"

namespace xgs {

namespace {

struct PipeRes {
  bool ready = false;
  cudaStream_t sp = nullptr, sa = nullptr;
  cudaEvent_t ev0 = nullptr, done = nullptr;
  cudaEvent_t evp[kMaxChunks], eva[kMaxChunks], evr[kMaxChunks];
};

constexpr int kMaxDevices = 16;
PipeRes g_res[kMaxDevices];
std::mutex g_mtx;   // the enqueue sequence below reuses per-device streams/events

cudaError_t res_for(int dev, PipeRes** out) {
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  PipeRes& r = g_res[dev];
  if (!r.ready) {
    cudaError_t e;
    // the prep of the next chunk gates the next screen: its stream gets the
    // highest priority, the accumulate stream the lowest (XGS_PIPE_PRIO=0: equal)
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    const char* pv = std::getenv("XGS_PIPE_PRIO");
    if (pv && pv[0] == '0') lo = hi = 0;
    if ((e = cudaStreamCreateWithPriority(&r.sp, cudaStreamNonBlocking, hi)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithPriority(&r.sa, cudaStreamNonBlocking, lo)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&r.ev0, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming)) != cudaSuccess) return e;
    for (int i = 0; i < kMaxChunks; i++) {
      if ((e = cudaEventCreateWithFlags(&r.evp[i], cudaEventDisableTiming)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&r.eva[i], cudaEventDisableTiming)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&r.evr[i], cudaEventDisableTiming)) != cudaSuccess) return e;
    }
    r.ready = true;
  }
  *out = &r;
  return cudaSuccess;
}

}  // namespace

int pipeline_chunks(int64_t n, int sm_count, int64_t* chunk_rows, bool host_src) {
  // a chunk is a whole number of screening waves (one 256-row tile per CTA pair)
  const int64_t wave = (int64_t)(sm_count / 2 > 0 ? sm_count / 2 : 1) * 256;
  const int64_t waves = (n + wave - 1) / wave;
  // Measured at C2 (B200): co-resident prep/accumulate blocks slow the
  // screening kernel about as much as they gain (2.27 ms/step at 1 chunk,
  // 2.33 at 4, 2.50 at 8), so the default is one chunk; XGS_PIPE_CHUNKS
  // overrides it for experiments.
  // Streaming rows from host memory: the H2D copy of chunk c+1 overlaps the
  // device work of chunk c (PCIe is ~20x slower than the step), so split.
  int chunks = host_src ? (int)(waves / 4 > 8 ? 8 : (waves / 4 < 1 ? 1 : waves / 4)) : 1;
  if (const char* env = std::getenv("XGS_PIPE_CHUNKS")) chunks = std::atoi(env);   // tuning override
  if (chunks > kMaxChunks) chunks = kMaxChunks;
  if (chunks < 1) chunks = 1;
  const int64_t wpc = (waves + chunks - 1) / chunks;
  *chunk_rows = wpc * wave;
  // never more rows than one slot of the screening buffers holds
  const int64_t cap = screen_chunk_rows(n);
  if (*chunk_rows > cap) *chunk_rows = cap;
  return (int)((n + *chunk_rows - 1) / *chunk_rows);
}

cudaError_t launch_assign_accumulate(const ScreenArgs& a, double* counts, double* sums, void* acc_ws,
                                     size_t acc_ws_bytes, cudaStream_t s, int32_t* host_stats, const void* x_host) {
  int64_t crows = 0;
  const int chunks = pipeline_chunks(a.n, a.sm_count, &crows, x_host != nullptr);
  std::lock_guard<std::mutex> lock(g_mtx);
  int dev = 0;
  cudaError_t e;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  PipeRes* r = nullptr;
  if ((e = res_for(dev, &r)) != cudaSuccess) return e;

  if ((e = screen_prepare(a, s)) != cudaSuccess) return e;
  if ((e = cudaEventRecord(r->ev0, s)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(r->sp, r->ev0, 0)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(r->sa, r->ev0, 0)) != cudaSuccess) return e;
  const size_t xrow = (size_t)a.ldx * dtype_size(a.dtype);
  for (int c = 0; c < chunks; c++) {
    const int64_t r0 = c * crows, r1 = (r0 + crows < a.n) ? r0 + crows : a.n;
    if (x_host) {   // rows [r0, r1) host -> device ahead of their prep, on the prep stream
      const size_t off = (size_t)r0 * xrow, bytes = (size_t)(r1 - r0) * xrow;
      if ((e = cudaMemcpyAsync(static_cast<char*>(const_cast<void*>(a.x)) + off,
                               static_cast<const char*>(x_host) + off, bytes, cudaMemcpyHostToDevice, r->sp)) !=
          cudaSuccess)
        return e;
    }
    // chunk c reuses the screening-buffer slot of chunk c - slots: its prep
    // waits until that chunk's screen and re-rank (which read the slot) ran
    const int slots = a.n > screen_chunk_rows(a.n) ? 2 : 1;
    if (c >= slots && (e = cudaStreamWaitEvent(r->sp, r->evr[c - slots], 0)) != cudaSuccess) return e;
    if ((e = screen_prep_rows(a, r0, r1, c, r->sp)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(r->evp[c], r->sp)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(s, r->evp[c], 0)) != cudaSuccess) return e;
    if ((e = screen_rows(a, r0, r1, c, s)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(r->eva[c], s)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(r->sa, r->eva[c], 0)) != cudaSuccess) return e;
    if ((e = screen_rerank(a, r0, r1, c, r->sa)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(r->evr[c], r->sa)) != cudaSuccess) return e;
    const void* xc = static_cast<const char*>(a.x) + (size_t)r0 * xrow;
    if ((e = launch_accumulate(xc, a.dtype, r1 - r0, a.d, a.ldx, a.codes + r0, nullptr, a.k, counts, sums, acc_ws,
                               acc_ws_bytes, a.sm_count, r->sa, c > 0)) != cudaSuccess)
      return e;
  }
  if ((e = cudaEventRecord(r->done, r->sa)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(s, r->done, 0)) != cudaSuccess) return e;
  return screen_finish(a, chunks, s, host_stats);
}

}  // namespace xgs
