// C-ABI entry points of libxgs (declared in include/xgs.h).
//
// Conventions: all buffers are caller-owned DEVICE memory; streams are passed
// as void* (cudaStream_t); scratch comes from a caller workspace sized by the
// matching *_workspace() query.  Return codes: 0 ok, 1 invalid input
// (-> InvalidInputError), 2 invalid state (-> InvalidStateError), 3 CUDA
// error, 4 not supported; xgs_last_error() holds the thread-local message.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "launchers.h"
#include "xgs.h"

using namespace xgs;

namespace xgs {
static std::atomic<long long> g_launches{0};
static std::atomic<int> g_prof_on{0};
static std::mutex g_prof_mu;
static std::map<std::string, std::vector<std::pair<cudaEvent_t, cudaEvent_t>>> g_prof;
static char g_prof_only[32] = {0};   // non-empty: only this tag records (no events between its kernels)

void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

ProfScope::ProfScope(const char* t, cudaStream_t st) : tag(t), s(st), ev0(nullptr) {
  if (!g_prof_on.load()) return;
  if (g_prof_only[0] && std::strcmp(g_prof_only, t) != 0) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) == cudaSuccess && cudaEventRecord(e, s) == cudaSuccess) ev0 = e;
}
ProfScope::~ProfScope() {
  if (!ev0) return;
  cudaEvent_t e1;
  if (cudaEventCreate(&e1) != cudaSuccess) return;
  cudaEventRecord(e1, s);
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof[tag].push_back({(cudaEvent_t)ev0, e1});
}
}  // namespace xgs

namespace {
thread_local std::string g_err;

int fail(int code, const char* msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return CUDA_ERROR;
}
int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}
bool valid_dtype(int dt) { return dt == F32 || dt == F64 || dt == BF16; }

int check_rows(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx) {
  if (!valid_dtype(dtype)) return fail(INVALID_INPUT, "unsupported dtype");
  if (n < 0 || d < 1 || ldx < d) return fail(INVALID_INPUT, "bad row shape");
  if (d > 8192) return fail(NOT_SUPPORTED, "feature dim > 8192");
  if (n > 0 && !x) return fail(INVALID_INPUT, "null rows");
  return OK;
}
}  // namespace

extern "C" {

int xgs_abi_version(void) { return 2; }

const char* xgs_last_error(void) { return g_err.c_str(); }

int xgs_device_sm_count(void) { return sm_count(); }

long long xgs_launch_count(void) { return g_launches.load(); }

int xgs_profile_only(const char* tag) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (tag && std::strlen(tag) >= sizeof(g_prof_only)) return fail(INVALID_INPUT, "profile tag too long");
  std::snprintf(g_prof_only, sizeof(g_prof_only), "%s", tag ? tag : "");
  return OK;
}

int xgs_profile_enable(int on) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  for (auto& kv : g_prof)
    for (auto& pr : kv.second) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  g_prof.clear();
  g_prof_on.store(on ? 1 : 0);
  return OK;
}

// Timeline of every profiled launch, "tag,start_ms,end_ms" relative to the
// earliest recorded event (streams overlap: this is how the row-chunk
// pipeline's concurrency is inspected).  Synchronises.
int xgs_profile_dump(const char* path) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  FILE* f = std::fopen(path, "w");
  if (!f) return fail(INVALID_INPUT, "cannot open profile dump path");
  cudaEvent_t base = nullptr;
  float best = 0.f;
  for (auto& kv : g_prof)
    for (auto& pr : kv.second) {
      if (cudaEventSynchronize(pr.second) != cudaSuccess) {
        std::fclose(f);
        return cuda_fail(cudaGetLastError(), "profile");
      }
      float ms = 0.f;
      if (!base || (cudaEventElapsedTime(&ms, base, pr.first) == cudaSuccess && ms < best)) {
        base = pr.first;
        best = 0.f;
      }
    }
  std::fprintf(f, "tag,start_ms,end_ms\n");
  for (auto& kv : g_prof)
    for (auto& pr : kv.second) {
      float a = 0.f, b = 0.f;
      cudaEventElapsedTime(&a, base, pr.first);
      cudaEventElapsedTime(&b, base, pr.second);
      std::fprintf(f, "%s,%.4f,%.4f\n", kv.first.c_str(), a, b);
    }
  std::fclose(f);
  return OK;
}

int xgs_profile_read(const char* tag, double* total_ms, long long* count) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  double tot = 0.0;
  long long c = 0;
  auto it = g_prof.find(tag ? tag : "");
  if (it != g_prof.end())
    for (auto& pr : it->second) {
      if (cudaEventSynchronize(pr.second) != cudaSuccess) return cuda_fail(cudaGetLastError(), "profile");
      float ms = 0.f;
      cudaEventElapsedTime(&ms, pr.first, pr.second);
      tot += ms;
      c++;
    }
  if (total_ms) *total_ms = tot;
  if (count) *count = c;
  return OK;
}

// ---------------------------------------------------------------- VQ

size_t xgs_vq_assign_workspace(int64_t n, int64_t k, int64_t d, int dtype, int64_t ldx) {
  return screen_workspace_bytes(n, k, d, dtype, ldx);
}

namespace {
// Rigorous screening bound (see vq_screen_sm100.cu): fp16 unit roundoff u
// on power-of-2-scaled operands (bf16 rows convert to scaled fp16 exactly,
// so only the codebook rounds), fp32 accumulation over Dp products (1 ulp =
// 2^-23 per add, covering round-to-nearest and truncation), fp32 epilogue
// rounding, subnormal term c4, 25% slack.
ScreenArgs screen_args(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, const double* E, int64_t k,
                       int64_t* codes, void* ws, size_t ws_bytes, const SumPlan* pd) {
  const double u = std::ldexp(1.0, -11);
  const double ux = dtype == BF16 ? 0.0 : u;
  const double dp = (double)((d + 63) / 64 * 64);
  const double gacc = (dp + 32.0) * std::ldexp(1.0, -23);
  const double c1 = 1.25 * (2.0 * ((ux + u + ux * u) + gacc * (1 + u) * (1 + u)) + std::ldexp(1.0, -21));
  const double c2 = 1.25 * std::ldexp(1.0, -21);
  const double c4 = 1.25 * 4.0 * std::sqrt(dp) * std::ldexp(1.0, -37);
  ScreenArgs a;
  a.x = x;
  a.dtype = dtype;
  a.n = n;
  a.d = d;
  a.ldx = ldx;
  a.E = E;
  a.k = k;
  a.codes = codes;
  a.ws = ws;
  a.ws_bytes = ws_bytes;
  a.c1 = (float)c1;
  a.c2 = (float)c2;
  a.c4 = (float)c4;
  a.pd = pd;
  a.sm_count = sm_count();
  return a;
}

int check_assign(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, const double* E, int64_t k,
                 int64_t* codes) {
  int rc = check_rows(x, dtype, n, d, ldx);
  if (rc) return rc;
  if (k == 0) return fail(INVALID_STATE, "cannot assign against an empty codebook");
  if (k < 0 || !E || (n > 0 && !codes)) return fail(INVALID_INPUT, "bad codebook or output");
  if (n > 0x7fffffff) return fail(NOT_SUPPORTED, "more than 2^31-1 rows per call");
  return OK;
}
}  // namespace

int xgs_vq_assign(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, const double* E, int64_t k,
                  int64_t* codes, void* ws, size_t ws_bytes, int32_t* stats_out, void* stream) {
  int rc = check_assign(x, dtype, n, d, ldx, E, k, codes);
  if (rc) return rc;
  if (n == 0) return OK;
  if (ws_bytes < screen_workspace_bytes(n, k, d, dtype, ldx)) return fail(INVALID_INPUT, "workspace too small");
  SumPlan pd;
  if (!build_sum_plan((int)d, &pd)) return fail(NOT_SUPPORTED, "feature dim too large for the exact plan");
  ScreenArgs a = screen_args(x, dtype, n, d, ldx, E, k, codes, ws, ws_bytes, &pd);
  cudaError_t e = launch_screen_assign(a, (cudaStream_t)stream, stats_out);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_vq_assign");
  if (stats_out && (e = cudaStreamSynchronize((cudaStream_t)stream)) != cudaSuccess)
    return cuda_fail(e, "xgs_vq_assign");
  return OK;
}

int xgs_vq_assign_dev(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, const double* E, int64_t k,
                      int64_t* codes, void* ws, size_t ws_bytes, const int64_t* n_dev, void* stream) {
  int rc = check_assign(x, dtype, n, d, ldx, E, k, codes);
  if (rc) return rc;
  if (!n_dev) return fail(INVALID_INPUT, "null device row count");
  if (n == 0) return OK;
  if (n > screen_chunk_rows(n) || n != screen_chunk_rows(n))
    return fail(NOT_SUPPORTED, "a device row count needs a single-chunk batch (n <= 2^21)");
  if (ws_bytes < screen_workspace_bytes(n, k, d, dtype, ldx)) return fail(INVALID_INPUT, "workspace too small");
  SumPlan pd;
  if (!build_sum_plan((int)d, &pd)) return fail(NOT_SUPPORTED, "feature dim too large for the exact plan");
  ScreenArgs a = screen_args(x, dtype, n, d, ldx, E, k, codes, ws, ws_bytes, &pd);
  a.n_dev = n_dev;
  cudaError_t e = launch_screen_assign(a, (cudaStream_t)stream, nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_vq_assign_dev");
  return OK;
}

size_t xgs_vq_step_workspace(int64_t n, int64_t k, int64_t d, int dtype, int64_t ldx) {
  const size_t a = (screen_workspace_bytes(n, k, d, dtype, ldx) + 1023) / 1024 * 1024;
  return a + accumulate_workspace_bytes(n, k);
}

int xgs_vq_assign_accumulate(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, const double* E,
                             int64_t k, int64_t* codes, double* counts, double* sums, void* ws, size_t ws_bytes,
                             int32_t* stats_out, void* stream) {
  return xgs_vq_assign_accumulate_h2d(nullptr, const_cast<void*>(x), dtype, n, d, ldx, E, k, codes, counts, sums, ws, ws_bytes,
                                      stats_out, stream);
}

int xgs_vq_assign_accumulate_h2d(const void* x_host, void* x, int dtype, int64_t n, int64_t d, int64_t ldx,
                                 const double* E, int64_t k, int64_t* codes, double* counts, double* sums, void* ws,
                                 size_t ws_bytes, int32_t* stats_out, void* stream) {
  int rc = check_assign(x, dtype, n, d, ldx, E, k, codes);
  if (rc) return rc;
  if (n == 0) return fail(INVALID_INPUT, "batch must be nonempty");
  if (!counts || !sums) return fail(INVALID_INPUT, "bad accumulate arguments");
  if (ws_bytes < xgs_vq_step_workspace(n, k, d, dtype, ldx)) return fail(INVALID_INPUT, "workspace too small");
  SumPlan pd;
  if (!build_sum_plan((int)d, &pd)) return fail(NOT_SUPPORTED, "feature dim too large for the exact plan");
  const size_t sbytes = (screen_workspace_bytes(n, k, d, dtype, ldx) + 1023) / 1024 * 1024;
  ScreenArgs a = screen_args(x, dtype, n, d, ldx, E, k, codes, ws, sbytes, &pd);
  void* acc_ws = static_cast<char*>(ws) + sbytes;
  cudaError_t e = launch_assign_accumulate(a, counts, sums, acc_ws, ws_bytes - sbytes, (cudaStream_t)stream,
                                           stats_out, x_host);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_vq_assign_accumulate");
  if (stats_out && (e = cudaStreamSynchronize((cudaStream_t)stream)) != cudaSuccess)
    return cuda_fail(e, "xgs_vq_assign_accumulate");
  return OK;
}

// Exact fp64 path: squared distances / codes / confidence mask / probabilities.
int xgs_vq_exact(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, const double* E, int64_t k,
                 int mode, double tau, double gamma, double* out_dist, double* out_prob, int64_t* codes,
                 uint8_t* mask, void* stream) {
  int rc = check_rows(x, dtype, n, d, ldx);
  if (rc) return rc;
  if (k == 0) return fail(INVALID_STATE, "cannot assign against an empty codebook");
  if (k < 0 || !E) return fail(INVALID_INPUT, "bad codebook");
  if (n == 0) return OK;
  if (((mode & EX_WRITE_DIST) && !out_dist) || ((mode & EX_WRITE_PROB) && !out_prob) ||
      ((mode & EX_WRITE_CODE) && !codes) || ((mode & EX_CONF_MASK) && !mask))
    return fail(INVALID_INPUT, "null output for requested mode");
  if ((mode & (EX_CONF_MASK | EX_WRITE_PROB)) && k > 16384) return fail(NOT_SUPPORTED, "confidence with K > 16384");
  if ((mode & (EX_CONF_MASK | EX_WRITE_PROB)) && !(tau > 0)) return fail(INVALID_INPUT, "tau must be positive");
  SumPlan pd, pk;
  if (!build_sum_plan((int)d, &pd)) return fail(NOT_SUPPORTED, "feature dim too large");
  if (!build_sum_plan((int)(k <= 8192 ? k : 0), &pk) && (mode & (EX_CONF_MASK | EX_WRITE_PROB)))
    return fail(NOT_SUPPORTED, "K too large for the exact softmax plan");
  if (k > 8192 && (mode & (EX_CONF_MASK | EX_WRITE_PROB))) return fail(NOT_SUPPORTED, "confidence with K > 8192");
  ExactArgs a{};
  a.x = x;
  a.dtype = dtype;
  a.n = n;
  a.d = d;
  a.ldx = ldx;
  a.E = E;
  a.k = k;
  a.mode = mode;
  a.tau = tau;
  a.gamma = gamma;
  a.out_dist = out_dist;
  a.out_prob = out_prob;
  a.codes = codes;
  a.mask = mask;
  cudaError_t e = launch_exact_rows(a, pd, pk, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_vq_exact");
  return OK;
}

size_t xgs_vq_accumulate_workspace(int64_t n, int64_t k) { return accumulate_workspace_bytes(n, k); }

// seed_from_samples (vq.py:126-147): K seed row indices, queued without a host sync.
size_t xgs_vq_seed_workspace(int64_t n) { return seed_workspace_bytes(n < 0 ? 0 : n); }
int xgs_vq_seed_farthest(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, int64_t k, int64_t* seeds,
                         void* ws, size_t ws_bytes, void* stream) {
  int rc = check_rows(x, dtype, n, d, ldx);
  if (rc) return rc;
  if (n == 0) return fail(INVALID_INPUT, "seed buffer must be nonempty");
  if (k < 0 || (k > 0 && !seeds)) return fail(INVALID_INPUT, "bad seed output");
  if (k == 0) return OK;
  if (!ws || ws_bytes < seed_workspace_bytes(n)) return fail(INVALID_INPUT, "seed workspace too small");
  SumPlan pd;
  if (!build_sum_plan((int)d, &pd)) return fail(NOT_SUPPORTED, "feature dim too large");
  cudaError_t e = launch_seed_farthest(x, dtype, n, d, ldx, k, seeds, ws, pd, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_vq_seed_farthest");
  return OK;
}

int xgs_vq_accumulate(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, const int64_t* codes,
                      const uint8_t* mask, int64_t k, double* counts, double* sums, void* ws, size_t ws_bytes,
                      void* stream) {
  int rc = check_rows(x, dtype, n, d, ldx);
  if (rc) return rc;
  if (k < 1 || !counts || !sums || (n > 0 && !codes)) return fail(INVALID_INPUT, "bad accumulate arguments");
  if (n > 0x7fffffff) return fail(NOT_SUPPORTED, "more than 2^31-1 rows per call");
  if (ws_bytes < accumulate_workspace_bytes(n, k)) return fail(INVALID_INPUT, "workspace too small");
  cudaError_t e = launch_accumulate(x, dtype, n, d, ldx, codes, mask, k, counts, sums, ws, ws_bytes, sm_count(),
                                    (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_vq_accumulate");
  return OK;
}

int xgs_vq_ema(double lam, double eps, int64_t k, int64_t d, const double* N, const double* M,
               const double* counts, const double* sums, double* N_out, double* M_out, double* E_out,
               void* stream) {
  if (!(lam >= 0.0 && lam < 1.0)) return fail(INVALID_INPUT, "EMA decay must lie in [0, 1)");
  if (k < 0 || d < 1) return fail(INVALID_INPUT, "bad codebook shape");
  if (k > 0 && (!N || !M || !counts || !sums || !N_out || !M_out || !E_out))
    return fail(INVALID_INPUT, "null buffer");
  cudaError_t e = launch_ema(lam, 1.0 - lam, eps, k, d, N, M, counts, sums, N_out, M_out, E_out,
                             (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_vq_ema");
  return OK;
}

int xgs_vq_revive(int64_t k, int64_t d, double eps, const double* ring, int64_t cap, const int64_t* dead_k,
                  const int64_t* ring_rows, int64_t n_dead, double* N, double* M, double* E, void* stream) {
  if (n_dead < 0 || n_dead > k || d < 1) return fail(INVALID_INPUT, "bad revive arguments");
  if (n_dead > 0 && (!ring || !dead_k || !ring_rows || !N || !M || !E)) return fail(INVALID_INPUT, "null buffer");
  const double n_new = 1.0 + eps;
  const double denom = n_new + eps;
  cudaError_t e = launch_revive(k, d, n_new, denom, ring, cap, dead_k, ring_rows, n_dead, N, M, E,
                                (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_vq_revive");
  return OK;
}

int xgs_vq_ring_write_dev(const void* x, int dtype, int64_t ldx, const int64_t* n_dev, int64_t n_max, int64_t d,
                          double* ring, int64_t cap, int64_t* start_dev, void* stream) {
  if (!valid_dtype(dtype)) return fail(INVALID_INPUT, "unsupported dtype");
  if (n_max < 0 || d < 1 || ldx < d || cap < 1) return fail(INVALID_INPUT, "bad ring write shape");
  if (n_max > 0 && (!x || !n_dev || !ring || !start_dev)) return fail(INVALID_INPUT, "null buffer");
  cudaError_t e = launch_ring_write_dev(x, dtype, ldx, n_dev, n_max, d, ring, cap, start_dev, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_vq_ring_write_dev");
  return OK;
}

int xgs_vq_ring_write(const void* x, int dtype, int64_t ldx, int64_t row0, int64_t nrows, int64_t d,
                      double* ring, int64_t cap, int64_t phys0, void* stream) {
  if (!valid_dtype(dtype) || nrows < 0 || row0 < 0 || cap < 1 || nrows > cap || phys0 < 0 || phys0 >= cap)
    return fail(INVALID_INPUT, "bad ring write");
  if (nrows > 0 && (!x || !ring)) return fail(INVALID_INPUT, "null buffer");
  cudaError_t e = launch_ring_write(x, dtype, ldx, row0, nrows, d, ring, cap, phys0, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_vq_ring_write");
  return OK;
}

int xgs_gather_rows_f64(const double* src, int64_t d, const int64_t* rows, int64_t n, double* dst, void* stream) {
  if (n < 0 || d < 1) return fail(INVALID_INPUT, "bad gather");
  if (n > 0 && (!src || !rows || !dst)) return fail(INVALID_INPUT, "null buffer");
  cudaError_t e = launch_gather_rows(src, d, rows, n, dst, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_gather_rows_f64");
  return OK;
}

// ---------------------------------------------------------------- GRID

int xgs_backproject(const double* R, const double* t, const double* intr4, const double* u, const double* v,
                    const double* d, int64_t n, double* out, void* stream) {
  if (n < 0 || !intr4) return fail(INVALID_INPUT, "bad backproject arguments");
  if (n > 0 && (!R || !t || !u || !v || !d || !out)) return fail(INVALID_INPUT, "null buffer");
  cudaError_t e = launch_backproject(R, t, intr4, 1.0, u, v, d, n, out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_backproject");
  return OK;
}

size_t xgs_gemm_f64_workspace(int64_t n, int64_t kr, int64_t m, int64_t nq, int softmax_rows) {
  return gemm_f64_workspace_bytes(n, m, nq, kr, softmax_rows != 0);
}

int xgs_gemm_f64(const double* A, int64_t n, int64_t kr, int64_t lda_r, int64_t lda_k, int softmax_rows,
                 const double* B, int64_t m, int64_t ldb_k, int64_t ldb_m, double* C, int64_t ldc, const double* Q,
                 int64_t nq, double tau, double eps, double* scores, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || kr < 1 || m < 0 || (n > 0 && (!A || !B))) return fail(INVALID_INPUT, "bad gemm operands");
  if (!C && !scores) return fail(INVALID_INPUT, "need an output (C or scores)");
  if (C && ldc < m) return fail(INVALID_INPUT, "ldc < m");
  if (scores && (!Q || nq < 2)) return fail(INVALID_INPUT, "relevance needs a positive and >= 1 negative query");
  if (nq > 16) return fail(NOT_SUPPORTED, "more than 16 query vectors");
  if (ws_bytes < gemm_f64_workspace_bytes(n, m, scores ? nq : 0, kr, softmax_rows != 0))
    return fail(INVALID_INPUT, "workspace too small");
  if (softmax_rows && (lda_k != 1 || lda_r != kr)) return fail(NOT_SUPPORTED, "softmax rows must be dense (lda_k == 1, lda_r == kr)");
  cudaError_t e = launch_gemm_f64(A, n, kr, lda_r, lda_k, softmax_rows != 0, B, m, ldb_k, ldb_m, C, ldc, Q,
                                  scores ? nq : 0, tau, eps, scores, ws, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_gemm_f64");
  return OK;
}

int xgs_pose_depths(const double* mu, int64_t n, const double* R9, const double* t3, double* z, uint64_t* key,
                    uint32_t* idx, void* stream) {
  if (n < 0 || !R9 || !t3) return fail(INVALID_INPUT, "bad pose_depths arguments");
  if (n > 0 && (!mu || !z)) return fail(INVALID_INPUT, "null buffer");
  if (key && !idx) return fail(INVALID_INPUT, "order keys need the index buffer");
  if (key && n > 0xffffffffll) return fail(NOT_SUPPORTED, "more than 2^32 points");
  cudaError_t e = launch_pose_depths(mu, n, R9, t3, z, key, idx, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_pose_depths");
  return OK;
}

int xgs_hashset_create(int64_t capacity, void** handle) {
  if (!handle || capacity < 0) return fail(INVALID_INPUT, "bad hashset arguments");
  HashSet* h = nullptr;
  cudaError_t e = hashset_create(capacity < 1024 ? 1024 : 2 * capacity, &h);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_hashset_create");
  *handle = h;
  return OK;
}

int xgs_hashset_destroy(void* handle) {
  hashset_destroy(static_cast<HashSet*>(handle));
  return OK;
}

int xgs_hashset_insert(void* handle, const uint64_t* keys, int64_t n, uint8_t* was_new, void* stream) {
  if (!handle || n < 0 || (n > 0 && !keys)) return fail(INVALID_INPUT, "bad hashset insert");
  cudaError_t e = hashset_insert(static_cast<HashSet*>(handle), keys, n, was_new, (cudaStream_t)stream);
  if (e == cudaErrorNotSupported)
    return fail(NOT_SUPPORTED, "the map was used by an XGS_GRID_ASYNC call (a CUDA graph may hold its table) and "
                               "cannot grow");
  if (e != cudaSuccess) return cuda_fail(e, "xgs_hashset_insert");
  return OK;
}

int xgs_hashset_contains(void* handle, const uint64_t* keys, int64_t n, uint8_t* out, void* stream) {
  if (!handle || n < 0 || (n > 0 && (!keys || !out))) return fail(INVALID_INPUT, "bad hashset query");
  cudaError_t e = hashset_contains(static_cast<HashSet*>(handle), keys, n, out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_hashset_contains");
  return OK;
}

int xgs_hashset_copy(void* dst, const void* src, void* stream) {
  if (!dst || !src) return fail(INVALID_INPUT, "bad hashset copy");
  if (dst == src) return OK;
  cudaError_t e = hashset_copy(static_cast<HashSet*>(dst), static_cast<const HashSet*>(src), (cudaStream_t)stream);
  if (e == cudaErrorInvalidValue) return fail(INVALID_INPUT, "hashset copy needs equal table capacities");
  if (e != cudaSuccess) return cuda_fail(e, "xgs_hashset_copy");
  return OK;
}

int xgs_hashset_size(void* handle, int64_t* n_out, void* stream) {
  if (!handle || !n_out) return fail(INVALID_INPUT, "bad hashset size");
  cudaError_t e = hashset_size(static_cast<HashSet*>(handle), n_out, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_hashset_size");
  return OK;
}

size_t xgs_grid_workspace(int64_t npix) { return grid_workspace_bytes(npix); }

int xgs_radix_sort_pairs_u64(uint64_t* keys, uint32_t* vals, int64_t n, int bits, void* ws, size_t ws_bytes,
                             void* stream) {
  if (n < 0 || bits < 0 || bits > 64 || (n > 0 && (!keys || !vals))) return fail(INVALID_INPUT, "bad sort");
  if (n > 0x7fffffff) return fail(NOT_SUPPORTED, "more than 2^31-1 items");
  if (ws_bytes < grid_workspace_bytes(n)) return fail(INVALID_INPUT, "workspace too small");
  if (n == 0) return OK;
  cudaError_t e = radix_sort_pairs(keys, vals, n, bits, ws, ws_bytes, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_radix_sort_pairs_u64");
  return OK;
}

static int grid_sample_call(const xgs_grid_frames* in, void* hashset, xgs_grid_result* out, void* ws, size_t ws_bytes,
                            void* stream, float* depth_dev, uint8_t* color_dev) {
  if (!in || !out || !hashset) return fail(INVALID_INPUT, "null argument");
  if (in->frames < 0 || in->height < 1 || in->width < 1) return fail(INVALID_INPUT, "bad frame shape");
  if (!(in->voxel > 0) || !(in->fx > 0) || !(in->fy > 0)) return fail(INVALID_INPUT, "voxel size and focal lengths must be positive");
  if (in->stride < 1) return fail(INVALID_INPUT, "stride must be >= 1");
  if (in->mode != 0 && in->mode != 1) return fail(INVALID_INPUT, "mode must be 0 (first) or 1 (mean)");
  const int64_t npix = in->frames * in->height * in->width;
  if (npix > 0x7fffffff) return fail(NOT_SUPPORTED, "more than 2^31-1 pixels per batch");
  if (npix > 0 && (!in->depth || !in->rot || !in->trans)) return fail(INVALID_INPUT, "null frame buffer");
  if (in->feat && (in->feat_c < 1 || in->feat_h < 1 || in->feat_w < 1 || !out->feat))
    return fail(INVALID_INPUT, "bad feature map");
  if (in->feat && out->feat_dtype != XGS_F32 && out->feat_dtype != XGS_F64)
    return fail(INVALID_INPUT, "feature output dtype must be XGS_F32 or XGS_F64");
  if (in->feat && in->mode == 1 && out->feat_dtype != XGS_F64)
    return fail(INVALID_INPUT, "mean-mode features are fp64 averages: feat_dtype must be XGS_F64");
  if (ws_bytes < grid_workspace_bytes(npix)) return fail(INVALID_INPUT, "workspace too small");
  GridIn gi;
  gi.frames = in->frames;
  gi.H = in->height;
  gi.W = in->width;
  if (depth_dev) {   // host frames, copied into the device staging buffers inside the call
    if (in->color && !color_dev) return fail(INVALID_INPUT, "colour staging buffer missing");
    gi.depth = depth_dev;
    gi.color = in->color ? color_dev : nullptr;
    gi.depth_host = in->depth;
    gi.color_host = in->color;
  } else {
    gi.depth = in->depth;
    gi.color = in->color;
  }
  gi.rot = in->rot;
  gi.trans = in->trans;
  gi.fx = in->fx;
  gi.fy = in->fy;
  gi.cx = in->cx;
  gi.cy = in->cy;
  gi.voxel = in->voxel;
  gi.stride = in->stride;
  gi.mode = in->mode;
  gi.min_scale = in->min_scale;
  gi.feat = in->feat;
  gi.fc = in->feat_c;
  gi.fh = in->feat_h;
  gi.fw = in->feat_w;
  gi.async = (in->flags & XGS_GRID_ASYNC) != 0;
  if (gi.async && (in->mode != 0 || depth_dev)) return fail(NOT_SUPPORTED, "XGS_GRID_ASYNC: first-pick, device frames only");
  GridOut go;
  go.capacity = out->capacity;
  go.key = out->key;
  go.pid = out->pid;
  go.mu = out->mu;
  go.color = out->color;
  go.scale = out->scale;
  go.depth = out->depth;
  go.feat = out->feat;
  go.feat64 = out->feat_dtype == XGS_F64;
  go.count = out->count;
  go.dev_status = out->dev_status;
  cudaError_t e = grid_sample(gi, static_cast<HashSet*>(hashset), go, ws, ws_bytes, sm_count(), (cudaStream_t)stream);
  if (e == cudaErrorNotSupported)
    return fail(NOT_SUPPORTED, gi.async ? "XGS_GRID_ASYNC needs the library state sized by an earlier synchronous "
                                          "batch of at least this size"
                                        : "the map was used by an XGS_GRID_ASYNC call (a CUDA graph may hold its "
                                          "table) and cannot grow: create it with room for the whole stream");
  out->n_new = go.n_new;
  out->n_valid = go.n_valid;
  out->n_voxels = go.n_voxels;
  out->n_sorted = go.n_sorted;
  out->sort_passes = go.sort_passes;
  if (e == cudaErrorInvalidValue && go.n_new > go.capacity) return fail(INVALID_INPUT, "output capacity too small");
  if (e != cudaSuccess) return cuda_fail(e, "xgs_grid_sample");
  return OK;
}

int xgs_grid_sample(const xgs_grid_frames* in, void* hashset, xgs_grid_result* out, void* ws, size_t ws_bytes,
                    void* stream) {
  return grid_sample_call(in, hashset, out, ws, ws_bytes, stream, nullptr, nullptr);
}

// Same, with in->depth / in->color in (pinned) host memory: copied into
// depth_dev [F,H,W] / color_dev [F,H,W,3] frame chunk by frame chunk, each
// chunk's front-end launch overlapping the next chunk's copy.
int xgs_grid_sample_h2d(const xgs_grid_frames* in, float* depth_dev, uint8_t* color_dev, void* hashset,
                        xgs_grid_result* out, void* ws, size_t ws_bytes, void* stream) {
  if (!depth_dev) return fail(INVALID_INPUT, "null depth staging buffer");
  return grid_sample_call(in, hashset, out, ws, ws_bytes, stream, depth_dev, color_dev);
}

int xgs_prefix_mask(const int64_t* n_dev, int64_t cap, uint8_t* mask, void* stream) {
  if (cap < 0 || (cap > 0 && (!n_dev || !mask))) return fail(INVALID_INPUT, "bad prefix mask");
  if (cap == 0) return OK;
  cudaError_t e = launch_prefix_mask(n_dev, cap, mask, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_prefix_mask");
  return OK;
}

// ---------------------------------------------------------------- SUPERVISION

int xgs_sup_gather(const void* P, int p_dtype, int64_t Hf, int64_t Wf, const int64_t* S, const double* Phi, int64_t R,
                   int64_t D, int64_t H, int64_t W, int64_t s, const int32_t* offs, int64_t n_off, int64_t Hp,
                   int64_t Wp, double* G, double* V, int* corrupt, void* stream) {
  if (s < 1) return fail(INVALID_INPUT, "stride must be >= 1");
  if (H < 1 || W < 1 || D < 0 || n_off < 0 || Hp < 0 || Wp < 0) return fail(INVALID_INPUT, "bad target shape");
  if (P && (Hf < 1 || Wf < 1 || (p_dtype != F32 && p_dtype != F64)))
    return fail(INVALID_INPUT, "feature source must be (D, H_f, W_f) with H_f, W_f >= 1");
  if (!P && (!S || (R > 0 && !Phi))) return fail(INVALID_INPUT, "need a feature source or an annotation");
  if (n_off > 65535) return fail(NOT_SUPPORTED, "more than 65535 offsets per call");
  if (n_off > 0 && (!offs || !G)) return fail(INVALID_INPUT, "null buffer");
  cudaError_t e = launch_sup_gather(P, p_dtype, Hf, Wf, S, Phi, R, D, H, W, s, offs, n_off, Hp, Wp, G, V, corrupt,
                                    (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_sup_gather");
  return OK;
}

int xgs_sup_loss(const double* pred, const double* G, const double* V, int64_t D, int64_t cells, double lam,
                 double* acc, double* cot, void* stream) {
  if (D < 1 || cells < 0) return fail(INVALID_INPUT, "prediction and target shapes disagree");
  if (cells > 0 && (!pred || !G || !V || !acc || !cot)) return fail(INVALID_INPUT, "null buffer");
  cudaError_t e = launch_sup_loss(pred, G, V, D, cells, lam, acc, cot, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_sup_loss");
  return OK;
}


// ------------------------------------------------------- codebook consumers

int xgs_softmax_rows(const double* logits, int64_t n, int64_t k, int mode, const double* upstream, double* out,
                     double* out_h, void* stream) {
  if (n < 0 || k < 1) return fail(INVALID_INPUT, "bad logits shape");
  if (k > 8192) return fail(NOT_SUPPORTED, "K > 8192");
  if (mode != CB_WEIGHTS && mode != CB_ENTROPY && mode != CB_VJP) return fail(INVALID_INPUT, "bad softmax mode");
  if (n == 0) return OK;
  if (!logits || ((mode != CB_ENTROPY) && !out) || (mode == CB_ENTROPY && !out_h) || (mode == CB_VJP && !upstream))
    return fail(INVALID_INPUT, "null buffer");
  SumPlan pk;
  if (!build_sum_plan((int)k, &pk)) return fail(NOT_SUPPORTED, "K too large for the pairwise plan");
  cudaStream_t s = (cudaStream_t)stream;
  // non-finite flag: a per-thread, per-device mapped pinned word the kernel
  // sets directly (no allocation, no copy per call)
  thread_local volatile int* hflag[16] = {};
  thread_local int* dflag[16] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess && (dev < 0 || dev >= 16)) e = cudaErrorInvalidDevice;
  if (e == cudaSuccess && !hflag[dev]) {
    void* h = nullptr;
    e = cudaHostAlloc(&h, 64, cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&dflag[dev]), h, 0);
    if (e == cudaSuccess) hflag[dev] = static_cast<volatile int*>(h);
  }
  if (e == cudaSuccess) {
    *hflag[dev] = 0;
    e = launch_softmax_rows(logits, n, k, mode, upstream, out, out_h, pk, dflag[dev], s);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_softmax_rows");
  if (*hflag[dev]) return fail(INVALID_INPUT, "logits must be finite");
  return OK;
}

int xgs_contrast_scores(const double* feats, int64_t n, int64_t d, const double* qvecs, int64_t nq, double tau,
                        double eps, double* scores, void* stream) {
  if (n < 0 || d < 1 || d > 8192) return fail(INVALID_INPUT, "bad feature shape");
  if (nq < 2) return fail(INVALID_INPUT, "query must carry at least one negative phrase");
  if (n == 0) return OK;
  if (!feats || !qvecs || !scores) return fail(INVALID_INPUT, "null buffer");
  SumPlan pd;
  if (!build_sum_plan((int)d, &pd)) return fail(NOT_SUPPORTED, "feature dim too large");
  cudaError_t e = launch_contrast(feats, n, d, qvecs, nq, tau, eps, scores, pd, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_contrast_scores");
  return OK;
}

int xgs_desc_order_keys(const double* v, int64_t n, uint64_t* keys, uint32_t* idx, void* stream) {
  if (n < 0 || n > 0xffffffffll) return fail(INVALID_INPUT, "bad length");
  if (n && (!v || !keys || !idx)) return fail(INVALID_INPUT, "null buffer");
  cudaError_t e = launch_desc_keys(v, n, keys, idx, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_desc_order_keys");
  return OK;
}

// First m entries of np.argsort(-v, kind="stable") (thinker.py:202) without
// sorting all n: top-16-bit bucket select + stable sort of the candidates.
size_t xgs_desc_top_m_workspace(int64_t n) { return topm_workspace_bytes(n < 0 ? 0 : n); }
int xgs_desc_top_m(const double* v, int64_t n, int64_t m, int64_t* out, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || n > 0x7fffffffll || m < 0 || m > n) return fail(INVALID_INPUT, "bad length");
  if (n && m && (!v || !out)) return fail(INVALID_INPUT, "null buffer");
  if (ws_bytes < topm_workspace_bytes(n)) return fail(INVALID_INPUT, "workspace too small");
  cudaError_t e = launch_desc_top_m(v, n, m, out, ws, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "xgs_desc_top_m");
  return OK;
}

// ------------------------------------------------------- lattice rasterizer

int xgs_raster_build(const xgs_raster_in* in, void** handle, int64_t* n_pairs, int64_t* blend_steps, void* stream) {
  if (!in || !handle) return fail(INVALID_INPUT, "null argument");
  *handle = nullptr;
  if (in->n < 0 || in->n > 0x7fffffffll || in->n_rows < 0 || in->n_cols < 0 || in->row_step < 1 || in->col_step < 1)
    return fail(INVALID_INPUT, "bad raster shape");
  if (in->n_rows * in->n_cols > 0x7fffffffll) return fail(NOT_SUPPORTED, "lattice too large");
  if (in->n > 0 && (!in->mu || !in->quat || !in->scale || !in->opacity)) return fail(INVALID_INPUT, "null field");
  if (!(in->fx > 0) || !(in->fy > 0) || !(in->near_z > 0 && in->near_z < in->far_z))
    return fail(INVALID_INPUT, "bad intrinsics");
  RasterIn r;
  r.n = in->n;
  r.mu = in->mu;
  r.quat = in->quat;
  r.scale = in->scale;
  r.opacity = in->opacity;
  std::memcpy(r.R, in->R, sizeof(r.R));
  std::memcpy(r.t, in->t, sizeof(r.t));
  r.fx = in->fx; r.fy = in->fy; r.cx = in->cx; r.cy = in->cy; r.near_z = in->near_z; r.far_z = in->far_z;
  r.n_rows = in->n_rows; r.row0 = in->row0; r.row_step = in->row_step;
  r.n_cols = in->n_cols; r.col0 = in->col0; r.col_step = in->col_step;
  r.term = in->term_threshold; r.cutoff = in->cutoff_sigma; r.eig_floor = in->eig_floor;
  r.all_pairs = in->all_pairs != 0;
  RasterState* st = nullptr;
  cudaError_t e = raster_build(r, &st, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    raster_free(st);
    return cuda_fail(e, "xgs_raster_build");
  }
  raster_stats(st, n_pairs, blend_steps, nullptr);
  *handle = st;
  return OK;
}

int xgs_raster_fetch(void* handle, int64_t* gauss, int64_t* pixel, double* weight, double* alpha_prime, double* t_before,
                     uint8_t* alive, double* depth, void* stream) {
  if (!handle) return fail(INVALID_INPUT, "null handle");
  cudaError_t e = raster_fetch(static_cast<RasterState*>(handle), gauss, pixel, weight, alpha_prime, t_before, alive,
                               depth, (cudaStream_t)stream);
  return e == cudaSuccess ? OK : cuda_fail(e, "xgs_raster_fetch");
}

int xgs_raster_accumulate(void* handle, const double* payload, int64_t C, double* out, double* alpha_out,
                          double* depth_out, void* stream) {
  if (!handle || C < 0 || (C > 0 && (!payload || !out))) return fail(INVALID_INPUT, "bad accumulate arguments");
  cudaError_t e = raster_accumulate(static_cast<RasterState*>(handle), payload, C, out, alpha_out, depth_out,
                                    (cudaStream_t)stream);
  return e == cudaSuccess ? OK : cuda_fail(e, "xgs_raster_accumulate");
}

int xgs_raster_argmax(void* handle, int64_t* out, void* stream) {
  if (!handle || !out) return fail(INVALID_INPUT, "bad argmax arguments");
  cudaError_t e = raster_argmax(static_cast<RasterState*>(handle), out, (cudaStream_t)stream);
  return e == cudaSuccess ? OK : cuda_fail(e, "xgs_raster_argmax");
}

int xgs_raster_vjp(void* handle, const double* upstream, int64_t D, double* feature_grads, void* stream) {
  if (!handle || D < 1 || !upstream || !feature_grads) return fail(INVALID_INPUT, "bad vjp arguments");
  cudaError_t e = raster_vjp(static_cast<RasterState*>(handle), upstream, D, feature_grads, (cudaStream_t)stream);
  return e == cudaSuccess ? OK : cuda_fail(e, "xgs_raster_vjp");
}

int xgs_raster_free(void* handle) {
  raster_free(static_cast<RasterState*>(handle));
  return OK;
}

}  // extern "C"
