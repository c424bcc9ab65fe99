// Host-side launchers shared between the kernel translation units and the
// C-ABI layer (capi.cu).  No torch types anywhere: plain pointers + sizes.
#pragma once

#include <cstdlib>

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include "common.cuh"

namespace xgs {

// ---------------- launch accounting + opt-in event profiler (capi.cu) ----------------
// Every kernel launch is counted; when profiling is on, the named kernels are
// bracketed by CUDA events recorded on their own stream.
void count_launches(int n);
struct ProfScope {
  ProfScope(const char* tag, cudaStream_t s);
  ~ProfScope();
  const char* tag;
  cudaStream_t s;
  void* ev0;
};

// ---------------- exact fp64 path (vq_exact.cu) ----------------
enum ExactMode : int {
  EX_WRITE_DIST = 1,   // out_dist[row*K + k] = exact squared distance
  EX_WRITE_CODE = 2,   // codes[row] = argmin (first minimum)
  EX_CONF_MASK = 4,    // mask[row] = max softmax(-sqrt(d)/tau) >= gamma
  EX_WRITE_PROB = 8,   // out_prob[row*K + k] = softmax probabilities
};
struct ExactArgs {
  const void* x;
  int dtype;
  int64_t n, d, ldx;
  const double* E;
  int64_t k;
  const int32_t* rows;      // optional row list (else rows 0..n-1)
  const int32_t* nrows_dev; // optional device count for the row list
  int mode;
  double tau, gamma;
  double* out_dist;
  double* out_prob;
  int64_t* codes;
  uint8_t* mask;
};
cudaError_t launch_exact_rows(const ExactArgs& a, const SumPlan& pd, const SumPlan& pk,
                              cudaStream_t s);

// Candidate re-rank queue entries written by the screening GEMM.
constexpr int kCandCap = 16;
struct RerankEntry {
  int32_t row;
  int32_t cnt;
  int32_t cand[kCandCap];
};
cudaError_t launch_rerank(const void* x, int dtype, int64_t d, int64_t ldx, const double* E,
                          const RerankEntry* q, const int32_t* qcount, int64_t qcap,
                          int64_t* codes, const SumPlan& pd, cudaStream_t s);

// ---------------- tcgen05 screening GEMM (vq_screen_sm100.cu) ----------------
struct ScreenArgs {
  const void* x;        // input rows (any dtype); scaled fp16 copy made per call
  int dtype;
  int64_t n, d, ldx;
  const double* E;      // fp64 master codebook (K x D)
  int64_t k;
  int64_t* codes;       // out: int64 codes for rows resolved in the epilogue
  void* ws;             // workspace (see screen_workspace_bytes)
  size_t ws_bytes;
  float c1, c2, c4;     // error-bound coefficients (host computed)
  const SumPlan* pd;
  int sm_count;
  const int64_t* n_dev = nullptr;   // nullable: rows [0, min(*n_dev, n)) only (single-chunk batches)
};
size_t screen_workspace_bytes(int64_t n, int64_t k, int64_t d, int dtype, int64_t ldx);
cudaError_t launch_screen_assign(const ScreenArgs& a, cudaStream_t s, int32_t* host_stats);
// staged form used by the row-chunk pipeline: codebook prep once, then per
// chunk of rows [r0, r1): operand prep, screen + re-rank + exact rescan
constexpr int kMaxChunks = 64;
// Rows per screening chunk (the unit the per-row screening buffers are sized
// for): the whole batch up to 2^21 rows, else 2^21 (or n / kMaxChunks rounded
// up to a 256-row tile pair when that is larger).
// XGS_SCREEN_CHUNK_ROWS overrides the 2^21 (tests drive the multi-chunk
// slot ring with small batches).
inline int64_t screen_chunk_rows(int64_t n) {
  static const int64_t env = [] {
    const char* v = std::getenv("XGS_SCREEN_CHUNK_ROWS");
    return v ? (int64_t)std::atoll(v) : (int64_t)0;
  }();
  const int64_t base = env >= 256 ? env / 256 * 256 : (int64_t)1 << 21;
  if (n <= base) return n > 0 ? n : 1;
  int64_t c = (n + kMaxChunks - 1) / kMaxChunks;
  c = (c + 255) / 256 * 256;
  return c > base ? c : base;
}
cudaError_t screen_prepare(const ScreenArgs& a, cudaStream_t s);
cudaError_t screen_prep_rows(const ScreenArgs& a, int64_t r0, int64_t r1, int chunk, cudaStream_t s);
cudaError_t screen_rows(const ScreenArgs& a, int64_t r0, int64_t r1, int chunk, cudaStream_t s);
cudaError_t screen_rerank(const ScreenArgs& a, int64_t r0, int64_t r1, int chunk, cudaStream_t s);
cudaError_t screen_finish(const ScreenArgs& a, int chunks, cudaStream_t s, int32_t* host_stats);

// ---------------- row-chunk pipelined assign + accumulate (vq_pipeline.cu) ----------------
int pipeline_chunks(int64_t n, int sm_count, int64_t* chunk_rows, bool host_src);
// x_host (nullable): rows are streamed from this (pinned) host copy into a.x
// chunk by chunk, each copy overlapping the previous chunk's device work
cudaError_t launch_assign_accumulate(const ScreenArgs& a, double* counts, double* sums, void* acc_ws,
                                     size_t acc_ws_bytes, cudaStream_t s, int32_t* host_stats,
                                     const void* x_host = nullptr);

// ---------------- codebook update (vq_update.cu) ----------------
size_t accumulate_workspace_bytes(int64_t n, int64_t k);

// farthest-point seeding (vq_seed.cu): K-1 launches, no host synchronisation
size_t seed_workspace_bytes(int64_t n);
cudaError_t launch_seed_farthest(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, int64_t k,
                                 int64_t* seeds, void* ws, const SumPlan& pd, cudaStream_t s);
// cont != 0 continues the per-(k, d) chains and counts from the values already
// in counts/sums (rows of this call follow, in row order, the rows of the
// previous call): chunked accumulation is bit-identical to one call.
cudaError_t launch_accumulate(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx,
                              const int64_t* codes, const uint8_t* mask, int64_t k,
                              double* counts, double* sums, void* ws, size_t ws_bytes,
                              int sm_count, cudaStream_t s, int cont = 0);
cudaError_t launch_ema(double lam, double one_minus_lam, double eps, int64_t k, int64_t d,
                       const double* N, const double* M, const double* counts, const double* sums,
                       double* N_out, double* M_out, double* E_out, cudaStream_t s);
cudaError_t launch_revive(int64_t k, int64_t d, double n_new, double denom, const double* ring,
                          int64_t cap, const int64_t* dead_k, const int64_t* ring_rows,
                          int64_t n_dead, double* N, double* M, double* E, cudaStream_t s);
cudaError_t launch_ring_write_dev(const void* x, int dtype, int64_t ldx, const int64_t* n_dev, int64_t n_max,
                                  int64_t d, double* ring, int64_t cap, int64_t* start_dev, cudaStream_t s);
cudaError_t launch_ring_write(const void* x, int dtype, int64_t ldx, int64_t row0, int64_t nrows,
                              int64_t d, double* ring, int64_t cap, int64_t phys0,
                              cudaStream_t s);
cudaError_t launch_gather_rows(const double* src, int64_t d, const int64_t* rows, int64_t n,
                               double* dst, cudaStream_t s);

// ---------------- voxel grid sampling (grid.cu) ----------------
struct HashSet;
cudaError_t hashset_create(int64_t capacity, HashSet** out);
void hashset_destroy(HashSet* h);
cudaError_t hashset_size(HashSet* h, int64_t* n, cudaStream_t s);
cudaError_t hashset_reserve(HashSet* h, int64_t extra, cudaStream_t s);
cudaError_t hashset_insert(HashSet* h, const uint64_t* keys, int64_t n, uint8_t* was_new, cudaStream_t s);
cudaError_t hashset_contains(HashSet* h, const uint64_t* keys, int64_t n, uint8_t* out, cudaStream_t s);
cudaError_t hashset_copy(HashSet* dst, const HashSet* src, cudaStream_t s);
cudaError_t launch_backproject(const double* R, const double* t, const double* intr4, double voxel, const double* u,
                               const double* v, const double* d, int64_t n, double* out, cudaStream_t s);
size_t grid_workspace_bytes(int64_t npix);
struct GridIn {
  int64_t frames, H, W;
  const float* depth;
  const uint8_t* color;
  // host frames (xgs_grid_sample_h2d): copied into depth / color inside the call
  const float* depth_host = nullptr;
  const uint8_t* color_host = nullptr;
  const double* rot;
  const double* trans;
  double fx, fy, cx, cy, voxel;
  int stride, mode;
  double min_scale;
  const float* feat;
  int64_t fc, fh, fw;
  bool async = false;       // XGS_GRID_ASYNC: no host sync / allocation (graph-capturable)
};
struct GridOut {
  int64_t capacity;
  uint64_t* key;
  int64_t* pid;
  double* mu;
  double* color;
  double* scale;
  double* depth;
  void* feat;               // [cap, C], fp32 (feat64 == 0, first-pick only) or fp64
  int feat64;
  double* count;
  int64_t* dev_status = nullptr;   // device {n_new, n_valid, n_voxels, error}
  int64_t n_new, n_valid, n_voxels;
  int64_t n_sorted, sort_passes;
};
cudaError_t launch_prefix_mask(const int64_t* n_dev, int64_t cap, uint8_t* mask, cudaStream_t s);
cudaError_t launch_pose_depths(const double* mu, int64_t n, const double* R9, const double* t3, double* z,
                               uint64_t* key, uint32_t* idx, cudaStream_t s);
cudaError_t grid_sample(const GridIn& in, HashSet* hs, GridOut& out, void* ws, size_t ws_bytes, int sms,
                        cudaStream_t s);
cudaError_t radix_sort_pairs(uint64_t* keys, uint32_t* vals, int64_t n, int bits, void* ws, size_t ws_bytes,
                             cudaStream_t s);
cudaError_t exclusive_scan_i32(const int32_t* in, int64_t n, int32_t* out, int32_t* block_sums, int32_t* grand,
                               cudaStream_t s);

// ---------------- supervision targets (supervision.cu) ----------------
cudaError_t launch_sup_gather(const void* P, int p_dtype, int64_t Hf, int64_t Wf, const int64_t* S, const double* Phi,
                              int64_t R, int64_t D, int64_t H, int64_t W, int64_t s, const int32_t* offs,
                              int64_t n_off, int64_t Hp, int64_t Wp, double* G, double* V, int* corrupt,
                              cudaStream_t st);
cudaError_t launch_sup_loss(const double* pred, const double* G, const double* V, int64_t D, int64_t cells, double lam,
                            double* acc, double* cot, cudaStream_t st);

// ---------------- lattice rasterizer (raster.cu) ----------------
struct RasterIn {
  int64_t n;
  const double* mu;
  const double* quat;
  const double* scale;
  const double* opacity;
  double R[9], t[3];
  double fx, fy, cx, cy, near_z, far_z;
  int64_t n_rows, row0, row_step, n_cols, col0, col_step;
  double term, cutoff, eig_floor;
  int all_pairs;   // 1: dead pairs too (build_blend_pairs), 0: alive prefix only
};
struct RasterState;
cudaError_t raster_build(const RasterIn& in, RasterState** out, cudaStream_t s);
void raster_free(RasterState* st);
void raster_stats(RasterState* st, int64_t* npairs, int64_t* blend_steps, int64_t* nvis);
cudaError_t raster_fetch(RasterState* st, int64_t* gauss, int64_t* pixel, double* weight, double* alpha, double* tb,
                         uint8_t* alive, double* depth, cudaStream_t s);
cudaError_t raster_accumulate(RasterState* st, const double* payload, int64_t C, double* out, double* alpha_out,
                              double* depth_out, cudaStream_t s);
cudaError_t raster_argmax(RasterState* st, int64_t* out, cudaStream_t s);
cudaError_t raster_vjp(RasterState* st, const double* upstream, int64_t D, double* fg, cudaStream_t s);

// ---------------- fp64 codeword contractions (decode_f64.cu) ----------------
size_t gemm_f64_workspace_bytes(int64_t n, int64_t m, int64_t nq, int64_t kr, bool softmax);
cudaError_t launch_gemm_f64(const double* A, int64_t n, int64_t kr, int64_t lda_r, int64_t lda_k, bool softmax,
                            const double* B, int64_t m, int64_t ldb_k, int64_t ldb_m, double* C, int64_t ldc,
                            const double* Q, int64_t nq, double tau, double eps, double* scores, void* ws,
                            cudaStream_t s);

// ---------------- codebook consumers (codebook.cu) ----------------
enum CbMode : int { CB_WEIGHTS = 1, CB_ENTROPY = 2, CB_VJP = 4 };
cudaError_t launch_softmax_rows(const double* logits, int64_t n, int64_t k, int mode, const double* up, double* out,
                                double* out_h, const SumPlan& pk, int* bad, cudaStream_t s);
cudaError_t launch_contrast(const double* F, int64_t n, int64_t d, const double* Q, int64_t nq, double tau, double eps,
                            double* scores, const SumPlan& pd, cudaStream_t s);
size_t topm_workspace_bytes(int64_t n);
cudaError_t launch_desc_top_m(const double* v, int64_t n, int64_t m, int64_t* out, void* ws, cudaStream_t s);
cudaError_t launch_desc_keys(const double* v, int64_t n, uint64_t* keys, uint32_t* idx, cudaStream_t s);

}  // namespace xgs
