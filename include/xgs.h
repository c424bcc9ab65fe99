/*
 * xgs.h — C ABI of libxgs, the B200 (sm_100a) implementation of the X-GS
 * per-frame hot path: online EMA vector quantisation and voxel grid sampling.
 *
 * The reference (semsplat 0.1.0) has no FFI: its boundary is the Python API of
 * semsplat.vq and semsplat.slam.  Each entry point below names the reference
 * function it replaces (file:line under /root/reference/pkg/src/semsplat).
 * The Python package paper_2603_09632_b200 binds these through ctypes and keeps
 * the reference signatures; INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - every array argument is caller-owned DEVICE memory (plain pointers and
 *     sizes, row-major, leading dimension in elements); `stream` is a
 *     cudaStream_t passed as void*; calls are asynchronous on that stream
 *     unless stated otherwise;
 *   - scratch memory is caller-provided, sized by the matching *_workspace();
 *   - return 0 on success, XGS_INVALID_INPUT (-> InvalidInputError),
 *     XGS_INVALID_STATE (-> InvalidStateError), XGS_CUDA_ERROR,
 *     XGS_NOT_SUPPORTED; xgs_last_error() returns a thread-local message;
 *   - re-entrant: no global mutable state besides opaque handles.
 */
#ifndef XGS_H_
#define XGS_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define XGS_API __attribute__((visibility("default")))
#else
#define XGS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum { XGS_OK = 0, XGS_INVALID_INPUT = 1, XGS_INVALID_STATE = 2, XGS_CUDA_ERROR = 3, XGS_NOT_SUPPORTED = 4 };
enum { XGS_F32 = 0, XGS_F64 = 1, XGS_BF16 = 2 };
/* modes of xgs_vq_exact (bit set) */
enum { XGS_EX_DIST = 1, XGS_EX_CODE = 2, XGS_EX_MASK = 4, XGS_EX_PROB = 8 };

XGS_API int xgs_abi_version(void);
XGS_API const char* xgs_last_error(void);
XGS_API int xgs_device_sm_count(void);
/* number of kernels libxgs has launched in this process (bench evidence) */
XGS_API long long xgs_launch_count(void);
/* opt-in profiler: CUDA events recorded on the launching stream around each
 * named kernel group ("vq_prep", "vq_screen", "vq_rerank", "vq_accumulate",
 * "vq_chain", "vq_ema", "grid_*"); enable(1) clears, read() synchronises. */
XGS_API int xgs_profile_enable(int on);
/* restrict the profiler to one tag (NULL / "" = every tag): e.g. "grid_batch"
 * alone times a whole grid batch without events between its kernels */
XGS_API int xgs_profile_only(const char* tag);
XGS_API int xgs_profile_read(const char* tag, double* total_ms, long long* count);
/* CSV "tag,start_ms,end_ms" of every profiled launch, relative to the earliest */
XGS_API int xgs_profile_dump(const char* path);

/* ------------------------------------------------------------------ VQ */

/* assign_batch (vq.py:84-87) / assign (vq.py:76-81): int64 codes of the
 * nearest fp64 codeword, ties to the lowest index, bit-identical to the
 * reference.  tcgen05 fp16 screening GEMM + exact fp64 re-rank.
 * stats_out (HOST, nullable): {rows re-ranked, rows rescanned exactly};
 * when given the call synchronises on `stream`.
 * Errors: K == 0 -> XGS_INVALID_STATE (vq.py:78-79, 85-86). */
XGS_API size_t xgs_vq_assign_workspace(int64_t n, int64_t k, int64_t d, int dtype, int64_t ldx);
XGS_API int xgs_vq_assign(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, const double* E, int64_t k,
                          int64_t* codes, void* ws, size_t ws_bytes, int32_t* stats_out, void* stream);
/* xgs_vq_assign on rows [0, min(*n_dev, n)) only, the count read on the device
 * (graph-capturable: a fixed-capacity window whose valid row count a previous
 * kernel wrote, e.g. the new points of a grid batch); codes of the rows past it
 * are not written.  Single-chunk batches (n <= 2^21). */
XGS_API int xgs_vq_assign_dev(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, const double* E,
                              int64_t k, int64_t* codes, void* ws, size_t ws_bytes, const int64_t* n_dev,
                              void* stream);

/* Exact fp64 path, one CTA per row:
 *   XGS_EX_DIST  squared_distances (vq.py:69-73) -> out_dist (n, k)
 *   XGS_EX_CODE  argmin -> codes (n)
 *   XGS_EX_MASK  confidence_mask (vq.py:121-124) -> mask (n) u8: 1 pass, 0 reject, 2 undecided (fl(1/S)
 *                within 1e-12 relative of gamma: CUDA exp and the host libm may differ by an ulp;
 *                the caller decides these rows with the reference's host expression)
 *   XGS_EX_PROB  confidence_scores (vq.py:112-118) -> out_prob (n, k) */
XGS_API int xgs_vq_exact(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, const double* E, int64_t k,
                         int mode, double tau, double gamma, double* out_dist, double* out_prob, int64_t* codes,
                         uint8_t* mask, void* stream);

/* accumulate (vq.py:90-100) given the codes: counts = bincount(codes[mask]),
 * sums = np.add.at(zeros, codes[mask], x[mask]) — bit-identical (sequential
 * fp64 chains per (k, d) in ascending row order).  mask may be NULL. */
/* seed_from_samples (vq.py:126-147): greedy farthest-point traversal from row
 * 0; seeds[t] = first argmax of min squared distance (NumPy pairwise order),
 * or t % n once that maximum is 0.  K-1 kernel launches on `stream`, no host
 * synchronisation; seeds (k int64) and ws (xgs_vq_seed_workspace(n) bytes)
 * are device memory.  n == 0 -> invalid input. */
XGS_API size_t xgs_vq_seed_workspace(int64_t n);
XGS_API int xgs_vq_seed_farthest(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, int64_t k,
                                 int64_t* seeds, void* ws, size_t ws_bytes, void* stream);

XGS_API size_t xgs_vq_accumulate_workspace(int64_t n, int64_t k);
XGS_API int xgs_vq_accumulate(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, const int64_t* codes,
                              const uint8_t* mask, int64_t k, double* counts, double* sums, void* ws,
                              size_t ws_bytes, void* stream);

/* assign_batch + accumulate of one online_step (vq.py:193-212, the
 * accumulate(batch[mask]) at :206 when the confidence mask is all-true):
 * codes, counts and sums bit-identical to xgs_vq_assign followed by
 * xgs_vq_accumulate (mask NULL).  Rows are processed in chunks whose operand
 * prep, screening GEMM and accumulate chains overlap on internal streams;
 * the fp64 chains continue across chunks in row order, so the sums keep the
 * np.add.at order.  Completion is ordered on `stream`.  stats_out as for
 * xgs_vq_assign.  The enqueue is serialised by an internal lock. */
XGS_API size_t xgs_vq_step_workspace(int64_t n, int64_t k, int64_t d, int dtype, int64_t ldx);
XGS_API int xgs_vq_assign_accumulate(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, const double* E,
                                     int64_t k, int64_t* codes, double* counts, double* sums, void* ws,
                                     size_t ws_bytes, int32_t* stats_out, void* stream);
/* The same step with the rows in (pinned) HOST memory: x_host is copied into
 * the device buffer x chunk by chunk on an internal stream, each chunk's copy
 * overlapping the previous chunk's prep / screen / accumulate (the end-to-end
 * path is PCIe-bound).  x_host may equal NULL (then x is already resident). */
XGS_API int xgs_vq_assign_accumulate_h2d(const void* x_host, void* x, int dtype, int64_t n, int64_t d, int64_t ldx,
                                         const double* E, int64_t k, int64_t* codes, double* counts, double* sums,
                                         void* ws, size_t ws_bytes, int32_t* stats_out, void* stream);

/* ema_step (vq.py:103-109): N' = lam N + (1-lam) c ; M' = lam M + (1-lam) s ;
 * E' = M' / (N' + eps).  Outputs may alias inputs. */
XGS_API int xgs_vq_ema(double lam, double eps, int64_t k, int64_t d, const double* N, const double* M,
                       const double* counts, const double* sums, double* N_out, double* M_out, double* E_out,
                       void* stream);

/* revive_dead_codes (vq.py:173-190) after the host drew the reservoir rows:
 * for i < n_dead: M[k_i] = ring[r_i]; N[k_i] = 1+eps; E[k_i] = M[k_i]/(N[k_i]+eps). */
XGS_API int xgs_vq_revive(int64_t k, int64_t d, double eps, const double* ring, int64_t cap, const int64_t* dead_k,
                          const int64_t* ring_rows, int64_t n_dead, double* N, double* M, double* E,
                          void* stream);

/* FeatureReservoir.extend (core.py:191-195) as a device ring buffer:
 * rows [row0, row0+nrows) of x -> ring[(phys0 + j) % cap] as fp64. */
XGS_API int xgs_vq_ring_write(const void* x, int dtype, int64_t ldx, int64_t row0, int64_t nrows, int64_t d,
                              double* ring, int64_t cap, int64_t phys0, void* stream);
/* xgs_vq_ring_write with the row count on the device (graph-capturable): rows
 * [0, min(*n_dev, n_max)) of x are appended to the ring at the device-resident
 * write position *start_dev, which is then advanced ((start + n) % cap; n >= cap
 * keeps the last cap rows at ring rows [0, cap) and resets it to 0).  The
 * caller mirrors the FIFO bookkeeping on the host after reading n. */
XGS_API int xgs_vq_ring_write_dev(const void* x, int dtype, int64_t ldx, const int64_t* n_dev, int64_t n_max,
                                  int64_t d, double* ring, int64_t cap, int64_t* start_dev, void* stream);
XGS_API int xgs_gather_rows_f64(const double* src, int64_t d, const int64_t* rows, int64_t n, double* dst,
                                void* stream);

/* ------------------------------------------------ lattice rasterizer */

/* build_blend_pairs (rasterizer.py:89-191): depth-sorted, 3-sigma-culled,
 * transmittance-terminated blend pairs of a Gaussian field on the lattice
 * rows = row0 + row_step*i (i < n_rows), cols = col0 + col_step*j (j < n_cols).
 * Gaussian arrays are DEVICE fp64 (mu (n,3), quat wxyz (n,4), scale (n,3),
 * opacity (n)); the pose (world->camera R row-major, t) and intrinsics are
 * host values.  The handle owns the pairs (pixel-segmented, depth order
 * within a pixel); build synchronises on `stream` to size them. */
typedef struct {
  int64_t n;
  const double* mu;
  const double* quat;
  const double* scale;
  const double* opacity;
  double R[9], t[3];
  double fx, fy, cx, cy, near_z, far_z;
  int64_t n_rows, row0, row_step, n_cols, col0, col_step;
  double term_threshold, cutoff_sigma, eig_floor;
  int32_t all_pairs;   /* 1: every culled pair incl. dead ones (build_blend_pairs);
                          0: only pairs in front of termination (renders / VJP) */
} xgs_raster_in;
XGS_API int xgs_raster_build(const xgs_raster_in* in, void** handle, int64_t* n_pairs, int64_t* blend_steps,
                             void* stream);
/* BlendPairs arrays (any may be NULL): gauss/pixel int64, weight, alpha',
 * T_before, depth fp64, alive u8, each of length n_pairs. */
XGS_API int xgs_raster_fetch(void* handle, int64_t* gauss, int64_t* pixel, double* weight, double* alpha_prime,
                             double* t_before, uint8_t* alive, double* depth, void* stream);
/* _accumulate_channels / render (rasterizer.py:194-244): out (C, P) =
 * sum of weight * payload[gauss, c] per lattice pixel (pair order, as
 * np.bincount); alpha_out / depth_out (P) nullable. */
XGS_API int xgs_raster_accumulate(void* handle, const double* payload, int64_t C, double* out, double* alpha_out,
                                  double* depth_out, void* stream);
/* render_argmax_ids (rasterizer.py:290-306): Gaussian of the largest blend
 * weight per pixel, -1 where uncovered. */
XGS_API int xgs_raster_argmax(void* handle, int64_t* out, void* stream);
/* feature_gradients' blend cotangents (rasterizer.py:309-335): fg (n, D) =
 * np.add.at over pairs of weight * upstream[:, pixel], upstream (D, P). */
XGS_API int xgs_raster_vjp(void* handle, const double* upstream, int64_t D, double* feature_grads, void* stream);
XGS_API int xgs_raster_free(void* handle);

/* ------------------------------------------------- codebook consumers */

/* One fp64 row op over (n, k) logits, NumPy order (row max, exp(l - max),
 * pairwise sums over k <= 8192):
 *   mode 1  mixture_weights (core.py:473-480)  -> out (n, k)
 *   mode 2  semantic_entropy (thinker.py:185-191) -> out_h (n)
 *   mode 4  softmax_vjp (core.py:483-487) with upstream (n, k) -> out (n, k)
 * Non-finite logits -> XGS_INVALID_INPUT (the reference raises); the call
 * synchronises on `stream` to read that flag. */
XGS_API int xgs_softmax_rows(const double* logits, int64_t n, int64_t k, int mode, const double* upstream,
                             double* out, double* out_h, void* stream);
/* _contrast_scores / relevance_per_gaussian (thinker.py:110-129) on decoded
 * features F (n, d): q = 1 positive + nq-1 negative unit vectors (nq, d). */
XGS_API int xgs_contrast_scores(const double* feats, int64_t n, int64_t d, const double* qvecs, int64_t nq,
                                double tau, double eps, double* scores, void* stream);
/* keys + indices for a stable descending argsort (np.argsort(-v, kind=
 * "stable"), thinker.py:171, :202) through xgs_radix_sort_pairs_u64 with 64
 * key bits; -0.0 ties with +0.0 as in NumPy. */
XGS_API int xgs_desc_order_keys(const double* v, int64_t n, uint64_t* keys, uint32_t* idx, void* stream);
/* The first m indices of np.argsort(-v, kind="stable") (sample_tokens,
 * thinker.py:194-206) without ordering all n: histogram of the descending
 * keys' top 16 bits, the bucket of the m-th key, an order-preserving
 * compaction of the keys up to it and a stable 64-bit radix sort of those.
 * out: m int64 (device).  One host synchronisation (the candidate count). */
XGS_API size_t xgs_desc_top_m_workspace(int64_t n);
XGS_API int xgs_desc_top_m(const double* v, int64_t n, int64_t m, int64_t* out, void* ws, size_t ws_bytes,
                           void* stream);

/* ------------------------------------------------------------- GRID */

/* slam.backproject (slam.py:594-598) for n points, bit-identical:
 * cam = ((u-cx)*d/fx, (v-cy)*d/fy, d); p = R^T (cam - t) with OpenBLAS
 * dgemv's FMA order.  R (3x3 row-major world->camera), t (3), u, v, d (n)
 * and out (n x 3) are DEVICE pointers; intr4 = {fx, fy, cx, cy} is HOST. */
XGS_API int xgs_backproject(const double* R, const double* t, const double* intr4, const double* u,
                            const double* v, const double* d, int64_t n, double* out, void* stream);

/* GPU hash set of occupied voxel keys (the map).  Opaque handle; open
 * addressing with 64-bit keys, load factor kept <= 1/2 (grows on demand --
 * except after an XGS_GRID_ASYNC call used it: a graph may hold its table, so
 * a call that would have to grow it returns XGS_NOT_SUPPORTED).
 * insert = insert-if-absent; was_new (nullable) reports keys that were absent. */
XGS_API int xgs_hashset_create(int64_t capacity, void** handle);
XGS_API int xgs_hashset_destroy(void* handle);
XGS_API int xgs_hashset_insert(void* handle, const uint64_t* keys, int64_t n, uint8_t* was_new, void* stream);
XGS_API int xgs_hashset_contains(void* handle, const uint64_t* keys, int64_t n, uint8_t* out, void* stream);
XGS_API int xgs_hashset_size(void* handle, int64_t* n_out, void* stream); /* synchronises */
/* snapshot / restore: dst's keys become src's (tables of equal capacity; stream-ordered copy) */
XGS_API int xgs_hashset_copy(void* dst, const void* src, void* stream);

/* In-house stable LSD radix sort of (u64 key, u32 value) pairs on bits [0, bits). */
XGS_API size_t xgs_grid_workspace(int64_t npix);
XGS_API int xgs_radix_sort_pairs_u64(uint64_t* keys, uint32_t* vals, int64_t n, int bits, void* ws,
                                     size_t ws_bytes, void* stream);

/* slam.pose_depths (slam.py:654-655): z (n) = camera depth of the Gaussian
 * centres mu (n, 3) fp64 under the world->camera pose R9 / t3 (HOST arrays),
 * in the reference's BLAS evaluation order.  With key / idx non-NULL also the
 * ascending IEEE order keys of z and the identity indices, ready for
 * xgs_radix_sort_pairs_u64 (the median fallback depth of densify_and_prune). */
XGS_API int xgs_pose_depths(const double* mu, int64_t n, const double* R9, const double* t3, double* z,
                            uint64_t* key, uint32_t* idx, void* stream);

/* Voxel grid sampling of a batch of frames (the insertion half of
 * densify_and_prune, slam.py:601-651, with the coverage render replaced by
 * the occupied-voxel hash set; SURVEY.md 8(a) g8 definitions):
 * valid pixel = stride lattice and depth > 0; key = floor(p/voxel) packed
 * 3x21 bits biased by 2^20; representative = lowest (frame, pixel) id of a
 * voxel (mode 0) or the pixel-order mean over the voxel's points in that
 * frame (mode 1); voxels already in `hashset` are rejected and the new ones
 * inserted; outputs in ascending (frame, pixel) id.  Synchronises twice
 * (batch bounding box, output count).  A capacity of F * ceil(H/stride) *
 * ceil(W/stride) rows can never overflow; with a smaller one the call returns
 * XGS_INVALID_INPUT ("output capacity too small") AFTER the batch's new voxels
 * were inserted into `hashset` (n_new reports how many): the map already holds
 * them, so a retry of the same frames would reject them as occupied. */
typedef struct {
  int64_t frames, height, width;
  const float* depth;      /* [F,H,W] */
  const uint8_t* color;    /* [F,H,W,3] or NULL */
  const double* rot;       /* [F,3,3] world->camera rotations, row-major */
  const double* trans;     /* [F,3] */
  double fx, fy, cx, cy;   /* u = row pairs fx/cx (core.py:5-9) */
  double voxel;
  int32_t stride;          /* pixel lattice stride (slam.py:621-623) */
  int32_t mode;            /* 0 first-pick, 1 mean */
  double min_scale;        /* size = max(min_scale, 0.5*stride*depth/fx) (slam.py:631) */
  const float* feat;       /* [F,C,Hf,Wf] or NULL, gathered by supervision.py:133-147 */
  int64_t feat_c, feat_h, feat_w;
  int32_t flags;           /* XGS_GRID_ASYNC: see below */
} xgs_grid_frames;

/* flags: XGS_GRID_ASYNC -- no host synchronisation and no allocation inside
 * the call, so it can be captured in a CUDA graph: first-pick mode, device
 * frames only, a library state sized by an earlier synchronous call on this
 * device (same or larger frame batch), and a hash set created with room for
 * every voxel the stream will insert (load <= 1/2).  n_new / n_valid /
 * n_voxels are NOT returned in the struct (set to -1); out->dev_status
 * (device int64[4]) receives {n_new, n_valid, n_voxels, error} when the
 * batch's last kernel ends; error != 0 (batch table or map probing overflow)
 * means the batch must be redone synchronously.  A captured graph holds the
 * addresses of the library's per-device grid state: after the first async
 * call those buffers are never freed (a synchronous batch that outgrows one
 * gets a new buffer; the old one stays allocated for the graphs) -- and the
 * state's counters are shared, so grid batches of one device must run on one
 * stream at a time. */
enum { XGS_GRID_ASYNC = 1 };

typedef struct {
  int64_t capacity;        /* rows of every output array */
  uint64_t* key;           /* [cap] */
  int64_t* pid;            /* [cap] frame*H*W + u*W + v */
  double* mu;              /* [cap,3] */
  double* color;           /* [cap,3] rgb/255 */
  double* scale;           /* [cap] */
  double* depth;           /* [cap] */
  void* feat;              /* [cap,C] or NULL; element type feat_dtype */
  double* count;           /* [cap] points averaged (mode 1) or 1, nullable */
  int64_t n_new, n_valid, n_voxels; /* written by the call */
  int64_t n_sorted, sort_passes;     /* radix-sort work of the call (items, 8-bit passes) */
  int32_t feat_dtype;      /* XGS_F32 (mode 0 only: the gathered value) or XGS_F64 (mode 0: widened;
                              mode 1: the fp64 pixel-order mean over the voxel's members) */
  int64_t* dev_status;     /* device int64[4] {n_new, n_valid, n_voxels, error}, nullable (XGS_GRID_ASYNC) */
} xgs_grid_result;

XGS_API int xgs_grid_sample(const xgs_grid_frames* in, void* hashset, xgs_grid_result* out, void* ws,
                            size_t ws_bytes, void* stream);
/* xgs_grid_sample with in->depth / in->color in (pinned) HOST memory: the
 * frames are copied into the caller's device staging buffers depth_dev
 * [F,H,W] / color_dev [F,H,W,3] inside the call, frame chunk by frame chunk on
 * a library copy stream, each chunk's front-end launch overlapping the copy of
 * the next; returns after the host frames were read. */
XGS_API int xgs_grid_sample_h2d(const xgs_grid_frames* in, float* depth_dev, uint8_t* color_dev, void* hashset,
                                xgs_grid_result* out, void* ws, size_t ws_bytes, void* stream);

/* mask[i] = i < *n_dev for i < cap (uint8): the valid-row mask of a
 * fixed-capacity batch whose row count is known only on the device (the
 * graph-captured stream step feeds the grid's new voxels to the VQ this way). */
XGS_API int xgs_prefix_mask(const int64_t* n_dev, int64_t cap, uint8_t* mask, void* stream);

/* fp64 codeword contraction on the fp64 tensor pipe (DMMA), SURVEY 8(f) #3:
 * C[n x m] = op(A)[n x kr] . B[kr x m], element (r, k) of A at A[r*lda_r +
 * k*lda_k], of B at B[k*ldb_k + j*ldb_m].  softmax_rows: A holds logits and
 * enters as softmax over each row (mixture_weights, core.py:473-480).
 *   decode_feature (core.py:490-496): A = logits (n x K), B = E (K x D), C out.
 *   relevance_per_gaussian (thinker.py:122-129): scores (n) = the contrast of
 *     the decoded rows against Q = [positive; negatives] (nq x m) with tau /
 *     eps, no (n x D) feature matrix (C may be NULL).
 *   feature_gradients (rasterizer.py:309-335): A = fg (n x D), B = E^T.
 * Workspace: xgs_gemm_f64_workspace(n, kr, m, nq or 0, softmax_rows).  Agrees with the
 * reference's BLAS dgemm to ~1e-15 relative (different summation order). */
XGS_API size_t xgs_gemm_f64_workspace(int64_t n, int64_t kr, int64_t m, int64_t nq, int softmax_rows);
XGS_API int xgs_gemm_f64(const double* A, int64_t n, int64_t kr, int64_t lda_r, int64_t lda_k, int softmax_rows,
                         const double* B, int64_t m, int64_t ldb_k, int64_t ldb_m, double* C, int64_t ldc,
                         const double* Q, int64_t nq, double tau, double eps, double* scores, void* ws,
                         size_t ws_bytes, void* stream);

/* ------------------------------------------- SUPERVISION */

/* Grid-sampled supervision targets for n_off lattice offsets in one launch
 * ("target prefetch"): build_target_continuous (supervision.py:138-147) when
 * P != NULL (P: [D, Hf, Wf], dtype XGS_F32/XGS_F64), else
 * build_target_discrete (supervision.py:118-130) from S [H, W] int64 region ids
 * (-1 background) and Phi [R, D] fp64.  offs: [n_off, 2] int32 (o_h, o_w).
 * G: [n_off, D, Hp, Wp] fp64, V: [n_off, Hp, Wp] fp64; cells beyond the
 * offset's (H_s, W_s) are padding (pad_target, supervision.py:208-221).
 * corrupt (device int, nullable) is set to 1 for region ids outside [-1, R). */
XGS_API int xgs_sup_gather(const void* P, int p_dtype, int64_t Hf, int64_t Wf, const int64_t* S, const double* Phi,
                           int64_t R, int64_t D, int64_t H, int64_t W, int64_t s, const int32_t* offs, int64_t n_off,
                           int64_t Hp, int64_t Wp, double* G, double* V, int* corrupt, void* stream);

/* masked_semantic_loss (supervision.py:150-184) on [D, cells] fp64 arrays:
 * acc (device, 3 doubles) <- {sum(1-cos), sum(l1/D), n_valid}; cot <- dloss/dpred. */
XGS_API int xgs_sup_loss(const double* pred, const double* G, const double* V, int64_t D, int64_t cells, double lam,
                         double* acc, double* cot, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* XGS_H_ */
