// Codebook consumers: the per-Gaussian softmax family of
// core.py and the relevance / entropy / token sampling of thinker.py.
//
//   cb_rows_kernel     : one warp per logit row (K <= 8192), fp64.  Row max,
//                        exp(l - max), NumPy pairwise sums over K (the same
//                        leaf/combine order as np.sum along a contiguous
//                        axis, see common.cuh), then per mode
//                          WEIGHTS  mixture_weights      (core.py:473-480)
//                          ENTROPY  semantic_entropy     (thinker.py:185-191),
//                                   now cb_entropy_kernel (two passes)
//                          VJP      softmax_vjp          (core.py:483-487)
//                        Non-finite logits set a flag (the reference raises).
//   cb_contrast_kernel : one warp per decoded feature row: pairwise L2 norm
//                        (np.linalg.norm), normalise by (norm + eps), dot with
//                        the positive and every negative query vector and take
//                        the min over negatives of the two-way softmax
//                        (thinker.py:110-129).
//   cb_desc_keys_kernel: order-preserving u64 keys for a stable DESCENDING
//                        argsort (np.argsort(-v, kind="stable")) through the
//                        in-house radix sort (grid.cu); -0.0 folds onto +0.0
//                        because NumPy's comparison sort treats them as ties.
// The codeword mixture itself, softmax(logits) @ E, is a plain fp64 GEMM and
// goes to cuBLAS from the host (core.decode_feature).
#include "launchers.h"

namespace xgs {

namespace {

constexpr int kCbWarps = 8;

// exp(l - max) of the row is evaluated once into per-warp shared memory
// (CACHE: K <= kCbCacheK) and reused by the sums and the outputs.  The entropy
// uses p = e * (1/S) and log p = (l - max) - log S instead of e / S and
// log(e / S) (one division and one log per row, not per element; each differs
// by a few ulps, inside the 1e-13 relative tolerance of the parity tests).
constexpr int kCbCacheK = 1024;

template <int MODE, bool CACHE>
__global__ void __launch_bounds__(kCbWarps * 32)
cb_rows_kernel(const double* __restrict__ L, int64_t n, int64_t k, const double* __restrict__ up,
               double* __restrict__ out, double* __restrict__ out_h, SumPlan pk, int* __restrict__ bad) {
  __shared__ double scratch_all[kCbWarps][kMaxLeaves];
  extern __shared__ double ecache_all[];   // CACHE: kCbWarps x k
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* scratch = scratch_all[warp];
  double* ec = CACHE ? ecache_all + (size_t)warp * k : nullptr;
  for (int64_t r = (int64_t)blockIdx.x * kCbWarps + warp; r < n; r += (int64_t)gridDim.x * kCbWarps) {
    const double* l = L + r * k;
    double m = -__longlong_as_double(0x7ff0000000000000ll);
    bool fin = true;
#pragma unroll 8
    for (int64_t i = lane; i < k; i += 32) {
      const double v = __ldg(l + i);
      fin = fin && isfinite(v);
      m = fmax(m, v);
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
    if (!__all_sync(FULL, fin)) {
      if (lane == 0) *(volatile int*)bad = 1;   // idempotent flag (may live in mapped host memory)
      continue;
    }
    if (CACHE) {
#pragma unroll 4   // independent exp chains per lane (the fp64 pipe is latency-bound otherwise)
      for (int64_t i = lane; i < k; i += 32) ec[i] = exp(dsub(__ldg(l + i), m));
      __syncwarp();
    }
    auto ex = [&](int i) { return CACHE ? ec[i] : exp(dsub(__ldg(l + i), m)); };
    // S = sum exp(l - max) in NumPy's pairwise order
    const double S = warp_pairwise(pk, ex, scratch, lane);
    if (MODE == CB_WEIGHTS) {
      for (int64_t i = lane; i < k; i += 32) out[r * k + i] = ddiv(ex((int)i), S);
    } else if (MODE == CB_ENTROPY) {
      const double logS = log(S), invS = ddiv(1.0, S);
      const double h = warp_pairwise(
          pk,
          [&](int i) {
            const double p = dmul(ex(i), invS);   // within 1 ulp of e / S
            return p > 0.0 ? dmul(p, dsub(dsub(__ldg(l + i), m), logS)) : 0.0;
          },
          scratch, lane);
      if (lane == 0) out_h[r] = -h;
    } else {   // CB_VJP: w * (up - sum(w * up))
      const double* u = up + r * k;
      const double inner = warp_pairwise(pk, [&](int i) { return dmul(ddiv(ex(i), S), __ldg(u + i)); }, scratch, lane);
      for (int64_t i = lane; i < k; i += 32) out[r * k + i] = dmul(ddiv(ex((int)i), S), dsub(__ldg(u + i), inner));
    }
    __syncwarp();   // the cache is rewritten by the next row
  }
}

// semantic_entropy in two passes over the logits (row max, then one fused
// exp pass): with d = l - max, e = exp(d), S = sum e and T = sum e*d,
//   H = -sum p log p = log S - T / S      (p = e / S, log p = d - log S),
// so no per-element division, log or cached exponentials.  The sums are warp
// reductions (not NumPy's pairwise order): the result differs from the
// reference by a few ulps of log S (inside the 1e-13 relative tolerance).
__global__ void __launch_bounds__(kCbWarps * 32)
cb_entropy_kernel(const double* __restrict__ L, int64_t n, int64_t k, double* __restrict__ out_h, int* __restrict__ bad) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t r = (int64_t)blockIdx.x * kCbWarps + warp; r < n; r += (int64_t)gridDim.x * kCbWarps) {
    const double* l = L + r * k;
    double m = -__longlong_as_double(0x7ff0000000000000ll);
    bool fin = true;
#pragma unroll 8
    for (int64_t i = lane; i < k; i += 32) {
      const double v = __ldg(l + i);
      fin = fin && isfinite(v);
      m = fmax(m, v);
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
    if (!__all_sync(FULL, fin)) {
      if (lane == 0) *(volatile int*)bad = 1;   // idempotent flag (may live in mapped host memory)
      continue;
    }
    double S = 0.0, T = 0.0;
#pragma unroll 4
    for (int64_t i = lane; i < k; i += 32) {
      const double d = dsub(__ldg(l + i), m);
      const double e = exp(d);
      S = dadd(S, e);
      T = fma(e, d, T);
    }
    for (int o = 16; o; o >>= 1) {
      S += __shfl_xor_sync(FULL, S, o);
      T += __shfl_xor_sync(FULL, T, o);
    }
    if (lane == 0) out_h[r] = dsub(log(S), ddiv(T, S));
  }
}

__global__ void __launch_bounds__(kCbWarps * 32)
cb_contrast_kernel(const double* __restrict__ F, int64_t n, int64_t d, const double* __restrict__ Q, int64_t nq,
                   double tau, double eps, double* __restrict__ scores, SumPlan pd) {
  __shared__ double scratch_all[kCbWarps][kMaxLeaves];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* scratch = scratch_all[warp];
  for (int64_t r = (int64_t)blockIdx.x * kCbWarps + warp; r < n; r += (int64_t)gridDim.x * kCbWarps) {
    const double* f = F + r * d;
    const double ss = warp_pairwise(
        pd,
        [&](int i) {
          const double v = __ldg(f + i);
          return dmul(v, v);
        },
        scratch, lane);
    const double den = dadd(sqrt(ss), eps);
    double pos = 0.0, score = 1.0;
    for (int64_t q = 0; q < nq; q++) {
      double acc = 0.0;
      for (int64_t i = lane; i < d; i += 32) acc = fma(ddiv(__ldg(f + i), den), __ldg(Q + q * d + i), acc);
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
      if (q == 0) {
        pos = acc;
      } else {
        const double margin = dmul(tau, dsub(pos, acc));
        score = fmin(score, ddiv(1.0, dadd(1.0, exp(-margin))));
      }
    }
    if (lane == 0) scores[r] = score;
  }
}

__global__ void cb_desc_keys_kernel(const double* __restrict__ v, int64_t n, uint64_t* __restrict__ keys,
                                    uint32_t* __restrict__ idx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double x = v[i];
    if (x == 0.0) x = 0.0;   // -0.0 == +0.0 for the comparison sort
    const uint64_t b = (uint64_t)__double_as_longlong(x);
    const uint64_t asc = (b >> 63) ? ~b : (b | 0x8000000000000000ull);   // ascending order of x
    keys[i] = ~asc;                                                      // descending
    idx[i] = (uint32_t)i;
  }
}

// Top-M of a stable descending order (np.argsort(-v, kind="stable")[:M]):
// histogram of the keys' top 16 bits, the bucket holding the M-th key, an
// order-preserving compaction of every key up to that bucket, and the full
// 64-bit stable radix sort of only those (ties keep ascending index order).
constexpr int kTopBits = 16;
constexpr int kTopBuckets = 1 << kTopBits;

__global__ void topm_hist_kernel(const uint64_t* __restrict__ keys, int64_t n, int32_t* __restrict__ hist) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i - threadIdx.x < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int bkt = i < n ? (int)(keys[i] >> (64 - kTopBits)) : -1;
    const unsigned peers = __match_any_sync(FULL, bkt);
    if (bkt >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(hist + bkt, __popc(peers));
  }
}

// one CTA: the smallest bucket b with (#keys in buckets <= b) >= m; out[0] = b,
// out[1] = #keys in buckets <= b
__global__ void __launch_bounds__(1024) topm_pick_kernel(const int32_t* __restrict__ hist, int64_t m, int32_t* out) {
  __shared__ int32_t wsum[32];
  constexpr int PER = kTopBuckets / 1024;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int32_t c[PER], s = 0;
#pragma unroll
  for (int j = 0; j < PER; j++) {
    c[j] = hist[t * PER + j];
    s += c[j];
  }
  int32_t x = s;
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int32_t w = wsum[lane];
    int32_t wx = w;
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(FULL, wx, o);
      if (lane >= o) wx += y;
    }
    wsum[lane] = wx - w;
  }
  __syncthreads();
  int64_t run = (int64_t)wsum[warp] + x - s;   // keys in buckets before this thread's
#pragma unroll
  for (int j = 0; j < PER; j++) {
    if (run < m && run + c[j] >= m) {   // exactly one thread / bucket satisfies this
      out[0] = t * PER + j;
      out[1] = (int32_t)(run + c[j]);
    }
    run += c[j];
  }
}

__global__ void topm_flag_kernel(const uint64_t* __restrict__ keys, int64_t n, const int32_t* __restrict__ pick,
                                 int32_t* __restrict__ flag) {
  const uint64_t b = (uint64_t)pick[0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (keys[i] >> (64 - kTopBits)) <= b ? 1 : 0;
}

__global__ void topm_compact_kernel(const uint64_t* __restrict__ keys, int64_t n, const int32_t* __restrict__ flag,
                                    const int32_t* __restrict__ pos, uint64_t* __restrict__ ck,
                                    uint32_t* __restrict__ cv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) {
      ck[pos[i]] = keys[i];
      cv[pos[i]] = (uint32_t)i;
    }
}

__global__ void topm_out_kernel(const uint32_t* __restrict__ cv, int64_t m, int64_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = cv[i];
}

unsigned cb_blocks(int64_t rows) {
  int64_t b = (rows + kCbWarps - 1) / kCbWarps;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace

cudaError_t launch_softmax_rows(const double* logits, int64_t n, int64_t k, int mode, const double* up, double* out,
                                double* out_h, const SumPlan& pk, int* bad, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  ProfScope prof("cb_rows", s);
  const bool cache = k <= kCbCacheK;
  const size_t smem = cache ? sizeof(double) * kCbWarps * (size_t)k : 0;
  cudaError_t ea = attr_once(kAttrCodebook, [] {
    cudaError_t r = cudaFuncSetAttribute(cb_rows_kernel<CB_WEIGHTS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kCbWarps * kCbCacheK * 8);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(cb_rows_kernel<CB_VJP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kCbWarps * kCbCacheK * 8);
    return r;
  });
  if (ea != cudaSuccess) return ea;
  const unsigned b = cb_blocks(n);
  const int T = kCbWarps * 32;
  if (mode == CB_ENTROPY) {
    cb_entropy_kernel<<<b, T, 0, s>>>(logits, n, k, out_h, bad);
    count_launches(1);
    return cudaGetLastError();
  }
  switch (mode * 2 + (cache ? 1 : 0)) {
    case CB_WEIGHTS * 2 + 1: cb_rows_kernel<CB_WEIGHTS, true><<<b, T, smem, s>>>(logits, n, k, up, out, out_h, pk, bad); break;
    case CB_WEIGHTS * 2: cb_rows_kernel<CB_WEIGHTS, false><<<b, T, 0, s>>>(logits, n, k, up, out, out_h, pk, bad); break;
    case CB_VJP * 2 + 1: cb_rows_kernel<CB_VJP, true><<<b, T, smem, s>>>(logits, n, k, up, out, out_h, pk, bad); break;
    default: cb_rows_kernel<CB_VJP, false><<<b, T, 0, s>>>(logits, n, k, up, out, out_h, pk, bad);
  }
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_contrast(const double* F, int64_t n, int64_t d, const double* Q, int64_t nq, double tau, double eps,
                            double* scores, const SumPlan& pd, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  ProfScope prof("cb_contrast", s);
  cb_contrast_kernel<<<cb_blocks(n), kCbWarps * 32, 0, s>>>(F, n, d, Q, nq, tau, eps, scores, pd); count_launches(1);
  return cudaGetLastError();
}

// workspace: keys (8n) + flags (4n) + positions (4n) + compact keys / ids
// (12n) + histogram + the radix sort's own workspace for n items
size_t topm_workspace_bytes(int64_t n) {
  const size_t nn = (size_t)(n > 0 ? n : 1);
  return align_up(8 * nn, 256) + align_up(4 * nn, 256) * 2 + align_up(8 * nn, 256) + align_up(4 * nn, 256) +
         align_up(4 * (size_t)kTopBuckets, 256) + 256 + grid_workspace_bytes(n);
}

cudaError_t launch_desc_top_m(const double* v, int64_t n, int64_t m, int64_t* out, void* ws, cudaStream_t s) {
  if (n == 0 || m == 0) return cudaSuccess;
  const size_t nn = (size_t)n;
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t b) { char* r = p; p += align_up(b, 256); return r; };
  uint64_t* keys = reinterpret_cast<uint64_t*>(take(8 * nn));
  int32_t* flag = reinterpret_cast<int32_t*>(take(4 * nn));
  int32_t* pos = reinterpret_cast<int32_t*>(take(4 * nn));
  uint64_t* ck = reinterpret_cast<uint64_t*>(take(8 * nn));
  uint32_t* cv = reinterpret_cast<uint32_t*>(take(4 * nn));
  int32_t* hist = reinterpret_cast<int32_t*>(take(4 * (size_t)kTopBuckets));
  int32_t* misc = reinterpret_cast<int32_t*>(take(256));   // [0] bucket, [1] selected count, [2] scan total
  void* sws = p;
  const size_t sws_bytes = grid_workspace_bytes(n);
  cudaError_t e;
  int64_t b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  cb_desc_keys_kernel<<<(unsigned)b, 256, 0, s>>>(v, n, keys, cv);
  if ((e = cudaMemsetAsync(hist, 0, 4 * (size_t)kTopBuckets, s)) != cudaSuccess) return e;
  topm_hist_kernel<<<(unsigned)b, 256, 0, s>>>(keys, n, hist);
  topm_pick_kernel<<<1, 1024, 0, s>>>(hist, m, misc);
  topm_flag_kernel<<<(unsigned)b, 256, 0, s>>>(keys, n, misc, flag);
  count_launches(4);
  if ((e = exclusive_scan_i32(flag, n, pos, reinterpret_cast<int32_t*>(sws), misc + 2, s)) != cudaSuccess) return e;
  topm_compact_kernel<<<(unsigned)b, 256, 0, s>>>(keys, n, flag, pos, ck, cv);
  count_launches(1);
  int32_t nsel = 0;
  if ((e = cudaMemcpyAsync(&nsel, misc + 1, 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  if ((e = radix_sort_pairs(ck, cv, nsel, 64, sws, sws_bytes, s)) != cudaSuccess) return e;
  topm_out_kernel<<<(unsigned)((m + 255) / 256 < 148 * 16 ? (m + 255) / 256 : 148 * 16), 256, 0, s>>>(cv, m, out);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_desc_keys(const double* v, int64_t n, uint64_t* keys, uint32_t* idx, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  int64_t b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  cb_desc_keys_kernel<<<(unsigned)b, 256, 0, s>>>(v, n, keys, idx); count_launches(1);
  return cudaGetLastError();
}

}  // namespace xgs
