// Exact fp64 VQ kernels (bit-identical to the reference's NumPy evaluation).
//
//   exact_rows_kernel : one CTA per row, 8 warps over the K codewords, each
//                       distance a warp-cooperative NumPy pairwise sum
//                       (vq.py:69-73); argmin with lowest-index ties
//                       (vq.py:84-87); optional confidence softmax
//                       (vq.py:112-124) with the row sum over K in the same
//                       pairwise order.  Used for squared_distances /
//                       confidence_scores, for the gamma > 1/K mask, and as the
//                       fallback for rows whose candidate list overflowed.
//   rerank_kernel     : one warp per queued row, exact distances of the 2..8
//                       screening candidates only.
#include "launchers.h"

namespace xgs {

namespace {

constexpr int kExactWarps = 8;

template <typename X>
__global__ void __launch_bounds__(kExactWarps * 32)
exact_rows_kernel(ExactArgs a, SumPlan pd, SumPlan pk) {
  extern __shared__ double smem[];
  double* scratch_all = smem;                                 // kExactWarps * 128
  double* dist = smem + kExactWarps * kMaxLeaves;            // K (if softmax needed)
  __shared__ double red_v[kExactWarps];
  __shared__ int red_k[kExactWarps];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* scratch = scratch_all + warp * kMaxLeaves;
  const bool need_soft = (a.mode & (EX_CONF_MASK | EX_WRITE_PROB)) != 0;
  const int64_t nrows = a.nrows_dev ? (int64_t)*a.nrows_dev : a.n;
  const X* xb = static_cast<const X*>(a.x);

  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int64_t row = a.rows ? (int64_t)a.rows[r] : r;
    const X* xr = xb + row * a.ldx;
    double bv = 0.0;
    int bk = -1;
    for (int k = warp; k < a.k; k += kExactWarps) {
      const double dk = warp_sqdist(xr, a.E + (int64_t)k * a.d, pd, scratch, lane);
      if (lane == 0) {
        if (bk < 0) { bv = dk; bk = k; } else argmin_merge(bv, bk, dk, k);
        if (a.mode & EX_WRITE_DIST) a.out_dist[row * a.k + k] = dk;
        if (need_soft) dist[k] = dk;
      }
    }
    if (lane == 0) { red_v[warp] = bv; red_k[warp] = bk; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = red_v[0];
      int kk = red_k[0];
      for (int w = 1; w < kExactWarps; w++)
        if (red_k[w] >= 0) {
          if (kk < 0) { v = red_v[w]; kk = red_k[w]; } else argmin_merge(v, kk, red_v[w], red_k[w]);
        }
      red_v[0] = v;
      red_k[0] = kk;
      if (a.mode & EX_WRITE_CODE) a.codes[row] = kk;
    }
    __syncthreads();
    if (need_soft) {
      // vq.py:114-118: d = sqrt(sq); logits = -d/tau; logits -= max; e = exp
      const double lmax = ddiv(-__dsqrt_rn(red_v[0]), a.tau);
      if (warp == 0) {
        const double S = warp_pairwise(
            pk,
            [&](int i) { return exp(dsub(ddiv(-__dsqrt_rn(dist[i]), a.tau), lmax)); },
            scratch, lane);
        if (lane == 0) {
          if (a.mode & EX_CONF_MASK) {
            // p.max = fl(1/S) (vq.py:118-124).  CUDA's exp and the host
            // libm's may differ in the last ulp, moving S by up to ~K ulps:
            // rows whose 1/S lies within 1e-12 relative of gamma are marked 2
            // and decided on the host with the reference's own NumPy ops.
            const double inv = ddiv(1.0, S);
            a.mask[row] = fabs(inv - a.gamma) <= 1e-12 * a.gamma ? 2 : (inv >= a.gamma ? 1 : 0);
          }
          red_v[1] = S;
        }
      }
      __syncthreads();
      if (a.mode & EX_WRITE_PROB) {
        const double S = red_v[1];
        for (int k = threadIdx.x; k < a.k; k += blockDim.x)
          a.out_prob[row * a.k + k] = ddiv(exp(dsub(ddiv(-__dsqrt_rn(dist[k]), a.tau), lmax)), S);
      }
      __syncthreads();
    }
  }
}

template <typename X>
__global__ void __launch_bounds__(256)
rerank_kernel(const X* __restrict__ x, int64_t d, int64_t ldx, const double* __restrict__ E,
              const RerankEntry* __restrict__ q, const int32_t* __restrict__ qcount,
              int64_t* __restrict__ codes, SumPlan pd) {
  __shared__ double scratch_all[8][kMaxLeaves];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* scratch = scratch_all[warp];
  const int n = *qcount;
  for (int i = blockIdx.x * 8 + warp; i < n; i += gridDim.x * 8) {
    const RerankEntry e = q[i];
    const X* xr = x + (int64_t)e.row * ldx;
    double bv = 0.0;
    int bk = -1;
    for (int c = 0; c < e.cnt; c++) {
      const int k = e.cand[c];
      const double dk = warp_sqdist(xr, E + (int64_t)k * d, pd, scratch, lane);
      if (bk < 0) { bv = dk; bk = k; } else argmin_merge(bv, bk, dk, k);
    }
    if (lane == 0) codes[e.row] = bk;
  }
}

template <typename X>
cudaError_t exact_rows_t(const ExactArgs& a, const SumPlan& pd, const SumPlan& pk, cudaStream_t s) {
  const bool need_soft = (a.mode & (EX_CONF_MASK | EX_WRITE_PROB)) != 0;
  size_t smem = sizeof(double) * (kExactWarps * kMaxLeaves + (need_soft ? a.k : 0));
  auto kern = exact_rows_kernel<X>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int64_t grid = a.nrows_dev ? 148 * 8 : a.n;
  if (grid > 148 * 64) grid = 148 * 64;
  if (grid < 1) grid = 1;
  kern<<<(unsigned)grid, kExactWarps * 32, smem, s>>>(a, pd, pk); count_launches(1);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_exact_rows(const ExactArgs& a, const SumPlan& pd, const SumPlan& pk, cudaStream_t s) {
  if (a.n == 0 && !a.nrows_dev) return cudaSuccess;
  switch (a.dtype) {
    case F32: return exact_rows_t<float>(a, pd, pk, s);
    case F64: return exact_rows_t<double>(a, pd, pk, s);
    default: return exact_rows_t<uint16_t>(a, pd, pk, s);
  }
}

cudaError_t launch_rerank(const void* x, int dtype, int64_t d, int64_t ldx, const double* E,
                          const RerankEntry* q, const int32_t* qcount, int64_t qcap,
                          int64_t* codes, const SumPlan& pd, cudaStream_t s) {
  if (qcap <= 0) return cudaSuccess;
  int64_t blocks = (qcap + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  switch (dtype) {
    case F32:
      rerank_kernel<float><<<(unsigned)blocks, 256, 0, s>>>((const float*)x, d, ldx, E, q, qcount, codes, pd); count_launches(1);
      break;
    case F64:
      rerank_kernel<double><<<(unsigned)blocks, 256, 0, s>>>((const double*)x, d, ldx, E, q, qcount, codes, pd); count_launches(1);
      break;
    default:
      rerank_kernel<uint16_t><<<(unsigned)blocks, 256, 0, s>>>((const uint16_t*)x, d, ldx, E, q, qcount, codes, pd); count_launches(1);
  }
  return cudaGetLastError();
}

}  // namespace xgs
