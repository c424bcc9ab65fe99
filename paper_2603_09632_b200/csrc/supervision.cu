// Grid-sampled semantic supervision targets (reference
// supervision.py:21-221), batched over lattice offsets ("target prefetch").
//
//   sup_gather_kernel : for every offset (o_h, o_w) and padded cell (m, n):
//                       u = o_h + m*s, v = o_w + n*s on the stride lattice;
//                       continuous source -> nearest-neighbour feature-map
//                       gather with the reference's fp64 index arithmetic
//                       floor(u*(H_f-1)/max(H-1,1) + 0.5) (supervision.py:
//                       133-147); discrete source -> region-table lookup with
//                       background -1 masked (supervision.py:118-130); cells
//                       beyond (H_s, W_s) are padding with V = 0
//                       (supervision.py:204-221).  Output (n_off, D, Hp, Wp)
//                       fp64, writes coalesced along the cell index.
//   sup_loss_kernel   : masked cosine + L1 per valid cell with the reference's
//                       sequential-over-D reductions, cotangent
//                       lam*(-dcos + sign(p-t)/D)/n (supervision.py:150-184).
#include "launchers.h"

namespace xgs {

namespace {

__device__ __forceinline__ int64_t grid_res(int64_t H, int64_t s, int64_t o) {
  const int64_t q = H - 1 - o;
  const int64_t fl = q >= 0 ? q / s : -((-q + s - 1) / s);   // floored division
  const int64_t r = 1 + fl;
  return r > 0 ? r : 0;
}

__device__ __forceinline__ int64_t nn_index(int64_t u, int64_t Hf, int64_t H) {
  const double den = (double)(H - 1 > 1 ? H - 1 : 1);
  return (int64_t)floor(dadd(ddiv(dmul((double)u, (double)(Hf - 1)), den), 0.5));
}

template <typename T>
__global__ void __launch_bounds__(256)
sup_gather_kernel(const T* __restrict__ P, int64_t Hf, int64_t Wf, const int64_t* __restrict__ S,
                  const double* __restrict__ Phi, int64_t R, int64_t D, int64_t H, int64_t W, int64_t s,
                  const int32_t* __restrict__ offs, int64_t Hp, int64_t Wp, double* __restrict__ G,
                  double* __restrict__ V, int* corrupt) {
  const int64_t cells = Hp * Wp;
  const int64_t o = blockIdx.y;
  const int64_t oh = offs[2 * o], ow = offs[2 * o + 1];
  const int64_t Hs = grid_res(H, s, oh), Ws = grid_res(W, s, ow);
  const int64_t d0 = (int64_t)blockIdx.z * 64, d1 = min(D, d0 + 64);
  double* Go = G + o * D * cells;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = c / Wp, n = c - m * Wp;
    bool valid = m < Hs && n < Ws;
    const T* src = nullptr;
    const double* row = nullptr;
    if (valid) {
      const int64_t u = oh + m * s, v = ow + n * s;
      if (P) {
        src = P + nn_index(u, Hf, H) * Wf + nn_index(v, Wf, W);
      } else {
        const int64_t r = S[u * W + v];
        if (r < -1 || r >= R) {
          atomicOr(corrupt, 1);
          valid = false;
        } else if (r == -1) {
          valid = false;
        } else {
          row = Phi + r * D;
        }
      }
    }
    if (blockIdx.z == 0 && V) V[o * cells + c] = valid ? 1.0 : 0.0;
    for (int64_t d = d0; d < d1; d++) {
      double g = 0.0;
      if (valid) g = src ? (double)src[d * Hf * Wf] : row[d];
      Go[d * cells + c] = g;
    }
  }
}

// Per valid cell: cos / L1 terms and the cotangent (needs the global valid
// count n, produced by the caller's first pass: mode 0 accumulates, mode 1 writes).
__global__ void __launch_bounds__(256)
sup_loss_kernel(const double* __restrict__ pred, const double* __restrict__ G, const double* __restrict__ V,
                int64_t D, int64_t cells, double lam, int mode, double* acc, double* __restrict__ cot) {
  double s_cos = 0.0, s_l1 = 0.0, cnt = 0.0;
  const double n = mode ? acc[2] : 0.0;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += (int64_t)gridDim.x * blockDim.x) {
    const bool valid = V[c] > 0.0;
    if (!valid) {
      if (mode)
        for (int64_t d = 0; d < D; d++) cot[d * cells + c] = 0.0;
      continue;
    }
    double pp = 0.0, tt = 0.0, dot = 0.0, l1 = 0.0;   // sequential over D, as NumPy's axis-0 reduce
    for (int64_t d = 0; d < D; d++) {
      const double p = pred[d * cells + c], t = G[d * cells + c];
      pp = dadd(pp, dmul(p, p));
      tt = dadd(tt, dmul(t, t));
      dot = dadd(dot, dmul(p, t));
      l1 = dadd(l1, fabs(dsub(p, t)));
    }
    const double np_ = __dsqrt_rn(pp), nt = __dsqrt_rn(tt);
    const double a = dadd(np_, 1e-8), b = dadd(nt, 1e-8);
    const bool both = np_ == 0.0 && nt == 0.0;
    const double cosv = both ? 1.0 : ddiv(dot, dmul(a, b));
    if (!mode) {
      s_cos = dadd(s_cos, dsub(1.0, cosv));
      s_l1 = dadd(s_l1, ddiv(l1, (double)D));
      cnt += 1.0;
      continue;
    }
    const double safe = np_ > 0.0 ? np_ : 1.0;
    const double ab = dmul(a, b);
    const double k = ddiv(dot, dmul(dmul(dmul(safe, a), a), b));
    for (int64_t d = 0; d < D; d++) {
      const double p = pred[d * cells + c], t = G[d * cells + c];
      double dc = both ? 0.0 : dsub(ddiv(t, ab), dmul(dmul(k, p), np_ > 0.0 ? 1.0 : 0.0));
      const double sg = p > t ? 1.0 : (p < t ? -1.0 : 0.0);
      cot[d * cells + c] = ddiv(dmul(lam, dadd(-dc, ddiv(sg, (double)D))), n);
    }
  }
  if (!mode) {
    for (int o = 16; o; o >>= 1) {
      s_cos += __shfl_xor_sync(FULL, s_cos, o);
      s_l1 += __shfl_xor_sync(FULL, s_l1, o);
      cnt += __shfl_xor_sync(FULL, cnt, o);
    }
    if ((threadIdx.x & 31) == 0 && cnt > 0) {
      atomicAdd(acc, s_cos);
      atomicAdd(acc + 1, s_l1);
      atomicAdd(acc + 2, cnt);
    }
  }
}

}  // namespace

cudaError_t launch_sup_gather(const void* P, int p_dtype, int64_t Hf, int64_t Wf, const int64_t* S, const double* Phi,
                              int64_t R, int64_t D, int64_t H, int64_t W, int64_t s, const int32_t* offs,
                              int64_t n_off, int64_t Hp, int64_t Wp, double* G, double* V, int* corrupt,
                              cudaStream_t st) {
  const int64_t cells = Hp * Wp;
  if (cells == 0 || n_off == 0 || D == 0) return cudaSuccess;
  int64_t bx = (cells + 255) / 256;
  if (bx > 4096) bx = 4096;
  dim3 grid((unsigned)bx, (unsigned)n_off, (unsigned)((D + 63) / 64));
  ProfScope prof("sup_gather", st);
  if (!P || p_dtype == F64)
    sup_gather_kernel<double><<<grid, 256, 0, st>>>((const double*)P, Hf, Wf, S, Phi, R, D, H, W, s, offs, Hp, Wp, G, V, corrupt);
  else
    sup_gather_kernel<float><<<grid, 256, 0, st>>>((const float*)P, Hf, Wf, S, Phi, R, D, H, W, s, offs, Hp, Wp, G, V, corrupt);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_sup_loss(const double* pred, const double* G, const double* V, int64_t D, int64_t cells, double lam,
                            double* acc, double* cot, cudaStream_t st) {
  if (cells == 0) return cudaSuccess;
  int64_t b = (cells + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  cudaError_t e = cudaMemsetAsync(acc, 0, 3 * sizeof(double), st);
  if (e != cudaSuccess) return e;
  sup_loss_kernel<<<(unsigned)b, 256, 0, st>>>(pred, G, V, D, cells, lam, 0, acc, cot); count_launches(1);
  sup_loss_kernel<<<(unsigned)b, 256, 0, st>>>(pred, G, V, D, cells, lam, 1, acc, cot); count_launches(1);
  return cudaGetLastError();
}

}  // namespace xgs
