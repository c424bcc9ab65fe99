// Lattice-only semantic rasterizer + VJP (reference
// rasterizer.py:89-335, the paper's "custom GPU kernel").
//
// build_blend_pairs (rasterizer.py:89-191) on the B200, in fp64 like the
// reference, as a tile-binned pipeline:
//   R1 raster_prep_kernel   : per Gaussian camera transform, near/far cull,
//                             projected centre, 3D covariance (quat, scale),
//                             Jacobian projection, 2x2 eigenvalue floor
//                             (core.py:402-448), inverse covariance and the
//                             3-sigma radius; depth sort key;
//   R2 in-house radix sort of (depth, index) -> ranks (ties to the lower index,
//                             the reference's stable argsort of z);
//   R3 raster_bin_kernel    : lattice bounding box of every splat -> the
//                             16x16-pixel lattice tiles it touches; (tile,
//                             rank) keys radix-sorted -> per-tile lists in
//                             depth order;
//   R4 raster_tile_kernel   : one CTA per tile, one thread per lattice pixel,
//                             the tile's splats staged through shared memory
//                             in depth order; pass COUNT counts the culled
//                             pairs (quad <= cutoff^2) per pixel, pass EMIT
//                             writes them pixel-segmented in depth order (the
//                             reference's pair order) with alpha' =
//                             opacity exp(-quad/2), the running log
//                             transmittance sum(max(log1p(-alpha'), log 1e-30)),
//                             T_before, alive = T_before >= threshold and the
//                             blend weight alpha' T_before (0 once dead);
//   R5 raster_accum_kernel  : _accumulate_channels / render (bincount order:
//                             sequential fp64 sums per pixel in pair order);
//   R6 raster_argmax_kernel : render_argmax_ids (largest weight, the last of
//                             equal weights as in the stable lexsort);
//   R7 raster_vjp_kernel    : feature_gradients' np.add.at (pairs stably sorted
//                             by Gaussian, one sequential fp64 chain per
//                             (Gaussian, channel) in pair order; Gaussians with
//                             more than 512 pairs: 32 in-order segment chains
//                             added in order, raster_vjp_long_kernel).
// The reference's transmittance comes from one global cumsum over all pairs;
// the per-pixel running sum here is the same quantity without the global
// rounding drift, so T and the weights agree to ~1e-12 relative (exp, log1p,
// atan2, cos, sin are libm vs CUDA ulps).
#include <cstring>

#include "launchers.h"

namespace xgs {

namespace {

constexpr int RT = 8;                  // lattice tile edge (pixels): one CTA of 64 threads per tile
constexpr int RT_THREADS = RT * RT;
constexpr double LOG_T_MIN = -69.07755278982137;   // log(1e-30), rasterizer.py:27

struct Prep {
  double* uc;
  double* vc;
  double* ia;
  double* ib;
  double* ic;
  double* rad;
  double* z;
  double* op;
};

__device__ __forceinline__ uint64_t z_key(double z) { return (uint64_t)__double_as_longlong(z); }   // z > 0

__global__ void raster_prep_kernel(RasterIn in, Prep p, uint64_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                   unsigned long long* nvis) {
  unsigned cnt = 0;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < in.n; g += (int64_t)gridDim.x * blockDim.x) {
    const double* m = in.mu + g * 3;
    double cam[3];
#pragma unroll
    for (int i = 0; i < 3; i++)   // pts @ R.T + t
      cam[i] = dadd(dadd(dadd(dmul(m[0], in.R[3 * i]), dmul(m[1], in.R[3 * i + 1])), dmul(m[2], in.R[3 * i + 2])),
                    in.t[i]);
    const double z = cam[2];
    const bool vis = (z > in.near_z) && (z < in.far_z);
    keys[g] = vis ? z_key(z) : ~0ull;
    vals[g] = (uint32_t)g;
    if (!vis) continue;
    cnt++;
    p.uc[g] = dadd(ddiv(dmul(in.fx, cam[0]), z), in.cx);
    p.vc[g] = dadd(ddiv(dmul(in.fy, cam[1]), z), in.cy);
    // Sigma = R diag(s^2) R^T (quat_to_rot, core.py:40-55 / :402-405)
    const double* q = in.quat + g * 4;
    const double w = q[0], x = q[1], y = q[2], zq = q[3];
    double Rq[9];
    Rq[0] = dsub(1.0, dmul(2.0, dadd(dmul(y, y), dmul(zq, zq))));
    Rq[1] = dmul(2.0, dsub(dmul(x, y), dmul(w, zq)));
    Rq[2] = dmul(2.0, dadd(dmul(x, zq), dmul(w, y)));
    Rq[3] = dmul(2.0, dadd(dmul(x, y), dmul(w, zq)));
    Rq[4] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(zq, zq))));
    Rq[5] = dmul(2.0, dsub(dmul(y, zq), dmul(w, x)));
    Rq[6] = dmul(2.0, dsub(dmul(x, zq), dmul(w, y)));
    Rq[7] = dmul(2.0, dadd(dmul(y, zq), dmul(w, x)));
    Rq[8] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(y, y))));
    const double* sc = in.scale + g * 3;
    const double s2[3] = {dmul(sc[0], sc[0]), dmul(sc[1], sc[1]), dmul(sc[2], sc[2])};
    double S[9];
#pragma unroll
    for (int i = 0; i < 3; i++)
#pragma unroll
      for (int k = 0; k < 3; k++) {
        double a = 0.0;
#pragma unroll
        for (int j = 0; j < 3; j++) a = dadd(a, dmul(dmul(Rq[3 * i + j], s2[j]), Rq[3 * k + j]));
        S[3 * i + k] = a;
      }
    // J (2x3) and JW = J @ W (core.py:437-444)
    const double z2 = dmul(z, z);
    const double J00 = ddiv(in.fx, z), J02 = -ddiv(dmul(in.fx, cam[0]), z2);
    const double J11 = ddiv(in.fy, z), J12 = -ddiv(dmul(in.fy, cam[1]), z2);
    double JW[6];
#pragma unroll
    for (int k = 0; k < 3; k++) {
      JW[k] = dadd(dmul(J00, in.R[k]), dmul(J02, in.R[6 + k]));
      JW[3 + k] = dadd(dmul(J11, in.R[3 + k]), dmul(J12, in.R[6 + k]));
    }
    double C[4];
#pragma unroll
    for (int i = 0; i < 2; i++)
#pragma unroll
      for (int l = 0; l < 2; l++) {
        double a = 0.0;
#pragma unroll
        for (int j = 0; j < 3; j++) {
          double t = 0.0;
#pragma unroll
          for (int k = 0; k < 3; k++) t = dadd(t, dmul(S[3 * j + k], JW[3 * l + k]));
          a = dadd(a, dmul(JW[3 * i + j], t));
        }
        C[2 * i + l] = a;
      }
    const double c01 = dmul(0.5, dadd(C[1], C[2]));
    const double a0 = dmul(0.5, dadd(C[0], C[0])), c0 = dmul(0.5, dadd(C[3], C[3]));
    // _floor_eigenvalues_2x2 (core.py:408-422)
    const double half_tr = dmul(0.5, dadd(a0, c0));
    const double hd = dmul(0.5, dsub(a0, c0));
    const double disc = sqrt(fmax(dadd(dmul(hd, hd), dmul(c01, c01)), 0.0));
    const double l1 = fmax(dadd(half_tr, disc), in.eig_floor), l2 = fmax(dsub(half_tr, disc), in.eig_floor);
    const double th = dmul(0.5, atan2(dmul(2.0, c01), dsub(a0, c0)));
    const double ct = cos(th), st = sin(th);
    const double A = dadd(dmul(dmul(l1, ct), ct), dmul(dmul(l2, st), st));
    const double Cc = dadd(dmul(dmul(l1, st), st), dmul(dmul(l2, ct), ct));
    const double B = dmul(dmul(dsub(l1, l2), ct), st);
    // inverse + radius (rasterizer.py:110-115)
    const double det = dsub(dmul(A, Cc), dmul(B, B));
    p.ia[g] = ddiv(Cc, det);
    p.ib[g] = ddiv(-B, det);
    p.ic[g] = ddiv(A, det);
    const double hd2 = dmul(0.5, dsub(A, Cc));
    const double lam = dadd(dmul(0.5, dadd(A, Cc)), sqrt(fmax(dadd(dmul(hd2, hd2), dmul(B, B)), 0.0)));
    p.rad[g] = dmul(in.cutoff, sqrt(lam));
    p.z[g] = z;
    p.op[g] = in.opacity[g];
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(nvis, (unsigned long long)cnt);
}

struct Ranked {   // splat parameters in depth order (rank r)
  double* uc;
  double* vc;
  double* ia;
  double* ib;
  double* ic;
  double* z;
  double* op;
  int32_t* gid;
  int32_t* box;   // 4 per rank: tile row lo/hi, tile col lo/hi (lo > hi: none)
};

// lattice index range of a splat (rasterizer.py:136-141, with a 1e-9 px guard:
// the exact quad test culls, the box only has to contain the ellipse)
__device__ __forceinline__ void lattice_range(double c, double r, const RasterIn& in, bool rows, int64_t* lo,
                                              int64_t* hi) {
  const int64_t n = rows ? in.n_rows : in.n_cols;
  const double o = (double)(rows ? in.row0 : in.col0), s = (double)(rows ? in.row_step : in.col_step);
  const double a = ceil((c - r - 1e-9 - o) / s), b = floor((c + r + 1e-9 - o) / s);
  *lo = a < 0.0 ? 0 : (a > (double)n ? n : (int64_t)a);
  *hi = b >= (double)(n - 1) ? n - 1 : (b < -1.0 ? -1 : (int64_t)b);
}

__global__ void raster_rank_kernel(RasterIn in, Prep p, const uint32_t* __restrict__ order, int64_t nvis, Ranked rk,
                                   int32_t* __restrict__ tcount, int64_t tiles_c) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nvis; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = order[r];
    const double uc = p.uc[g], vc = p.vc[g], rad = p.rad[g];
    rk.uc[r] = uc;
    rk.vc[r] = vc;
    rk.ia[r] = p.ia[g];
    rk.ib[r] = p.ib[g];
    rk.ic[r] = p.ic[g];
    rk.z[r] = p.z[g];
    rk.op[r] = p.op[g];
    rk.gid[r] = (int32_t)g;
    int64_t m0, m1, n0, n1;
    lattice_range(uc, rad, in, true, &m0, &m1);
    lattice_range(vc, rad, in, false, &n0, &n1);
    int32_t* b = rk.box + r * 4;
    if (m1 < m0 || n1 < n0) {
      b[0] = 1;
      b[1] = 0;
      b[2] = 1;
      b[3] = 0;
      tcount[r] = 0;
    } else {
      b[0] = (int32_t)(m0 / RT);
      b[1] = (int32_t)(m1 / RT);
      b[2] = (int32_t)(n0 / RT);
      b[3] = (int32_t)(n1 / RT);
      tcount[r] = (b[1] - b[0] + 1) * (b[3] - b[2] + 1);
    }
    (void)tiles_c;
  }
}

__global__ void raster_bin_kernel(const Ranked rk, int64_t nvis, const int32_t* __restrict__ toff, int64_t tiles_c,
                                  uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nvis; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t* b = rk.box + r * 4;
    int64_t o = toff[r];
    for (int ty = b[0]; ty <= b[1]; ty++)
      for (int tx = b[2]; tx <= b[3]; tx++) {
        keys[o] = ((uint64_t)(ty * tiles_c + tx) << 32) | (uint64_t)r;
        vals[o] = (uint32_t)r;
        o++;
      }
  }
}

__global__ void raster_tile_ranges_kernel(const uint64_t* __restrict__ keys, int64_t n, int32_t* __restrict__ tstart,
                                          int64_t ntiles) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i < n ? (int64_t)(keys[i] >> 32) : ntiles;
    const int64_t tp = i > 0 ? (int64_t)(keys[i - 1] >> 32) : -1;
    for (int64_t u = tp + 1; u <= t; u++) tstart[u] = (int32_t)i;
  }
}

struct PairsOut {
  int32_t* gauss;
  int32_t* pixel;
  double* weight;
  double* alpha;
  double* tb;
  uint8_t* alive;
  double* depth;
};

// EMIT == false: count pairs per lattice pixel; true: write them.
// ALL: every culled pair, dead ones included (build_blend_pairs' arrays);
// otherwise only the alive prefix of each pixel (T_before >= threshold; T is
// non-increasing in depth order, so the first dead pair ends the pixel), which
// is all the renders, argmax and VJP consume (dead pairs have weight 0), and
// the tile stops once all of its pixels are dead.
template <bool EMIT, bool ALL>
__global__ void __launch_bounds__(RT_THREADS)
raster_tile_kernel(RasterIn in, Ranked rk, const uint32_t* __restrict__ tlist, const int32_t* __restrict__ tstart,
                   int64_t tiles_c, int32_t* __restrict__ pcount, const int32_t* __restrict__ poff, PairsOut po,
                   unsigned long long* blend_steps) {
  __shared__ double s_uc[RT_THREADS], s_vc[RT_THREADS], s_ia[RT_THREADS], s_ib[RT_THREADS], s_ic[RT_THREADS];
  __shared__ double s_op[RT_THREADS], s_z[RT_THREADS];
  __shared__ int32_t s_gid[RT_THREADS];
  const int64_t tile = blockIdx.x;
  const int64_t ty = tile / tiles_c, tx = tile - ty * tiles_c;
  const int64_t mi = ty * RT + threadIdx.x / RT, ni = tx * RT + threadIdx.x % RT;
  const bool live = mi < in.n_rows && ni < in.n_cols;
  const double row = (double)(in.row0 + mi * in.row_step), col = (double)(in.col0 + ni * in.col_step);
  const int64_t pix = mi * in.n_cols + ni;
  const double cut2 = dmul(in.cutoff, in.cutoff);
  const int32_t b0 = tstart[tile], b1 = tstart[tile + 1];
  constexpr bool NEED_T = EMIT || !ALL;
  int32_t cnt = 0;
  int64_t o = (EMIT && live) ? poff[pix] : 0;
  double logT = 0.0;
  unsigned steps = 0;
  bool done = !live;
  for (int32_t base = b0; base < b1; base += RT_THREADS) {
    const int32_t nb = min(RT_THREADS, b1 - base);
    if (!ALL) {
      if (__syncthreads_and(done)) break;   // every pixel of the tile is past termination
    } else {
      __syncthreads();
    }
    if ((int)threadIdx.x < nb) {
      const uint32_t r = tlist[base + threadIdx.x];
      s_uc[threadIdx.x] = rk.uc[r];
      s_vc[threadIdx.x] = rk.vc[r];
      s_ia[threadIdx.x] = rk.ia[r];
      s_ib[threadIdx.x] = rk.ib[r];
      s_ic[threadIdx.x] = rk.ic[r];
      if (NEED_T) s_op[threadIdx.x] = rk.op[r];
      if (EMIT) {
        s_z[threadIdx.x] = rk.z[r];
        s_gid[threadIdx.x] = rk.gid[r];
      }
    }
    __syncthreads();
    if (done) continue;
    for (int j = 0; j < nb; j++) {
      const double du = dsub(row, s_uc[j]), dv = dsub(col, s_vc[j]);
      // inv_a du du + 2 inv_b du dv + inv_c dv dv, left to right (rasterizer.py:147)
      const double quad = dadd(dadd(dmul(dmul(s_ia[j], du), du), dmul(dmul(dmul(2.0, s_ib[j]), du), dv)),
                               dmul(dmul(s_ic[j], dv), dv));
      if (!(quad <= cut2)) continue;
      if (!NEED_T) {
        cnt++;
        continue;
      }
      const double a = dmul(s_op[j], exp(dmul(-0.5, quad)));
      const double T = exp(logT);
      const bool alive = T >= in.term;
      if (!ALL && !alive) {
        done = true;
        break;
      }
      if (EMIT) {
        po.gauss[o] = s_gid[j];
        po.pixel[o] = (int32_t)pix;
        po.weight[o] = alive ? dmul(a, T) : 0.0;
        po.alpha[o] = a;
        po.tb[o] = T;
        po.alive[o] = alive ? 1 : 0;
        po.depth[o] = s_z[j];
        o++;
      } else {
        cnt++;
      }
      steps += alive ? 1u : 0u;
      logT = dadd(logT, fmax(log1p(-a), LOG_T_MIN));
    }
  }
  if (!EMIT && live) pcount[pix] = cnt;
  if (EMIT) {
    for (int k = 16; k; k >>= 1) steps += __shfl_xor_sync(FULL, steps, k);
    if ((threadIdx.x & 31) == 0 && steps) atomicAdd(blend_steps, (unsigned long long)steps);
  }
}

// warp per lattice pixel, lanes over channels; sums in pair order (np.bincount)
__global__ void raster_accum_kernel(const int32_t* __restrict__ poff, int64_t npix, const int32_t* __restrict__ gauss,
                                    const double* __restrict__ weight, const double* __restrict__ depth,
                                    const double* __restrict__ payload, int64_t C, double* __restrict__ out,
                                    double* __restrict__ alpha_out, double* __restrict__ depth_out) {
  const int lane = threadIdx.x & 31;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < npix;
       p += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t a = poff[p], b = poff[p + 1];
    for (int64_t c0 = 0; c0 < C; c0 += 32) {
      const int64_t c = c0 + lane;
      double acc = 0.0;
      if (c < C)
        for (int32_t i = a; i < b; i++) acc = dadd(acc, dmul(weight[i], payload[(int64_t)gauss[i] * C + c]));
      if (c < C) out[c * npix + p] = acc;
    }
    if (lane == 0 && (alpha_out || depth_out)) {
      double sa = 0.0, sd = 0.0;
      for (int32_t i = a; i < b; i++) {
        sa = dadd(sa, weight[i]);
        sd = dadd(sd, dmul(weight[i], depth[i]));
      }
      if (alpha_out) alpha_out[p] = sa;
      if (depth_out) depth_out[p] = sd;
    }
  }
}

__global__ void raster_argmax_kernel(const int32_t* __restrict__ poff, int64_t npix, const int32_t* __restrict__ gauss,
                                     const double* __restrict__ weight, int64_t* __restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = poff[p], b = poff[p + 1];
    int32_t best = -1;
    double bw = 0.0;
    for (int32_t i = a; i < b; i++)
      if (best < 0 || weight[i] >= bw) {   // stable lexsort: the last of equal weights ends the segment
        best = i;
        bw = weight[i];
      }
    out[p] = (best >= 0 && bw > 0.0) ? (int64_t)gauss[best] : -1;
  }
}

__global__ void raster_gauss_keys_kernel(const int32_t* __restrict__ gauss, int64_t np, uint64_t* __restrict__ keys,
                                         uint32_t* __restrict__ vals) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = (uint64_t)(uint32_t)gauss[i];
    vals[i] = (uint32_t)i;
  }
}

// (D, P) -> (P, D) so the per-pair upstream rows are contiguous
__global__ void raster_transpose_kernel(const double* __restrict__ in, int64_t D, int64_t P, double* __restrict__ out) {
  __shared__ double t[32][33];
  for (int64_t bp = (int64_t)blockIdx.x * 32; bp < P; bp += (int64_t)gridDim.x * 32)
    for (int64_t bd = (int64_t)blockIdx.y * 32; bd < D; bd += (int64_t)gridDim.y * 32) {
      for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t d = bd + k, p = bp + threadIdx.x;
        t[k][threadIdx.x] = (d < D && p < P) ? in[d * P + p] : 0.0;
      }
      __syncthreads();
      for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t p = bp + k, d = bd + threadIdx.x;
        if (p < P && d < D) out[p * D + d] = t[threadIdx.x][k];
      }
      __syncthreads();
    }
}

// feature_grads[g, d] = sum over g's pairs (pair order) of weight * up[pixel, d].
// One warp per (Gaussian, 32-channel chunk): each lane owns one channel's
// sequential fp64 chain (np.add.at order), so a splat covering many pixels is
// spread over D/32 warps instead of serialising one; pair metadata is fetched
// 32 pairs at a time and broadcast by shuffles.
// One lane's chain over pairs [a, b) of a Gaussian (channel dd of upT).
__device__ __forceinline__ double vjp_chain(const uint32_t* __restrict__ pidx, const int32_t* __restrict__ pixel,
                                            const double* __restrict__ weight, const double* __restrict__ upT,
                                            int64_t D, int64_t dd, int32_t a, int32_t b, int lane) {
  double acc = 0.0;
  for (int32_t i0 = a; i0 < b; i0 += 32) {
    int32_t mp = 0;
    double mw = 0.0;
    if (i0 + lane < b) {
      const uint32_t q = pidx[i0 + lane];
      mp = pixel[q];
      mw = weight[q];
    }
    const int cnt = min(32, b - i0);
#pragma unroll 8
    for (int j = 0; j < cnt; j++) {
      const int64_t px = __shfl_sync(FULL, mp, j);
      const double w = __shfl_sync(FULL, mw, j);
      acc = dadd(acc, dmul(w, __ldg(upT + px * D + dd)));
    }
  }
  return acc;
}

// Gaussians with more than kVjpLong pairs (large splats near the camera: up to
// ~20K lattice pixels) go to raster_vjp_long_kernel: one sequential chain per
// lane there set the whole kernel's time (4.1 ms at the bench's 2^18
// Gaussians).  A classify pass lists the short and the long Gaussians with
// pairs (list order is irrelevant: every item is computed on its own), so no
// warp walks the Gaussians without pairs (a (Gaussian, chunk) item each had
// cost 0.6 ms of dependent range loads).
constexpr int32_t kVjpLong = 512;
__global__ void raster_vjp_classify_kernel(const int32_t* __restrict__ gstart, int64_t n,
                                           int32_t* __restrict__ short_list, int32_t* __restrict__ short_count,
                                           int32_t* __restrict__ long_list, int32_t* __restrict__ long_count) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
    const int32_t len = gstart[g + 1] - gstart[g];
    if (len > kVjpLong) long_list[atomicAdd(long_count, 1)] = (int32_t)g;
    else if (len > 0) short_list[atomicAdd(short_count, 1)] = (int32_t)g;
  }
}

__global__ void __launch_bounds__(256)
raster_vjp_kernel(const uint32_t* __restrict__ pidx, const int32_t* __restrict__ pixel,
                  const double* __restrict__ weight, const double* __restrict__ upT, int64_t D,
                  const int32_t* __restrict__ gstart, const int32_t* __restrict__ short_list,
                  const int32_t* __restrict__ short_count, double* __restrict__ fg) {
  const int lane = threadIdx.x & 31;
  const int64_t chunks = (D + 31) / 32;
  const int64_t items = (int64_t)*short_count * chunks;
  for (int64_t wi = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < items;
       wi += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t g = short_list[wi / chunks], d = (wi % chunks) * 32 + lane;
    const int32_t a = gstart[g], b = gstart[g + 1];
    double acc = 0.0;
    for (int32_t i0 = a; i0 < b; i0 += 32) {
      int32_t mp = 0;
      double mw = 0.0;
      if (i0 + lane < b) {
        const uint32_t q = pidx[i0 + lane];
        mp = pixel[q];
        mw = weight[q];
      }
      const int cnt = min(32, b - i0);
      const int64_t dd = d < D ? d : D - 1;   // every lane shuffles; tail lanes read a valid channel and drop it
#pragma unroll 8
      for (int j = 0; j < cnt; j++) {
        const int64_t px = __shfl_sync(FULL, mp, j);
        const double w = __shfl_sync(FULL, mw, j);
        acc = dadd(acc, dmul(w, __ldg(upT + px * D + dd)));
      }
    }
    if (d < D && b > a) fg[g * D + d] = acc;
  }
}

// A long Gaussian's (chunk of 32 channels) per block: the 32 warps sum 32
// contiguous segments of its pairs, then warp 0 adds the 32 partials in segment
// order -- deterministic; the reassociation differs from one sequential chain
// by ~1e-16 relative (the pair weights themselves carry ~1e-12).
constexpr int kVjpSegs = 32;
__global__ void __launch_bounds__(32 * kVjpSegs)
raster_vjp_long_kernel(const uint32_t* __restrict__ pidx, const int32_t* __restrict__ pixel,
                       const double* __restrict__ weight, const double* __restrict__ upT, int64_t D,
                       const int32_t* __restrict__ gstart, const int32_t* __restrict__ long_list,
                       const int32_t* __restrict__ long_count, double* __restrict__ fg) {
  __shared__ double part[kVjpSegs][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t chunks = (D + 31) / 32;
  const int64_t items = (int64_t)*long_count * chunks;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t g = long_list[it / chunks], d = (it % chunks) * 32 + lane;
    const int64_t dd = d < D ? d : D - 1;
    const int32_t a = gstart[g], b = gstart[g + 1];
    const int32_t len = b - a;
    const int32_t s0 = a + (int32_t)((int64_t)len * warp / kVjpSegs),
                  s1 = a + (int32_t)((int64_t)len * (warp + 1) / kVjpSegs);
    part[warp][lane] = vjp_chain(pidx, pixel, weight, upT, D, dd, s0, s1, lane);
    __syncthreads();
    if (warp == 0 && d < D) {
      double acc = part[0][lane];
#pragma unroll
      for (int w = 1; w < kVjpSegs; w++) acc = dadd(acc, part[w][lane]);
      fg[g * D + d] = acc;
    }
    __syncthreads();
  }
}

__global__ void raster_gauss_ranges_kernel(const uint64_t* __restrict__ keys, int64_t np, int32_t* __restrict__ gstart,
                                           int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= np; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i < np ? (int64_t)keys[i] : n;
    const int64_t tp = i > 0 ? (int64_t)keys[i - 1] : -1;
    for (int64_t u = tp + 1; u <= t; u++) gstart[u] = (int32_t)i;
  }
}

__global__ void i32_to_i64_kernel(const int32_t* __restrict__ a, int64_t n, int64_t* __restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

unsigned blocks_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

int bits_for_count(int64_t v) {
  int b = 1;
  while ((1ll << b) <= v) b++;
  return b;
}

template <typename T>
cudaError_t dalloc(T** p, int64_t n, cudaStream_t s) {
  return cudaMallocAsync(reinterpret_cast<void**>(p), sizeof(T) * (size_t)(n > 0 ? n : 1), s);
}

}  // namespace

struct RasterState {
  int64_t n = 0, npix = 0, np = 0, nvis = 0;
  unsigned long long blend_steps = 0;
  int32_t* poff = nullptr;     // npix + 1
  PairsOut po{};
  cudaStream_t s = nullptr;
};

void raster_free(RasterState* st) {
  if (!st) return;
  cudaStream_t s = st->s;
  cudaFreeAsync(st->poff, s);
  cudaFreeAsync(st->po.gauss, s);
  cudaFreeAsync(st->po.pixel, s);
  cudaFreeAsync(st->po.weight, s);
  cudaFreeAsync(st->po.alpha, s);
  cudaFreeAsync(st->po.tb, s);
  cudaFreeAsync(st->po.alive, s);
  cudaFreeAsync(st->po.depth, s);
  delete st;
}

// Keep freed stream-ordered allocations in the device pool across the
// build's synchronisations (the default release threshold of 0 hands them back
// to the driver at every sync, making each cudaMallocAsync a real allocation).
void keep_pool() {
  static bool done[16] = {false};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;
    if (cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr) == cudaSuccess) done[dev] = true;
  }
  done[dev] = true;
}

cudaError_t raster_build(const RasterIn& in, RasterState** out, cudaStream_t s) {
  keep_pool();
  RasterState* st = new RasterState();
  st->s = s;
  st->n = in.n;
  st->npix = in.n_rows * in.n_cols;
  *out = st;
  cudaError_t e = cudaSuccess;
#define RCHK(x)                        \
  do {                                 \
    if ((e = (x)) != cudaSuccess) goto done; \
  } while (0)
  {
    ProfScope prof("raster_build", s);
    const int64_t n = in.n, npix = st->npix;
    const int64_t tiles_r = (in.n_rows + RT - 1) / RT, tiles_c = (in.n_cols + RT - 1) / RT, ntiles = tiles_r * tiles_c;
    Prep p{};
    Ranked rk{};
    uint64_t *k0 = nullptr, *tk = nullptr;
    uint32_t *v0 = nullptr, *tv = nullptr;
    int32_t *tcount = nullptr, *ssum = nullptr, *grand = nullptr, *tstart = nullptr, *pcount = nullptr;
    unsigned long long* cnt = nullptr;
    void* ws = nullptr;
    size_t wsb = 0;
    unsigned long long hc[2] = {0, 0};
    int32_t hg = 0;
    RCHK(dalloc(&st->poff, npix + 1, s));
    RCHK(cudaMemsetAsync(st->poff, 0, sizeof(int32_t) * (size_t)(npix + 1), s));
    if (n == 0 || npix == 0) goto done;
    RCHK(dalloc(&cnt, 2, s));
    RCHK(cudaMemsetAsync(cnt, 0, 16, s));
    RCHK(dalloc(&p.uc, 8 * n, s));
    p.vc = p.uc + n; p.ia = p.vc + n; p.ib = p.ia + n; p.ic = p.ib + n; p.rad = p.ic + n; p.z = p.rad + n; p.op = p.z + n;
    RCHK(dalloc(&k0, n, s));
    RCHK(dalloc(&v0, n, s));
    raster_prep_kernel<<<blocks_for(n, 128), 128, 0, s>>>(in, p, k0, v0, cnt); count_launches(1);
    RCHK(cudaGetLastError());
    wsb = grid_workspace_bytes(n);
    RCHK(cudaMallocAsync(&ws, wsb, s));
    RCHK(radix_sort_pairs(k0, v0, n, 64, ws, wsb, s));
    RCHK(cudaMemcpyAsync(hc, cnt, 8, cudaMemcpyDeviceToHost, s));
    RCHK(cudaStreamSynchronize(s));
    st->nvis = (int64_t)hc[0];
    if (st->nvis > 0) {
      const int64_t nv = st->nvis;
      RCHK(dalloc(&rk.uc, 7 * nv, s));
      rk.vc = rk.uc + nv; rk.ia = rk.vc + nv; rk.ib = rk.ia + nv; rk.ic = rk.ib + nv; rk.z = rk.ic + nv; rk.op = rk.z + nv;
      RCHK(dalloc(&rk.gid, nv, s));
      RCHK(dalloc(&rk.box, 4 * nv, s));
      RCHK(dalloc(&tcount, nv, s));
      RCHK(dalloc(&ssum, nv / 4096 + npix / 4096 + 8, s));
      RCHK(dalloc(&grand, 2, s));
      raster_rank_kernel<<<blocks_for(nv, 128), 128, 0, s>>>(in, p, v0, nv, rk, tcount, tiles_c); count_launches(1);
      RCHK(cudaGetLastError());
      RCHK(exclusive_scan_i32(tcount, nv, tcount, ssum, grand, s));
      RCHK(cudaMemcpyAsync(&hg, grand, 4, cudaMemcpyDeviceToHost, s));
      RCHK(cudaStreamSynchronize(s));
      const int64_t nt = hg;
      RCHK(dalloc(&tstart, ntiles + 1, s));
      if (nt > 0) {
        RCHK(dalloc(&tk, nt, s));
        RCHK(dalloc(&tv, nt, s));
        raster_bin_kernel<<<blocks_for(nv, 128), 128, 0, s>>>(rk, nv, tcount, tiles_c, tk, tv); count_launches(1);
        RCHK(cudaGetLastError());
        if ((size_t)grid_workspace_bytes(nt) > wsb) {
          cudaFreeAsync(ws, s);
          wsb = grid_workspace_bytes(nt);
          RCHK(cudaMallocAsync(&ws, wsb, s));
        }
        RCHK(radix_sort_pairs(tk, tv, nt, 32 + bits_for_count(ntiles), ws, wsb, s));
        raster_tile_ranges_kernel<<<blocks_for(nt + 1, 256), 256, 0, s>>>(tk, nt, tstart, ntiles); count_launches(1);
        RCHK(cudaGetLastError());
        RCHK(dalloc(&pcount, npix, s));
        RCHK(cudaMemsetAsync(pcount, 0, sizeof(int32_t) * (size_t)npix, s));
        if (in.all_pairs)
          raster_tile_kernel<false, true><<<(unsigned)ntiles, RT_THREADS, 0, s>>>(in, rk, tv, tstart, tiles_c, pcount,
                                                                                  nullptr, PairsOut{}, nullptr);
        else
          raster_tile_kernel<false, false><<<(unsigned)ntiles, RT_THREADS, 0, s>>>(in, rk, tv, tstart, tiles_c, pcount,
                                                                                   nullptr, PairsOut{}, nullptr);
        count_launches(1);
        RCHK(cudaGetLastError());
        RCHK(exclusive_scan_i32(pcount, npix, st->poff, ssum, grand, s));
        RCHK(cudaMemcpyAsync(&hg, grand, 4, cudaMemcpyDeviceToHost, s));
        RCHK(cudaStreamSynchronize(s));
        st->np = hg;
        RCHK(cudaMemcpyAsync(st->poff + npix, grand, 4, cudaMemcpyDeviceToDevice, s));
        const int64_t npairs = st->np;
        RCHK(dalloc(&st->po.gauss, npairs, s));
        RCHK(dalloc(&st->po.pixel, npairs, s));
        RCHK(dalloc(&st->po.weight, npairs, s));
        RCHK(dalloc(&st->po.alpha, npairs, s));
        RCHK(dalloc(&st->po.tb, npairs, s));
        RCHK(dalloc(&st->po.alive, npairs, s));
        RCHK(dalloc(&st->po.depth, npairs, s));
        if (npairs > 0) {
          if (in.all_pairs)
            raster_tile_kernel<true, true><<<(unsigned)ntiles, RT_THREADS, 0, s>>>(in, rk, tv, tstart, tiles_c, nullptr,
                                                                                   st->poff, st->po, cnt + 1);
          else
            raster_tile_kernel<true, false><<<(unsigned)ntiles, RT_THREADS, 0, s>>>(in, rk, tv, tstart, tiles_c,
                                                                                    nullptr, st->poff, st->po, cnt + 1);
          count_launches(1);
          RCHK(cudaGetLastError());
        }
        RCHK(cudaMemcpyAsync(hc, cnt, 16, cudaMemcpyDeviceToHost, s));
        RCHK(cudaStreamSynchronize(s));
        st->blend_steps = hc[1];
      }
    }
    cudaFreeAsync(cnt, s);
    cudaFreeAsync(p.uc, s);
    cudaFreeAsync(k0, s);
    cudaFreeAsync(v0, s);
    cudaFreeAsync(ws, s);
    cudaFreeAsync(rk.uc, s);
    cudaFreeAsync(rk.gid, s);
    cudaFreeAsync(rk.box, s);
    cudaFreeAsync(tcount, s);
    cudaFreeAsync(ssum, s);
    cudaFreeAsync(grand, s);
    cudaFreeAsync(tstart, s);
    cudaFreeAsync(tk, s);
    cudaFreeAsync(tv, s);
    cudaFreeAsync(pcount, s);
  }
done:
#undef RCHK
  return e;
}

cudaError_t raster_fetch(RasterState* st, int64_t* gauss, int64_t* pixel, double* weight, double* alpha,
                         double* tb, uint8_t* alive, double* depth, cudaStream_t s) {
  const int64_t np = st->np;
  if (np == 0) return cudaSuccess;
  if (gauss) { i32_to_i64_kernel<<<blocks_for(np, 256), 256, 0, s>>>(st->po.gauss, np, gauss); count_launches(1); }
  if (pixel) { i32_to_i64_kernel<<<blocks_for(np, 256), 256, 0, s>>>(st->po.pixel, np, pixel); count_launches(1); }
  cudaError_t e = cudaSuccess;
  if (weight && (e = cudaMemcpyAsync(weight, st->po.weight, 8 * np, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
  if (alpha && (e = cudaMemcpyAsync(alpha, st->po.alpha, 8 * np, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
  if (tb && (e = cudaMemcpyAsync(tb, st->po.tb, 8 * np, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
  if (alive && (e = cudaMemcpyAsync(alive, st->po.alive, np, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
  if (depth && (e = cudaMemcpyAsync(depth, st->po.depth, 8 * np, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t raster_accumulate(RasterState* st, const double* payload, int64_t C, double* out, double* alpha_out,
                              double* depth_out, cudaStream_t s) {
  ProfScope prof("raster_accum", s);
  const int64_t npix = st->npix;
  if (npix == 0) return cudaSuccess;
  raster_accum_kernel<<<blocks_for(npix * 32, 256), 256, 0, s>>>(st->poff, npix, st->po.gauss, st->po.weight,
                                                                st->po.depth, payload, C, out, alpha_out, depth_out);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t raster_argmax(RasterState* st, int64_t* out, cudaStream_t s) {
  if (st->npix == 0) return cudaSuccess;
  raster_argmax_kernel<<<blocks_for(st->npix, 256), 256, 0, s>>>(st->poff, st->npix, st->po.gauss, st->po.weight, out);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t raster_vjp(RasterState* st, const double* upstream, int64_t D, double* fg, cudaStream_t s) {
  ProfScope prof("raster_vjp", s);
  const int64_t n = st->n, np = st->np, P = st->npix;
  cudaError_t e;
  if ((e = cudaMemsetAsync(fg, 0, sizeof(double) * (size_t)n * (size_t)D, s)) != cudaSuccess) return e;
  if (np == 0 || n == 0) return cudaSuccess;
  uint64_t* keys = nullptr;
  uint32_t* vals = nullptr;
  double* upT = nullptr;
  int32_t* gstart = nullptr;
  void* ws = nullptr;
  const size_t wsb = grid_workspace_bytes(np);
  if ((e = dalloc(&keys, np, s)) != cudaSuccess) return e;
  if ((e = dalloc(&vals, np, s)) != cudaSuccess) return e;
  if ((e = dalloc(&upT, P * D, s)) != cudaSuccess) return e;
  if ((e = dalloc(&gstart, n + 1, s)) != cudaSuccess) return e;
  // [n] Gaussians with more than kVjpLong pairs, [n] the others with pairs, then the two counts
  int32_t* long_list = nullptr;
  if ((e = dalloc(&long_list, 2 * n + 2, s)) != cudaSuccess) return e;
  int32_t* short_list = long_list + n;
  int32_t* counts = long_list + 2 * n;   // {long, short}
  if ((e = cudaMemsetAsync(counts, 0, 2 * sizeof(int32_t), s)) != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&ws, wsb, s)) != cudaSuccess) return e;
  raster_gauss_keys_kernel<<<blocks_for(np, 256), 256, 0, s>>>(st->po.gauss, np, keys, vals); count_launches(1);
  if ((e = radix_sort_pairs(keys, vals, np, bits_for_count(n), ws, wsb, s)) != cudaSuccess) return e;
  raster_gauss_ranges_kernel<<<blocks_for(np + 1, 256), 256, 0, s>>>(keys, np, gstart, n); count_launches(1);
  {
    dim3 tb(32, 8), gb((unsigned)((P + 31) / 32 < 4096 ? (P + 31) / 32 : 4096), (unsigned)((D + 31) / 32 < 64 ? (D + 31) / 32 : 64));
    raster_transpose_kernel<<<gb, tb, 0, s>>>(upstream, D, P, upT); count_launches(1);
  }
  raster_vjp_classify_kernel<<<blocks_for(n, 256), 256, 0, s>>>(gstart, n, short_list, counts + 1, long_list, counts);
  count_launches(1);
  raster_vjp_kernel<<<blocks_for(np * ((D + 31) / 32) * 32, 256), 256, 0, s>>>(vals, st->po.pixel, st->po.weight, upT,
                                                                              D, gstart, short_list, counts + 1, fg);
  count_launches(1);
  raster_vjp_long_kernel<<<148 * 2, 32 * kVjpSegs, 0, s>>>(vals, st->po.pixel, st->po.weight, upT, D, gstart, long_list,
                                                           counts, fg); count_launches(1);
  e = cudaGetLastError();
  cudaFreeAsync(keys, s);
  cudaFreeAsync(vals, s);
  cudaFreeAsync(upT, s);
  cudaFreeAsync(gstart, s);
  cudaFreeAsync(long_list, s);
  cudaFreeAsync(ws, s);
  return e;
}

void raster_stats(RasterState* st, int64_t* npairs, int64_t* blend_steps, int64_t* nvis) {
  if (npairs) *npairs = st->np;
  if (blend_steps) *blend_steps = (int64_t)st->blend_steps;
  if (nvis) *nvis = st->nvis;
}

}  // namespace xgs
