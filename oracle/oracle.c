/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's hot-path
 * arithmetic (semsplat 0.1.0, /root/reference/pkg/src/semsplat).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library, and only as the checker or the timed CPU baseline.
 * The product path (paper_2603_09632_b200) never links or calls it.
 *
 * Single-threaded by design: callers parallelise over row ranges (ctypes
 * releases the GIL).  Compiled with -O2 -ffp-contract=off (no implicit FMA),
 * so every double operation below rounds exactly as NumPy's scalar loops do.
 *
 * Restated functions:
 *   sqdist_pairwise   vq.py:69-73  np.sum((x-e)*(x-e), axis=2): NumPy's
 *                     pairwise_sum (8 accumulators, block 128, split at
 *                     n/2 rounded down to a multiple of 8)
 *   assign            vq.py:84-87  np.argmin -> first (lowest) index of min
 *   accumulate        vq.py:90-100 bincount + np.add.at (sequential fp64 chain
 *                     per (k,d) in ascending row order, starting from +0.0)
 *   backproject       slam.py:594-598  cam=((u-cx)*d/fx, (v-cy)*d/fy, d);
 *                     p = R^T (cam - t), with OpenBLAS dgemv's FMA order
 *                     fma(R2i,w2, fma(R1i,w1, R0i*w0)) (pinned by golden vectors)
 *   voxel keys        SURVEY.md 8(a) g8 definitions (builder-owned: no
 *                     reference code exists for them)
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>

enum { DT_F32 = 0, DT_F64 = 1, DT_BF16 = 2 };

static inline double load_elem(const void* x, int dtype, int64_t i) {
  if (dtype == DT_F32) return (double)((const float*)x)[i];
  if (dtype == DT_F64) return ((const double*)x)[i];
  uint32_t b = ((uint32_t)((const uint16_t*)x)[i]) << 16;
  float f;
  memcpy(&f, &b, 4);
  return (double)f;
}

/* NumPy pairwise_sum over a[0..n) (numpy/_core/src/umath/loops_utils.h.src). */
static double pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; i++) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    int64_t i;
    for (int j = 0; j < 8; j++) r[j] = a[j];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise(a, n2) + pairwise(a + n2, n - n2);
  }
}

double xgs_oracle_pairwise_sum(const double* a, int64_t n) { return pairwise(a, n); }

/* One squared distance, vq.py:71-73: diff = x - e; sum(diff*diff). */
static double sqdist_row(const double* xr, const double* e, int64_t D, double* tmp) {
  for (int64_t d = 0; d < D; d++) {
    double df = xr[d] - e[d];
    tmp[d] = df * df;
  }
  return pairwise(tmp, D);
}

/* Full (N,K) matrix, vq.py:69-73. */
int xgs_oracle_sqdist(const void* x, int dtype, int64_t N, int64_t D, const double* E,
                      int64_t K, double* out) {
  {
    double* xr = (double*)malloc(sizeof(double) * (size_t)(D > 0 ? D : 1));
    double* tmp = (double*)malloc(sizeof(double) * (size_t)(D > 0 ? D : 1));
    for (int64_t n = 0; n < N; n++) {
      for (int64_t d = 0; d < D; d++) xr[d] = load_elem(x, dtype, n * D + d);
      for (int64_t k = 0; k < K; k++) out[n * K + k] = sqdist_row(xr, E + k * D, D, tmp);
    }
    free(xr);
    free(tmp);
  }
  return 0;
}

/* vq.py:84-87: argmin over the fp64 distances, first minimum wins. */
int xgs_oracle_assign(const void* x, int dtype, int64_t N, int64_t D, const double* E,
                      int64_t K, int64_t* codes) {
  {
    double* xr = (double*)malloc(sizeof(double) * (size_t)(D > 0 ? D : 1));
    double* tmp = (double*)malloc(sizeof(double) * (size_t)(D > 0 ? D : 1));
    for (int64_t n = 0; n < N; n++) {
      for (int64_t d = 0; d < D; d++) xr[d] = load_elem(x, dtype, n * D + d);
      double best = 0.0;
      int64_t bk = 0;
      for (int64_t k = 0; k < K; k++) {
        double v = sqdist_row(xr, E + k * D, D, tmp);
        /* np.argmin: NaN wins (first NaN), else strict < keeps the first min */
        if (k == 0 || v < best || (isnan(v) && !isnan(best))) {
          if (k == 0 || !isnan(best)) { best = v; bk = k; }
        }
      }
      codes[n] = bk;
    }
    free(xr);
    free(tmp);
  }
  return 0;
}

/* vq.py:90-100 after the assignment: counts = bincount, sums = np.add.at. */
int xgs_oracle_accumulate(const void* x, int dtype, int64_t N, int64_t D,
                          const int64_t* codes, int64_t K, double* counts, double* sums) {
  for (int64_t k = 0; k < K; k++) counts[k] = 0.0;
  for (int64_t i = 0; i < K * D; i++) sums[i] = 0.0;
  for (int64_t n = 0; n < N; n++) {
    int64_t k = codes[n];
    counts[k] += 1.0;
    for (int64_t d = 0; d < D; d++) sums[k * D + d] = sums[k * D + d] + load_elem(x, dtype, n * D + d);
  }
  return 0;
}

/* slam.py:594-598 for one pixel. intr = {fx, fy, cx, cy} (u=row pairs fx/cx). */
static inline void backproject1(const double* R, const double* t, const double* intr,
                                double u, double v, double depth, double* p) {
  double c0 = (u - intr[2]) * depth / intr[0];
  double c1 = (v - intr[3]) * depth / intr[1];
  double c2 = depth;
  double w0 = c0 - t[0], w1 = c1 - t[1], w2 = c2 - t[2];
  for (int i = 0; i < 3; i++) p[i] = fma(R[6 + i], w2, fma(R[3 + i], w1, R[i] * w0));
}

int xgs_oracle_backproject(const double* R, const double* t, const double* intr,
                           const double* u, const double* v, const double* depth,
                           int64_t n, double* out) {
  for (int64_t i = 0; i < n; i++) backproject1(R, t, intr, u[i], v[i], depth[i], out + 3 * i);
  return 0;
}

#define XGS_KEY_BIAS (1LL << 20)
#define XGS_KEY_INVALID 0xFFFFFFFFFFFFFFFFULL

/* Per-pixel voxel key: depth>0 on the stride lattice,
 * ix = floor(p/vs), 21-bit biased fields; out-of-range -> invalid. */
int xgs_oracle_grid_keys(const float* depth, int64_t H, int64_t W, int64_t stride,
                         const double* intr, const double* R, const double* t, double voxel,
                         uint64_t* keys, double* pts) {
  for (int64_t u = 0; u < H; u++) {
    for (int64_t v = 0; v < W; v++) {
      int64_t i = u * W + v;
      double* p = pts + 3 * i;
      keys[i] = XGS_KEY_INVALID;
      p[0] = p[1] = p[2] = 0.0;
      if ((u % stride) != 0 || (v % stride) != 0) continue;
      float d32 = depth[i];
      if (!(d32 > 0.0f)) continue;
      backproject1(R, t, intr, (double)u, (double)v, (double)d32, p);
      int64_t q[3];
      int ok = 1;
      for (int a = 0; a < 3; a++) {
        double f = floor(p[a] / voxel);
        if (!(f >= -(double)XGS_KEY_BIAS && f < (double)XGS_KEY_BIAS)) { ok = 0; break; }
        q[a] = (int64_t)f + XGS_KEY_BIAS;
      }
      if (!ok) continue;
      keys[i] = ((uint64_t)q[0] << 42) | ((uint64_t)q[1] << 21) | (uint64_t)q[2];
    }
  }
  return 0;
}
