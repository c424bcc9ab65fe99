// fp64 codeword contractions of the codebook consumers,
// fused on the fp64 tensor pipe (DMMA.8x8x4, mma.sync m8n8k4 f64):
//
//   decode_feature  (core.py:490-496)     C = softmax(L) . E            (n x K)(K x D)
//   relevance_per_gaussian (thinker.py:122-129)
//                                         score = contrast(softmax(L) . E)  -- no (n x D)
//                                         feature matrix: the epilogue keeps, per row and
//                                         column tile, |f|^2 and f . q_j for the query
//                                         vectors; a finish kernel combines the tiles
//   relevance_per_pixel (thinker.py:132-156)  W given (K x P, read transposed)
//   feature_gradients (rasterizer.py:309-335) fg . E^T (B read transposed)
//
// C[n x m] = A[n x kr] . B[kr x m] with arbitrary strides on A and B.  With
// `softmax` the A operand is a row of logits and each element enters the MMA
// as exp(l - max_row) * (1 / sum_row exp(l - max_row)), the row statistics
// computed by a first pass (the reference's mixture_weights, core.py:473-480).
//
// Tile: 64 rows x 256 columns per CTA, 16 warps each owning 32 x 32 (4 x 4
// MMA tiles, 32 fp64 accumulators per lane); K-chunks of 32 staged in shared
// memory, double-buffered by cp.async (chunks of 16: one barrier per 16 k,
// 71.8 vs 69.2 ms at the relevance benchmark).
// Shared-memory row strides are 4 (mod 16) doubles so the fragment loads
// (A: lane -> (row l/4, k l%4); B: lane -> (k l%4, col l/4)) are conflict-free.
//
// The reference contracts with BLAS dgemm; both sum in fp64 in a different
// order, so results agree to ~1e-15 relative (tests: 1e-12), not bitwise --
// the same contract the cuBLAS path had.
#include "launchers.h"

namespace xgs {

namespace {

constexpr int kGBM = 64, kGBN = 256, kGKC = 32, kGThreads = 512;   // 16 warps: 2 (rows) x 8 (columns)
constexpr int kGAStride = kGKC + 4;      // 36 == 4 (mod 16)
constexpr int kGBStride = kGBN + 4;      // 260 == 4 (mod 16)
constexpr int kGMaxQ = 16;               // query vectors in the relevance epilogue
constexpr size_t kGSmem = sizeof(double) * (2 * kGBM * kGAStride + 2 * kGKC * kGBStride);
constexpr int64_t kGRowChunk = 1 << 18;  // softmax weights staged per 2^18-row chunk (2^18 x K fp64)

struct GemmArgs {
  const double* A;
  int64_t n, kr, lda_r, lda_k;
  const double* B;
  int64_t m, ldb_k, ldb_m;
  double* C;              // [n x m] (ldc) or null
  int64_t ldc;
  const double* Q;        // [nq x m] (relevance) or null
  int nq;
  double* part;           // [n x tiles x (1 + nq)] partials (relevance)
  int64_t tiles;
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__global__ void __launch_bounds__(kGThreads, 1) gemm_f64_kernel(GemmArgs a) {
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                                  // [2][kGBM][kGAStride]
  double* Bs = gsm + 2 * kGBM * kGAStride;           // [2][kGKC][kGBStride]
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wr = warp >> 3, wc = warp & 7;           // warp tile: rows wr*32.., columns wc*32..
  const int64_t r0 = (int64_t)blockIdx.x * kGBM;
  const int64_t c0 = (int64_t)blockIdx.y * kGBN;
  const int64_t nrows = a.n - r0 < kGBM ? a.n - r0 : kGBM;
  const int64_t ncols = a.m - c0 < kGBN ? a.m - c0 : kGBN;
  const bool a_cp = a.lda_k == 1 && (a.lda_r % 2) == 0 && (reinterpret_cast<uintptr_t>(a.A) % 16) == 0 &&
                    nrows == kGBM;
  const bool b_cp = a.ldb_m == 1 && (a.ldb_k % 2) == 0 && (c0 % 2) == 0 &&
                    (reinterpret_cast<uintptr_t>(a.B) % 16) == 0 && ncols == kGBN;
  auto stage = [&](int buf, int64_t k0) {
    double* as = As + buf * kGBM * kGAStride;
    double* bs = Bs + buf * kGKC * kGBStride;
    const bool full_k = k0 + kGKC <= a.kr;
    if (a_cp && full_k) {   // kGBM rows x kGKC doubles in 16-byte copies
#pragma unroll
      for (int i = 0; i < kGBM * kGKC / 2 / kGThreads; i++) {
        const int idx = t + kGThreads * i;
        const int rr = idx / (kGKC / 2), kk = (idx % (kGKC / 2)) * 2;
        cp_async16(as + rr * kGAStride + kk, a.A + (r0 + rr) * a.lda_r + (k0 + kk));
      }
    } else {
      for (int idx = t; idx < kGBM * kGKC; idx += kGThreads) {
        const int rr = a.lda_k == 1 ? idx / kGKC : idx % kGBM, kk = a.lda_k == 1 ? idx % kGKC : idx / kGBM;
        as[rr * kGAStride + kk] =
            (rr < nrows && k0 + kk < a.kr) ? a.A[(r0 + rr) * a.lda_r + (k0 + kk) * a.lda_k] : 0.0;
      }
    }
    if (b_cp && full_k) {   // kGKC rows x kGBN doubles in 16-byte copies
#pragma unroll
      for (int i = 0; i < kGKC * kGBN / 2 / kGThreads; i++) {
        const int idx = t + kGThreads * i;
        const int kk = idx / (kGBN / 2), cc = (idx % (kGBN / 2)) * 2;
        cp_async16(bs + kk * kGBStride + cc, a.B + (k0 + kk) * a.ldb_k + (c0 + cc));
      }
    } else if (a.ldb_m == 1) {
      for (int idx = t; idx < kGKC * kGBN; idx += kGThreads) {
        const int kk = idx / kGBN, cc = idx % kGBN;
        bs[kk * kGBStride + cc] = (k0 + kk < a.kr && cc < ncols) ? a.B[(k0 + kk) * a.ldb_k + (c0 + cc)] : 0.0;
      }
    } else {   // B^T layout: walk k (contiguous), store transposed
      for (int idx = t; idx < kGKC * kGBN; idx += kGThreads) {
        const int kk = idx % kGKC, cc = idx / kGKC;
        bs[kk * kGBStride + cc] =
            (k0 + kk < a.kr && cc < ncols) ? a.B[(k0 + kk) * a.ldb_k + (c0 + cc) * a.ldb_m] : 0.0;
      }
    }
    cp_async_commit();
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int64_t nchunks = (a.kr + kGKC - 1) / kGKC;
  stage(0, 0);
  for (int64_t ch = 0; ch < nchunks; ch++) {
    const int buf = (int)(ch & 1);
    cp_async_wait_all();
    __syncthreads();   // chunk ch staged; chunk ch-1's buffer is free
    if (ch + 1 < nchunks) stage(buf ^ 1, (ch + 1) * kGKC);
    const double* as = As + buf * kGBM * kGAStride + wr * 32 * kGAStride;
    const double* bs = Bs + buf * kGKC * kGBStride + wc * 32;
#pragma unroll
    for (int ks = 0; ks < kGKC / 4; ks++) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; i++) af[i] = as[(i * 8 + (lane >> 2)) * kGAStride + ks * 4 + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; j++) bf[j] = bs[(ks * 4 + (lane & 3)) * kGBStride + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  // ---- epilogue: lane holds rows wr*32 + i*8 + lane/4, columns wc*32 + j*8 + 2*(lane%4) + {0,1}
  if (a.C) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int64_t r = wr * 32 + i * 8 + (lane >> 2);
      if (r >= nrows) continue;
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int64_t c = wc * 32 + j * 8 + 2 * (lane & 3) + h;
          if (c < ncols) a.C[(r0 + r) * a.ldc + c0 + c] = acc[i][j][h];
        }
    }
  }
  if (a.part) {
    // per row: |f|^2 and f . q_j over this tile's columns, summed over the 4
    // lanes of a row (xor 1, 2) and then over the 8 column warps in shared
    // memory (the A staging buffers are free now)
    double* red = gsm;   // [kGBM][1 + nq]
    const int nv = 1 + a.nq;
    __syncthreads();
    for (int i = t; i < kGBM * nv; i += kGThreads) red[i] = 0.0;
    __syncthreads();
    for (int q = 0; q < nv; q++) {
      const double* qv = q ? a.Q + (int64_t)(q - 1) * a.m + c0 : nullptr;
#pragma unroll
      for (int i = 0; i < 4; i++) {
        double x = 0.0;
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int64_t c = wc * 32 + j * 8 + 2 * (lane & 3) + h;
            if (c < ncols) x = fma(acc[i][j][h], q ? qv[c] : acc[i][j][h], x);
          }
        x += __shfl_xor_sync(FULL, x, 1);
        x += __shfl_xor_sync(FULL, x, 2);
        if ((lane & 3) == 0) atomicAdd(&red[(wr * 32 + i * 8 + (lane >> 2)) * nv + q], x);
      }
    }
    __syncthreads();
    for (int i = t; i < kGBM * nv; i += kGThreads) {
      const int r = i / nv, q = i % nv;
      if (r < nrows) a.part[((r0 + r) * a.tiles + blockIdx.y) * nv + q] = red[i];
    }
  }
}

// thinker.py:110-129: f_hat = f / (|f| + eps); score = min over negatives of
// 1 / (1 + exp(-tau (f_hat . pos - f_hat . neg))), starting from 1
__global__ void relevance_finish_kernel(const double* __restrict__ part, int64_t n, int64_t tiles, int nq, double tau,
                                        double eps, double* __restrict__ scores) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double s[1 + kGMaxQ];
    for (int q = 0; q <= nq; q++) s[q] = 0.0;
    for (int64_t tt = 0; tt < tiles; tt++)
      for (int q = 0; q <= nq; q++) s[q] += part[(r * tiles + tt) * (1 + nq) + q];
    const double den = sqrt(s[0]) + eps;
    const double pos = s[1] / den;
    double sc = 1.0;
    for (int q = 2; q <= nq; q++) sc = fmin(sc, 1.0 / (1.0 + exp(-(tau * (pos - s[q] / den)))));
    scores[r] = sc;
  }
}

}  // namespace

size_t gemm_f64_workspace_bytes(int64_t n, int64_t m, int64_t nq, int64_t kr, bool softmax) {
  const int64_t tiles = (m + kGBN - 1) / kGBN;
  const int64_t chunk = n < kGRowChunk ? n : kGRowChunk;
  return sizeof(double) * (size_t)(n * tiles * (1 + nq) + (softmax ? chunk * kr : 0)) + 256;
}

cudaError_t launch_gemm_f64(const double* A, int64_t n, int64_t kr, int64_t lda_r, int64_t lda_k, bool softmax,
                            const double* B, int64_t m, int64_t ldb_k, int64_t ldb_m, double* C, int64_t ldc,
                            const double* Q, int64_t nq, double tau, double eps, double* scores, void* ws,
                            cudaStream_t s) {
  if (n == 0 || m == 0) return cudaSuccess;
  if (nq > kGMaxQ) return cudaErrorInvalidValue;
  cudaError_t e = attr_once(kAttrGemmF64, [] {
    return cudaFuncSetAttribute(gemm_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGSmem);
  });
  if (e != cudaSuccess) return e;
  const int64_t tiles = (m + kGBN - 1) / kGBN;
  double* part = static_cast<double*>(ws);
  double* wbuf = part + (scores ? n * tiles * (1 + nq) : 0);
  int* bad = reinterpret_cast<int*>(wbuf + (softmax ? (n < kGRowChunk ? n : kGRowChunk) * kr : 0));
  SumPlan pk;
  if (softmax && !build_sum_plan((int)kr, &pk)) return cudaErrorInvalidValue;
  // softmax rows: the weights of a row chunk (the exact NumPy-order
  // mixture_weights of xgs_softmax_rows) are staged in the workspace, then
  // contracted; otherwise one pass over all rows
  const int64_t step = softmax ? kGRowChunk : n;
  for (int64_t c = 0; c < n; c += step) {
    const int64_t rows = n - c < step ? n - c : step;
    GemmArgs g{};
    g.n = rows;
    g.kr = kr;
    if (softmax) {
      if ((e = launch_softmax_rows(A + c * lda_r, rows, kr, CB_WEIGHTS, nullptr, wbuf, nullptr, pk, bad, s)) !=
          cudaSuccess)
        return e;
      g.A = wbuf;
      g.lda_r = kr;
      g.lda_k = 1;
    } else {
      g.A = A + c * lda_r;
      g.lda_r = lda_r;
      g.lda_k = lda_k;
    }
    g.B = B;
    g.m = m;
    g.ldb_k = ldb_k;
    g.ldb_m = ldb_m;
    g.C = C ? C + c * ldc : nullptr;
    g.ldc = ldc;
    g.Q = Q;
    g.nq = (int)nq;
    g.tiles = tiles;
    g.part = scores ? part + c * tiles * (1 + nq) : nullptr;
    ProfScope prof("decode_gemm", s);
    const dim3 grid((unsigned)((rows + kGBM - 1) / kGBM), (unsigned)tiles);
    gemm_f64_kernel<<<grid, kGThreads, kGSmem, s>>>(g);
    count_launches(1);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (scores) {
    const int64_t blocks = (n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16;
    relevance_finish_kernel<<<(unsigned)blocks, 256, 0, s>>>(part, n, tiles, (int)nq, tau, eps, scores);
    count_launches(1);
  }
  return cudaGetLastError();
}

}  // namespace xgs
