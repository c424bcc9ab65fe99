// Greedy farthest-point seeding (vq.py:126-147, seed_from_samples) without a
// host round trip per seed.
//
// The reference keeps min_d = min over chosen seeds of the squared distance
// (np.sum((buffer - s)**2, axis=1): NumPy pairwise order over D), takes
// j = argmax(min_d) (first maximum; NumPy puts the first NaN ahead of every
// number), and appends buffer[len(seeds) % n] instead of buffer[j] once the
// maximum is 0 (fewer distinct rows than K; min_d stays all-zero from then on,
// so every later seed cycles too).
//
// seed_persistent_kernel runs all K-1 passes in one cooperative launch (one
// grid barrier per seed); where a cooperative launch of that size is not
// possible, seed_step_kernel(t) runs one launch per seed: it reads seed t-1
// from device memory, folds its distances into min_d (one warp per row, exact
// fp64 pairwise sums), reduces a per-block (max, index) and the last block to
// finish reduces the block partials and writes seed t.  Either way nothing
// synchronises with the host.
#include <cstdlib>

#include "launchers.h"

namespace xgs {

namespace {

constexpr int kSeedWarps = 8;

// argmax order of NumPy: NaN first, then larger value, then lower index
__device__ __forceinline__ bool seed_before(double a, int64_t ia, double b, int64_t ib) {
  const bool na = isnan(a), nb = isnan(b);
  if (na != nb) return na;
  if (!na && a != b) return a > b;
  return ia < ib;
}

// np.minimum propagates NaN (fmin would drop it)
__device__ __forceinline__ double np_minimum(double a, double b) {
  if (isnan(a)) return a;
  if (isnan(b)) return b;
  return b < a ? b : a;
}

struct SeedWs {
  double* min_d;   // n
  double* pv;      // per-block partial maxima
  int64_t* pi;
  unsigned* counter;
  int* cycling;    // set once the maximum hit 0
};

__device__ __forceinline__ void block_argmax(double& v, int64_t& i, double* sv, int64_t* si) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int o = 16; o; o >>= 1) {
    const double v2 = __shfl_xor_sync(FULL, v, o);
    const int64_t i2 = __shfl_xor_sync(FULL, i, o);
    if (seed_before(v2, i2, v, i)) {
      v = v2;
      i = i2;
    }
  }
  if (lane == 0) {
    sv[warp] = v;
    si[warp] = i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++)
      if (seed_before(sv[w], si[w], v, i)) {
        v = sv[w];
        i = si[w];
      }
  }
}

template <typename X>
__global__ void __launch_bounds__(kSeedWarps * 32)
seed_step_kernel(const X* __restrict__ x, int64_t n, int64_t d, int64_t ldx, int64_t t, int64_t* __restrict__ seeds,
                 SeedWs w, SumPlan pd) {
  extern __shared__ double srow[];   // the previous seed row, fp64
  __shared__ double scratch_all[kSeedWarps][kMaxLeaves];
  __shared__ double sv[kSeedWarps];
  __shared__ int64_t si[kSeedWarps];
  __shared__ bool last;
  if (*(volatile int*)w.cycling) {   // min_d is all zero: seeds cycle through the buffer
    if (blockIdx.x == 0 && threadIdx.x == 0) seeds[t] = t % n;
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t cur = seeds[t - 1];
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) srow[i] = ld64(x + cur * ldx, i);
  __syncthreads();
  double* scratch = scratch_all[warp];
  double v = -__longlong_as_double(0x7ff0000000000000ll);
  int64_t vi = INT64_MAX;
  for (int64_t r = (int64_t)blockIdx.x * kSeedWarps + warp; r < n; r += (int64_t)gridDim.x * kSeedWarps) {
    const X* xr = x + r * ldx;
    const double dist = warp_pairwise(
        pd,
        [&](int i) {
          const double df = dsub(ld64(xr, i), srow[i]);
          return dmul(df, df);
        },
        scratch, lane);
    const double m = t == 1 ? dist : np_minimum(w.min_d[r], dist);
    if (lane == 0) w.min_d[r] = m;
    if (seed_before(m, r, v, vi)) {
      v = m;
      vi = r;
    }
  }
  block_argmax(v, vi, sv, si);
  if (threadIdx.x == 0) {
    w.pv[blockIdx.x] = v;
    w.pi[blockIdx.x] = vi;
    __threadfence();
    last = atomicAdd(w.counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  v = -__longlong_as_double(0x7ff0000000000000ll);
  vi = INT64_MAX;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
    const double v2 = __ldcg(w.pv + b);
    const int64_t i2 = __ldcg(w.pi + b);
    if (seed_before(v2, i2, v, vi)) {
      v = v2;
      vi = i2;
    }
  }
  __syncthreads();   // sv/si reuse
  block_argmax(v, vi, sv, si);
  if (threadIdx.x == 0) {
    if (v == 0.0) {   // vq.py:141-143
      seeds[t] = t % n;
      *w.cycling = 1;
    } else {
      seeds[t] = vi;
    }
    *w.counter = 0;
  }
}

// All K-1 passes in one cooperative launch (every block co-resident): per
// pass the blocks fold their rows' distances into min_d, publish a block
// (max, index) into one of two partial buffers, meet at a counter barrier,
// and then each block reduces all partials itself (same order, same result in
// every block), so one grid barrier per seed.
// 16 warps per block and at most 2 blocks per SM: few blocks meet at each
// barrier (one counter atomic each) while enough warps share the rows.
constexpr int kPersistWarps = 16;

template <typename X>
__global__ void __launch_bounds__(kPersistWarps * 32)
seed_persistent_kernel(const X* __restrict__ x, int64_t n, int64_t d, int64_t ldx, int64_t k,
                       int64_t* __restrict__ seeds, SeedWs w, SumPlan pd) {
  extern __shared__ double srow[];
  __shared__ double scratch_all[kPersistWarps][kMaxLeaves];
  __shared__ double sv[kPersistWarps];
  __shared__ int64_t si[kPersistWarps];
  __shared__ double s_v;
  __shared__ int64_t s_j;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned nb = gridDim.x;
  double* scratch = scratch_all[warp];
  int64_t cur = 0;
  for (int64_t t = 1; t < k; t++) {
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) srow[i] = ld64(x + cur * ldx, i);
    __syncthreads();
    double v = -__longlong_as_double(0x7ff0000000000000ll);
    int64_t vi = INT64_MAX;
    for (int64_t r = (int64_t)blockIdx.x * kPersistWarps + warp; r < n; r += (int64_t)nb * kPersistWarps) {
      const X* xr = x + r * ldx;
      const double dist = warp_pairwise(
          pd,
          [&](int i) {
            const double df = dsub(ld64(xr, i), srow[i]);
            return dmul(df, df);
          },
          scratch, lane);
      const double m = t == 1 ? dist : np_minimum(w.min_d[r], dist);
      if (lane == 0) w.min_d[r] = m;
      if (seed_before(m, r, v, vi)) {
        v = m;
        vi = r;
      }
    }
    block_argmax(v, vi, sv, si);
    double* pv = w.pv + (t & 1) * nb;
    int64_t* pi = w.pi + (t & 1) * nb;
    if (threadIdx.x == 0) {
      pv[blockIdx.x] = v;
      pi[blockIdx.x] = vi;
      __threadfence();
      atomicAdd(w.counter, 1u);
      while (*(volatile unsigned*)w.counter < (unsigned)t * nb) {
      }
      __threadfence();
    }
    __syncthreads();
    v = -__longlong_as_double(0x7ff0000000000000ll);
    vi = INT64_MAX;
    for (unsigned b = threadIdx.x; b < nb; b += blockDim.x) {
      const double v2 = __ldcg(pv + b);
      const int64_t i2 = __ldcg(pi + b);
      if (seed_before(v2, i2, v, vi)) {
        v = v2;
        vi = i2;
      }
    }
    __syncthreads();   // sv / si reuse
    block_argmax(v, vi, sv, si);
    if (threadIdx.x == 0) {
      s_v = v;
      s_j = vi;
    }
    __syncthreads();
    if (s_v == 0.0) {   // vq.py:141-143: min_d is all zero from here on, the seeds cycle
      if (blockIdx.x == 0)
        for (int64_t u = t + threadIdx.x; u < k; u += blockDim.x) seeds[u] = u % n;
      return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) seeds[t] = s_j;
    cur = s_j;
    __syncthreads();   // srow is rewritten by the next pass
  }
}

unsigned seed_blocks(int64_t n) {
  int64_t b = (n + kSeedWarps - 1) / kSeedWarps;
  if (b > 148 * 8) b = 148 * 8;
  return (unsigned)(b < 1 ? 1 : b);
}

template <typename X>
cudaError_t seed_launch(const void* x, int64_t n, int64_t d, int64_t ldx, int64_t k, int64_t* seeds, const SeedWs& w,
                        const SumPlan& pd, cudaStream_t s) {
  const size_t smem = sizeof(double) * (size_t)d;
  static int per_sm = 0;   // occupancy of the persistent kernel (identical B200s: same on every device)
  cudaError_t ea = attr_once(kAttrSeed, [] {
    cudaError_t r = cudaFuncSetAttribute(seed_step_kernel<X>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(seed_persistent_kernel<X>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8);
    return r;
  });
  if (ea != cudaSuccess) return ea;
  int dev = 0, sms = 148, coop = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, seed_persistent_kernel<X>, kPersistWarps * 32, smem) !=
      cudaSuccess)
    per_sm = 0;
  if (per_sm > 2) per_sm = 2;
  const unsigned want = (unsigned)((n + kPersistWarps - 1) / kPersistWarps);
  const unsigned nb = (unsigned)((int64_t)per_sm * sms < (int64_t)want ? per_sm * sms : want);
  const char* no_coop = std::getenv("XGS_SEED_NO_COOP");   // tests: exercise the per-launch path
  if (coop && nb >= 1 && k > 1 && !(no_coop && no_coop[0] == '1')) {
    const X* xp = static_cast<const X*>(x);
    SeedWs ww = w;
    SumPlan pp = pd;
    void* args[] = {(void*)&xp, (void*)&n, (void*)&d, (void*)&ldx, (void*)&k, (void*)&seeds, (void*)&ww, (void*)&pp};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)seed_persistent_kernel<X>, dim3(nb), dim3(kPersistWarps * 32),
                                                args, smem, s);
    if (e == cudaSuccess) {
      count_launches(1);
      return cudaSuccess;
    }
    cudaGetLastError();   // not co-resident here: fall back to one launch per seed
  }
  const unsigned b = seed_blocks(n);
  for (int64_t t = 1; t < k; t++) {
    seed_step_kernel<X><<<b, kSeedWarps * 32, smem, s>>>(static_cast<const X*>(x), n, d, ldx, t, seeds, w, pd);
    count_launches(1);
  }
  return cudaGetLastError();
}

}  // namespace

size_t seed_workspace_bytes(int64_t n) {
  const size_t nb = seed_blocks(n);
  return align_up(sizeof(double) * (size_t)n, 256) + align_up(sizeof(double) * 2 * nb, 256) +
         align_up(sizeof(int64_t) * 2 * nb, 256) + 256;   // partials double-buffered (persistent kernel)
}

cudaError_t launch_seed_farthest(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx, int64_t k,
                                 int64_t* seeds, void* ws, const SumPlan& pd, cudaStream_t s) {
  ProfScope prof("vq_seed", s);
  const size_t nb = seed_blocks(n);
  char* p = static_cast<char*>(ws);
  SeedWs w;
  w.min_d = reinterpret_cast<double*>(p);
  p += align_up(sizeof(double) * (size_t)n, 256);
  w.pv = reinterpret_cast<double*>(p);
  p += align_up(sizeof(double) * 2 * nb, 256);
  w.pi = reinterpret_cast<int64_t*>(p);
  p += align_up(sizeof(int64_t) * 2 * nb, 256);
  w.counter = reinterpret_cast<unsigned*>(p);
  w.cycling = reinterpret_cast<int*>(p + 128);
  cudaError_t e;
  if ((e = cudaMemsetAsync(p, 0, 256, s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(seeds, 0, sizeof(int64_t), s)) != cudaSuccess) return e;   // seeds[0] = row 0
  switch (dtype) {
    case F32: return seed_launch<float>(x, n, d, ldx, k, seeds, w, pd, s);
    case F64: return seed_launch<double>(x, n, d, ldx, k, seeds, w, pd, s);
    default: return seed_launch<uint16_t>(x, n, d, ldx, k, seeds, w, pd, s);
  }
}

}  // namespace xgs
