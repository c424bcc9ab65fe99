// Shared device helpers for libxgs (sm_100a).
//
// The exact-arithmetic helpers reproduce the reference's NumPy fp64 evaluation
// order bit for bit:
//   * squared distance (vq.py:69-73): diff = x - e; sum(diff*diff) with NumPy's
//     pairwise_sum over D (8 strided accumulators per leaf of <= 128 elements,
//     leaves split at n/2 rounded down to a multiple of 8);
//   * every add/mul/div uses the __d*_rn intrinsics so nvcc can never contract
//     them into an FMA.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <atomic>

namespace xgs {

enum Status : int { OK = 0, INVALID_INPUT = 1, INVALID_STATE = 2, CUDA_ERROR = 3, NOT_SUPPORTED = 4 };
enum DType : int { F32 = 0, F64 = 1, BF16 = 2 };

constexpr unsigned FULL = 0xffffffffu;

// Programmatic dependent launch: a kernel launched with launch_pdl may start
// while the previous kernel in the stream drains (its launch latency hides
// behind the predecessor's tail); it must call pdl_wait() before touching
// anything the predecessor writes.  Chains of short dependent kernels (the
// radix-sort passes, select, emit) lose the per-boundary launch gap.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Kernel attributes (cudaFuncSetAttribute) belong to the device context that
// is current when they are set, so a process driving several GPUs must set
// them on each: attr_once runs a site's setter once per (site, device) and
// records it only when it succeeded.
enum AttrSite : int {
  kAttrScreen0 = 0, kAttrScreen1, kAttrScreen2, kAttrSeed, kAttrUpdate, kAttrGridFront, kAttrGridSort,
  kAttrGridHash, kAttrCodebook, kAttrGemmF64, kAttrSites
};
inline std::atomic<uint32_t>* attr_table() {
  static std::atomic<uint32_t> done[64];
  return done;
}
template <typename F>
inline cudaError_t attr_once(int site, F&& set) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return set();
  std::atomic<uint32_t>& m = attr_table()[dev];
  if (m.load(std::memory_order_acquire) & (1u << site)) return cudaSuccess;
  e = set();
  if (e == cudaSuccess) m.fetch_or(1u << site, std::memory_order_acq_rel);
  return e;
}

inline size_t dtype_size(int dtype) { return dtype == F64 ? 8 : dtype == F32 ? 4 : 2; }
inline size_t align_up(size_t b, size_t a) { return (b + a - 1) / a * a; }

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// Element load with exact widening to fp64 (fp32 / bf16 -> fp64 is exact).
__device__ __forceinline__ double ld64(const float* p, int64_t i) { return (double)__ldg(p + i); }
__device__ __forceinline__ double ld64(const double* p, int64_t i) { return __ldg(p + i); }
__device__ __forceinline__ double ld64(const uint16_t* p, int64_t i) {
  return (double)__uint_as_float(((uint32_t)__ldg(p + i)) << 16);
}
__device__ __forceinline__ float ld32(const float* p, int64_t i) { return __ldg(p + i); }
__device__ __forceinline__ float ld32(const double* p, int64_t i) { return (float)__ldg(p + i); }
__device__ __forceinline__ float ld32(const uint16_t* p, int64_t i) {
  return __uint_as_float(((uint32_t)__ldg(p + i)) << 16);
}

// NumPy pairwise-sum evaluation plan for a fixed length n: leaves (offset,len)
// in order plus a postfix program (leaf index >= 0, -1 = add the two tops).
constexpr int kMaxLeaves = 128;   // n <= 8192
constexpr int kMaxOps = 2 * kMaxLeaves;
struct SumPlan {
  int n;
  int n_leaves;
  int n_ops;
  int16_t leaf_off[kMaxLeaves];
  int16_t leaf_len[kMaxLeaves];
  int16_t ops[kMaxOps];
};

// Host: build the plan (mirrors numpy/_core/src/umath/loops_utils.h.src).
inline bool build_sum_plan(int n, SumPlan* p) {
  p->n = n;
  p->n_leaves = 0;
  p->n_ops = 0;
  struct Rec {
    static bool go(SumPlan* p, int off, int len) {
      if (len <= 128) {
        if (p->n_leaves >= kMaxLeaves || p->n_ops >= kMaxOps) return false;
        p->leaf_off[p->n_leaves] = (int16_t)off;
        p->leaf_len[p->n_leaves] = (int16_t)len;
        p->ops[p->n_ops++] = (int16_t)p->n_leaves++;
        return true;
      }
      int n2 = len / 2;
      n2 -= n2 % 8;
      if (!go(p, off, n2) || !go(p, off + n2, len - n2)) return false;
      if (p->n_ops >= kMaxOps) return false;
      p->ops[p->n_ops++] = -1;
      return true;
    }
  };
  return n >= 0 && n <= 8192 && Rec::go(p, 0, n);
}

// Warp-cooperative pairwise sum of f(i), i in [0, plan.n).  Lanes are grouped
// 8 per leaf (lane j of a group owns accumulator r[j]); the 3-level xor
// shuffle reproduces ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) exactly.  `scratch`
// is per-warp shared memory of >= n_leaves doubles.  Result valid in all lanes.
template <typename F>
__device__ __forceinline__ double warp_pairwise(const SumPlan& P, F f, double* scratch, int lane) {
  const int grp = lane >> 3, j = lane & 7;
  for (int l0 = 0; l0 < P.n_leaves; l0 += 4) {
    const int l = l0 + grp;
    const bool active = l < P.n_leaves;
    const int off = active ? P.leaf_off[l] : 0;
    const int n = active ? P.leaf_len[l] : 0;
    const int main = n >= 8 ? n - (n & 7) : 0;
    double acc = 0.0;
    if (n >= 8) {
      // all of the lane's terms are evaluated (loads issued) before the
      // sequential chain, which adds them in the same order as before
      double v[16];   // leaf length <= 128 -> <= 16 terms per lane
#pragma unroll
      for (int i = 0; i < 16; i++) v[i] = 8 * i < main ? f(off + 8 * i + j) : 0.0;
      acc = v[0];
#pragma unroll
      for (int i = 1; i < 16; i++)
        if (8 * i < main) acc = dadd(acc, v[i]);
    }
    double t = dadd(acc, __shfl_xor_sync(FULL, acc, 1));
    t = dadd(t, __shfl_xor_sync(FULL, t, 2));
    t = dadd(t, __shfl_xor_sync(FULL, t, 4));
    if (j == 0 && active) {
      double r = n >= 8 ? t : 0.0;
      for (int i = main; i < n; i++) r = dadd(r, f(off + i));
      scratch[l] = r;
    }
  }
  __syncwarp();
  double res = 0.0;
  if (lane == 0) {
    double st[24];
    int sp = 0;
    for (int o = 0; o < P.n_ops; o++) {
      const int op = P.ops[o];
      if (op >= 0) {
        st[sp++] = scratch[op];
      } else {
        const double b = st[--sp];
        const double a = st[--sp];
        st[sp++] = dadd(a, b);
      }
    }
    res = sp ? st[0] : 0.0;
  }
  __syncwarp();
  return __shfl_sync(FULL, res, 0);
}

// Exact fp64 squared distance of one row against one codeword (vq.py:69-73).
template <typename X>
__device__ __forceinline__ double warp_sqdist(const X* __restrict__ x, const double* __restrict__ e,
                                              const SumPlan& P, double* scratch, int lane) {
  return warp_pairwise(
      P,
      [&](int i) {
        const double d = dsub(ld64(x, i), __ldg(e + i));
        return dmul(d, d);
      },
      scratch, lane);
}

// Lexicographic (value, index) minimum: NumPy argmin keeps the first minimum.
__device__ __forceinline__ void argmin_merge(double& v, int& k, double v2, int k2) {
  if (v2 < v || (v2 == v && k2 < k)) {
    v = v2;
    k = k2;
  }
}

}  // namespace xgs
