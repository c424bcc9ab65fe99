// Micro-benchmark (measurement only, not part of libxgs): cost of the batch
// dedup-table insert pattern on B200 for a C3-like item stream.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o insert_bench insert_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

constexpr unsigned long long EMPTY = ~0ull;
__device__ __forceinline__ uint32_t dd_hash(uint64_t key) {
  uint32_t h = (uint32_t)key * 0x9E3779B1u ^ (uint32_t)(key >> 32) * 0x85EBCA77u;
  h ^= h >> 15; h *= 0x2C1B3C6Du; return h ^ (h >> 13);
}
__device__ __forceinline__ ulonglong2 slot_ld(const unsigned long long* s, uint64_t h) {
  return __ldcg(reinterpret_cast<const ulonglong2*>(s + 2 * h));
}
template <int MODE>  // 0 full insert, 1 read-only probe, 2 CAS-only (no min)
__global__ void __launch_bounds__(256) ins(const uint64_t* keys, const uint32_t* pids, int n, unsigned long long* slots,
                                           uint64_t mask, int* ovf) {
  for (int i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += 4 * gridDim.x * blockDim.x) {
    uint64_t k[4], h[4]; uint32_t p[4]; ulonglong2 c[4]; bool v[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      int i = i0 + j * gridDim.x * blockDim.x; v[j] = i < n;
      if (v[j]) { k[j] = keys[i]; p[j] = pids[i]; h[j] = dd_hash(k[j]) & mask; c[j] = slot_ld(slots, h[j]); }
    }
#pragma unroll
    for (int j = 0; j < 4; j++) {
      if (!v[j]) continue;
      uint64_t hh = h[j]; ulonglong2 cur = c[j];
      for (int t = 0; t < 256; t++) {
        if (cur.x == EMPTY) {
          if (MODE == 1) break;
          unsigned long long prev = atomicCAS(slots + 2 * hh, EMPTY, (unsigned long long)k[j]);
          cur.x = prev == EMPTY ? k[j] : prev;
        }
        if (cur.x == k[j]) break;
        hh = (hh + 1) & mask; cur = slot_ld(slots, hh);
      }
      if (MODE == 0 && (uint32_t)cur.y > p[j]) atomicMin(reinterpret_cast<unsigned*>(slots + 2 * hh + 1), p[j]);
      if (MODE == 1 && cur.x != k[j]) *ovf = 1;
    }
  }
}
__global__ void fill(unsigned long long* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = EMPTY;
}

int main() {
  const int nvox = 162000, rep = 27, n = nvox * rep;
  std::mt19937_64 rng(1);
  std::vector<uint64_t> vk(nvox);
  for (auto& x : vk) x = rng() >> 1;
  // "frame order": 16 frames, each frame a contiguous chunk holding each voxel ~rep/16 times, voxel order random per frame
  std::vector<uint64_t> keys(n); std::vector<uint32_t> pids(n);
  int o = 0;
  for (int f = 0; f < 16; f++) {
    std::vector<int> idx;
    for (int v = 0; v < nvox; v++) for (int r = f * rep / 16; r < (f + 1) * rep / 16; r++) idx.push_back(v);
    std::shuffle(idx.begin(), idx.end(), rng);
    for (int v : idx) { if (o < n) { keys[o] = vk[v]; pids[o] = o; o++; } }
  }
  const int nn = o;
  std::vector<uint64_t> sk(keys.begin(), keys.begin() + nn);
  std::vector<uint32_t> sp(pids.begin(), pids.begin() + nn);
  // sorted-by-key variant (all repeats of a key adjacent)
  std::vector<int> perm(nn); for (int i = 0; i < nn; i++) perm[i] = i;
  std::sort(perm.begin(), perm.end(), [&](int a, int b) { return sk[a] < sk[b] || (sk[a] == sk[b] && a < b); });
  std::vector<uint64_t> sk2(nn); std::vector<uint32_t> sp2(nn);
  for (int i = 0; i < nn; i++) { sk2[i] = sk[perm[i]]; sp2[i] = sp[perm[i]]; }
  uint64_t *dk, *dk2; uint32_t *dp, *dp2; unsigned long long* slots; int* ovf;
  const int64_t cap = 1 << 20;
  cudaMalloc(&dk, nn * 8); cudaMalloc(&dp, nn * 4); cudaMalloc(&dk2, nn * 8); cudaMalloc(&dp2, nn * 4);
  cudaMalloc(&slots, cap * 16); cudaMalloc(&ovf, 4);
  cudaMemcpy(dk, sk.data(), nn * 8, cudaMemcpyHostToDevice); cudaMemcpy(dp, sp.data(), nn * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dk2, sk2.data(), nn * 8, cudaMemcpyHostToDevice); cudaMemcpy(dp2, sp2.data(), nn * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto kern, const uint64_t* k, const uint32_t* p, int grid, bool refill) {
    float best = 1e9;
    for (int it = 0; it < 5; it++) {
      if (refill) fill<<<1184, 256>>>(slots, cap * 2);
      cudaEventRecord(a);
      kern<<<grid, 256>>>(k, p, nn, slots, cap - 1, ovf);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
    }
    printf("%-40s grid %5d  %.1f us  (%.2f G items/s)\n", name, grid, best * 1e3, nn / (best * 1e-3) / 1e9);
  };
  for (int g : {148 * 8, 148 * 16, 148 * 32}) {
    run("insert frame-order", ins<0>, dk, dp, g, true);
    run("insert key-sorted", ins<0>, dk2, dp2, g, true);
    run("CAS-only frame-order", ins<2>, dk, dp, g, true);
    run("read-only probe (populated)", ins<1>, dk, dp, g, false);
  }
  printf("items %d, voxels %d, err %s\n", nn, nvox, cudaGetErrorString(cudaGetLastError()));
}
