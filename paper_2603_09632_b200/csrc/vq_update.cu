// Codebook-update kernels: accumulate (vq.py:90-100), EMA (vq.py:103-109),
// dead-code revival (vq.py:173-190) and the reservoir ring (core.py:178-203).
//
// accumulate is bit-identical to bincount + np.add.at: np.add.at adds rows
// into sums[code] sequentially in ascending row order, i.e. one fp64 chain per
// (k, d) starting from +0.0.  We (1) count rows per (tile, code), (2) scan to
// per-(tile, code) offsets, (3) stably scatter row ids into code-sorted order
// (warp match_any ranks, tiles walked in order) and (4) run one chain per
// (k, d) over the sorted row ids: lanes own consecutive d so each row read is
// a coalesced 128-512 B segment.  HBM traffic ~ one read of X + 8 B/row.
#include <algorithm>
#include <cstdlib>

#include "launchers.h"

namespace xgs {

namespace {

constexpr int kTileTarget = 2048;  // number of row tiles (bounds the T x K table)
// block-per-tile path: ~256 tiles of >= 256 rows, 8 warps per tile while the
// per-warp shared counter rows fit (W * K * 4 B <= kScatterSmem)
constexpr int kBlockTileTarget = 256;
constexpr int64_t kScatterSmem = 160 * 1024;
constexpr int64_t kBlockTileMaxK = kScatterSmem / 4;
inline bool block_tiles(int64_t k) { return k <= kBlockTileMaxK; }
inline int scatter_warps(int64_t k) {
  const int64_t w = kScatterSmem / (4 * (k > 0 ? k : 1));
  return (int)(w >= 8 ? 8 : (w < 1 ? 1 : w));
}

struct AccPlan {
  int64_t tile_rows, tiles;
  size_t off_tile_counts, off_code_count, off_code_start, off_sorted, off_order, total;
};

AccPlan acc_plan(int64_t n, int64_t k) {
  AccPlan p;
  int64_t tr;
  if (block_tiles(k)) {
    tr = (n + kBlockTileTarget - 1) / kBlockTileTarget;
    if (tr < 256) tr = 256;
    tr = (tr + 255) / 256 * 256;
  } else {
    tr = (n + kTileTarget - 1) / kTileTarget;
    if (tr < 256) tr = 256;
    tr = (tr + 31) / 32 * 32;
  }
  p.tile_rows = tr;
  p.tiles = n > 0 ? (n + tr - 1) / tr : 1;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o += (bytes + 255) / 256 * 256; return r; };
  p.off_tile_counts = take(sizeof(int32_t) * (size_t)p.tiles * (size_t)k);
  p.off_code_count = take(sizeof(int32_t) * (size_t)k);
  p.off_code_start = take(sizeof(int32_t) * (size_t)(k + 1));
  p.off_sorted = take(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  p.off_order = take(sizeof(int32_t) * (size_t)k);
  p.total = o;
  return p;
}

__device__ __forceinline__ int row_code(const int64_t* codes, const uint8_t* mask, int64_t r) {
  if (mask && !mask[r]) return -1;
  return (int)codes[r];
}

// (1) per-(tile, code) counts; one warp per tile.
__global__ void acc_hist_kernel(const int64_t* __restrict__ codes, const uint8_t* __restrict__ mask,
                                int64_t n, int64_t k, int64_t tile_rows, int32_t* tile_counts) {
  const int64_t t = blockIdx.x;
  const int lane = threadIdx.x;
  int32_t* tc = tile_counts + t * k;
  const int64_t r0 = t * tile_rows, r1 = min(n, r0 + tile_rows);
  for (int64_t base = r0; base < r1; base += 32) {
    const int64_t r = base + lane;
    const int c = r < r1 ? row_code(codes, mask, r) : -1;
    const unsigned peers = __match_any_sync(FULL, c);
    if (c >= 0 && lane == __ffs(peers) - 1) tc[c] += __popc(peers);
    __syncwarp();
  }
}

// (2a) exclusive scan over tiles for 32 codes per block; writes per-code totals.
__global__ void __launch_bounds__(1024)
acc_scan_tiles_kernel(int32_t* tile_counts, int64_t tiles, int64_t k, int32_t* code_count) {
  pdl_wait();
  __shared__ int32_t part[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t code = (int64_t)blockIdx.x * 32 + lane;
  const int64_t per = (tiles + 31) / 32;
  const int64_t t0 = warp * per, t1 = min(tiles, t0 + per);
  int32_t s = 0;
  if (code < k)
    for (int64_t t = t0; t < t1; t++) s += tile_counts[t * k + code];
  part[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    int32_t run = 0;
    for (int w = 0; w < 32; w++) {
      const int32_t v = part[w][lane];
      part[w][lane] = run;
      run += v;
    }
    if (code < k) code_count[code] = run;
  }
  __syncthreads();
  int32_t run = part[warp][lane];
  if (code < k)
    for (int64_t t = t0; t < t1; t++) {
      const int32_t v = tile_counts[t * k + code];
      tile_counts[t * k + code] = run;
      run += v;
    }
}

// (2b) exclusive scan of the K code totals -> code_start[0..K] (one block,
// warp-shuffle scan of per-thread partials).
__global__ void __launch_bounds__(1024)
acc_scan_codes_kernel(const int32_t* __restrict__ code_count, int64_t k, int32_t* code_start) {
  pdl_wait();
  __shared__ int32_t wsum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t per = (k + 1023) / 1024;
  const int64_t c0 = threadIdx.x * per, c1 = min(k, c0 + per);
  int32_t s = 0;
  for (int64_t c = c0; c < c1; c++) s += code_count[c];
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
    if (lane == 31) code_start[k] = wx;
  }
  __syncthreads();
  int32_t run = wsum[warp] + x - s;
  for (int64_t c = c0; c < c1; c++) {
    code_start[c] = run;
    run += code_count[c];
  }
}

// (2c) codes by descending row count (ties by index): the serial chains of the
// biggest codes start first, so the largest code overlaps the rest of the work.
// Counts are staged through shared memory in 4096-code slabs.
__global__ void __launch_bounds__(256)
acc_order_kernel(const int32_t* __restrict__ code_count, int64_t k, int32_t* order) {
  __shared__ int32_t cc[4096];
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t mine = c < k ? code_count[c] : 0;
  int32_t rank = 0;
  for (int64_t j0 = 0; j0 < k; j0 += 4096) {
    const int64_t m = min((int64_t)4096, k - j0);
    __syncthreads();
    for (int64_t j = threadIdx.x; j < m; j += blockDim.x) cc[j] = code_count[j0 + j];
    __syncthreads();
    if (c < k)
      for (int64_t j = 0; j < m; j++) {
        const int32_t o = cc[j];
        rank += (o > mine) || (o == mine && j0 + j < c);
      }
  }
  if (c < k) order[rank] = (int32_t)c;
}

// (3) stable scatter of row ids into code-sorted order; one warp per tile.
__global__ void acc_scatter_kernel(const int64_t* __restrict__ codes, const uint8_t* __restrict__ mask,
                                   int64_t n, int64_t k, int64_t tile_rows, int32_t* tile_off,
                                   const int32_t* __restrict__ code_start, int32_t* sorted) {
  const int64_t t = blockIdx.x;
  const int lane = threadIdx.x;
  int32_t* to = tile_off + t * k;
  const int64_t r0 = t * tile_rows, r1 = min(n, r0 + tile_rows);
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t base = r0; base < r1; base += 32) {
    const int64_t r = base + lane;
    const int c = r < r1 ? row_code(codes, mask, r) : -1;
    const unsigned peers = __match_any_sync(FULL, c);
    if (c >= 0) {
      const int32_t pos = code_start[c] + to[c] + __popc(peers & lt);
      sorted[pos] = (int32_t)r;
    }
    __syncwarp();
    if (c >= 0 && lane == __ffs(peers) - 1) to[c] += __popc(peers);
    __syncwarp();
  }
}

// Block-per-tile variant of (1)-(3) (K <= kBlockTileMaxK): per-tile counters
// live in shared memory instead of global read-modify-write chains, a tile
// is 8 warps wide, and the codes-by-count order is one warp per code.
//
// (1') per-tile code histogram (shared atomics, one add per distinct code per
//      32 rows), written out as one coalesced row of the tile table.
__global__ void __launch_bounds__(256)
acc_hist_block_kernel(const int64_t* __restrict__ codes, const uint8_t* __restrict__ mask, int64_t n, int64_t k,
                      int64_t tile_rows, int32_t* __restrict__ tile_counts) {
  pdl_wait();
  extern __shared__ int32_t cnt[];   // k
  const int64_t t = blockIdx.x;
  for (int64_t c = threadIdx.x; c < k; c += blockDim.x) cnt[c] = 0;
  __syncthreads();
  const int64_t r0 = t * tile_rows, r1 = min(n, r0 + tile_rows);
  const int lane = threadIdx.x & 31;
#pragma unroll 4
  for (int64_t base = r0; base < r1; base += blockDim.x) {
    const int64_t r = base + threadIdx.x;
    const int c = r < r1 ? row_code(codes, mask, r) : -1;
    const unsigned peers = __match_any_sync(FULL, c);
    if (c >= 0 && lane == __ffs(peers) - 1) atomicAdd(&cnt[c], __popc(peers));
  }
  __syncthreads();
  for (int64_t c = threadIdx.x; c < k; c += blockDim.x) tile_counts[t * k + c] = cnt[c];
}

// (2c') codes by descending row count (ties by index), one warp per code.
__global__ void __launch_bounds__(256)
acc_order_warp_kernel(const int32_t* __restrict__ code_count, int64_t k, int32_t* order) {
  pdl_wait();
  __shared__ int32_t cc[4096];
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int32_t mine = c < k ? code_count[c] : 0;
  int32_t rank = 0;
  for (int64_t j0 = 0; j0 < k; j0 += 4096) {
    const int64_t m = min((int64_t)4096, k - j0);
    __syncthreads();
    for (int64_t j = threadIdx.x; j < m; j += blockDim.x) cc[j] = code_count[j0 + j];
    __syncthreads();
    for (int64_t j = lane; j < m; j += 32) {
      const int32_t o = cc[j];
      rank += (o > mine) || (o == mine && j0 + j < c);
    }
  }
  for (int o = 16; o; o >>= 1) rank += __shfl_xor_sync(FULL, rank, o);
  if (c < k && lane == 0) order[rank] = (int32_t)c;
}

// (3') stable scatter, one block per tile: warp w owns the w-th contiguous
// slice of the tile.  Pass 1 counts each slice per code into its own shared
// row; a column scan turns the rows into the slice's first output slot per
// code (code_start + the tile's offset + earlier slices); pass 2 re-walks the
// slice in row order placing each row at slot + its rank among equal codes.
__global__ void acc_scatter_block_kernel(const int64_t* __restrict__ codes, const uint8_t* __restrict__ mask,
                                         int64_t n, int64_t k, int64_t tile_rows,
                                         const int32_t* __restrict__ tile_off, const int32_t* __restrict__ code_start,
                                         int32_t* __restrict__ sorted) {
  pdl_wait();
  extern __shared__ int32_t sc[];   // warps x k
  const int W = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t = blockIdx.x;
  const int64_t r0 = t * tile_rows, r1 = min(n, r0 + tile_rows);
  const int64_t slice = ((tile_rows + W - 1) / W + 31) / 32 * 32;
  const int64_t s0 = min(r1, r0 + warp * slice), s1 = min(r1, s0 + slice);
  int32_t* mine = sc + (int64_t)warp * k;
  for (int64_t i = threadIdx.x; i < (int64_t)W * k; i += blockDim.x) sc[i] = 0;
  __syncthreads();
#pragma unroll 4
  for (int64_t base = s0; base < s1; base += 32) {
    const int64_t r = base + lane;
    const int c = r < s1 ? row_code(codes, mask, r) : -1;
    const unsigned peers = __match_any_sync(FULL, c);
    if (c >= 0 && lane == __ffs(peers) - 1) mine[c] += __popc(peers);
  }
  __syncthreads();
  for (int64_t c = threadIdx.x; c < k; c += blockDim.x) {
    int32_t run = code_start[c] + tile_off[t * k + c];
    for (int w = 0; w < W; w++) {
      const int32_t v = sc[(int64_t)w * k + c];
      sc[(int64_t)w * k + c] = run;
      run += v;
    }
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t base = s0; base < s1; base += 32) {
    const int64_t r = base + lane;
    const int c = r < s1 ? row_code(codes, mask, r) : -1;
    const unsigned peers = __match_any_sync(FULL, c);
    if (c >= 0) sorted[mine[c] + __popc(peers & lt)] = (int32_t)r;
    __syncwarp();
    if (c >= 0 && lane == __ffs(peers) - 1) mine[c] += __popc(peers);
    __syncwarp();
  }
}

// Raw vector loads (no widening) so a warp can keep U rows in flight; the
// loads are volatile asm so ptxas keeps them ahead of the dependent adds.
template <typename X, int VEC>
struct Raw;
template <> struct Raw<float, 2> {
  uint32_t w[2];
  __device__ __forceinline__ void load(const float* p) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.b32 {%0, %1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "l"(p));
  }
  __device__ __forceinline__ void pin() { asm volatile("" : "+r"(w[0]), "+r"(w[1])); }
  __device__ __forceinline__ double get(int i) const { return (double)__uint_as_float(w[i]); }
};
template <> struct Raw<uint16_t, 8> {
  uint32_t w[4];
  __device__ __forceinline__ void load(const uint16_t* p) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "l"(p));
  }
  __device__ __forceinline__ void pin() { asm volatile("" : "+r"(w[0]), "+r"(w[1]), "+r"(w[2]), "+r"(w[3])); }
  __device__ __forceinline__ double get(int i) const {
    return (double)__uint_as_float((i & 1) ? (w[i >> 1] & 0xffff0000u) : (w[i >> 1] << 16));
  }
};
template <> struct Raw<double, 2> {
  double w[2];
  __device__ __forceinline__ void load(const double* p) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(w[0]), "=d"(w[1]) : "l"(p));
  }
  __device__ __forceinline__ void pin() { asm volatile("" : "+d"(w[0]), "+d"(w[1])); }
  __device__ __forceinline__ double get(int i) const { return w[i]; }
};
template <> struct Raw<float, 1> {
  uint32_t w;
  __device__ __forceinline__ void load(const float* p) {
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(w) : "l"(p));
  }
  __device__ __forceinline__ void pin() { asm volatile("" : "+r"(w)); }
  __device__ __forceinline__ double get(int) const { return (double)__uint_as_float(w); }
};
template <> struct Raw<uint16_t, 2> {
  uint32_t w;
  __device__ __forceinline__ void load(const uint16_t* p) {
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(w) : "l"(p));
  }
  __device__ __forceinline__ void pin() { asm volatile("" : "+r"(w)); }
  __device__ __forceinline__ double get(int i) const {
    return (double)__uint_as_float(i ? (w & 0xffff0000u) : (w << 16));
  }
};
template <typename X> struct Raw<X, 1> {
  double w;
  __device__ __forceinline__ void load(const X* p) { w = ld64(p, 0); }
  __device__ __forceinline__ void pin() { asm volatile("" : "+d"(w)); }
  __device__ __forceinline__ double get(int) const { return w; }
};

// (4) one sequential fp64 chain per (k, d): warp = (code, 32*VEC dims).  A
// chain is inherently serial, so a warp's speed is its memory-level
// parallelism: U rows are loaded ahead (U*32*VEC*sizeof(X) bytes in flight per
// warp) before the U dependent adds.
constexpr int kChainWarps = 8;
constexpr int64_t kLongCodes = 32;
template <typename X, int VEC, int U>
__device__ __forceinline__ void chain_run(const X* __restrict__ x, int64_t d, int64_t ldx, int64_t code, int64_t d0,
                                          int lane, const int32_t* __restrict__ code_start,
                                          const int32_t* __restrict__ sorted, double* __restrict__ counts,
                                          double* __restrict__ sums, int cont) {
  static_assert(U <= 32 || U % 32 == 0, "row batch: <= 32 or whole warps of ids");
  constexpr int NI = U > 32 ? U / 32 : 1;   // sorted-index loads per lane per batch
  const bool live = d0 < d;
  const int32_t beg = code_start[code], end = code_start[code + 1];
  double acc[VEC];
#pragma unroll
  for (int v = 0; v < VEC; v++) acc[v] = (cont && live && d0 + v < d) ? sums[code * d + d0 + v] : 0.0;
  const X* xd = x + (live ? d0 : 0);
  int32_t b = beg;
  // the next batch's row ids are loaded one batch ahead, so each batch waits
  // on one memory latency (the row values), not two (ids, then values)
  int32_t rn[NI];
#pragma unroll
  for (int q = 0; q < NI; q++) {
    const int i = q * 32 + lane;
    rn[q] = (i < U && b + i < end) ? __ldg(sorted + b + i) : 0;
  }
  for (; b + U <= end; b += U) {
    Raw<X, VEC> val[U];
    int32_t rows[U];
#pragma unroll
    for (int t = 0; t < U; t++) rows[t] = __shfl_sync(FULL, rn[t >> 5], t & 31);
#pragma unroll
    for (int u = 0; u < U; u++) val[u].load(xd + (int64_t)rows[u] * ldx);
#pragma unroll
    for (int q = 0; q < NI; q++) {
      const int i = q * 32 + lane;
      rn[q] = (i < U && b + U + i < end) ? __ldg(sorted + b + U + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; u++) val[u].pin();   // all U loads issue before the first add
#pragma unroll
    for (int u = 0; u < U; u++)
#pragma unroll
      for (int v = 0; v < VEC; v++) acc[v] = dadd(acc[v], val[u].get(v));
  }
  for (; b < end; b++) {
    Raw<X, VEC> val;
    val.load(xd + (int64_t)sorted[b] * ldx);
#pragma unroll
    for (int v = 0; v < VEC; v++) acc[v] = dadd(acc[v], val.get(v));
  }
  if (live) {
#pragma unroll
    for (int v = 0; v < VEC; v++) sums[code * d + d0 + v] = acc[v];
  }
  if (d0 == 0) counts[code] = (cont ? counts[code] : 0.0) + (double)(end - beg);   // integer-valued: exact
}

// Codes come in descending-count order.  The first n_long codes (the longest
// chains, which bound the kernel) run on the first long_blocks blocks with
// narrower column slices (VL) and twice the rows in flight (UL): fewer
// dependent memory round trips per chain; the rest use (VEC, U).
template <typename X, int VEC, int U, int VL, int UL>
__global__ void __launch_bounds__(kChainWarps * 32, 2)
acc_chain_kernel(const X* __restrict__ x, int64_t d, int64_t ldx, int64_t k,
                 const int32_t* __restrict__ code_start, const int32_t* __restrict__ sorted,
                 const int32_t* __restrict__ order, double* __restrict__ counts, double* __restrict__ sums,
                 int cont, int64_t n_long, unsigned long_blocks) {
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (blockIdx.x < long_blocks) {
    const int64_t gw = (int64_t)blockIdx.x * kChainWarps + warp;
    const int64_t nch = (d + 32 * VL - 1) / (32 * VL);
    if (gw / nch >= n_long) return;
    chain_run<X, VL, UL>(x, d, ldx, order[gw / nch], (gw % nch) * 32 * VL + (int64_t)lane * VL, lane, code_start,
                         sorted, counts, sums, cont);
  } else {
    const int64_t gw = (int64_t)(blockIdx.x - long_blocks) * kChainWarps + warp;
    const int64_t nch = (d + 32 * VEC - 1) / (32 * VEC);
    if (gw / nch >= k - n_long) return;
    chain_run<X, VEC, U>(x, d, ldx, order[n_long + gw / nch], (gw % nch) * 32 * VEC + (int64_t)lane * VEC, lane,
                         code_start, sorted, counts, sums, cont);
  }
}

// Small batches (n <= kSmallRows, e.g. the per-frame C4 stream): one launch,
// one warp per (code, group of kSmallG 32-dim chunks) walking the rows in
// ascending order, 256 at a time (each lane reads 8 codes, eight ballots mark
// the rows of the warp's code, the set bits are added lowest first) -- the same
// per-(k, d) sequential chains in row order (np.add.at) without the
// counting-sort kernels.  Each hit row costs the warp one load latency (the
// chain is serial), so the path stays for batches of at most 1024 rows: with
// a device-side row count over a 16K-row window (the C4 graph) it measured
// 0.189 vs 0.177 ms per frame against the counting sort.
constexpr int64_t kSmallRows = 1024;
constexpr int kSmallG = 8;
template <typename X>
__global__ void __launch_bounds__(256)
acc_small_kernel(const X* __restrict__ x, int64_t n, int64_t d, int64_t ldx, const int64_t* __restrict__ codes,
                 const uint8_t* __restrict__ mask, int64_t k, double* __restrict__ counts, double* __restrict__ sums,
                 int cont) {
  const int lane = threadIdx.x & 31;
  const int64_t groups = ((d + 31) / 32 + kSmallG - 1) / kSmallG;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= k * groups) return;   // warp-uniform
  const int64_t code = w / groups, j0 = (w - code * groups) * kSmallG * 32 + lane;
  const int64_t nn = n;
  double acc[kSmallG];
#pragma unroll
  for (int c = 0; c < kSmallG; c++) acc[c] = (cont && j0 + 32 * c < d) ? sums[code * d + j0 + 32 * c] : 0.0;
  int64_t cnt = 0;
  for (int64_t r0 = 0; r0 < nn; r0 += 256) {
    unsigned b[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int64_t r = r0 + 32 * u + lane;
      b[u] = __ballot_sync(0xffffffffu, r < nn && row_code(codes, mask, r) == (int)code);
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      cnt += __popc(b[u]);
      while (b[u]) {
        const int i = __ffs(b[u]) - 1;
        b[u] &= b[u] - 1;
        const X* row = x + (r0 + 32 * u + i) * ldx;
#pragma unroll
        for (int c = 0; c < kSmallG; c++)
          if (j0 + 32 * c < d) acc[c] = dadd(acc[c], ld64(row, j0 + 32 * c));
      }
    }
  }
#pragma unroll
  for (int c = 0; c < kSmallG; c++)
    if (j0 + 32 * c < d) sums[code * d + j0 + 32 * c] = acc[c];
  if (j0 == 0) counts[code] = (cont ? counts[code] : 0.0) + (double)cnt;
}

template <typename X, int VEC, int VL, int UL>
cudaError_t launch_chain(const X* x, int64_t d, int64_t ldx, int64_t k, const int32_t* cs,
                         const int32_t* sorted, const int32_t* order, double* counts, double* sums,
                         cudaStream_t s, int cont) {
  constexpr int U = VEC >= 4 ? 16 : 32;
  // the largest codes take the long-chain path (VL == 0: none)
  // Measured: fp32 rows at C2 (K=1024) are fastest with the larger half of
  // the codes on the long path (chains 0.43 ms with none, 0.39 with 32, 0.37
  // with 512); bf16 rows at the C5 shard (K=4096) with 32 (4.65 ms vs 5.18 at
  // 2048).  XGS_LONG_CODES overrides for tuning.
  static const int64_t long_env = [] {
    const char* e = std::getenv("XGS_LONG_CODES");
    return e ? (int64_t)std::atoll(e) : (int64_t)-1;
  }();
  const int64_t long_codes = long_env >= 0 ? long_env : (sizeof(X) == 4 ? k / 2 : kLongCodes);
  const int64_t n_long = VL > 0 ? (k < long_codes ? k : long_codes) : 0;
  constexpr int VLx = VL > 0 ? VL : VEC, ULx = VL > 0 ? UL : U;
  const int64_t lw = n_long * ((d + 32 * VLx - 1) / (32 * VLx));
  const unsigned lb = (unsigned)((lw + kChainWarps - 1) / kChainWarps);
  const int64_t warps = (k - n_long) * ((d + 32 * VEC - 1) / (32 * VEC));
  ProfScope prof("vq_chain", s);
  count_launches(1);
  return launch_pdl(acc_chain_kernel<X, VEC, U, VLx, ULx>, dim3(lb + (unsigned)((warps + kChainWarps - 1) / kChainWarps)),
                    dim3(kChainWarps * 32), 0, s, x, d, ldx, k, cs, sorted, order, counts, sums, cont, n_long, lb);
}

// EMA (vq.py:103-109): N' = lam*N + (1-lam)*c ; M' = lam*M + (1-lam)*s ;
// E' = M' / (N' + eps).  One CTA per code row; safe in place.
__global__ void ema_kernel(double lam, double oml, double eps, int64_t d, const double* N, const double* M,
                           const double* __restrict__ counts, const double* __restrict__ sums,
                           double* N_out, double* M_out, double* E_out) {
  const int64_t k = blockIdx.x;
  __shared__ double nk;
  if (threadIdx.x == 0) nk = dadd(dmul(lam, N[k]), dmul(oml, counts[k]));
  __syncthreads();
  const double den = dadd(nk, eps);
  for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
    const int64_t e = k * d + j;
    const double m = dadd(dmul(lam, M[e]), dmul(oml, sums[e]));
    M_out[e] = m;
    E_out[e] = ddiv(m, den);
  }
  if (threadIdx.x == 0) N_out[k] = nk;
}

// Revival (vq.py:184-188): M_k = x ; N_k = 1+eps ; E_k = M_k / (N_k + eps).
__global__ void revive_kernel(int64_t d, double n_new, double denom, const double* __restrict__ ring,
                              const int64_t* __restrict__ dead_k, const int64_t* __restrict__ ring_rows,
                              double* N, double* M, double* E) {
  const int64_t i = blockIdx.x;
  const int64_t k = dead_k[i];
  const double* src = ring + ring_rows[i] * d;
  for (int64_t j = threadIdx.x; j < d; j += blockDim.x) {
    const double v = src[j];
    M[k * d + j] = v;
    E[k * d + j] = ddiv(v, denom);
  }
  if (threadIdx.x == 0) N[k] = n_new;
}

template <typename X>
__global__ void ring_write_kernel(const X* __restrict__ x, int64_t ldx, int64_t row0, int64_t d,
                                  double* ring, int64_t cap, int64_t phys0) {
  const int64_t j = blockIdx.x;
  double* dst = ring + ((phys0 + j) % cap) * d;
  const X* src = x + (row0 + j) * ldx;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) dst[i] = ld64(src, i);
}

// The same with the row count and the ring's write position on the device
// (a graph-captured step whose batch size is known only on the device): one
// block per potential row (n_max), rows >= n exit.  n >= cap keeps the last cap
// rows at ring rows [0, cap).  ring_advance_kernel then moves the position.
template <typename X>
__global__ void ring_write_dev_kernel(const X* __restrict__ x, int64_t ldx, const int64_t* __restrict__ n_dev,
                                      int64_t n_max, int64_t d, double* ring, int64_t cap,
                                      const int64_t* __restrict__ start_dev) {
  pdl_wait();
  const int64_t n = min(*n_dev, n_max);
  const int64_t start = *start_dev;
  // rows strided over a bounded grid: n_max (the caller's capacity) is usually
  // far above the frame's n, and a block per potential row paid for the empty ones
  for (int64_t j = max((int64_t)0, n - cap) + blockIdx.x; j < n; j += gridDim.x) {
    const int64_t phys = n >= cap ? j - (n - cap) : (start + j) % cap;
    double* dst = ring + phys * d;
    const X* src = x + j * ldx;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) dst[i] = ld64(src, i);
  }
}

__global__ void ring_advance_kernel(const int64_t* __restrict__ n_dev, int64_t n_max, int64_t cap, int64_t* start_dev) {
  pdl_wait();
  const int64_t n = min(*n_dev, n_max);
  *start_dev = n >= cap ? 0 : (*start_dev + n) % cap;
}

__global__ void gather_rows_kernel(const double* __restrict__ src, int64_t d, const int64_t* __restrict__ rows,
                                   double* dst) {
  const int64_t i = blockIdx.x;
  for (int64_t j = threadIdx.x; j < d; j += blockDim.x) dst[i * d + j] = src[rows[i] * d + j];
}

}  // namespace

size_t accumulate_workspace_bytes(int64_t n, int64_t k) { return acc_plan(n, k).total; }

cudaError_t launch_accumulate(const void* x, int dtype, int64_t n, int64_t d, int64_t ldx,
                              const int64_t* codes, const uint8_t* mask, int64_t k, double* counts,
                              double* sums, void* ws, size_t ws_bytes, int sm_count, cudaStream_t s, int cont) {
  (void)sm_count;
  const AccPlan p = acc_plan(n, k);
  if (ws_bytes < p.total) return cudaErrorInvalidValue;
  char* w = static_cast<char*>(ws);
  int32_t* tile_counts = reinterpret_cast<int32_t*>(w + p.off_tile_counts);
  int32_t* code_count = reinterpret_cast<int32_t*>(w + p.off_code_count);
  int32_t* code_start = reinterpret_cast<int32_t*>(w + p.off_code_start);
  int32_t* sorted = reinterpret_cast<int32_t*>(w + p.off_sorted);
  int32_t* order = reinterpret_cast<int32_t*>(w + p.off_order);
  ProfScope prof("vq_accumulate", s);
  if (n <= kSmallRows) {
    const int64_t warps = k * (((d + 31) / 32 + kSmallG - 1) / kSmallG);
    const unsigned blocks = (unsigned)((warps + 7) / 8);
    switch (dtype) {
      case F32: acc_small_kernel<float><<<blocks, 256, 0, s>>>((const float*)x, n, d, ldx, codes, mask, k, counts, sums, cont); break;
      case F64: acc_small_kernel<double><<<blocks, 256, 0, s>>>((const double*)x, n, d, ldx, codes, mask, k, counts, sums, cont); break;
      default: acc_small_kernel<uint16_t><<<blocks, 256, 0, s>>>((const uint16_t*)x, n, d, ldx, codes, mask, k, counts, sums, cont);
    }
    count_launches(1);
    return cudaGetLastError();
  }
  cudaError_t e;
  if (block_tiles(k)) {
    cudaError_t ea = attr_once(kAttrUpdate, [] {
      cudaError_t r = cudaFuncSetAttribute(acc_hist_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kScatterSmem);
      if (r == cudaSuccess)
        r = cudaFuncSetAttribute(acc_scatter_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kScatterSmem);
      return r;
    });
    if (ea != cudaSuccess) return ea;
    const int W = scatter_warps(k);
    if (n > 0) {
      if ((e = launch_pdl(acc_hist_block_kernel, dim3((unsigned)p.tiles), dim3(256), sizeof(int32_t) * (size_t)k, s,
                          codes, mask, n, k, p.tile_rows, tile_counts)) != cudaSuccess)
        return e;
      count_launches(1);
    } else if ((e = cudaMemsetAsync(tile_counts, 0, sizeof(int32_t) * (size_t)k, s)) != cudaSuccess) {
      return e;
    }
    if ((e = launch_pdl(acc_scan_tiles_kernel, dim3((unsigned)((k + 31) / 32)), dim3(1024), 0, s, tile_counts, p.tiles,
                        k, code_count)) != cudaSuccess)
      return e;
    if ((e = launch_pdl(acc_scan_codes_kernel, dim3(1), dim3(1024), 0, s, (const int32_t*)code_count, k,
                        code_start)) != cudaSuccess)
      return e;
    if ((e = launch_pdl(acc_order_warp_kernel, dim3((unsigned)((k + 7) / 8)), dim3(256), 0, s,
                        (const int32_t*)code_count, k, order)) != cudaSuccess)
      return e;
    count_launches(3);
    if (n > 0) {
      if ((e = launch_pdl(acc_scatter_block_kernel, dim3((unsigned)p.tiles), dim3(32 * W),
                          sizeof(int32_t) * (size_t)W * (size_t)k, s, codes, mask, n, k, p.tile_rows,
                          (const int32_t*)tile_counts, (const int32_t*)code_start, sorted)) != cudaSuccess)
        return e;
      count_launches(1);
    }
  } else {
    if ((e = cudaMemsetAsync(tile_counts, 0, sizeof(int32_t) * (size_t)p.tiles * (size_t)k, s)) != cudaSuccess)
      return e;
    if (n > 0) {
      acc_hist_kernel<<<(unsigned)p.tiles, 32, 0, s>>>(codes, mask, n, k, p.tile_rows, tile_counts); count_launches(1);
    }
    acc_scan_tiles_kernel<<<(unsigned)((k + 31) / 32), 1024, 0, s>>>(tile_counts, p.tiles, k, code_count); count_launches(1);
    acc_scan_codes_kernel<<<1, 1024, 0, s>>>(code_count, k, code_start); count_launches(1);
    acc_order_kernel<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(code_count, k, order); count_launches(1);
    if (n > 0) {
      acc_scatter_kernel<<<(unsigned)p.tiles, 32, 0, s>>>(codes, mask, n, k, p.tile_rows, tile_counts,
                                                          code_start, sorted); count_launches(1);
    }
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const uintptr_t xa = reinterpret_cast<uintptr_t>(x);
  switch (dtype) {
    case F32:
      if (d % 2 == 0 && ldx % 2 == 0 && xa % 8 == 0)
        return launch_chain<float, 2, 1, 64>((const float*)x, d, ldx, k, code_start, sorted, order, counts, sums, s, cont);
      return launch_chain<float, 1, 0, 0>((const float*)x, d, ldx, k, code_start, sorted, order, counts, sums, s, cont);
    case F64:
      if (d % 2 == 0 && ldx % 2 == 0 && xa % 16 == 0)
        return launch_chain<double, 2, 0, 0>((const double*)x, d, ldx, k, code_start, sorted, order, counts, sums, s, cont);
      return launch_chain<double, 1, 0, 0>((const double*)x, d, ldx, k, code_start, sorted, order, counts, sums, s, cont);
    default:
      if (d % 8 == 0 && ldx % 8 == 0 && xa % 16 == 0)
        return launch_chain<uint16_t, 8, 2, 64>((const uint16_t*)x, d, ldx, k, code_start, sorted, order, counts, sums, s, cont);
      return launch_chain<uint16_t, 1, 0, 0>((const uint16_t*)x, d, ldx, k, code_start, sorted, order, counts, sums, s, cont);
  }
}

cudaError_t launch_ema(double lam, double one_minus_lam, double eps, int64_t k, int64_t d, const double* N,
                       const double* M, const double* counts, const double* sums, double* N_out,
                       double* M_out, double* E_out, cudaStream_t s) {
  if (k == 0) return cudaSuccess;
  ProfScope prof("vq_ema", s);
  ema_kernel<<<(unsigned)k, 128, 0, s>>>(lam, one_minus_lam, eps, d, N, M, counts, sums, N_out, M_out, E_out); count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_revive(int64_t k, int64_t d, double n_new, double denom, const double* ring, int64_t cap,
                          const int64_t* dead_k, const int64_t* ring_rows, int64_t n_dead, double* N,
                          double* M, double* E, cudaStream_t s) {
  (void)k;
  (void)cap;
  if (n_dead == 0) return cudaSuccess;
  revive_kernel<<<(unsigned)n_dead, 128, 0, s>>>(d, n_new, denom, ring, dead_k, ring_rows, N, M, E); count_launches(1);
  return cudaGetLastError();
}

constexpr int64_t kRingBlocks = 148 * 8;
cudaError_t launch_ring_write_dev(const void* x, int dtype, int64_t ldx, const int64_t* n_dev, int64_t n_max,
                                  int64_t d, double* ring, int64_t cap, int64_t* start_dev, cudaStream_t s) {
  if (n_max <= 0) return cudaSuccess;
  cudaError_t e;
  switch (dtype) {
    case F32:
      e = launch_pdl(ring_write_dev_kernel<float>, dim3((unsigned)std::min<int64_t>(n_max, kRingBlocks)), dim3(256), 0, s, (const float*)x, ldx, n_dev,
                     n_max, d, ring, cap, (const int64_t*)start_dev);
      break;
    case F64:
      e = launch_pdl(ring_write_dev_kernel<double>, dim3((unsigned)std::min<int64_t>(n_max, kRingBlocks)), dim3(256), 0, s, (const double*)x, ldx,
                     n_dev, n_max, d, ring, cap, (const int64_t*)start_dev);
      break;
    default:
      e = launch_pdl(ring_write_dev_kernel<uint16_t>, dim3((unsigned)std::min<int64_t>(n_max, kRingBlocks)), dim3(256), 0, s, (const uint16_t*)x, ldx,
                     n_dev, n_max, d, ring, cap, (const int64_t*)start_dev);
  }
  if (e != cudaSuccess) return e;
  count_launches(1);
  e = launch_pdl(ring_advance_kernel, dim3(1), dim3(1), 0, s, n_dev, n_max, cap, start_dev);
  count_launches(1);
  return e;
}

cudaError_t launch_ring_write(const void* x, int dtype, int64_t ldx, int64_t row0, int64_t nrows, int64_t d,
                              double* ring, int64_t cap, int64_t phys0, cudaStream_t s) {
  if (nrows == 0) return cudaSuccess;
  switch (dtype) {
    case F32: ring_write_kernel<float><<<(unsigned)nrows, 128, 0, s>>>((const float*)x, ldx, row0, d, ring, cap, phys0); count_launches(1); break;
    case F64: ring_write_kernel<double><<<(unsigned)nrows, 128, 0, s>>>((const double*)x, ldx, row0, d, ring, cap, phys0); count_launches(1); break;
    default: ring_write_kernel<uint16_t><<<(unsigned)nrows, 128, 0, s>>>((const uint16_t*)x, ldx, row0, d, ring, cap, phys0); count_launches(1);
  }
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const double* src, int64_t d, const int64_t* rows, int64_t n, double* dst,
                               cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  gather_rows_kernel<<<(unsigned)n, 128, 0, s>>>(src, d, rows, dst); count_launches(1);
  return cudaGetLastError();
}

}  // namespace xgs
