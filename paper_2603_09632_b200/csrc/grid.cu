// Voxel grid sampling of back-projected RGB-D frames (sm_100a).
//
// Turns a batch of F depth frames into new Gaussians, one per voxel that is
// not yet occupied in the map, in ascending (frame, pixel) order:
//   G1 grid_front_kernel / grid_keys_kernel: depth loads, back-projection in
//                            the reference's operation order (slam.py:594-598),
//                            floor(p / voxel) -> 63-bit biased voxel key; the
//                            fused front end also drops pixels whose left or
//                            upper neighbour has the same key and compacts the
//                            survivors in pixel order;
//   G2' first-pick mode: dd_insert_kernel + dd_scan_kernel, a batch hash table
//                            (per-voxel atomicMin of the pixel id) gives each
//                            voxel's lowest pixel id; the scan runs the map
//                            test and flags new voxels;
//   G2 mean mode (or XGS_GRID_SORT=1): in-house LSD radix sort of (key, pixel
//                            id) on the bbox-relative key (ceil(bits/8) passes
//                            of upsweep / scan / stable downsweep), then
//   G3 grid_select_kernel  : segment heads = lowest pixel id per voxel;
//                            insert-if-absent into the GPU hash set of the map;
//   G4 hash set            : open addressing, 64-bit keys, linear probing,
//                            power-of-two capacity at load <= 1/2;
//   G5 grid_emit_kernel    : pixel-order compaction (exclusive scan of the
//                            new-head flags) and the GaussianField-compatible
//                            outputs (mu, rgb/255, iso scale, depth, feature).
// Semantics are pinned by oracle/grid.py.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "launchers.h"

namespace xgs {

namespace {

constexpr uint64_t KEY_INVALID = ~0ull;
constexpr int64_t KEY_BIAS = 1ll << 20;
constexpr uint64_t EMPTY = ~0ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Insert-if-absent; true when the key was not present before.
__device__ __forceinline__ bool hs_insert(unsigned long long* table, uint64_t mask, uint64_t key) {
  uint64_t h = mix64(key) & mask;
  while (true) {
    const unsigned long long prev = atomicCAS(table + h, (unsigned long long)EMPTY, (unsigned long long)key);
    if (prev == EMPTY) return true;
    if (prev == key) return false;
    h = (h + 1) & mask;
  }
}
// Same result, probing with plain loads first: a key already in the map (most
// segment heads at steady state) costs no atomic; only an empty slot is
// claimed with atomicCAS (a lost race to another key moves on to the next
// slot).  Slots never go back to EMPTY, so a stale non-empty read is exact.
__device__ __forceinline__ bool hs_insert_probe(unsigned long long* table, uint64_t mask, uint64_t key) {
  uint64_t h = mix64(key) & mask;
  while (true) {
    unsigned long long v = __ldcg(table + h);
    if (v == EMPTY) {
      v = atomicCAS(table + h, (unsigned long long)EMPTY, (unsigned long long)key);
      if (v == EMPTY) return true;
    }
    if (v == key) return false;
    h = (h + 1) & mask;
  }
}
__device__ __forceinline__ bool hs_contains(const unsigned long long* table, uint64_t mask, uint64_t key) {
  uint64_t h = mix64(key) & mask;
  while (true) {
    const unsigned long long v = table[h];
    if (v == key) return true;
    if (v == EMPTY) return false;
    h = (h + 1) & mask;
  }
}

struct Cam {
  double fx, fy, cx, cy, voxel, inv_voxel;
};

// slam.py:594-598 with the dgemv FMA order (oracle/oracle.c backproject1).
__device__ __forceinline__ void backproject(const double* __restrict__ R, const double* __restrict__ t, const Cam& c,
                                            double u, double v, double d, double* p) {
  const double c0 = ddiv(dmul(dsub(u, c.cx), d), c.fx);
  const double c1 = ddiv(dmul(dsub(v, c.cy), d), c.fy);
  const double w0 = dsub(c0, t[0]), w1 = dsub(c1, t[1]), w2 = dsub(d, t[2]);
#pragma unroll
  for (int i = 0; i < 3; i++) p[i] = __fma_rn(R[6 + i], w2, __fma_rn(R[3 + i], w1, dmul(R[i], w0)));
}

// floor(RN(p / vs)) without a division in the common case: q = RN(p * RN(1/vs))
// is within 3*2^-53*|p/vs| of RN(p/vs), so unless q lies within that band of an
// integer both floors agree; inside the band fall back to the exact quotient.
__device__ __forceinline__ double floor_div(double p, double vs, double inv) {
  const double q = dmul(p, inv);
  const double f = floor(q);
  const double band = fabs(q) * 1e-15 + 1e-300;
  if (dsub(q, f) > band && dsub(dadd(f, 1.0), q) > band) return f;
  return floor(ddiv(p, vs));
}

__device__ __forceinline__ bool voxel_of(const double* p, double voxel, int64_t* q, double inv) {
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const double f = floor_div(p[a], voxel, inv);
    if (!(f >= -(double)KEY_BIAS && f < (double)KEY_BIAS)) return false;
    q[a] = (int64_t)f + KEY_BIAS;
  }
  return true;
}

// ---------------------------------------------------------------- G1
// One thread per 4 consecutive pixels of a row (float4 depth load when W % 4
// == 0); 32-bit index math (npix < 2^31 is checked by the C ABI).
__global__ void __launch_bounds__(256)
grid_keys_kernel(const float* __restrict__ depth, int64_t npix, int64_t H, int64_t W, int stride,
                 const double* __restrict__ rot, const double* __restrict__ trans, Cam cam,
                 uint64_t* __restrict__ keys, uint32_t* __restrict__ vals, int* bbox, unsigned long long* nvalid,
                 bool vec4) {
  int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
  unsigned cnt = 0;
  const uint32_t HW = (uint32_t)(H * W), Wu = (uint32_t)W, su = (uint32_t)stride;
  const uint32_t nq = (uint32_t)(vec4 ? npix / 4 : npix);
  const int per = vec4 ? 4 : 1;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    float dv[4];
    uint32_t p0;
    if (vec4) {
      const float4 d4 = __ldg(reinterpret_cast<const float4*>(depth) + q);
      dv[0] = d4.x; dv[1] = d4.y; dv[2] = d4.z; dv[3] = d4.w;
      p0 = q * 4;
    } else {
      dv[0] = __ldg(depth + q);
      p0 = q;
    }
    const uint32_t f = p0 / HW, rem = p0 - f * HW;
    const uint32_t u = rem / Wu, v0 = rem - u * Wu;
    const bool row_on = (u % su) == 0;
    const double* R = rot + (size_t)f * 9;
    const double* T = trans + (size_t)f * 3;
    uint64_t kout[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      if (j >= per) break;
      const uint32_t v = v0 + j;
      uint64_t key = KEY_INVALID;
      const float d32 = dv[j];
      if (row_on && (v % su) == 0 && d32 > 0.f) {
        double p[3];
        backproject(R, T, cam, (double)u, (double)v, (double)d32, p);
        int64_t qv[3];
        if (voxel_of(p, cam.voxel, qv, cam.inv_voxel)) {
          key = ((uint64_t)qv[0] << 42) | ((uint64_t)qv[1] << 21) | (uint64_t)qv[2];
#pragma unroll
          for (int a = 0; a < 3; a++) {
            lo[a] = min(lo[a], (int)qv[a]);
            hi[a] = max(hi[a], (int)qv[a]);
          }
          cnt++;
        }
      }
      kout[j] = key;
    }
    if (vec4) {
      reinterpret_cast<ulonglong2*>(keys)[(size_t)q * 2] = make_ulonglong2(kout[0], kout[1]);
      reinterpret_cast<ulonglong2*>(keys)[(size_t)q * 2 + 1] = make_ulonglong2(kout[2], kout[3]);
      if (vals) reinterpret_cast<uint4*>(vals)[q] = make_uint4(p0, p0 + 1, p0 + 2, p0 + 3);
    } else {
      keys[p0] = kout[0];
      if (vals) vals[p0] = p0;
    }
  }
#pragma unroll
  for (int a = 0; a < 3; a++)
    for (int o = 16; o; o >>= 1) {
      lo[a] = min(lo[a], __shfl_xor_sync(FULL, lo[a], o));
      hi[a] = max(hi[a], __shfl_xor_sync(FULL, hi[a], o));
    }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
  if ((threadIdx.x & 31) == 0) {
    if (cnt) {
#pragma unroll
      for (int a = 0; a < 3; a++) {
        atomicMin(bbox + a, lo[a]);
        atomicMax(bbox + 3 + a, hi[a]);
      }
    }
    atomicAdd(nvalid, (unsigned long long)cnt);
  }
}

__global__ void init_bbox_kernel(int* bbox, unsigned long long* nvalid) {
  if (threadIdx.x < 3) {
    bbox[threadIdx.x] = INT_MAX;
    bbox[3 + threadIdx.x] = INT_MIN;
  }
  if (threadIdx.x < 6) nvalid[threadIdx.x] = 0;   // nvalid, nvox, items, and the scratch counters after them
}

// First-pick mode: compact the per-pixel keys before the sort.  A pixel whose
// key equals the previous pixel's (keys[p-1], pixel order) is dropped -- the
// earlier one has the lower pixel id -- and invalid pixels go too.  The
// survivors are written IN PIXEL ORDER by a single-pass decoupled look-back
// over 4096-pixel tiles (dynamic tile ids, so earlier tiles are always in
// flight).  After the stable sort the first item of every voxel segment is
// therefore its lowest pixel id.
constexpr int CT_THREADS = 256, CT_ITEMS = 16, CT_TILE = CT_THREADS * CT_ITEMS;
constexpr unsigned long long LB_AGG = 1ull << 62, LB_PRE = 2ull << 62, LB_VAL = (1ull << 62) - 1;

__global__ void __launch_bounds__(CT_THREADS)
compact_keys_kernel(const uint64_t* __restrict__ kin, int64_t n, int64_t W, uint64_t* __restrict__ kout,
                    uint32_t* __restrict__ vout, unsigned* tile_counter, unsigned long long* status, int64_t ntiles,
                    unsigned long long* n_items) {
  __shared__ unsigned s_tile;
  __shared__ uint32_t wtot[CT_THREADS / 32];
  __shared__ uint32_t s_excl;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const unsigned t = s_tile;
    __syncthreads();
    if (t >= ntiles) break;
    // warp w owns items [tile + w*512, +512), round r covers 32 consecutive items
    const int64_t base = (int64_t)t * CT_TILE + (int64_t)warp * (CT_TILE / 8);
    // drop a pixel whose key equals its left (p-1) or upper (p-W) neighbour's: any
    // earlier pixel of the same voxel may stand in, so the lowest pixel id of
    // every voxel always survives
    uint64_t k[CT_ITEMS], pk[CT_ITEMS], uk[CT_ITEMS];
#pragma unroll
    for (int r = 0; r < CT_ITEMS; r++) {
      const int64_t i = base + r * 32 + lane;
      k[r] = i < n ? __ldg(kin + i) : KEY_INVALID;
      pk[r] = (i > 0 && i <= n) ? __ldg(kin + i - 1) : KEY_INVALID;
      uk[r] = (i >= W && i - W < n) ? __ldg(kin + i - W) : KEY_INVALID;
    }
    uint32_t keep = 0, roff[CT_ITEMS], wsum = 0;
#pragma unroll
    for (int r = 0; r < CT_ITEMS; r++) {
      const bool kp = k[r] != KEY_INVALID && k[r] != pk[r] && k[r] != uk[r];
      const unsigned b = __ballot_sync(FULL, kp);
      roff[r] = wsum + __popc(b & ((1u << lane) - 1u));
      wsum += __popc(b);
      keep |= (kp ? 1u : 0u) << r;
    }
    if (lane == 0) wtot[warp] = wsum;
    __syncthreads();
    if (warp == 0) {
      uint32_t wv = lane < CT_THREADS / 32 ? wtot[lane] : 0, wx = wv;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, wx, o);
        if (lane >= o) wx += y;
      }
      const uint32_t agg = __shfl_sync(FULL, wx, CT_THREADS / 32 - 1);
      if (lane < CT_THREADS / 32) wtot[lane] = wx - wv;   // exclusive warp offsets
      if (lane == 0) {
        unsigned long long excl = 0;
        if (t == 0) {
          atomicExch(status, LB_PRE | agg);
        } else {
          atomicExch(status + t, LB_AGG | agg);
          for (int64_t j = (int64_t)t - 1; j >= 0; j--) {
            unsigned long long sv;
            do {
              sv = *reinterpret_cast<volatile unsigned long long*>(status + j);
            } while ((sv & ~LB_VAL) == 0);
            excl += sv & LB_VAL;
            if (sv & LB_PRE) break;
          }
          atomicExch(status + t, LB_PRE | (excl + agg));
        }
        s_excl = (uint32_t)excl;
        if (t == ntiles - 1) *n_items = excl + agg;
      }
    }
    __syncthreads();
    const uint32_t wbase = s_excl + wtot[warp];
#pragma unroll
    for (int r = 0; r < CT_ITEMS; r++)
      if (keep & (1u << r)) {
        kout[wbase + roff[r]] = k[r];
        vout[wbase + roff[r]] = (uint32_t)(base + r * 32 + lane);
      }
  }
}


// ---------------------------------------------------------------- batch dedup table
// First-pick mode needs only every voxel's lowest pixel id, which a batch
// table {key, min pixel id} produces in any insertion order (one claim per
// voxel, an atomicMin of the pixel id only when the slot's current id is
// larger), so the front end inserts its surviving pixels straight from
// shared memory: no item list is materialised in HBM.
constexpr int kDedupProbe = 256;
// Table slot = 16 bytes {key u64, pixel id u32, pad u32} (all ones = empty),
// so one 16-byte load returns a slot's key and pixel id together (each probe
// costs one L2 sector).  Inserts are issued four per thread with their table
// loads together.

__device__ __forceinline__ ulonglong2 slot_ld(const unsigned long long* slots, uint64_t h) {
  return __ldcg(reinterpret_cast<const ulonglong2*>(slots + 2 * h));
}
__device__ __forceinline__ uint32_t* slot_pid(unsigned long long* slots, uint64_t h) {
  return reinterpret_cast<uint32_t*>(slots + 2 * h + 1);
}

__device__ __forceinline__ uint32_t dd_hash(uint64_t key) {
  uint32_t h = (uint32_t)key * 0x9E3779B1u ^ (uint32_t)(key >> 32) * 0x85EBCA77u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  return h ^ (h >> 13);
}

// finish one insert whose first slot `cur` (at h) was already loaded
__device__ __forceinline__ void dd_insert_finish(unsigned long long* slots, uint64_t mask, uint64_t h, ulonglong2 cur,
                                                 uint64_t key, uint32_t pid, int* overflow) {
  int t = 0;
  for (; t < kDedupProbe; t++) {
    if (cur.x == EMPTY) {
      const unsigned long long prev = atomicCAS(slots + 2 * h, (unsigned long long)EMPTY, (unsigned long long)key);
      cur.x = prev == EMPTY ? key : prev;
    }
    if (cur.x == key) break;
    h = (h + 1) & mask;
    cur = slot_ld(slots, h);
  }
  if (t == kDedupProbe) {
    *overflow = 1;
    return;
  }
  // a stale pid read is >= the slot's current pid (pids only decrease), so
  // skipping the atomic when it is already <= pid is exact
  if ((uint32_t)cur.y > pid) atomicMin(slot_pid(slots, h), pid);
}


// ---------------------------------------------------------------- G1 fused front end
// First-pick mode on W % 4 == 0, W <= 4 * kFrontMaxThreads: keys, left/up dedup
// and ordered compaction in one pass over the depth.  A block owns FK_ROWS rows
// of one frame (thread t = columns 4t..4t+3) plus the row above as the halo,
// and streams over them: per row, each warp compacts its surviving (key,
// column) items into its own shared-memory segment (warp ballots, no block
// barrier), so only the previous row's keys stay in registers.  The segments
// are laid out in (row, warp) = pixel order; after one barrier an exclusive
// scan of the segment counts gives every segment its offset inside the block's
// fixed output slot plus the block's item count.  FRONT_SORT: the sort's
// rekey pass gathers the slots densely (no block waits on another), so the
// items enter the sort in ascending pixel order, exactly as the two-kernel
// path writes them.  FRONT_INSERT (first-pick hash path): each warp inserts its
// segments' items into the batch dedup table instead, densely (no divergence)
// and four table loads in flight per lane; while a block waits on L2 the other
// resident blocks compute, so no item list goes through HBM.  A pixel is dropped when its left neighbour (same warp) or
// upper neighbour has the same key: any earlier pixel of the same voxel may
// stand in, so the lowest pixel id of every voxel always survives (a warp's
// first column keeps its item; the dedup downstream removes the repeat).
//
// Keys are evaluated in fp32 with a rigorous error bound first.  The
// back-projection is regrouped as p_i = d * P_i + Q_i with
//   P_i = R_0i (u - cx)/fx + R_1i (v - cy)/fy + R_2i   (row part + column part)
//   Q_i = -(R_0i t_0 + R_1i t_1 + R_2i t_2)            (per frame)
// and its magnitude bound M_i = d * C_i + D_i, C_i = |R_0i| (|u|+|cx|)/fx +
// |R_1i| (|v|+|cy|)/fy + |R_2i|, D_i = sum_j |R_ji| |t_j|.  Every fp32
// rounding on that path (cx, 1/fx, R and t conversions, the products and
// sums) is bounded by u = 2^-24 times a term of M_i, about 8 of them in total,
// and the reference's fp64 evaluation (slam.py:594-598) is within ~2^-50 M_i
// of exact, so |p32_i - p64_i| <= 2^-20 M_i.  One bound serves the three axes:
// M = d * (max_i Crow_i + max_i Ccol_i) + max_i D_i >= M_i (all pre-scaled by
// 1/voxel), dl = M * (2^-20 * 1.002 + 2^-21) + 2^-40.  With q = p32 / voxel,
// x = RD(q + 2^23 + 2^20) = floor(q) + 2^23 + 2^20 exactly (|q| < 2^20), so
// fl = x - (2^23 + 2^20) and fr = q - fl are exact; if dl < fr < 1 - dl on all
// three axes, floor(p64 / voxel) == fl, and the low 21 bits of x's encoding are
// the biased key field fl + 2^20.  Otherwise (voxel faces, non-finite values,
// out of key range) the pixel takes the exact fp64 path (backproject +
// floor_div), bit-identical to the reference.
constexpr int FK_ROWS = 5;   // rows per front block (A/B at C3 1 cm: 4 0.157, 5 0.151, 6 0.157, 7 0.160 ms)
constexpr int kInsILP = 4;   // table loads in flight per lane in FRONT_INSERT's tail (8: spills, 0.213 vs 0.199 ms)
constexpr int kFrontPend = 256;    // per-block queue of pixels for the exact path (overflow: segment scan)
// thread t covers columns 4t..4t+3 (W <= 4 * kFrontMaxThreads)
constexpr int kFrontMaxThreads = 320;
constexpr int kFrontWarps = kFrontMaxThreads / 32;
constexpr int kPendW = kFrontPend / kFrontWarps;   // FRONT_INSERT: per-warp share of that queue
constexpr int kFrontBlocksPerSM = FK_ROWS <= 6 ? 3 : 2;   // bounded by the staged segments (FK_ROWS * 11.5 KB)
constexpr int kFrontSeg = 128;     // items per (row, warp) segment: the warp's columns
// a segment in shared memory: 128 keys (8 B) then 128 columns inside the warp's span (1 B),
// so item o = seg * 128 + i sits at a compile-time stride from its segment (no block-size math)
constexpr int kSegBytes = kFrontSeg * 9;
constexpr size_t front_smem_bytes(int64_t nw) { return (size_t)FK_ROWS * nw * kSegBytes; }

struct CamF {
  float cx, cy, rfx, rfy, inv_voxel;
};

__device__ __forceinline__ uint64_t key_exact(const double* R, const double* T, const Cam& cam, uint32_t u,
                                              uint32_t v, float d32) {
  double p[3];
  backproject(R, T, cam, (double)u, (double)v, (double)d32, p);
  int64_t q[3];
  if (!voxel_of(p, cam.voxel, q, cam.inv_voxel)) return KEY_INVALID;
  return ((uint64_t)q[0] << 42) | ((uint64_t)q[1] << 21) | (uint64_t)q[2];
}

// sm_100 paired fp32 arithmetic on {lo, hi} = {pixel j, pixel j + 1}
using u64 = unsigned long long;
__device__ __forceinline__ u64 f2(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float lane_of(u64 v, int h) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return h ? b : a;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 add2_rd(u64 a, u64 b) {
  u64 r;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 sub2_rd(u64 a, u64 b) {
  u64 r;
  asm("sub.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
constexpr float kDl = 0x1p-20f * 1.002f + 0x1p-21f;

enum FrontMode : int { FRONT_SORT = 1, FRONT_INSERT = 2 };

// the front end's pre-key -> the packed voxel key (see the keying loop)
__host__ __device__ constexpr uint64_t pre_to_key(uint64_t k) {
  return ((uint64_t)((uint32_t)(k >> 32) - 0x96000u) << 32) | (uint32_t)((uint32_t)k - 0x4B000000u);
}
// staged image of the PEND sentinel (pre_to_key is injective; bit 63 set, so no real key)
constexpr uint64_t kPendStaged = pre_to_key(KEY_INVALID - 1);
__device__ __forceinline__ uint64_t& seg_key(uint8_t* smem, uint32_t o) {
  return *reinterpret_cast<uint64_t*>(smem + (o / kFrontSeg) * kSegBytes + (o % kFrontSeg) * 8);
}
__device__ __forceinline__ uint8_t& seg_col(uint8_t* smem, uint32_t o) {
  return smem[(o / kFrontSeg) * kSegBytes + kFrontSeg * 8 + (o % kFrontSeg)];
}

template <int MODE, int DIAG>
__global__ void __launch_bounds__(kFrontMaxThreads, kFrontBlocksPerSM)
grid_front_kernel(const float* __restrict__ depth, int64_t H, int64_t W, int stride, const double* __restrict__ rot,
                  const double* __restrict__ trans, Cam cam, CamF cf, uint64_t* __restrict__ kout,
                  uint32_t* __restrict__ vout, int* bbox, unsigned long long* cnts, int32_t* __restrict__ block_count,
                  unsigned bid0, unsigned long long* __restrict__ slots, uint64_t mask, int* overflow,
                  bool halo, int csplit) {
  constexpr int diag = DIAG;   // neighbour dedup width (compile time: no per-pixel predicates)
  constexpr bool BOX = MODE == FRONT_SORT;
  constexpr int NR = FK_ROWS;
  constexpr float XB = 9437184.f;   // 2^23 + 2^20
  // PEND marks a pixel the fp32 filter could not decide: it compares unequal to
  // every key (so it and its neighbours are kept) and is resolved exactly below.
  constexpr uint64_t PEND = KEY_INVALID - 1;
  __shared__ float4 s_row[NR + 1];            // per row: P_row (3, pre-scaled) + max_i C_row
  __shared__ float s_frame[8];                // R1 / voxel (3), Q / voxel (3), max_i D_i, max_i |R1| / voxel
  __shared__ uint32_t s_cnt[NR * kFrontWarps];   // segment counts
  __shared__ uint32_t s_off[NR * kFrontWarps];   // their exclusive scan
  __shared__ uint32_t s_run;
  __shared__ int s_box[6];
  __shared__ uint32_t s_npend;
  __shared__ uint32_t s_pend[kFrontPend];     // staged slots of pixels left to the exact path
  extern __shared__ __align__(16) uint8_t front_smem[];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
  const int nseg = NR * nw;
  const uint32_t smem_base = (uint32_t)__cvta_generic_to_shared(front_smem);
  const unsigned bid = bid0 + blockIdx.x;   // bid0: first block of this launch (frame-chunked launches)
  // csplit blocks side by side per row band (FRONT_INSERT): each covers
  // blockDim.x * 4 columns from colbase; shorter blocks shorten the last wave
  const unsigned bb = bid / (unsigned)csplit;
  const uint32_t colbase = (bid % (unsigned)csplit) * blockDim.x * 4;
  const int rbf = (int)((H + NR - 1) / NR);   // row blocks per frame
  const int f = (int)(bb / (unsigned)rbf);
  const int r0 = (int)(bb % (unsigned)rbf) * NR;
  const int nr = (int)min((int64_t)NR, H - r0);
  const double* Rd = rot + (size_t)f * 9;
  const double* Td = trans + (size_t)f * 3;
  const float iv = cf.inv_voxel;
  // ---- per-frame and per-row constants: threads 0..NR the rows, thread NR+1 the frame ----
  if (t <= NR + 1) {
    float R0[3], R1[3], R2[3];
#pragma unroll
    for (int i = 0; i < 3; i++) {
      R0[i] = (float)Rd[i] * iv;
      R1[i] = (float)Rd[3 + i] * iv;
      R2[i] = (float)Rd[6 + i] * iv;
    }
    if (t <= NR) {
      const float uu = (float)(r0 - 1 + t);
      const float ru = (uu - cf.cx) * cf.rfx, bu = (uu + fabsf(cf.cx)) * cf.rfx;
      float4 rc;
      rc.x = fmaf(R0[0], ru, R2[0]);
      rc.y = fmaf(R0[1], ru, R2[1]);
      rc.z = fmaf(R0[2], ru, R2[2]);
      rc.w = fmaxf(fmaxf(fmaf(fabsf(R0[0]), bu, fabsf(R2[0])), fmaf(fabsf(R0[1]), bu, fabsf(R2[1]))),
                   fmaf(fabsf(R0[2]), bu, fabsf(R2[2])));
      s_row[t] = rc;
    } else {
      const float t0 = (float)Td[0], t1 = (float)Td[1], t2 = (float)Td[2];
      float dm = 0.f;
#pragma unroll
      for (int i = 0; i < 3; i++) {
        const float r0f = (float)Rd[i], r1f = (float)Rd[3 + i], r2f = (float)Rd[6 + i];
        s_frame[i] = R1[i];
        s_frame[3 + i] = -fmaf(r2f, t2, fmaf(r1f, t1, r0f * t0)) * iv;
        dm = fmaxf(dm, fmaf(fabsf(r2f), fabsf(t2), fmaf(fabsf(r1f), fabsf(t1), fabsf(r0f) * fabsf(t0))) * iv);
      }
      s_frame[6] = dm;
      s_frame[7] = fmaxf(fmaxf(fabsf(R1[0]), fabsf(R1[1])), fabsf(R1[2]));
      s_npend = 0;
      if (BOX) {
#pragma unroll
        for (int a = 0; a < 6; a++) s_box[a] = a < 3 ? INT_MAX : INT_MIN;
      }
    }
  }
  __syncthreads();
  const uint32_t Wu = (uint32_t)W, su = (uint32_t)stride;
  const uint32_t c0 = colbase + (uint32_t)t * 4;
  unsigned colmask = 0;
  // column parts: P_col_i = R1_i / voxel * cv (fused into the row part per pixel), C_col = max_i |R1_i| / voxel * bv
  float cv[4], Cc[4];
  const float Qs0 = s_frame[3], Qs1 = s_frame[4], Qs2 = s_frame[5], Dmax = s_frame[6];
  const float R10 = s_frame[0], R11 = s_frame[1], R12 = s_frame[2];
  {
    const float A1 = s_frame[7];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const float vv = (float)(c0 + j);
      cv[j] = (vv - cf.cy) * cf.rfy;
      Cc[j] = A1 * ((vv + fabsf(cf.cy)) * cf.rfy);
      if (c0 + j < Wu && (su == 1 || ((c0 + j) % su) == 0)) colmask |= 1u << j;
    }
  }
  const float4* dframe = reinterpret_cast<const float4*>(depth + (size_t)f * H * W);
  const uint32_t w4 = Wu >> 2;
  unsigned cnt = 0;
  uint32_t wpend = 0;   // FRONT_INSERT: this warp's queued pending pixels (warp-uniform)
  // previous row's keys: the halo row's (rr = 0) when it is keyed, else none --
  // without the halo (halo == false, or the frame's first row) the block's first
  // row is deduplicated within the row only (more table inserts, one row fewer keyed)
  uint64_t kp[4] = {KEY_INVALID, KEY_INVALID, KEY_INVALID, KEY_INVALID};
  const int rr0 = (r0 > 0 && halo) ? 0 : 1;
  float4 dn = make_float4(0.f, 0.f, 0.f, 0.f), dn2 = dn;
  // row pointer stepped by one row per iteration (no per-row 64-bit index math);
  // two rows in flight ahead of the one being keyed
  const float4* dptr = dframe + (size_t)(r0 - 1 + rr0) * w4 + colbase / 4 + t;
  if (colmask) {
    dn = __ldg(dptr);
    dptr += w4;
    if (rr0 + 1 <= nr) {
      dn2 = __ldg(dptr);
      dptr += w4;
    }
  }
#pragma unroll 1
  for (int rr = rr0; rr <= nr; rr++) {
    const int r = r0 - 1 + rr;
    const float4 d4 = dn;
    dn = dn2;
    if (rr + 1 < nr && colmask) {
      dn2 = __ldg(dptr);
      dptr += w4;
    }
    const unsigned rowmask = (r >= 0 && (su == 1 || ((uint32_t)r % su) == 0)) ? colmask : 0u;
    const float4 rc = s_row[rr];
    const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
    uint64_t k[4];
    unsigned vb = 0, pb = 0;   // per column j: valid pixel / left to the exact path (PEND)
    // two pixels per instruction (sm_100 paired fp32: FFMA2 / FADD2, IEEE per lane,
    // same roundings as the scalar expressions in the comments)
#pragma unroll
    for (int jp = 0; jp < 4; jp += 2) {
      const u64 d2 = f2(dv[jp], dv[jp + 1]);
      const u64 M = fma2(d2, add2(f2(rc.w, rc.w), f2(Cc[jp], Cc[jp + 1])), f2(Dmax, Dmax));   // d*(Crow+Ccol)+Dmax
      const u64 dl = fma2(M, f2(kDl, kDl), f2(0x1p-40f, 0x1p-40f));
      const u64 omd = sub2_rd(f2(1.f, 1.f), dl);                                               // RD(1 - dl)
      const u64 cv2 = f2(cv[jp], cv[jp + 1]);
      const u64 q0 = fma2(d2, fma2(f2(R10, R10), cv2, f2(rc.x, rc.x)), f2(Qs0, Qs0));          // d*(R1*cv+Prow)+Q
      const u64 q1 = fma2(d2, fma2(f2(R11, R11), cv2, f2(rc.y, rc.y)), f2(Qs1, Qs1));
      const u64 q2 = fma2(d2, fma2(f2(R12, R12), cv2, f2(rc.z, rc.z)), f2(Qs2, Qs2));
      const u64 xb = f2(XB, XB);
      const u64 x0 = add2_rd(q0, xb), x1 = add2_rd(q1, xb), x2 = add2_rd(q2, xb);             // floor(q) + XB
      const u64 g0 = sub2(q0, sub2(x0, xb)), g1 = sub2(q1, sub2(x1, xb)), g2 = sub2(q2, sub2(x2, xb));  // exact fractions
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int j = jp + h;
        const float f0 = lane_of(g0, h), f1 = lane_of(g1, h), f2v = lane_of(g2, h);
        const float lo = fminf(fminf(f0, f1), f2v), hi = fmaxf(fmaxf(f0, f1), f2v);
        const bool valid = ((rowmask >> j) & 1u) && dv[j] > 0.f;
        const bool ok = lane_of(M, h) < 1048000.f && lo > lane_of(dl, h) && hi < lane_of(omd, h);
        // pre-key: the key packing without masking the constant exponent bits
        // of x = b + 2^23 + 2^20 (bits(x) = 0x4B000000 + b): lo = key_lo +
        // 0x4B000000, hi = key_hi + 0x96000 (each mod 2^32) -- injective, so
        // the neighbour dedup compares pre-keys; staging converts (pre_to_key)
        const uint32_t u0 = __float_as_uint(lane_of(x0, h)), u1 = __float_as_uint(lane_of(x1, h)),
                       u2 = __float_as_uint(lane_of(x2, h));
        const uint64_t key = ((uint64_t)(u0 * 1024u + (u1 >> 11)) << 32) | (uint64_t)(u1 * 0x200000u + u2);
        k[j] = !valid ? KEY_INVALID : ok ? key : PEND;
        vb |= valid ? 1u << j : 0u;
        pb |= (valid && !ok) ? 1u << j : 0u;
      }
    }
    if (rr > 0) {
      // ---- left/up dedup, warp-local compaction into segment (row, warp) ----
      // A pixel may be dropped when ANY earlier pixel of the frame carries its
      // key (that pixel, or the one it was dropped for, stands in; the
      // voxel's lowest pixel id never has one): left and upper neighbours,
      // plus -- `diag` -- the upper-left / upper-right diagonals, which catch
      // most of the repeats the depth noise scatters around voxel faces.
      const uint64_t left = __shfl_up_sync(FULL, k[3], 1);
      uint64_t ul = KEY_INVALID, ur = KEY_INVALID;
      if (diag) {
        ul = __shfl_up_sync(FULL, kp[3], 1);
        ur = __shfl_down_sync(FULL, kp[0], 1);
        if (lane == 0) ul = KEY_INVALID;
        if (lane == 31) ur = KEY_INVALID;
      }
      // wide (diag > 1): also the pixels two columns away in this row (left) and
      // in the row above (both sides) -- still only the two rows held in registers
      uint64_t ll = KEY_INVALID, ul2 = KEY_INVALID, ur2 = KEY_INVALID;
      if (diag > 1) {
        ll = __shfl_up_sync(FULL, k[2], 1);
        ul2 = __shfl_up_sync(FULL, kp[2], 1);
        ur2 = __shfl_down_sync(FULL, kp[1], 1);
        if (lane == 0) ll = ul2 = KEY_INVALID;
        if (lane == 31) ur2 = KEY_INVALID;
      }
      cnt += __popc(vb & ~pb);
      unsigned dupm = 0;
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const uint64_t kk = k[j];
        const uint64_t lk = j == 0 ? (lane > 0 ? left : KEY_INVALID) : k[j - 1];
        bool dup = kk == lk || kk == kp[j];
        if (diag) dup = dup || kk == (j == 0 ? ul : kp[j - 1]) || kk == (j == 3 ? ur : kp[j + 1]);
        if (diag > 1) {
          const uint64_t l2 = j == 0 ? ll : j == 1 ? (lane > 0 ? left : KEY_INVALID) : k[j - 2];
          const uint64_t a2 = j == 0 ? ul2 : j == 1 ? ul : kp[j - 2];
          const uint64_t b2 = j == 3 ? ur2 : j == 2 ? ur : kp[j + 2];
          dup = dup || kk == l2 || kk == a2 || kk == b2;
        }
        dupm |= dup ? 1u << j : 0u;
      }
      // kept: valid and not a repeat, or undecided (PEND compares equal to a
      // PEND neighbour above, but is always kept); invalid pixels never
      const unsigned keep = vb & (pb | ~dupm), pend = pb;
      const unsigned lt = (1u << lane) - 1u;
      unsigned below = 0, total = 0;
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const unsigned b = __ballot_sync(FULL, keep & (1u << j));
        below += __popc(b & lt);
        total += __popc(b);
      }
      const int seg = (rr - 1) * nw + warp;
      const uint32_t o0 = (uint32_t)seg * kFrontSeg + below;
      // predicated st.shared (a C++ `if` here becomes four branches that each
      // rematerialise the segment address under the 64-register cap)
      const uint32_t segs = smem_base + (uint32_t)seg * kSegBytes;
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const uint32_t i = below + __popc(keep & ((1u << j) - 1u));
        const uint64_t sv = pre_to_key(k[j]);   // PEND -> kPendStaged
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t"
            "@p st.shared.u64 [%1], %2;\n\t@p st.shared.u8 [%3], %4;\n\t}"
            ::"r"(keep & (1u << j)), "r"(segs + i * 8), "l"(sv), "r"(segs + kFrontSeg * 8 + i),
            "r"((uint32_t)(lane * 4 + j)) : "memory");
      }
      if (__any_sync(FULL, pend)) {   // rare: queue the undecided pixels for the exact path
        if constexpr (MODE == FRONT_INSERT) {
          // the warp's own queue (no block barrier before the inserts)
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const unsigned b = __ballot_sync(FULL, (pend >> j) & 1u);
            const uint32_t pi = wpend + __popc(b & lt);
            if (((pend >> j) & 1u) && pi < (uint32_t)kPendW)
              s_pend[warp * kPendW + pi] = o0 + __popc(keep & ((1u << j) - 1u));
            wpend += __popc(b);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 4; j++)
            if ((pend >> j) & 1u) {
              const uint32_t pi = atomicAdd(&s_npend, 1u);
              if (pi < kFrontPend) s_pend[pi] = o0 + __popc(keep & ((1u << j) - 1u));
            }
        }
      }
      if (lane == 0) s_cnt[seg] = total;
    }
#pragma unroll
    for (int j = 0; j < 4; j++) kp[j] = k[j];
  }
  // ---- exact fp64 keys of the pending pixels, one lane each ----
  const uint32_t fbase = (uint32_t)((size_t)f * H * W);
  auto resolve = [&](uint32_t o) {
    const int seg = (int)(o / kFrontSeg);
    const uint32_t u = (uint32_t)(r0 + seg / nw), v = colbase + (uint32_t)(seg % nw) * kFrontSeg +
                                                     seg_col(front_smem, o);
    const uint64_t key = key_exact(Rd, Td, cam, u, v, depth[fbase + u * Wu + v]);
    seg_key(front_smem, o) = key;
    cnt += key != KEY_INVALID ? 1u : 0u;
  };
  if constexpr (MODE == FRONT_INSERT) {
    // each warp resolves its own pending pixels (its queue, or on overflow a
    // scan of its own segments) -- no block barrier
    __syncwarp();
    if (wpend <= (uint32_t)kPendW) {
      for (uint32_t i = lane; i < wpend; i += 32) resolve(s_pend[warp * kPendW + i]);
    } else {
      for (int rr = 0; rr < nr; rr++) {
        const int sg = rr * nw + warp;
        for (uint32_t i = lane; i < s_cnt[sg]; i += 32) {
          const uint32_t o = (uint32_t)sg * kFrontSeg + i;
          if (seg_key(front_smem, o) == kPendStaged) resolve(o);
        }
      }
    }
    __syncwarp();
  } else {
  // rows past the frame's last row: empty segments
  for (int s = nr * nw + t; s < nseg; s += blockDim.x) s_cnt[s] = 0;
  __syncthreads();
  {
    const uint32_t np = s_npend;
    if (np <= (uint32_t)kFrontPend) {
      for (uint32_t i = t; i < np; i += blockDim.x) resolve(s_pend[i]);
    } else {
      for (int s = warp; s < nseg; s += nw)
        for (uint32_t i = lane; i < s_cnt[s]; i += 32) {
          const uint32_t o = (uint32_t)s * kFrontSeg + i;
          if (seg_key(front_smem, o) == kPendStaged) resolve(o);
        }
    }
  }
  }
  if (MODE == FRONT_INSERT) {
    // ---- this warp's segments (rows rr, warp) into the batch table ----
    uint32_t segc[NR], tot = 0;
#pragma unroll
    for (int rr = 0; rr < NR; rr++) {
      segc[rr] = rr < nr ? s_cnt[rr * nw + warp] : 0u;
      tot += segc[rr];
    }
    int ovf = 0;
    const uint32_t pcol = fbase + colbase + (uint32_t)warp * kFrontSeg;
    for (uint32_t q0 = lane; q0 < tot; q0 += kInsILP * 32) {
      uint64_t key[kInsILP], h[kInsILP];
      uint32_t pid[kInsILP];
      ulonglong2 cur[kInsILP];
#pragma unroll
      for (int j = 0; j < kInsILP; j++) {
        uint32_t q = q0 + 32 * j;
        key[j] = KEY_INVALID;
        if (q < tot) {
          int rr = 0;
#pragma unroll
          for (int i = 0; i < NR - 1; i++)
            if (rr == i && q >= segc[i]) {
              q -= segc[i];
              rr = i + 1;
            }
          const uint32_t o = (uint32_t)(rr * nw + warp) * kFrontSeg + q;
          key[j] = seg_key(front_smem, o);
          pid[j] = pcol + (uint32_t)(r0 + rr) * Wu + seg_col(front_smem, o);
        }
        if (key[j] != KEY_INVALID) {
          h[j] = dd_hash(key[j]) & mask;
          cur[j] = slot_ld(slots, h[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < kInsILP; j++)
        if (key[j] != KEY_INVALID) dd_insert_finish(slots, mask, h[j], cur[j], key[j], pid[j], &ovf);
    }
    cnt = __reduce_add_sync(FULL, cnt);
    if (lane == 0) {
      if (cnt) atomicAdd(cnts, (unsigned long long)cnt);
      if (tot) atomicAdd(cnts + 2, (unsigned long long)tot);
    }
    if (__any_sync(FULL, ovf) && lane == 0) *overflow = 1;
    return;
  }
  // ---- exclusive scan of the segment counts (warp 0; nseg <= 96) ----
  if (warp == 0) {
    uint32_t v[3], run = 0;
#pragma unroll
    for (int i = 0; i < 3; i++) {
      const int s = lane * 3 + i;
      v[i] = s < nseg ? s_cnt[s] : 0u;
      run += v[i];
    }
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    uint32_t e = x - run;
#pragma unroll
    for (int i = 0; i < 3; i++) {
      const int s = lane * 3 + i;
      if (s < nseg) s_off[s] = e;
      e += v[i];
    }
    if (lane == 31) s_run = x;
  }
  cnt = __reduce_add_sync(FULL, cnt);
  if (lane == 0 && cnt) atomicAdd(cnts, (unsigned long long)cnt);
  __syncthreads();
  const uint32_t run = s_run;
  if (t == 0) {
    block_count[bid] = (int32_t)run;
    if (run) atomicAdd(cnts + 2, (unsigned long long)run);
  }
  // ---- copy out to this block's slot (FK_ROWS * W items), one warp per segment ----
  // Pixels resolved to invalid stay as KEY_INVALID items (they sort last / are
  // skipped by the dedup).  The voxel bounding box over the survivors equals
  // the box over all valid pixels (every dropped pixel repeats a survivor's key).
  const size_t gbase = ((size_t)f * H + r0) * (size_t)W;
  int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
  for (int rr = 0; rr < nr; rr++) {   // the warp copies its own segments
    const int s = rr * nw + warp;
    const uint32_t beg = s_off[s], end = beg + s_cnt[s];
    const uint32_t pbase = fbase + (uint32_t)(r0 + rr) * Wu + (uint32_t)warp * kFrontSeg;
    for (uint32_t i = lane; i < end - beg; i += 32) {
      const uint32_t o = (uint32_t)s * kFrontSeg + i;
      const uint64_t key = seg_key(front_smem, o);
      kout[gbase + beg + i] = key;
      vout[gbase + beg + i] = pbase + seg_col(front_smem, o);
      if (BOX && key != KEY_INVALID) {
        const int q[3] = {(int)(key >> 42), (int)((key >> 21) & 0x1fffff), (int)(key & 0x1fffff)};
#pragma unroll
        for (int a = 0; a < 3; a++) {
          lo[a] = min(lo[a], q[a]);
          hi[a] = max(hi[a], q[a]);
        }
      }
    }
  }
  if (BOX) {
#pragma unroll
    for (int a = 0; a < 3; a++) {
      lo[a] = __reduce_min_sync(FULL, lo[a]);
      hi[a] = __reduce_max_sync(FULL, hi[a]);
    }
    if (lane == 0 && lo[0] != INT_MAX) {
#pragma unroll
      for (int a = 0; a < 3; a++) {
        atomicMin(&s_box[a], lo[a]);
        atomicMax(&s_box[3 + a], hi[a]);
      }
    }
    __syncthreads();
    if (t == 0 && s_box[0] != INT_MAX) {
#pragma unroll
      for (int a = 0; a < 3; a++) {
        atomicMin(bbox + a, s_box[a]);
        atomicMax(bbox + 3 + a, s_box[3 + a]);
      }
    }
  }
}

// ---------------------------------------------------------------- G2 radix sort
// The sort key is the bbox-relative packing of the biased voxel fields:
// rel = ((x-x0) << (by+bz)) | ((y-y0) << bz) | (z-z0); invalid keys map to
// all ones and sort last.  Only the ordering matters (grouping by voxel).
struct RelKey {
  uint32_t x0, y0, z0;
  int by, bz;
  __device__ __forceinline__ uint64_t operator()(uint64_t key) const {
    if (key == KEY_INVALID) return ~0ull;
    const uint64_t m = (1ull << 21) - 1;
    const uint64_t x = (key >> 42) - x0, y = ((key >> 21) & m) - y0, z = (key & m) - z0;
    return (x << (by + bz)) | (y << bz) | z;
  }
};

constexpr int SORT_THREADS = 256;
constexpr int SORT_ITEMS = 16;                       // per thread
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS; // 4096
constexpr int RADIX = 256;
constexpr int STAGE_BYTES_SORT = SORT_TILE * 12;   // u64 keys + u32 values (u32 keys use 8 B)

cudaError_t sort_init();
cudaError_t front_init();

template <typename K>
__global__ void __launch_bounds__(SORT_THREADS)
sort_upsweep_kernel(const K* __restrict__ keys, int64_t n, int shift, int32_t* tile_hist, int64_t tiles) {
  pdl_wait();
  __shared__ int32_t h[8][RADIX];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 8 * RADIX; i += SORT_THREADS) (&h[0][0])[i] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * SORT_TILE + (int64_t)warp * (SORT_TILE / 8);
  K k[SORT_ITEMS];
#pragma unroll
  for (int r = 0; r < SORT_ITEMS; r++) {   // all loads first (memory-level parallelism)
    const int64_t i = base + r * 32 + lane;
    k[r] = i < n ? __ldg(keys + i) : (K)0;
  }
#pragma unroll
  for (int r = 0; r < SORT_ITEMS; r++) {
    const bool ok = base + r * 32 + lane < n;
    const int dg = ok ? (int)((k[r] >> shift) & (RADIX - 1)) : -1;
    const unsigned peers = __match_any_sync(FULL, dg);   // one smem atomic per distinct digit
    if (dg >= 0 && lane == __ffs(peers) - 1) atomicAdd(&h[warp][dg], __popc(peers));
  }
  __syncthreads();
  for (int d = threadIdx.x; d < RADIX; d += SORT_THREADS) {
    int32_t s = 0;
    for (int w = 0; w < 8; w++) s += h[w][d];
    tile_hist[(int64_t)d * tiles + blockIdx.x] = s;   // digit-major
  }
}

// bbox-relative sort keys, computed once before the passes (K = u32 when the
// relative key fits 32 bits: 4-byte keys halve the sort's key traffic)
template <typename K>
__global__ void rekey_kernel(const uint64_t* __restrict__ kin, int64_t n, RelKey rk, K* __restrict__ kout) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    kout[i] = (K)rk(kin[i]);
}

// fused front end: gather the per-block slots densely (block order = pixel
// order) while converting to relative keys; block_off = exclusive scan of the
// block counts, n = total items
template <typename K>
__global__ void rekey_gather_kernel(const uint64_t* __restrict__ slot_k, const uint32_t* __restrict__ slot_v,
                                    const int32_t* __restrict__ block_off, int64_t nblocks, int64_t H, int64_t W,
                                    int64_t n, RelKey rk, K* __restrict__ kout, uint32_t* __restrict__ vout) {
  pdl_wait();
  const int64_t rbf = (H + FK_ROWS - 1) / FK_ROWS;
  for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
    const int64_t o = block_off[b], e = b + 1 < nblocks ? block_off[b + 1] : n;
    const int64_t base = ((b / rbf) * H + (b % rbf) * FK_ROWS) * W;   // the block's first pixel
    const uint64_t* sk = slot_k + base;
    const uint32_t* sv = slot_v + base;
    for (int64_t i = threadIdx.x; i < e - o; i += blockDim.x) {
      kout[o + i] = (K)rk(sk[i]);
      vout[o + i] = sv[i];
    }
  }
}

// back to the biased 63-bit voxel keys after the sort (select / emit use them)
template <typename K>
__global__ void unrekey_kernel(const K* __restrict__ kin, int64_t n, RelKey rk, int bits, uint64_t* __restrict__ kout) {
  pdl_wait();
  const uint64_t all = bits >= 64 ? ~0ull : ((1ull << bits) - 1);
  const uint64_t mz = (1ull << rk.bz) - 1, my = (1ull << rk.by) - 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = (uint64_t)kin[i];
    if ((r & all) == all) {
      kout[i] = KEY_INVALID;
      continue;
    }
    const uint64_t z = (r & mz) + rk.z0, y = ((r >> rk.bz) & my) + rk.y0, x = (r >> (rk.by + rk.bz)) + rk.x0;
    kout[i] = (x << 42) | (y << 21) | z;
  }
}

// Per-digit exclusive scan over the tiles (one CTA per digit): tile offsets
// within the digit plus the digit total; the downsweep adds the digit base
// (exclusive scan of the 256 totals) itself, so a pass has one scan launch.
__global__ void __launch_bounds__(1024)
sort_scan_digits_kernel(int32_t* __restrict__ hist, int64_t tiles, int32_t* __restrict__ digit_tot) {
  pdl_wait();
  __shared__ int32_t sm[32];
  const int d = blockIdx.x;
  int32_t* row = hist + (int64_t)d * tiles;
  const int64_t per = (tiles + blockDim.x - 1) / blockDim.x;
  const int64_t t0 = (int64_t)threadIdx.x * per, t1 = min(tiles, t0 + per);
  int32_t sum = 0;
  for (int64_t t = t0; t < t1; t++) sum += row[t];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t x = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int32_t w = lane < (int)(blockDim.x >> 5) ? sm[lane] : 0, wx = w;
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(FULL, wx, o);
      if (lane >= o) wx += y;
    }
    sm[lane] = wx - w;
    if (lane == 31) digit_tot[d] = wx;
  }
  __syncthreads();
  int32_t run = sm[warp] + x - sum;
  for (int64_t t = t0; t < t1; t++) {
    const int32_t c = row[t];
    row[t] = run;
    run += c;
  }
}

// Stable downsweep: warp w owns tile items [w*512, w*512+512) in input order;
// ranks come from match_any per 32-item round + per-warp digit counters.  The
// tile is then re-ordered by digit in shared memory so the global writes are
// contiguous runs per digit (coalesced) instead of 32 scattered addresses.
template <typename K>
__global__ void __launch_bounds__(SORT_THREADS, 3)
sort_downsweep_kernel(const K* __restrict__ kin, const uint32_t* __restrict__ vin, int64_t n, int shift,
                      const int32_t* __restrict__ scanned, const int32_t* __restrict__ digit_tot, int64_t tiles,
                      K* __restrict__ kout, uint32_t* __restrict__ vout) {
  pdl_wait();
  __shared__ int32_t wc[8][RADIX];
  __shared__ int32_t toff[RADIX];
  __shared__ int32_t gbase[RADIX];
  __shared__ int32_t dbase[RADIX];
  extern __shared__ __align__(16) uint8_t stage_smem[];   // SORT_TILE keys + values (dynamic)
  K* sk = reinterpret_cast<K*>(stage_smem);
  uint32_t* sv = reinterpret_cast<uint32_t*>(stage_smem + SORT_TILE * sizeof(K));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (int i = threadIdx.x; i < 8 * RADIX; i += SORT_THREADS) (&wc[0][0])[i] = 0;
  __syncthreads();
  const int64_t tile0 = (int64_t)blockIdx.x * SORT_TILE;
  const int64_t base = tile0 + (int64_t)warp * (SORT_TILE / 8);
  K k[SORT_ITEMS];
  uint32_t v[SORT_ITEMS];
  int16_t rank[SORT_ITEMS];
  uint8_t dg[SORT_ITEMS];
#pragma unroll
  for (int r = 0; r < SORT_ITEMS; r++) {   // all loads first (memory-level parallelism)
    const int64_t i = base + r * 32 + lane;
    k[r] = i < n ? __ldg(kin + i) : (K)0;
    v[r] = i < n ? __ldg(vin + i) : 0u;
  }
#pragma unroll
  for (int r = 0; r < SORT_ITEMS; r++) {
    const bool ok = base + r * 32 + lane < n;
    const int d = ok ? (int)((k[r] >> shift) & (RADIX - 1)) : -1;
    const unsigned peers = __match_any_sync(FULL, d);
    int rr = -1;
    if (d >= 0) rr = wc[warp][d] + __popc(peers & lt);
    __syncwarp();
    if (d >= 0 && lane == __ffs(peers) - 1) wc[warp][d] += __popc(peers);
    __syncwarp();
    rank[r] = (int16_t)rr;
    dg[r] = (uint8_t)(d < 0 ? 0 : d);
  }
  __syncthreads();
  // per digit: exclusive prefix over warps (input order), tile total, global base
  {
    const int d = threadIdx.x;   // SORT_THREADS == RADIX
    int32_t run = 0;
    for (int w = 0; w < 8; w++) {
      const int32_t c = wc[w][d];
      wc[w][d] = run;
      run += c;
    }
    toff[d] = run;   // tile count of digit d (scanned below)
    gbase[d] = scanned[(int64_t)d * tiles + blockIdx.x];
    dbase[d] = digit_tot[d];
  }
  __syncthreads();
  // digit bases: exclusive scan of the 256 digit totals
  if (warp == 0) {
    int32_t c[8], s2 = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      c[j] = dbase[lane * 8 + j];
      s2 += c[j];
    }
    int32_t x = s2;
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    int32_t run = x - s2;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      dbase[lane * 8 + j] = run;
      run += c[j];
    }
  }
  __syncthreads();
  gbase[threadIdx.x] += dbase[threadIdx.x];
  // exclusive scan of the 256 tile counts -> tile-local digit offsets
  if (warp == 0) {
    int32_t c[8], s = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      c[j] = toff[lane * 8 + j];
      s += c[j];
    }
    int32_t x = s;
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    int32_t run = x - s;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      toff[lane * 8 + j] = run;
      run += c[j];
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < SORT_ITEMS; r++) {
    if (rank[r] >= 0) {
      const int pos = toff[dg[r]] + wc[warp][dg[r]] + rank[r];
      sk[pos] = k[r];
      sv[pos] = v[r];
    }
  }
  __syncthreads();
  const int cnt = (int)min((int64_t)SORT_TILE, n - tile0);
  for (int i = threadIdx.x; i < cnt; i += SORT_THREADS) {
    const K key = sk[i];
    const int d = (int)((key >> shift) & (RADIX - 1));
    const int64_t pos = (int64_t)gbase[d] + (i - toff[d]);
    kout[pos] = key;
    vout[pos] = sv[i];
  }
}

bool sort_forced() {
  const char* force_sort = std::getenv("XGS_GRID_SORT");
  return force_sort && force_sort[0] == '1';
}

cudaError_t front_init() {
  return attr_once(kAttrGridFront, [] {
    const int bytes = (int)front_smem_bytes(kFrontWarps);
    cudaError_t e = cudaFuncSetAttribute(grid_front_kernel<FRONT_SORT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         bytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(grid_front_kernel<FRONT_INSERT, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(grid_front_kernel<FRONT_INSERT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(grid_front_kernel<FRONT_INSERT, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    return e;
  });
}

cudaError_t sort_init() {
  return attr_once(kAttrGridSort, [] {
    cudaError_t e = cudaFuncSetAttribute(sort_downsweep_kernel<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         STAGE_BYTES_SORT);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(sort_downsweep_kernel<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               SORT_TILE * 8);
    return e;
  });
}

// ---------------------------------------------------------------- exclusive scan (int32)
constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <typename T>
__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t* sm, int32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int32_t w = lane < (int)(blockDim.x >> 5) ? sm[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(FULL, w, o);
      if (lane >= o) w += y;
    }
    sm[lane] = w;
  }
  __syncthreads();
  const int32_t before = (warp ? sm[warp - 1] : 0) + x - v;
  *total = sm[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before;
}

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS) scan_reduce_kernel(const T* __restrict__ in, int64_t n, int32_t* sums) {
  pdl_wait();
  __shared__ int32_t sm[32];
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int32_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++)
    if (base + i < n) s += (int32_t)in[base + i];
  int32_t total;
  block_excl_scan<T>(s, sm, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) scan_sums_kernel(int32_t* sums, int64_t nb, int32_t* grand) {
  pdl_wait();
  __shared__ int32_t sm[32];
  const int64_t per = (nb + 1023) / 1024;
  const int64_t b0 = threadIdx.x * per, b1 = min(nb, b0 + per);
  int32_t s = 0;
  for (int64_t b = b0; b < b1; b++) s += sums[b];
  int32_t total;
  int32_t run = block_excl_scan<int32_t>(s, sm, &total);
  for (int64_t b = b0; b < b1; b++) {
    const int32_t c = sums[b];
    sums[b] = run;
    run += c;
  }
  if (threadIdx.x == 0 && grand) *grand = total;
}

template <typename T>
__global__ void __launch_bounds__(SCAN_THREADS)
scan_apply_kernel(const T* __restrict__ in, int64_t n, const int32_t* __restrict__ sums, int32_t* __restrict__ out) {
  pdl_wait();
  __shared__ int32_t sm[32];
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int32_t vals[SCAN_ITEMS];
  int32_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    vals[i] = base + i < n ? (int32_t)in[base + i] : 0;
    s += vals[i];
  }
  int32_t total;
  int32_t run = block_excl_scan<T>(s, sm, &total) + sums[blockIdx.x];
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    if (base + i < n) out[base + i] = run;
    run += vals[i];
  }
}

// one-CTA in-place exclusive scan for short arrays (one launch instead of three)
__global__ void __launch_bounds__(1024) scan_small_kernel(int32_t* a, int64_t n, int32_t* grand) {
  pdl_wait();
  __shared__ int32_t sm[32];
  const int64_t per = (n + 1023) / 1024;
  const int64_t b0 = threadIdx.x * per, b1 = min(n, b0 + per);
  int32_t s = 0;
  for (int64_t b = b0; b < b1; b++) s += a[b];
  int32_t total;
  int32_t run = block_excl_scan<int32_t>(s, sm, &total);
  for (int64_t b = b0; b < b1; b++) {
    const int32_t c = a[b];
    a[b] = run;
    run += c;
  }
  if (threadIdx.x == 0 && grand) *grand = total;
}

template <typename T>
cudaError_t exclusive_scan(const T* in, int64_t n, int32_t* out, int32_t* block_sums, int32_t* grand, cudaStream_t s) {
  const int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (nb == 0) return cudaSuccess;
  if (n <= 65536 && (const void*)in == (const void*)out && sizeof(T) == 4) {
    count_launches(1);
    return launch_pdl(scan_small_kernel, dim3(1), dim3(1024), 0, s, out, n, grand);
  }
  cudaError_t e;
  if ((e = launch_pdl(scan_reduce_kernel<T>, dim3((unsigned)nb), dim3(SCAN_THREADS), 0, s, in, n, block_sums)) !=
      cudaSuccess)
    return e;
  if ((e = launch_pdl(scan_sums_kernel, dim3(1), dim3(1024), 0, s, block_sums, nb, grand)) != cudaSuccess) return e;
  count_launches(3);
  return launch_pdl(scan_apply_kernel<T>, dim3((unsigned)nb), dim3(SCAN_THREADS), 0, s, in, n,
                    (const int32_t*)block_sums, out);
}

// ---------------------------------------------------------------- G3 select
// Over the sorted (key, pid) items: a segment head (first item of a voxel, i.e.
// its lowest pixel id -- the input is in pixel order and the sort is stable)
// inserts its key into the map set; if the key was absent the head pixel is
// flagged new and remembers its sorted position.
__global__ void __launch_bounds__(256)
grid_select_kernel(const uint64_t* __restrict__ k, const uint32_t* __restrict__ v, int64_t n,
                   unsigned long long* table, uint64_t mask, unsigned long long* set_count, unsigned* flag_bits,
                   int32_t* head_pos, unsigned long long* nvox) {
  pdl_wait();
  unsigned newc = 0, vox = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = k[i];
    if (key == KEY_INVALID) continue;
    if (i > 0 && k[i - 1] == key) continue;
    vox++;
    if (hs_insert_probe(table, mask, key)) {
      const uint32_t pid = v[i];
      atomicOr(flag_bits + (pid >> 5), 1u << (pid & 31));
      head_pos[pid] = (int32_t)i;
      newc++;
    }
  }
  for (int o = 16; o; o >>= 1) {
    newc += __shfl_xor_sync(FULL, newc, o);
    vox += __shfl_xor_sync(FULL, vox, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (newc) atomicAdd(set_count, (unsigned long long)newc);
    if (vox) atomicAdd(nvox, (unsigned long long)vox);
  }
}

// ---------------------------------------------------------------- G5 emit
struct EmitArgs {
  const float* depth;
  const uint8_t* color;     // [F*H*W*3] or null
  const double* rot;
  const double* trans;
  Cam cam;
  int64_t H, W;
  int stride, mode;
  double min_scale;
  const float* feat;        // [F, C, Hf, Wf] or null
  int64_t fc, fh, fw;
  const uint64_t* skeys;    // sorted keys / pids (mean mode walks segments)
  const uint32_t* svals;
  int64_t n;
  // outputs
  uint64_t* key;
  int64_t* pid;
  double* mu;
  double* col;
  double* scale;
  double* dep;
  void* ofeat;              // [cap, fc]: float (feat64 == 0) or double
  int feat64;
  double* count;
  int32_t* cell;            // first-pick with features: [cap] feature-map cell of each voxel (emit -> feat kernel)
};

// One new voxel: output row o, representative pixel p (frame * H * W + u * W + v).
__device__ __forceinline__ void emit_one(int64_t o, int64_t p, const int32_t* __restrict__ head_pos,
                                         const EmitArgs& a) {
  const int64_t HW = a.H * a.W;
  const int64_t f = p / HW, rem = p - f * HW;
  const int64_t u = rem / a.W, v = rem - u * a.W;
  const double d = (double)a.depth[p];
  a.dep[o] = d;
  // iso size max(min_scale, 0.5*s*depth/fx)  (slam.py:631)
  const double sz = ddiv(dmul(dmul(0.5, (double)a.stride), d), a.cam.fx);
  a.scale[o] = fmax(a.min_scale, sz);
  if (a.mode == 0) {
    double mu[3];
    backproject(a.rot + f * 9, a.trans + f * 3, a.cam, (double)u, (double)v, d, mu);
    int64_t q[3];
    voxel_of(mu, a.cam.voxel, q, a.cam.inv_voxel);
    a.key[o] = ((uint64_t)q[0] << 42) | ((uint64_t)q[1] << 21) | (uint64_t)q[2];
    for (int c = 0; c < 3; c++) {
      a.mu[o * 3 + c] = mu[c];
      a.col[o * 3 + c] = a.color ? ddiv((double)a.color[p * 3 + c], 255.0) : 0.0;
    }
    if (a.count) a.count[o] = 1.0;
    if (a.cell) {   // the gather rule's cell (supervision.py:133-147), once per voxel for the feature kernel
      const double su = (double)(a.fh - 1), sv = (double)(a.fw - 1);
      const double hu = (double)max(a.H - 1, (int64_t)1), hv = (double)max(a.W - 1, (int64_t)1);
      const int64_t uu = (int64_t)floor(ddiv(dmul((double)u, su), hu) + 0.5);
      const int64_t vv = (int64_t)floor(ddiv(dmul((double)v, sv), hv) + 0.5);
      a.cell[o] = (int32_t)(uu * a.fw + vv);
    }
  } else {
    // mean over the voxel's points in the head's frame, sequential in pid order
    const int64_t i0 = head_pos[p];
    const uint64_t key = a.skeys[i0];
    a.key[o] = key;
    double sm[3] = {0.0, 0.0, 0.0}, sc[3] = {0.0, 0.0, 0.0};
    double cnt = 0.0;
    for (int64_t i = i0; i < a.n && a.skeys[i] == key; i++) {
      const int64_t q = a.svals[i];
      if (q / HW != f) continue;
      const int64_t r2 = q - f * HW;
      const int64_t uq = r2 / a.W, vq = r2 - uq * a.W;
      double mu[3];
      backproject(a.rot + f * 9, a.trans + f * 3, a.cam, (double)uq, (double)vq, (double)a.depth[q], mu);
      for (int c = 0; c < 3; c++) {
        sm[c] = dadd(sm[c], mu[c]);
        if (a.color) sc[c] = dadd(sc[c], ddiv((double)a.color[q * 3 + c], 255.0));
      }
      cnt = dadd(cnt, 1.0);
    }
    for (int c = 0; c < 3; c++) {
      a.mu[o * 3 + c] = ddiv(sm[c], cnt);
      a.col[o * 3 + c] = ddiv(sc[c], cnt);
    }
    if (a.count) a.count[o] = cnt;
  }
}

// One thread per new voxel; the count comes from device memory (the scan's
// total), so the emit is queued before the host reads it back.
__global__ void __launch_bounds__(128)
grid_emit_kernel(const int32_t* __restrict__ head_pos, const int32_t* __restrict__ nnew_dev, int64_t capacity,
                 EmitArgs a) {
  pdl_wait();
  const int64_t nnew = min((int64_t)*nnew_dev, capacity);
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < nnew; o += (int64_t)gridDim.x * blockDim.x)
    emit_one(o, a.pid[o], head_pos, a);
}

// First-pick features with the cells already computed by the emission: a work
// item is 32 voxels x 64 channels.  Lanes gather one channel plane at the 32
// voxels' cells (voxels in pid order sit on nearby cells, so a warp load
// touches few sectors; eight loads in flight per thread), a shared-memory
// transpose, then warps write voxel rows 64 channels wide.  (The thread-per-
// (voxel, channel) kernel below reads 32 planes 19 KB apart per warp load:
// one sector per element.)
constexpr int kFeatTV = 32, kFeatTC = 64;
template <typename T>
__global__ void __launch_bounds__(256)
grid_emit_feat_tile_kernel(const int32_t* __restrict__ nnew_dev, int64_t capacity, EmitArgs a) {
  pdl_wait();
  __shared__ float tile[kFeatTC][kFeatTV + 1];
  const int64_t nnew = min((int64_t)*nnew_dev, capacity);
  const int64_t nch = (a.fc + kFeatTC - 1) / kFeatTC;
  const int64_t items = (nnew + kFeatTV - 1) / kFeatTV * nch;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t HW = a.H * a.W, plane = a.fh * a.fw;
  T* out = static_cast<T*>(a.ofeat);
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t o0 = it / nch * kFeatTV, c0 = it % nch * kFeatTC;
    const int nv = (int)min((int64_t)kFeatTV, nnew - o0);
    int64_t base = 0;
    if (lane < nv) {
      const int64_t p = a.pid[o0 + lane];
      base = p / HW * a.fc * plane + a.cell[o0 + lane];
    }
    float x[kFeatTC / 8];
#pragma unroll
    for (int k = 0; k < kFeatTC / 8; k++) {
      const int64_t c = c0 + warp + 8 * k;
      x[k] = (lane < nv && c < a.fc) ? __ldg(a.feat + base + c * plane) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < kFeatTC / 8; k++) tile[warp + 8 * k][lane] = x[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kFeatTV / 8; k++) {
      const int v = warp + 8 * k;
#pragma unroll
      for (int h = 0; h < kFeatTC / 32; h++) {
        const int64_t c = c0 + 32 * h + lane;
        if (v < nv && c < a.fc) out[(o0 + v) * a.fc + c] = (T)tile[32 * h + lane][v];
      }
    }
    __syncthreads();
  }
}

__global__ void prefix_mask_kernel(const int64_t* __restrict__ n_dev, int64_t cap, uint8_t* __restrict__ mask) {
  pdl_wait();
  const int64_t n = *n_dev;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += (int64_t)gridDim.x * blockDim.x)
    mask[i] = i < n ? 1 : 0;
}

// Per-voxel features (supervision.py:133-147 nearest-lattice gather rule), one
// thread per (new voxel, channel) -- consecutive threads write consecutive
// channels of a row.  First-pick: the representative pixel's value; mean: the
// fp64 sum of the members' gathered values in ascending pid order (the voxel's
// points in the representative's frame, as for mu), / count.  (A thread per
// voxel copying all C channels serialises C strided loads: 0.45 ms for ~2.8K
// voxels x 768 channels at C4.)
__global__ void __launch_bounds__(256)
grid_emit_feat_kernel(const int32_t* __restrict__ head_pos, const int32_t* __restrict__ nnew_dev, int64_t capacity,
                      EmitArgs a) {
  pdl_wait();
  const int64_t nnew = min((int64_t)*nnew_dev, capacity);
  const int64_t total = nnew * a.fc;
  const int64_t HW = a.H * a.W;
  const double su = (double)(a.fh - 1), sv = (double)(a.fw - 1);
  const double hu = (double)max(a.H - 1, (int64_t)1), hv = (double)max(a.W - 1, (int64_t)1);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = i / a.fc, c = i - o * a.fc;
    const int64_t p = a.pid[o];
    const int64_t f = p / HW, rem = p - f * HW;
    const float* plane = a.feat + (f * a.fc + c) * a.fh * a.fw;
    if (a.mode == 0) {
      int64_t cell;
      if (a.cell) {
        cell = a.cell[o];   // computed once per voxel by the emission
      } else {
        const int64_t u = rem / a.W, v = rem - u * a.W;
        const int64_t uu = (int64_t)floor(ddiv(dmul((double)u, su), hu) + 0.5);
        const int64_t vv = (int64_t)floor(ddiv(dmul((double)v, sv), hv) + 0.5);
        cell = uu * a.fw + vv;
      }
      const float x = plane[cell];
      if (a.feat64) static_cast<double*>(a.ofeat)[i] = (double)x;
      else static_cast<float*>(a.ofeat)[i] = x;
    } else {
      const int64_t i0 = head_pos[p];
      const uint64_t key = a.skeys[i0];
      double acc = 0.0, cnt = 0.0;
      for (int64_t j = i0; j < a.n && a.skeys[j] == key; j++) {
        const int64_t q = a.svals[j];
        if (q / HW != f) continue;
        const int64_t r2 = q - f * HW;
        const int64_t uq = r2 / a.W, vq = r2 - uq * a.W;
        const int64_t uu = (int64_t)floor(ddiv(dmul((double)uq, su), hu) + 0.5);
        const int64_t vv = (int64_t)floor(ddiv(dmul((double)vq, sv), hv) + 0.5);
        acc = dadd(acc, (double)plane[uu * a.fw + vv]);
        cnt = dadd(cnt, 1.0);
      }
      static_cast<double*>(a.ofeat)[i] = ddiv(acc, cnt);
    }
  }
}

__global__ void fill_u64_kernel(unsigned long long* p, int64_t n, unsigned long long v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void rehash_kernel(const unsigned long long* old, int64_t oldcap, unsigned long long* table, uint64_t mask) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < oldcap; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = old[i];
    if (k != EMPTY) hs_insert(table, mask, k);
  }
}

__global__ void hs_insert_kernel(unsigned long long* table, uint64_t mask, const uint64_t* keys, int64_t n,
                                 uint8_t* was_new, unsigned long long* count) {
  unsigned c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const bool nw = keys[i] != KEY_INVALID && hs_insert_probe(table, mask, keys[i]);
    if (was_new) was_new[i] = nw;
    c += nw;
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}

__global__ void hs_contains_kernel(const unsigned long long* table, uint64_t mask, const uint64_t* keys, int64_t n,
                                   uint8_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = keys[i] != KEY_INVALID && hs_contains(table, mask, keys[i]);
}

__global__ void backproject_kernel(const double* R, const double* t, Cam cam, const double* u, const double* v,
                                   const double* d, int64_t n, double* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    backproject(R, t, cam, u[i], v[i], d[i], out + 3 * i);
}

// slam.py:654-655 pose_depths: camera z of every centre, pose.transform(mu)[:, 2]
// = (mu @ R.T + t)[:, 2]; the BLAS evaluation is fma(m2,R22, fma(m1,R21, m0*R20))
// + t2 (pinned against the reference on 200,000 points, tests/test_grid_gpu.py).
// `key` (nullable): the ascending order key of z (IEEE total order as uint64)
// for the in-house radix sort -> median.
__global__ void pose_depths_kernel(const double* __restrict__ mu, int64_t n, double R20, double R21, double R22,
                                   double t2, double* __restrict__ z, uint64_t* __restrict__ key,
                                   uint32_t* __restrict__ idx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double* m = mu + 3 * i;
    const double v = dadd(__fma_rn(m[2], R22, __fma_rn(m[1], R21, dmul(m[0], R20))), t2);
    z[i] = v;
    if (key) {
      const uint64_t b = (uint64_t)__double_as_longlong(v);
      key[i] = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
      idx[i] = (uint32_t)i;
    }
  }
}

unsigned grid_blocks(int64_t n, int threads, int sms) {
  int64_t b = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)sms * 16;
  if (b > cap) b = cap;
  return (unsigned)(b < 1 ? 1 : b);
}

int bits_for(int64_t range) {  // bits to hold values 0..range
  int b = 1;
  while ((1ll << b) <= range) b++;
  return b;
}

}  // namespace

// ---------------------------------------------------------------- host API (C++)

struct HashSet {
  unsigned long long* table = nullptr;
  int64_t cap = 0;
  unsigned long long* count_dev = nullptr;
  int64_t count_ub = 0;   // host upper bound of the key count (no sync needed to size the table)
  bool pinned = false;    // an XGS_GRID_ASYNC call used it: a graph may hold the table address, never regrow
};

cudaError_t hashset_create(int64_t capacity, HashSet** out) {
  int64_t cap = 1024;
  while (cap < capacity) cap <<= 1;
  HashSet* h = new HashSet();
  cudaError_t e = cudaMalloc(&h->table, sizeof(unsigned long long) * cap);
  if (e == cudaSuccess) e = cudaMalloc(&h->count_dev, sizeof(unsigned long long));
  if (e != cudaSuccess) {
    cudaFree(h->table);
    delete h;
    return e;
  }
  h->cap = cap;
  fill_u64_kernel<<<grid_blocks(cap, 256, 148), 256>>>(h->table, cap, EMPTY); count_launches(1);
  cudaMemset(h->count_dev, 0, sizeof(unsigned long long));
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return e;
  *out = h;
  return cudaSuccess;
}

void hashset_destroy(HashSet* h) {
  if (!h) return;
  cudaFree(h->table);
  cudaFree(h->count_dev);
  delete h;
}

cudaError_t hashset_size(HashSet* h, int64_t* n, cudaStream_t s) {
  unsigned long long c = 0;
  cudaError_t e = cudaMemcpyAsync(&c, h->count_dev, sizeof(c), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  *n = (int64_t)c;
  return e;
}

// grow so that `extra` more keys keep the load factor <= 1/2
cudaError_t hashset_reserve(HashSet* h, int64_t extra, cudaStream_t s) {
  cudaError_t e;
  if (2 * (h->count_ub + extra) <= h->cap) return cudaSuccess;   // bound suffices: no read-back
  int64_t cur = 0;
  if ((e = hashset_size(h, &cur, s)) != cudaSuccess) return e;
  h->count_ub = cur;
  if (2 * (cur + extra) <= h->cap) return cudaSuccess;
  if (h->pinned) return cudaErrorNotSupported;   // a captured graph would keep using the old table
  int64_t cap = h->cap;
  while (2 * (cur + extra) > cap) cap <<= 1;
  unsigned long long* t = nullptr;
  if ((e = cudaMallocAsync(&t, sizeof(unsigned long long) * cap, s)) != cudaSuccess) return e;
  fill_u64_kernel<<<grid_blocks(cap, 256, 148), 256, 0, s>>>(t, cap, EMPTY); count_launches(1);
  rehash_kernel<<<grid_blocks(h->cap, 256, 148), 256, 0, s>>>(h->table, h->cap, t, (uint64_t)cap - 1); count_launches(1);
  cudaFreeAsync(h->table, s);
  h->table = t;
  h->cap = cap;
  return cudaGetLastError();
}

cudaError_t hashset_insert(HashSet* h, const uint64_t* keys, int64_t n, uint8_t* was_new, cudaStream_t s) {
  cudaError_t e = hashset_reserve(h, n, s);
  if (e != cudaSuccess || n == 0) return e;
  hs_insert_kernel<<<grid_blocks(n, 256, 148), 256, 0, s>>>(h->table, (uint64_t)h->cap - 1, keys, n, was_new,
                                                           h->count_dev); count_launches(1);
  h->count_ub += n;
  return cudaGetLastError();
}

// snapshot / restore: dst takes src's keys (same capacity: the table is copied as is)
cudaError_t hashset_copy(HashSet* dst, const HashSet* src, cudaStream_t s) {
  if (dst->cap != src->cap) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemcpyAsync(dst->table, src->table, sizeof(unsigned long long) * src->cap,
                                  cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(dst->count_dev, src->count_dev, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s);
  dst->count_ub = src->count_ub;
  return e;
}

cudaError_t hashset_contains(HashSet* h, const uint64_t* keys, int64_t n, uint8_t* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  hs_contains_kernel<<<grid_blocks(n, 256, 148), 256, 0, s>>>(h->table, (uint64_t)h->cap - 1, keys, n, out); count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_pose_depths(const double* mu, int64_t n, const double* R9, const double* t3, double* z,
                               uint64_t* key, uint32_t* idx, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  pose_depths_kernel<<<grid_blocks(n, 256, 148), 256, 0, s>>>(mu, n, R9[6], R9[7], R9[8], t3[2], z, key, idx);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_backproject(const double* R, const double* t, const double* intr4, double voxel, const double* u,
                               const double* v, const double* d, int64_t n, double* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  Cam cam{intr4[0], intr4[1], intr4[2], intr4[3], voxel, 1.0 / voxel};
  backproject_kernel<<<grid_blocks(n, 256, 148), 256, 0, s>>>(R, t, cam, u, v, d, n, out); count_launches(1);
  return cudaGetLastError();
}

// LSD passes over bits [0, bits) of K keys (ping-pong k0/k1, v0/v1); on
// return k0/v0 hold the sorted pairs.
template <typename K>
cudaError_t lsd_passes(K*& k0, uint32_t*& v0, K*& k1, uint32_t*& v1, int64_t n, int bits, int32_t* hist,
                       int32_t* ssum, cudaStream_t s) {
  const int64_t tiles = (n + SORT_TILE - 1) / SORT_TILE;
  const int stage = SORT_TILE * (int)(sizeof(K) + 4);
  for (int shift = 0; shift < bits; shift += 8) {
    cudaError_t e;
    if ((e = launch_pdl(sort_upsweep_kernel<K>, dim3((unsigned)tiles), dim3(SORT_THREADS), 0, s, k0, n, shift, hist,
                        tiles)) != cudaSuccess)
      return e;
    if ((e = launch_pdl(sort_scan_digits_kernel, dim3(RADIX), dim3(1024), 0, s, hist, tiles, ssum)) != cudaSuccess)
      return e;
    if ((e = launch_pdl(sort_downsweep_kernel<K>, dim3((unsigned)tiles), dim3(SORT_THREADS), (size_t)stage, s, k0, v0, n,
                        shift, hist, ssum, tiles, k1, v1)) != cudaSuccess)
      return e;
    count_launches(3);
    K* tk = k0; k0 = k1; k1 = tk;
    uint32_t* tv = v0; v0 = v1; v1 = tv;
  }
  return cudaGetLastError();
}

// Workspace layout for one batch of npix pixels.
struct GridWs {
  size_t off_k0, off_v0, off_k1, off_v1, off_hist, off_scan_sums, off_flag, off_pos, off_head, off_lb, off_misc, total;
  int64_t tiles, lb_entries;
};

GridWs grid_ws(int64_t npix) {
  GridWs w;
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o += (b + 255) / 256 * 256; return r; };
  const size_t n = (size_t)(npix > 0 ? npix : 1);
  w.tiles = (npix + SORT_TILE - 1) / SORT_TILE;
  if (w.tiles < 1) w.tiles = 1;
  w.off_k0 = take(n * 8);
  w.off_v0 = take(n * 4);
  w.off_k1 = take(n * 8);
  w.off_v1 = take(n * 4);
  w.off_hist = take((size_t)RADIX * w.tiles * 4);
  const size_t scan_n = n > (size_t)RADIX * w.tiles ? n : (size_t)RADIX * w.tiles;
  size_t ss = ((scan_n + SCAN_TILE - 1) / SCAN_TILE + 1) * 4;
  if (ss < (size_t)RADIX * 4) ss = (size_t)RADIX * 4;   // also the sort's digit totals
  w.off_scan_sums = take(ss);
  w.off_flag = take((n / 32 + 1) * 4);
  w.off_pos = take(n * 4);
  w.off_head = take(n * 4);
  // look-back status: compaction tiles or fused front-end blocks
  w.lb_entries = (int64_t)(n / 16 + 64);
  if (w.lb_entries < (int64_t)(n / CT_TILE + 2)) w.lb_entries = (int64_t)(n / CT_TILE + 2);
  w.off_lb = take((size_t)w.lb_entries * 8);
  w.off_misc = take(256);
  w.total = o;
  return w;
}

size_t grid_workspace_bytes(int64_t npix) { return grid_ws(npix).total; }

// ---------------------------------------------------------------- G2' hash first-pick
// First-pick mode does not need the items in voxel order, only each voxel's
// lowest pixel id: a batch table (open addressing on the voxel key, one
// atomicMin of the pixel id per slot) finds it in one pass over the items
// instead of the radix sort + segment-head select.  Pass 1 claims / finds the
// key's slot and lowers its pixel id; pass 2 scans the table (one occupied
// slot per voxel), runs the map test (insert-if-absent into the occupancy
// set), flags new voxels in the pixel bitmask -- from which the emit stage
// writes the outputs in ascending pixel order exactly as before -- and empties
// the slot, so the table starts every batch empty without a memset.  Probing
// is bounded; an overflow (table too small for the batch's distinct voxels)
// skips pass 2 (the map is untouched) and the host retries with a table sized
// for every item.

// Other frame shapes (W > 4 * kFrontMaxThreads): the per-pixel keys of
// grid_keys_kernel inserted directly (left-neighbour dedup only).
__global__ void __launch_bounds__(256)
dd_insert_pixels_kernel(const uint64_t* __restrict__ keys, int64_t n, int64_t W, unsigned long long* slots,
                        uint64_t mask, unsigned long long* cnts, int* overflow) {
  pdl_wait();
  unsigned nitems = 0;
  int ovf = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = __ldg(keys + i);
    if (key == KEY_INVALID) continue;
    if (i % W != 0 && __ldg(keys + i - 1) == key) continue;
    const uint64_t h = dd_hash(key) & mask;
    dd_insert_finish(slots, mask, h, slot_ld(slots, h), key, (uint32_t)i, &ovf);
    nitems++;
  }
  nitems = __reduce_add_sync(FULL, nitems);
  if ((threadIdx.x & 31) == 0 && nitems) atomicAdd(cnts + 2, (unsigned long long)nitems);
  if (__any_sync(FULL, ovf) && (threadIdx.x & 31) == 0) *overflow = 1;
}

// Pass 2 over the table (each occupied slot = one voxel of the batch with its
// lowest pixel id): map test (insert-if-absent into the occupancy set), new
// voxels flagged in the pixel bitmask, slot emptied for the next batch.  Four
// slots per thread per step with their map probes issued together.  Also
// clears the emission look-back statuses for grid_pidlist_lb_kernel.
constexpr int kScanILP = 8;
constexpr int kMapProbe = 1 << 16;

__global__ void __launch_bounds__(256, 3)
dd_scan_map_kernel(unsigned long long* slots, int64_t cap, const int* overflow, unsigned long long* table,
                   uint64_t tmask, unsigned long long* set_count, unsigned* flag_bits, unsigned long long* nvox,
                   unsigned long long* lb_status, int64_t lb_tiles) {
  pdl_wait();
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = gt; i < lb_tiles; i += gs) lb_status[i] = 0ull;
  unsigned newc = 0, vox = 0;
  for (int64_t h0 = gt; h0 < cap; h0 += kScanILP * gs) {
    ulonglong2 sl[kScanILP];
    uint64_t th[kScanILP];
    unsigned long long tv[kScanILP];
#pragma unroll
    for (int j = 0; j < kScanILP; j++) {
      const int64_t hh = h0 + j * gs;
      sl[j] = hh < cap ? slot_ld(slots, (uint64_t)hh) : make_ulonglong2(EMPTY, EMPTY);
    }
    if (h0 == gt && *(volatile const int*)overflow) return;   // the host resets the whole table
#pragma unroll
    for (int j = 0; j < kScanILP; j++)
      if (sl[j].x != EMPTY) {
        th[j] = mix64(sl[j].x) & tmask;
        tv[j] = __ldcg(table + th[j]);
      }
#pragma unroll
    for (int j = 0; j < kScanILP; j++) {
      if (sl[j].x == EMPTY) continue;
      vox++;
      const uint64_t key = sl[j].x;
      uint64_t hh = th[j];
      unsigned long long v = tv[j];
      bool isnew = false;
      for (int probe = 0;; probe++) {
        if (v == EMPTY) {
          v = atomicCAS(table + hh, (unsigned long long)EMPTY, (unsigned long long)key);
          if (v == EMPTY) {
            isnew = true;
            break;
          }
        }
        if (v == key) break;
        if (probe == kMapProbe) {   // map set (nearly) full: report, never spin
          atomicOr(const_cast<int*>(overflow), 2);
          break;
        }
        hh = (hh + 1) & tmask;
        v = __ldcg(table + hh);
      }
      if (isnew) {
        const uint32_t pid = (uint32_t)sl[j].y;
        atomicOr(flag_bits + (pid >> 5), 1u << (pid & 31));
        newc++;
      }
      *reinterpret_cast<ulonglong2*>(slots + 2 * (h0 + j * gs)) = make_ulonglong2(~0ull, ~0ull);
    }
  }
  newc = __reduce_add_sync(FULL, newc);
  vox = __reduce_add_sync(FULL, vox);
  if ((threadIdx.x & 31) == 0) {
    if (newc) atomicAdd(set_count, (unsigned long long)newc);
    if (vox) atomicAdd(nvox, (unsigned long long)vox);
  }
}

// New-voxel pixel ids in ascending order in ONE pass over the bitmask: each
// block takes the next 2048-word tile (dynamic tile ids, so every earlier tile
// is running or done), reduces its popcounts, finds its output offset by a
// decoupled look-back over the earlier tiles' published sums, writes the set
// bits' pixel ids and clears the words (the bitmask is library-owned and
// starts every batch zeroed).  The last tile publishes the grand total for
// the emit kernel, copies the batch counters into the caller's mapped host
// status words and resets them for the next batch.
constexpr int kLbThreads = 256, kLbFlat = 1024;
// words per thread: 8 (2048-word tiles) when that still gives a tile per SM,
// else 1 (256-word tiles: a single small frame gets tens of blocks, not a few)
__host__ __device__ constexpr int64_t lb_tiles_for(int64_t nwords, int words) {
  return (nwords + (int64_t)kLbThreads * words - 1) / ((int64_t)kLbThreads * words);
}
inline int lb_words_for(int64_t nwords, int sms) { return lb_tiles_for(nwords, 8) >= sms ? 8 : 1; }

template <int kLbWords>
__global__ void __launch_bounds__(kLbThreads)
grid_pidlist_lb_kernel(unsigned* __restrict__ flag_bits, int64_t nwords, unsigned long long* lb_status,
                       unsigned long long* cnts, int64_t capacity, int64_t* __restrict__ pid_out,
                       int32_t* grand, volatile unsigned long long* host_status, int64_t* dev_status, EmitArgs ea,
                       bool fuse) {
  __shared__ unsigned s_tile;
  __shared__ uint32_t s_wsum[kLbThreads / 32];
  __shared__ uint32_t s_base, s_agg;
  pdl_wait();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t == 0) s_tile = atomicAdd(reinterpret_cast<unsigned*>(cnts + 6), 1u);
  __syncthreads();
  constexpr int kLbTile = kLbThreads * kLbWords;
  const int64_t tile = s_tile, ntiles = (nwords + kLbTile - 1) / kLbTile;
  const int64_t w0 = tile * kLbTile + (int64_t)t * kLbWords;
  unsigned w[kLbWords];
  if (kLbWords == 8 && w0 + kLbWords <= nwords) {
    const uint4 a = *reinterpret_cast<const uint4*>(flag_bits + w0), b = *reinterpret_cast<const uint4*>(flag_bits + w0 + 4);
    const unsigned ww[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int j = 0; j < kLbWords; j++) w[j] = ww[j];
    if (a.x | a.y | a.z | a.w) *reinterpret_cast<uint4*>(flag_bits + w0) = make_uint4(0, 0, 0, 0);
    if (b.x | b.y | b.z | b.w) *reinterpret_cast<uint4*>(flag_bits + w0 + 4) = make_uint4(0, 0, 0, 0);
  } else {
#pragma unroll
    for (int j = 0; j < kLbWords; j++) {
      w[j] = w0 + j < nwords ? flag_bits[w0 + j] : 0u;
      if (w[j]) flag_bits[w0 + j] = 0u;
    }
  }
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < kLbWords; j++) c += __popc(w[j]);
  uint32_t x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const uint32_t wv = lane < kLbThreads / 32 ? s_wsum[lane] : 0u;
    uint32_t wx = wv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, wx, o);
      if (lane >= o) wx += y;
    }
    const uint32_t agg = __shfl_sync(FULL, wx, kLbThreads / 32 - 1);
    if (lane < kLbThreads / 32) s_wsum[lane] = wx - wv;
    // look-back: lanes read 32 predecessors at a time.  Up to kLbFlat tiles
    // every tile simply sums ALL its predecessors' aggregates (published as
    // soon as each tile is reduced -- no chain of inclusive prefixes through
    // the tiles of one wave); beyond, the decoupled look-back stops at the
    // nearest inclusive prefix.
    unsigned long long excl = 0;
    if (ntiles <= kLbFlat) {
      if (lane == 0) atomicExch(lb_status + tile, LB_AGG | agg);
      // every lane loads its share of the predecessors at once (up to 32 each)
      unsigned long long v = 0;
      for (int64_t j0 = lane; j0 < tile; j0 += 32 * 8) {
        unsigned long long sv[8];
#pragma unroll
        for (int i = 0; i < 8; i++) {
          const int64_t jj = j0 + 32 * i;
          sv[i] = jj < tile ? *reinterpret_cast<volatile unsigned long long*>(lb_status + jj) : (unsigned long long)(1ull << 62);
        }
#pragma unroll
        for (int i = 0; i < 8; i++) {
          const int64_t jj = j0 + 32 * i;
          while ((sv[i] & ~LB_VAL) == 0) sv[i] = *reinterpret_cast<volatile unsigned long long*>(lb_status + jj);
          v += sv[i] & LB_VAL;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
      excl = v;
    } else if (tile == 0) {
      if (lane == 0) atomicExch(lb_status, LB_PRE | agg);
    } else {
      if (lane == 0) atomicExch(lb_status + tile, LB_AGG | agg);
      int64_t j = tile - 1;
      while (true) {
        const int64_t jj = j - lane;
        unsigned long long sv = 0;
        if (jj >= 0) {
          do {
            sv = *reinterpret_cast<volatile unsigned long long*>(lb_status + jj);
          } while ((sv & ~LB_VAL) == 0);
        }
        const unsigned pre = __ballot_sync(FULL, jj >= 0 && (sv & LB_PRE));
        // lanes up to (and including) the nearest prefix contribute
        const int stop = pre ? __ffs(pre) - 1 : 31;
        unsigned long long v = (lane <= stop && jj >= 0) ? (sv & LB_VAL) : 0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        excl += v;
        if (pre || j - 32 < 0) break;
        j -= 32;
      }
      if (lane == 0) atomicExch(lb_status + tile, LB_PRE | (excl + agg));
    }
    if (lane == 0) {
      s_base = (uint32_t)excl;
      s_agg = agg;
      if (tile == ntiles - 1) {
        const unsigned long long total = excl + agg;
        *grand = (int32_t)total;
        host_status[0] = cnts[0];   // valid pixels
        host_status[1] = cnts[1];   // distinct voxels of the batch
        host_status[2] = cnts[2];   // items inserted / sorted
        host_status[3] = total;     // new voxels
        host_status[4] = cnts[5];   // table overflow flag
        if (dev_status) {
          dev_status[0] = (int64_t)total;
          dev_status[1] = (int64_t)cnts[0];
          dev_status[2] = (int64_t)cnts[1];
          dev_status[3] = (int64_t)(cnts[5] & 0xffffffffull);
        }
        for (int i = 0; i < 7; i++) cnts[i] = 0ull;
        __threadfence_system();
      }
    }
  }
  __syncthreads();
  int64_t o = (int64_t)s_base + s_wsum[warp] + (x - c);
#pragma unroll
  for (int j = 0; j < kLbWords; j++) {
    unsigned word = w[j];
    while (word) {
      const int b = __ffs(word) - 1;
      word &= word - 1;
      if (o < capacity) pid_out[o] = (w0 + j) * 32 + b;
      o++;
    }
  }
  if (fuse) {
    // first-pick emission of this tile's new voxels, spread over the block's
    // threads (the pid list entries the block just wrote): no separate emit launch
    __syncthreads();
    const int64_t beg = s_base, end = min((int64_t)s_base + (int64_t)s_agg, capacity);
    for (int64_t oo = beg + t; oo < end; oo += kLbThreads) emit_one(oo, pid_out[oo], nullptr, ea);
  }
}

// copy stream + events of the host-frame pipeline (per device)
constexpr int kHostChunks = 8;
struct HostCopy {
  bool ready = false;
  cudaStream_t cs = nullptr;
  cudaEvent_t start = nullptr, done = nullptr, chunk[kHostChunks];
};
HostCopy g_hostcopy[16];
std::mutex g_hostcopy_mu;

cudaError_t host_copy_res(HostCopy** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
  HostCopy& h = g_hostcopy[dev];
  if (!h.ready) {
    if ((e = cudaStreamCreateWithFlags(&h.cs, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&h.start, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&h.done, cudaEventDisableTiming)) != cudaSuccess) return e;
    for (int i = 0; i < kHostChunks; i++)
      if ((e = cudaEventCreateWithFlags(&h.chunk[i], cudaEventDisableTiming)) != cudaSuccess) return e;
    h.ready = true;
  }
  *out = &h;
  return cudaSuccess;
}

// Per-device grid state (library-owned; every grid_sample call on the device
// holds g_dedup_mu): the batch dedup table (empty between batches), the
// new-voxel pixel bitmask (zero between batches: the pid-list pass clears the
// words it reads), the emission look-back statuses, the batch counters (reset
// by the last emission tile) and the mapped pinned host status words the last
// tile writes, so a batch ends with one stream synchronisation and no copy.
struct DedupTable {
  unsigned long long* slots = nullptr;   // 2 x cap words
  int64_t cap = 0;
  int64_t last_nvox = -1;
  unsigned* flags = nullptr;             // pixel bitmask words
  int64_t flag_words = 0;
  unsigned long long* lb = nullptr;      // look-back status per emission tile
  int64_t lb_tiles = 0;
  char* misc = nullptr;                  // bbox int[6] at +0, counters u64[8] at +64, grand at +128
  unsigned long long* host_st = nullptr;      // mapped pinned [8]
  unsigned long long* host_st_dev = nullptr;  // its device alias
  bool dirty = false;                    // a batch stopped before its counters were reset
  // set by the first XGS_GRID_ASYNC call: CUDA graphs may hold these buffers'
  // addresses from then on, so a buffer the synchronous path outgrows is
  // retired (kept allocated, never reused) instead of freed, and the batch
  // table is no longer shrunk
  bool pinned = false;
  std::vector<void*> retired;
  void release(void* p) {
    if (!p) return;
    if (pinned) retired.push_back(p);
    else cudaFree(p);
  }
};
constexpr int kDedupDevices = 16;
DedupTable g_dedup[kDedupDevices];
std::mutex g_dedup_mu;

cudaError_t grid_state(int64_t npix, cudaStream_t s, DedupTable** out, bool may_alloc = true) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kDedupDevices) return cudaErrorInvalidDevice;
  DedupTable& t = g_dedup[dev];
  if (!may_alloc && (!t.misc || t.flag_words < (npix + 31) / 32 + 8 || t.dirty || !t.slots))
    return cudaErrorNotSupported;
  if (!t.misc) {
    if ((e = cudaMalloc(&t.misc, 256)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(t.misc, 0, 256, s)) != cudaSuccess) return e;
    if ((e = cudaHostAlloc(reinterpret_cast<void**>(&t.host_st), 64, cudaHostAllocMapped)) != cudaSuccess) return e;
    if ((e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&t.host_st_dev), t.host_st, 0)) != cudaSuccess)
      return e;
  }
  const int64_t nwords = (npix + 31) / 32 + 8;
  if (t.flag_words < nwords) {
    if (t.flags) {
      if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
      t.release(t.flags);
      t.flags = nullptr;
    }
    const int64_t words = nwords + nwords / 4;
    if ((e = cudaMalloc(&t.flags, (size_t)words * 4)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(t.flags, 0, (size_t)words * 4, s)) != cudaSuccess) return e;
    t.flag_words = words;
    const int64_t tiles = lb_tiles_for(words, 1);   // the most tiles any word count per thread needs
    t.release(t.lb);
    if ((e = cudaMalloc(&t.lb, (size_t)tiles * 8)) != cudaSuccess) return e;
    t.lb_tiles = tiles;
  }
  if (t.dirty) {
    if ((e = cudaMemsetAsync(t.misc, 0, 256, s)) != cudaSuccess) return e;
    t.dirty = false;
  }
  *out = &t;
  return cudaSuccess;
}

// Table size: 4x the previous batch's distinct voxels (load <= 1/4 when the
// scene changes slowly), the item count for the first batch (front-end items
// repeat each voxel several times), 2x the item count after an overflow
// (`all`: every item could be a distinct voxel).
cudaError_t dedup_table(DedupTable& t, int64_t nitems, bool all, cudaStream_t s) {
  cudaError_t e;
  const int64_t want = all ? 2 * nitems : (t.last_nvox < 0 ? nitems : 4 * t.last_nvox);
  int64_t cap = 1 << 20;
  while (cap < want) cap <<= 1;
  // keep the table when it is big enough but not over 2x too big (probes stay L2-resident)
  if (t.slots && t.cap >= cap && (t.cap <= 2 * cap || t.pinned)) return cudaSuccess;
  if (t.slots) {
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;   // earlier batches may still use it
    t.release(t.slots);
    t.slots = nullptr;
  }
  if ((e = cudaMalloc(&t.slots, sizeof(unsigned long long) * 2 * cap)) != cudaSuccess) return e;
  t.cap = cap;
  fill_u64_kernel<<<grid_blocks(2 * cap, 256, 148), 256, 0, s>>>(t.slots, 2 * cap, ~0ull); count_launches(1);
  return cudaGetLastError();
}

// per-thread, per-device pinned landing buffer for the final read-back
// (a pageable destination would stage every copy through a driver buffer)
cudaError_t pinned_status(unsigned long long** out) {
  thread_local unsigned long long* buf[16] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 16) return cudaErrorInvalidDevice;
  if (!buf[dev] && (e = cudaHostAlloc(reinterpret_cast<void**>(&buf[dev]), 128, cudaHostAllocDefault)) != cudaSuccess)
    return e;
  *out = buf[dev];
  return cudaSuccess;
}

// G5: new-voxel pixel ids in ascending order (one look-back pass over the
// bitmask) and the GaussianField-compatible outputs (one thread per row, the
// count read from device memory), then the batch's single synchronisation:
// the last emission tile already wrote the counters into mapped host memory.
cudaError_t emit_outputs(const GridIn& in, const Cam& cam, DedupTable* st, const int32_t* head, const uint64_t* sk,
                         const uint32_t* sv, int64_t nitems, GridOut& out, int sms, cudaStream_t s, HostCopy* hcp,
                         bool sync = true) {
  ProfScope prof("grid_emit", s);
  cudaError_t e;
  const int64_t npix = in.frames * in.H * in.W;
  const int64_t nwords = (npix + 31) / 32;
  const int lbw = lb_words_for(nwords, sms);
  const int64_t lb_tiles = lb_tiles_for(nwords, lbw);
  unsigned long long* cnts = reinterpret_cast<unsigned long long*>(st->misc + 64);
  int32_t* grand = reinterpret_cast<int32_t*>(st->misc + 128);
  EmitArgs ea;
  ea.depth = in.depth;
  ea.color = in.color;
  ea.rot = in.rot;
  ea.trans = in.trans;
  ea.cam = cam;
  ea.H = in.H;
  ea.W = in.W;
  ea.stride = in.stride;
  ea.mode = in.mode;
  ea.min_scale = in.min_scale;
  ea.feat = in.feat;
  ea.fc = in.fc;
  ea.fh = in.fh;
  ea.fw = in.fw;
  ea.skeys = sk;
  ea.svals = sv;
  ea.n = nitems;   // mean mode only
  ea.key = out.key;
  ea.pid = out.pid;
  ea.mu = out.mu;
  ea.col = out.color;
  ea.scale = out.scale;
  ea.dep = out.depth;
  ea.ofeat = out.feat;
  ea.feat64 = out.feat64;
  ea.count = out.count;
  // first-pick features: the emission records each voxel's feature-map cell in
  // the (otherwise unused on this path) per-pixel head buffer
  ea.cell = (in.feat && in.mode == 0 && head) ? const_cast<int32_t*>(head) : nullptr;
  // first-pick: the pid-list kernel emits each tile's voxels itself (the colour
  // copy of a host-frame batch is waited for first); mean mode: separate emit
  // (only with at least one look-back tile per SM: a small frame has a few
  // 65K-pixel tiles, whose blocks would emit every voxel between them)
  static const int fe = [] {   // tuning knob, read once: -1 auto, 0 off, 1 on
    const char* v = std::getenv("XGS_GRID_FUSE_EMIT");
    return v ? (v[0] == '0' ? 0 : v[0] == '1' ? 1 : -1) : -1;
  }();
  const bool fuse = in.mode == 0 && fe != 0 && (lb_tiles >= sms || fe == 1);
  if (fuse && hcp && (e = cudaStreamWaitEvent(s, hcp->done, 0)) != cudaSuccess) return e;   // colour
  if ((e = launch_pdl(lbw == 8 ? grid_pidlist_lb_kernel<8> : grid_pidlist_lb_kernel<1>, dim3((unsigned)lb_tiles),
                      dim3(kLbThreads), 0, s, st->flags, nwords,
                      st->lb, cnts, (int64_t)out.capacity, out.pid, grand, st->host_st_dev, out.dev_status, ea,
                      fuse)) != cudaSuccess)
    return e;
  count_launches(1);
  if (!fuse) {
    if (hcp && (e = cudaStreamWaitEvent(s, hcp->done, 0)) != cudaSuccess) return e;   // colour
    if ((e = launch_pdl(grid_emit_kernel, dim3(grid_blocks(out.capacity, 128, sms)), dim3(128), 0, s, head,
                        (const int32_t*)grand, (int64_t)out.capacity, ea)) != cudaSuccess)
      return e;
    count_launches(1);
  }
  if (in.feat && ea.cell) {
    const int64_t items = (out.capacity + kFeatTV - 1) / kFeatTV * ((in.fc + kFeatTC - 1) / kFeatTC);
    const dim3 g((unsigned)std::min<int64_t>(std::max<int64_t>(items, 1), (int64_t)sms * 8));
    e = ea.feat64 ? launch_pdl(grid_emit_feat_tile_kernel<double>, g, dim3(256), 0, s, (const int32_t*)grand,
                               (int64_t)out.capacity, ea)
                  : launch_pdl(grid_emit_feat_tile_kernel<float>, g, dim3(256), 0, s, (const int32_t*)grand,
                               (int64_t)out.capacity, ea);
    if (e != cudaSuccess) return e;
    count_launches(1);
  } else if (in.feat) {
    if ((e = launch_pdl(grid_emit_feat_kernel, dim3(grid_blocks(out.capacity * in.fc, 256, sms)), dim3(256), 0, s,
                        head, (const int32_t*)grand, (int64_t)out.capacity, ea)) != cudaSuccess)
      return e;
    count_launches(1);
  }
  return sync ? cudaStreamSynchronize(s) : cudaGetLastError();
}

cudaError_t launch_prefix_mask(const int64_t* n_dev, int64_t cap, uint8_t* mask, cudaStream_t s) {
  cudaError_t e = launch_pdl(prefix_mask_kernel, dim3(grid_blocks(cap, 256, 148)), dim3(256), 0, s, n_dev, cap, mask);
  count_launches(1);
  return e;
}

cudaError_t grid_sample(const GridIn& in, HashSet* hs, GridOut& out, void* ws, size_t ws_bytes, int sms,
                        cudaStream_t s) {
  const int64_t npix = in.frames * in.H * in.W;
  const GridWs w = grid_ws(npix);
  if (ws_bytes < w.total) return cudaErrorInvalidValue;
  char* b = static_cast<char*>(ws);
  uint64_t* k0 = reinterpret_cast<uint64_t*>(b + w.off_k0);
  uint32_t* v0 = reinterpret_cast<uint32_t*>(b + w.off_v0);
  uint64_t* k1 = reinterpret_cast<uint64_t*>(b + w.off_k1);
  uint32_t* v1 = reinterpret_cast<uint32_t*>(b + w.off_v1);
  int32_t* hist = reinterpret_cast<int32_t*>(b + w.off_hist);
  int32_t* ssum = reinterpret_cast<int32_t*>(b + w.off_scan_sums);
  int32_t* head = reinterpret_cast<int32_t*>(b + w.off_head);
  unsigned long long* lb_status = reinterpret_cast<unsigned long long*>(b + w.off_lb);
  int32_t* block_count = reinterpret_cast<int32_t*>(lb_status);   // fused front end (sort path): per-block item counts
  out.n_new = out.n_valid = out.n_voxels = 0;
  out.n_sorted = out.sort_passes = 0;
  if (npix == 0) return cudaSuccess;
  cudaError_t e;
  std::lock_guard<std::mutex> st_lock(g_dedup_mu);
  ProfScope prof_batch("grid_batch", s);   // device span of the whole call (first launch .. status sync)
  DedupTable* st = nullptr;
  if ((e = grid_state(npix, s, &st, !in.async)) != cudaSuccess) return e;
  int* bbox = reinterpret_cast<int*>(st->misc);
  unsigned long long* cnts = reinterpret_cast<unsigned long long*>(st->misc + 64);   // nvalid, nvox, items, -, -, ovf, tile
  int* overflow = reinterpret_cast<int*>(cnts + 5);
  unsigned* flag = st->flags;
  const Cam cam{in.fx, in.fy, in.cx, in.cy, in.voxel, 1.0 / in.voxel};
  const bool compact = in.mode == 0;   // first-pick
  const int64_t nwords = (npix + 31) / 32;
  const int64_t lb_tiles = lb_tiles_for(nwords, lb_words_for(nwords, sms));
  // Host frames (xgs_grid_sample_h2d): depth is copied frame chunk by frame
  // chunk on a copy stream and each chunk's front-end launch waits only for
  // its own chunk, so the copies of later frames overlap the earlier frames'
  // keys; the colour follows and is waited for before the emit.
  const bool host_frames = in.depth_host != nullptr;
  HostCopy* hcp = nullptr;
  std::unique_lock<std::mutex> hc_lock(g_hostcopy_mu, std::defer_lock);
  struct CopyDone {   // the call returns only after the host frames were read
    HostCopy*& h;
    ~CopyDone() {
      if (h) cudaEventSynchronize(h->done);
    }
  } copy_done{hcp};
  if (host_frames) {
    hc_lock.lock();
    if ((e = host_copy_res(&hcp)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(hcp->start, s)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(hcp->cs, hcp->start, 0)) != cudaSuccess) return e;
  }
  const int64_t fpx = in.H * in.W;
  const int64_t fper = host_frames ? (in.frames + kHostChunks - 1) / kHostChunks : in.frames;
  const int nchunk = (int)((in.frames + fper - 1) / fper);   // every chunk non-empty
  if (host_frames) {
    for (int c = 0; c < nchunk; c++) {
      const int64_t f0 = c * fper, f1 = f0 + fper < in.frames ? f0 + fper : in.frames;
      if ((e = cudaMemcpyAsync(const_cast<float*>(in.depth) + f0 * fpx, in.depth_host + f0 * fpx,
                               sizeof(float) * (size_t)((f1 - f0) * fpx), cudaMemcpyHostToDevice, hcp->cs)) !=
          cudaSuccess)
        return e;
      if ((e = cudaEventRecord(hcp->chunk[c], hcp->cs)) != cudaSuccess) return e;
    }
    if (in.color && in.color_host) {
      if ((e = cudaMemcpyAsync(const_cast<uint8_t*>(in.color), in.color_host, (size_t)(in.frames * fpx * 3),
                               cudaMemcpyHostToDevice, hcp->cs)) != cudaSuccess)
        return e;
    }
    if ((e = cudaEventRecord(hcp->done, hcp->cs)) != cudaSuccess) return e;
  }
  const bool vec4 = (in.W % 4 == 0) && (reinterpret_cast<uintptr_t>(in.depth) % 16 == 0);
  const bool front_ok = vec4 && in.W <= 4 * kFrontMaxThreads;   // the fused front end (float4 rows)
  // first-pick takes the hash path; XGS_GRID_SORT=1 forces the radix sort +
  // select path (mean mode always sorts: its per-voxel sums run in pixel
  // order over the voxel's segment)
  const bool hashed = compact && !sort_forced();
  if (in.async && !hashed) return cudaErrorNotSupported;
  if (in.async) {   // a graph may capture this call: keep the state's buffers alive, never regrow the map
    st->pinned = true;
    hs->pinned = true;
  }
  st->dirty = true;
  if (hashed) {
    // ---------------- G1+G2': front end inserting into the batch table, table scan + map test
    if (!in.async) {   // async: the caller sized the map; the batch table exists (grid_state checked)
      if ((e = dedup_table(*st, npix / 16, false, s)) != cudaSuccess) return e;
      // the scan adds at most one key per occupied batch-table slot (an overflowing
      // batch is redone on a larger table, reserved again below): room for
      // min(pixels, table slots) new keys keeps the map's load <= 1/2 (a bound of
      // one key per pixel grew the C3 map to 64M slots, 512 MB, for 4M keys)
      if ((e = hashset_reserve(hs, std::min<int64_t>(npix, st->cap), s)) != cudaSuccess) return e;
    }
    out.sort_passes = 0;
    const CamF cf{(float)in.cx, (float)in.cy, (float)(1.0 / in.fx), (float)(1.0 / in.fy), (float)(1.0 / in.voxel)};
    if (front_ok && (e = front_init()) != cudaSuccess) return e;
    for (int attempt = 0;; attempt++) {
      const uint64_t mask = (uint64_t)st->cap - 1;
      {
        ProfScope prof("grid_keys", s);
        if (front_ok) {
          const int64_t rbf = (in.H + FK_ROWS - 1) / FK_ROWS;
          // tuning knobs, read once.  Neighbour dedup: 0 left/up, 1 (default) +
          // diagonals, 2 + two columns away.  C3 1 cm: 1 and 2 tie (2 cuts the
          // table inserts 2.82M -> 1.92M but costs three 64-bit compares per
          // pixel); 5 cm, where left/up already catch most repeats: 0.100 (1) vs
          // 0.109 ms (2); C4 unchanged
          static const int diag = [] {
            const char* v = std::getenv("XGS_GRID_DIAG");
            return v ? (v[0] == '0' ? 0 : v[0] == '1' ? 1 : 2) : 1;
          }();
          static const bool halo = [] {
            const char* v = std::getenv("XGS_GRID_HALO");
            return !(v && v[0] == '0');
          }();
          // Blocks per row band (each a whole number of 128-column warps): the
          // smallest split giving >= 16 blocks per SM, else one warp per block --
          // short-lived blocks shorten the last wave, and a single 640-wide frame
          // (80 bands) needs the split to fill the GPU at all.  C3 (16 x 1280x720):
          // 2; C4 (640x480): 5.
          static const int cs = [] {
            const char* v = std::getenv("XGS_GRID_CSPLIT");
            return v ? std::atoi(v) : 0;
          }();
          int csplit = 1;
          if (cs > 0) {
            csplit = cs;
          } else if (in.W % 128 == 0) {
            const int64_t nwr = in.W / 128, blocks1 = in.frames * rbf;
            csplit = (int)nwr;
            for (int64_t dd = 1; dd <= nwr; dd++)
              if (nwr % dd == 0 && blocks1 * dd >= 16 * (int64_t)sms) {
                csplit = (int)dd;
                break;
              }
          }
          if (csplit < 1 || in.W / 4 / csplit < 32) csplit = 1;
          const unsigned ntc = (unsigned)((in.W / 4 + 32 * csplit - 1) / (32 * csplit) * 32);
          for (int c = 0; c < nchunk; c++) {
            const int64_t f0 = c * fper, f1 = f0 + fper < in.frames ? f0 + fper : in.frames;
            if (f1 <= f0) break;
            if (host_frames && attempt == 0 && (e = cudaStreamWaitEvent(s, hcp->chunk[c], 0)) != cudaSuccess) return e;
            auto kern = diag == 0 ? grid_front_kernel<FRONT_INSERT, 0>
                                  : diag == 1 ? grid_front_kernel<FRONT_INSERT, 1> : grid_front_kernel<FRONT_INSERT, 2>;
            kern<<<(unsigned)((f1 - f0) * rbf * csplit), ntc, front_smem_bytes(ntc / 32), s>>>(
                in.depth, in.H, in.W, in.stride, in.rot, in.trans, cam, cf, nullptr, nullptr, bbox, cnts, nullptr,
                (unsigned)(f0 * rbf * csplit), st->slots, mask, overflow, halo, csplit);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
            count_launches(1);
          }
        } else {
          if (host_frames && attempt == 0 && (e = cudaStreamWaitEvent(s, hcp->done, 0)) != cudaSuccess) return e;
          grid_keys_kernel<<<grid_blocks(vec4 ? npix / 4 : npix, 256, sms), 256, 0, s>>>(
              in.depth, npix, in.H, in.W, in.stride, in.rot, in.trans, cam, k1, nullptr, bbox, cnts, vec4);
          count_launches(1);
          if ((e = launch_pdl(dd_insert_pixels_kernel, dim3(grid_blocks(npix, 256, sms)), dim3(256), 0, s,
                              (const uint64_t*)k1, npix, in.W, st->slots, mask, cnts, overflow)) != cudaSuccess)
            return e;
          count_launches(1);
        }
      }
      {
        ProfScope prof("grid_select", s);
        const int64_t sblocks = (st->cap + kScanILP * 256 - 1) / (kScanILP * 256);
        if ((e = launch_pdl(dd_scan_map_kernel, dim3((unsigned)(sblocks < 3 * sms ? sblocks : 3 * sms)), dim3(256), 0, s,
                            st->slots, st->cap, (const int*)overflow, hs->table, (uint64_t)hs->cap - 1,
                            hs->count_dev, flag, cnts + 1, st->lb, lb_tiles)) != cudaSuccess)
          return e;
        count_launches(1);
      }
      if ((e = emit_outputs(in, cam, st, head, k0, v0, 0, out, sms, s, host_frames ? hcp : nullptr, !in.async)) !=
          cudaSuccess)
        return e;
      if (in.async) {   // counts on the device (out.dev_status); the map bound grows by the pixel count
        out.n_new = out.n_valid = out.n_voxels = out.n_sorted = -1;
        hs->count_ub += std::min<int64_t>(npix, st->cap);
        st->dirty = false;
        return cudaGetLastError();
      }
      const unsigned long long* hst = st->host_st;
      out.n_valid = (int64_t)hst[0];
      out.n_voxels = (int64_t)hst[1];
      out.n_sorted = (int64_t)hst[2];
      out.n_new = (int64_t)hst[3];
      if (hst[4] & 2) return cudaErrorUnknown;   // the map set is full (reserve keeps load <= 1/2: not reached)
      if (!hst[4]) break;
      // the table was too small for this batch's distinct voxels: the scan did
      // not run (map untouched, nothing flagged or emitted); reset the partly
      // filled table and redo the batch on one sized for every pixel
      if (attempt > 0) return cudaErrorUnknown;
      fill_u64_kernel<<<grid_blocks(2 * st->cap, 256, sms), 256, 0, s>>>(st->slots, 2 * st->cap, ~0ull);
      count_launches(1);
      if ((e = dedup_table(*st, npix, true, s)) != cudaSuccess) return e;
      if ((e = hashset_reserve(hs, std::min<int64_t>(npix, st->cap), s)) != cudaSuccess) return e;
    }
    st->last_nvox = out.n_voxels;
  } else {
    // ---------------- G1 keys, G2 radix sort, G3 select (mean mode / forced sort)
    bool fused = false;
    int64_t fblocks = 0;
    {
      ProfScope prof("grid_keys", s);
      init_bbox_kernel<<<1, 32, 0, s>>>(bbox, cnts); count_launches(1);   // also zeroes cnts[0..5]
      fblocks = in.frames * ((in.H + FK_ROWS - 1) / FK_ROWS);
      fused = compact && vec4 && front_ok && fblocks <= w.lb_entries;
      if (host_frames && !fused) {   // the two-kernel front end reads every frame: wait for all of them
        if ((e = cudaStreamWaitEvent(s, hcp->done, 0)) != cudaSuccess) return e;
      }
      if (fused) {
        const CamF cf{(float)in.cx, (float)in.cy, (float)(1.0 / in.fx), (float)(1.0 / in.fy), (float)(1.0 / in.voxel)};
        const unsigned nt = (unsigned)((in.W / 4 + 31) / 32 * 32);
        const size_t fsmem = front_smem_bytes(nt / 32);
        if ((e = front_init()) != cudaSuccess) return e;
        const int64_t rbf = (in.H + FK_ROWS - 1) / FK_ROWS;
        for (int c = 0; c < nchunk; c++) {
          const int64_t f0 = c * fper, f1 = f0 + fper < in.frames ? f0 + fper : in.frames;
          if (f1 <= f0) break;
          if (host_frames && (e = cudaStreamWaitEvent(s, hcp->chunk[c], 0)) != cudaSuccess) return e;
          grid_front_kernel<FRONT_SORT, 1><<<(unsigned)((f1 - f0) * rbf), nt, fsmem, s>>>(
              in.depth, in.H, in.W, in.stride, in.rot, in.trans, cam, cf, k0, v0, bbox, cnts, block_count,
              (unsigned)(f0 * rbf), nullptr, 0, nullptr, true, 1);
          count_launches(1);
        }
      } else {
        grid_keys_kernel<<<grid_blocks(vec4 ? npix / 4 : npix, 256, sms), 256, 0, s>>>(
            in.depth, npix, in.H, in.W, in.stride, in.rot, in.trans, cam, compact ? k1 : k0, compact ? nullptr : v0,
            bbox, cnts, vec4); count_launches(1);
      }
      if (compact && !fused) {
        const int64_t ntiles = (npix + CT_TILE - 1) / CT_TILE;
        unsigned* tile_counter = reinterpret_cast<unsigned*>(cnts + 4);
        cudaMemsetAsync(tile_counter, 0, 4, s);
        cudaMemsetAsync(lb_status, 0, sizeof(unsigned long long) * ntiles, s);
        compact_keys_kernel<<<grid_blocks(ntiles * CT_THREADS, CT_THREADS, sms), CT_THREADS, 0, s>>>(
            k1, npix, in.W, k0, v0, tile_counter, lb_status, ntiles, cnts + 2); count_launches(1);
      }
    }
    // bbox (misc + 0) and the counters (misc + 64) in one copy to pinned memory
    int hb[8];
    unsigned long long hc[3] = {0, 0, 0};
    {
      unsigned long long* hst = nullptr;
      if ((e = pinned_status(&hst)) != cudaSuccess) return e;
      if ((e = cudaMemcpyAsync(hst, bbox, 88, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
      if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
      std::memcpy(hb, hst, 6 * sizeof(int));
      std::memcpy(hc, hst + 8, 24);
    }
    out.n_valid = (int64_t)hc[0];
    if (hc[0] == 0) {
      if ((e = cudaMemsetAsync(st->misc, 0, 256, s)) != cudaSuccess) return e;
      st->dirty = false;
      return cudaSuccess;
    }
    const int64_t nitems = compact ? (int64_t)hc[2] : npix;   // items to sort
    if ((e = hashset_reserve(hs, nitems, s)) != cudaSuccess) return e;
    // bbox-relative key width; +1 on x keeps the all-ones invalid key above every valid key
    RelKey rk;
    rk.x0 = (uint32_t)hb[0];
    rk.y0 = (uint32_t)hb[1];
    rk.z0 = (uint32_t)hb[2];
    const int bx = bits_for((int64_t)hb[3] - hb[0] + 1), by = bits_for((int64_t)hb[4] - hb[1]),
              bz = bits_for((int64_t)hb[5] - hb[2]);
    rk.by = by;
    rk.bz = bz;
    int bits = bx + by + bz;
    if (bits > 64) {  // degenerate extent: sort the raw biased keys (identity packing)
      rk.x0 = rk.y0 = rk.z0 = 0;
      rk.by = rk.bz = 21;
      bits = 64;
    }
    if ((e = sort_init()) != cudaSuccess) return e;
    out.n_sorted = nitems;
    out.sort_passes = (bits + 7) / 8;
    if ((e = cudaMemsetAsync(st->lb, 0, (size_t)lb_tiles * 8, s)) != cudaSuccess) return e;
    if (nitems > 0) {
      ProfScope prof("grid_sort", s);
      // relative keys once (u32 when they fit), LSD passes, biased keys back into k0
      const unsigned rb = grid_blocks(nitems, 256, sms);
      if (fused) {   // block slots -> dense: exclusive scan of the block counts
        if ((e = exclusive_scan_i32(block_count, fblocks, block_count, ssum, nullptr, s)) != cudaSuccess) return e;
      }
      if (bits <= 32) {
        uint32_t* r0 = reinterpret_cast<uint32_t*>(k1);
        uint32_t* r1 = r0 + nitems;
        if (fused) {   // items land in (r0, v1); the slots in (k0, v0) are dead afterwards
          if ((e = launch_pdl(rekey_gather_kernel<uint32_t>, dim3(grid_blocks(fblocks, 1, sms)), dim3(256), 0, s, k0, v0,
                              block_count, fblocks, in.H, in.W, nitems, rk, r0, v1)) != cudaSuccess)
            return e;
          count_launches(1);
          uint32_t* t = v0; v0 = v1; v1 = t;
        } else {
          rekey_kernel<uint32_t><<<rb, 256, 0, s>>>(k0, nitems, rk, r0); count_launches(1);
        }
        if ((e = lsd_passes<uint32_t>(r0, v0, r1, v1, nitems, bits, hist, ssum, s)) != cudaSuccess) return e;
        if ((e = launch_pdl(unrekey_kernel<uint32_t>, dim3(rb), dim3(256), 0, s, r0, nitems, rk, bits, k0)) != cudaSuccess)
          return e;
        count_launches(1);
      } else {
        if (fused) {
          rekey_gather_kernel<uint64_t><<<grid_blocks(fblocks, 1, sms), 256, 0, s>>>(k0, v0, block_count, fblocks, in.H, in.W,
                                                                                     nitems, rk, k1, v1); count_launches(1);
          uint32_t* t = v0; v0 = v1; v1 = t;
        } else {
          rekey_kernel<uint64_t><<<rb, 256, 0, s>>>(k0, nitems, rk, k1); count_launches(1);
        }
        uint64_t* r0 = k1;
        uint64_t* r1 = k0;
        if ((e = lsd_passes<uint64_t>(r0, v0, r1, v1, nitems, bits, hist, ssum, s)) != cudaSuccess) return e;
        if (r0 == k0) {   // sorted relative keys landed in k0's buffer: unpack through k1
          unrekey_kernel<uint64_t><<<rb, 256, 0, s>>>(r0, nitems, rk, bits, k1); count_launches(1);
          uint64_t* t = k0; k0 = k1; k1 = t;
        } else {
          unrekey_kernel<uint64_t><<<rb, 256, 0, s>>>(r0, nitems, rk, bits, k0); count_launches(1);
        }
      }
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      ProfScope prof2("grid_select", s);
      if ((e = launch_pdl(grid_select_kernel, dim3(grid_blocks(nitems, 256, sms)), dim3(256), 0, s, (const uint64_t*)k0,
                          (const uint32_t*)v0, nitems, hs->table, (uint64_t)hs->cap - 1, hs->count_dev, flag, head,
                          cnts + 1)) != cudaSuccess)
        return e;
      count_launches(1);
    }
    if ((e = emit_outputs(in, cam, st, head, k0, v0, nitems, out, sms, s, host_frames ? hcp : nullptr)) != cudaSuccess)
      return e;
    out.n_voxels = (int64_t)st->host_st[1];
    out.n_new = (int64_t)st->host_st[3];
  }
  st->dirty = false;
  hs->count_ub += out.n_new;
  if (out.n_new > out.capacity) return cudaErrorInvalidValue;
  return cudaGetLastError();
}

// exclusive scan of int32 counts (out may alias in); block_sums needs
// n / 4096 + 2 entries; *grand (device, nullable) receives the total
cudaError_t exclusive_scan_i32(const int32_t* in, int64_t n, int32_t* out, int32_t* block_sums, int32_t* grand,
                               cudaStream_t s) {
  return exclusive_scan<int32_t>(in, n, out, block_sums, grand, s);
}

// standalone in-house radix sort of (u64 key, u32 value) pairs on bits [0, bits)
cudaError_t radix_sort_pairs(uint64_t* keys, uint32_t* vals, int64_t n, int bits, void* ws, size_t ws_bytes,
                             cudaStream_t s) {
  const GridWs w = grid_ws(n);
  if (ws_bytes < w.total) return cudaErrorInvalidValue;
  char* b = static_cast<char*>(ws);
  uint64_t* k1 = reinterpret_cast<uint64_t*>(b + w.off_k1);
  uint32_t* v1 = reinterpret_cast<uint32_t*>(b + w.off_v1);
  int32_t* hist = reinterpret_cast<int32_t*>(b + w.off_hist);
  int32_t* ssum = reinterpret_cast<int32_t*>(b + w.off_scan_sums);
  uint64_t* k0 = keys;
  uint32_t* v0 = vals;
  cudaError_t e = sort_init();
  if (e != cudaSuccess) return e;
  if ((e = lsd_passes<uint64_t>(k0, v0, k1, v1, n, bits, hist, ssum, s)) != cudaSuccess) return e;
  if (k0 != keys) {
    if ((e = cudaMemcpyAsync(keys, k0, n * 8, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(vals, v0, n * 4, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace xgs
