// Streaming copy / in-place kernel with a rolling register pipeline.
//
// Profiling the register-staged kernel (4 vectors per thread) on config 1
// showed it latency-bound (long-scoreboard stalls ~50%, DRAM ~58% of peak):
// every CTA lives ~2.8 us regardless of how much it writes, so throughput is
// set by the bytes in flight per SM. This kernel doubles them without
// doubling registers: each thread issues kSV = 8 independent 128-bit loads up
// front (128 B in flight per thread, 128 KiB per SM at 4 CTAs/SM), then
// classifies, repairs and stores the vectors one at a time, keeping the
// flags of only two vectors live (the shuffle halo of vector k needs the low
// flags of vector k+1 from lane 0, and the high flags of vector k-1 from
// lane 31, which it carries over).
//
// Edge tiles (the first and the last tile of a job) run the same code with
// out-of-range units substituted by their halo rule (patch_edges) and
// per-unit stores for vectors that straddle the range.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "u16m_internal.h"
#include "u16m_repair.cuh"

namespace u16m {

constexpr int kSV = 8;                        // vectors per thread
constexpr int kSThreads = 256;
constexpr int kSWarpVecs = 32 * kSV;          // 256 vectors = 4 KiB per warp
constexpr int kSCtaVecs = (kSThreads / 32) * kSWarpVecs;  // 2048 vectors = 32 KiB per CTA

// CTA-level sum of `counted` added to *count: one atomic per CTA (per-warp
// atomics on one address serialise at the L2 slice). All threads call it.
__device__ __forceinline__ void cta_count_add(uint32_t counted, unsigned long long* count) {
  __shared__ uint32_t warp_counts[kSThreads / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) counted += __shfl_xor_sync(kFull, counted, o);
  if ((threadIdx.x & 31) == 0) warp_counts[threadIdx.x / 32] = counted;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long c = 0;
#pragma unroll
    for (int w = 0; w < kSThreads / 32; w++) c += warp_counts[w];
    if (c) atomicAdd(count, c);
  }
}

// One tile of the stream kernel. kEdge = false: every vector of the tile lies
// inside [lo, hi) (the hot path: no per-vector range tests, 128-bit stores
// only; the warp tile's outer halo unit is the only thing that may come from
// the halo rule). kEdge = true: the first / last tile of a job, with range
// patches and per-unit stores for vectors that straddle [lo, hi). Two
// separate bodies so that none of the edge bookkeeping is computed on the
// hot path (it was hoisted into it when both shared one loop: ~20 extra
// instructions per vector).
template <bool kEdge, bool kInPlace, int kGran, int kSV, bool kBE, bool kCount, bool kNoStore>
__device__ __forceinline__ void stream_tile(const Span& s, uint64_t tv0, uint64_t vend, int lane,
                                            uint32_t lane_off, uint32_t& counted) {
  constexpr int kSWarpVecs = 32 * kSV;
  const uint64_t v0 = tv0 + lane_off;  // this lane's vector k sits at v0 + 32k
  uint4 v[kSV];
  uint32_t halo = 0;
  if constexpr (!kEdge) {
    const uint4* src = s.in + v0;
#pragma unroll
    for (int k = 0; k < kSV; k++) v[k] = ld_stream(src + k * 32);
    const uint16_t* src16 = reinterpret_cast<const uint16_t*>(src);
    const int64_t wa = static_cast<int64_t>((v0 - lane) * 8);  // the warp tile's first unit
    if (lane == 0)
      halo = wa > static_cast<int64_t>(s.lo) ? to_mem<kBE>(src16[-1]) : unit_at(s, wa - 1);
    if (lane == 31) {
      const int64_t a = wa + kSWarpVecs * 8;
      halo = a < static_cast<int64_t>(s.hi) ? to_mem<kBE>(src16[(kSV - 1) * 32 * 8 + 8]) : unit_at(s, a);
    }
  } else {
#pragma unroll
    for (int k = 0; k < kSV; k++) {
      const uint64_t vi = v0 + k * 32;
      v[k] = vi < vend ? ld_stream(s.in + vi) : make_uint4(0, 0, 0, 0);
    }
    // unit_at returns unit values for halos but raw memory words in range.
    const uint64_t warp_v0 = v0 - lane;
    if (lane == 0) {
      const int64_t a = static_cast<int64_t>(warp_v0 * 8) - 1;
      halo = unit_at(s, a);
      if (a >= static_cast<int64_t>(s.lo)) halo = to_mem<kBE>(halo);
    }
    if (lane == 31) {
      const int64_t a = static_cast<int64_t>((warp_v0 + kSWarpVecs) * 8);
      halo = unit_at(s, a);
      if (a < static_cast<int64_t>(s.hi)) halo = to_mem<kBE>(halo);
    }
#pragma unroll
    for (int k = 0; k < kSV; k++) {
      const uint64_t vi = v0 + k * 32;
      if (vi * 8 < s.lo || vi * 8 + 8 > s.hi) patch_edges<kBE>(s, vi, v[k]);
    }
  }

  // Rolling pipeline over k: flags of vector k (cur) and k+1 (nxt) live.
  Flags cur = classify8<kBE>(v[0]);
  uint32_t hp_carry = hflag_hi(halo);  // lane 0: H flags of the unit before vector 0
  const uint32_t halo_l = lflag_lo(halo);
  const int up_lane = (lane + 31) & 31, dn_lane = (lane + 1) & 31;
  uint4* dst = s.out + v0;
#pragma unroll
  for (int k = 0; k < kSV; k++) {
    Flags nxt;
    if (k + 1 < kSV) nxt = classify8<kBE>(v[k + 1]);
    const uint32_t up = __shfl_sync(kFull, cur.H1, up_lane);  // lane 0 gets lane 31's (vector k)
    const uint32_t dn = __shfl_sync(kFull, cur.L0, dn_lane);
    uint32_t ln = dn;
    if (k + 1 < kSV) {
      const uint32_t dn_next = __shfl_sync(kFull, nxt.L0, dn_lane);  // lane 31 gets lane 0's (vector k+1)
      if (lane == 31) ln = dn_next;
    } else if (lane == 31) {
      ln = halo_l;
    }
    const uint32_t hp = lane ? up : hp_carry;
    hp_carry = up;  // lane 0: lane 31's H flags of vector k precede vector k+1
    uint32_t B0, B1;
    bad8(cur, hp, ln, B0, B1);
    const bool store = kInPlace ? group_dirty<kGran>((B0 | B1) != 0, lane) : true;
    if constexpr (!kEdge) {
      if constexpr (kCount) counted += __popc(B0) + __popc(B1);
      if constexpr (!kNoStore) {
        if (store) st_stream(dst + k * 32, blend<kBE>(v[k], B0, B1));
      }
    } else {
      const uint64_t vi = v0 + k * 32;
      if constexpr (kCount) {
        uint32_t c0 = B0, c1 = B1;
        mask_outside(s, vi, c0, c1);
        if (vi < vend) counted += __popc(c0) + __popc(c1);
      }
      if constexpr (!kNoStore) {
        if (vi * 8 >= s.lo && vi * 8 + 8 <= s.hi) {
          if (store) st_stream(dst + k * 32, blend<kBE>(v[k], B0, B1));
        } else if (store && vi < vend) {
          const uint4 r = blend<kBE>(v[k], B0, B1);
#pragma unroll
          for (int j = 0; j < 8; j++) {
            const uint64_t a = vi * 8 + j;
            if (a >= s.lo && a < s.hi) {
              const uint32_t u = get_unit(r, j);
              if (!kInPlace || u != get_unit(v[k], j)) s.out_units[a - s.lo] = static_cast<uint16_t>(u);
            }
          }
        }
      }
    }
    if (k + 1 < kSV) cur = nxt;
  }
}

// kBE: units are big-endian in memory (fused byte-order handling, §8(f-3));
// kCount: add the number of rewritten units to *count (CTA reduction, one
// atomic per CTA); kNoStore: validation only.
template <bool kInPlace, int kGran, int kSV = 8, int kMinBlocks = 4, bool kBE = false, bool kCount = false,
          bool kNoStore = false>
__global__ void __launch_bounds__(kSThreads, kMinBlocks) stream_kernel(Span s, unsigned long long* count,
                                                                      uint32_t* half_tile_counts) {
  // validation: the offsets scan's prefix kernel is a programmatic dependent
  if constexpr (kCount && kNoStore) asm volatile("griddepcontrol.launch_dependents;");
  constexpr int kSWarpVecs = 32 * kSV;
  constexpr int kSCtaVecs = (kSThreads / 32) * kSWarpVecs;
  const int lane = threadIdx.x & 31;
  const uint32_t lane_off = threadIdx.x / 32 * kSWarpVecs + lane;
  const uint64_t vbeg = s.lo / 8;
  const uint64_t vend = (s.hi + 7) / 8;
  const uint64_t ntiles = (vend - vbeg + kSCtaVecs - 1) / kSCtaVecs;
  uint64_t nwork = ntiles;
  if (s.tile_sel == kTilesEdges) nwork = ntiles < 2 ? ntiles : 2;
  if (s.tile_sel == kTilesInterior) nwork = ntiles > 2 ? ntiles - 2 : 0;
  uint32_t counted = 0;
  uint64_t count_tile = 0;
  // One tile per CTA (persistent grids measured 15-20 % slower: profiles/README.md).
  for (uint64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    // The last tile goes first: a ragged last tile runs the edge code path
    // (range patches, per-unit stores), whose cold instruction fetch made it
    // finish ~14 us after everything else when it was dispatched last.
    uint64_t tile = w == 0 ? ntiles - 1 : w - 1;
    if (s.tile_sel == kTilesEdges) tile = w == 0 ? 0 : ntiles - 1;
    if (s.tile_sel == kTilesInterior) tile = w + 1;
    count_tile = tile;
    const uint64_t tv0 = vbeg + tile * kSCtaVecs;
    if (s.prefetch_tiles > 0 && threadIdx.x == 0) {
      // One bulk L2 prefetch of the tile a later wave of CTAs will stream: extra
      // bytes in flight without registers (TMA prefetch, no smem, no barrier).
      const uint64_t pv = tv0 + static_cast<uint64_t>(s.prefetch_tiles) * kSCtaVecs;
      if (pv + kSCtaVecs <= vend)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s.in + pv), "r"(kSCtaVecs * 16) : "memory");
    }
    // "interior": every vector of the tile lies fully inside [lo, hi) — also the
    // first and last tile of a job whose ends are 16-byte aligned; only their
    // outer halo units come from the halo rule instead of memory.
    if (tv0 * 8 >= s.lo && (tv0 + kSCtaVecs) * 8 <= s.hi)
      stream_tile<false, kInPlace, kGran, kSV, kBE, kCount, kNoStore>(s, tv0, vend, lane, lane_off, counted);
    else
      stream_tile<true, kInPlace, kGran, kSV, kBE, kCount, kNoStore>(s, tv0, vend, lane, lane_off, counted);
  }  // tile loop
  if constexpr (kCount) {
    // CTA-level reduction, one atomic per CTA (per-warp atomics on one
    // address serialise at the L2 slice).
    __shared__ uint32_t warp_counts[kSThreads / 32];
#pragma unroll
    for (int o = 16; o; o >>= 1) counted += __shfl_xor_sync(kFull, counted, o);
    if (lane == 0) warp_counts[threadIdx.x / 32] = counted;
    __syncthreads();
    if (threadIdx.x == 0) {
      if (half_tile_counts) {
        // Per 8192-unit half tile (warps 0-3 / 4-7): the tile counts of the
        // offsets scan, in the general kernel's tile geometry (u16m_kernels.cu).
        uint32_t c0 = 0, c1 = 0;
#pragma unroll
        for (int w = 0; w < kSThreads / 64; w++) {
          c0 += warp_counts[w];
          c1 += warp_counts[w + kSThreads / 64];
        }
        // (one tile per CTA in this mode; the tile is not blockIdx.x: the last goes first)
        half_tile_counts[2 * count_tile] = c0;
        half_tile_counts[2 * count_tile + 1] = c1;
        // ... and the total of every chunk of 32768 half tiles (count[chunk]), so
        // that tile_prefix_kernel can scan the chunks in parallel, one CTA each
        if (count && (c0 | c1)) atomicAdd(count + (count_tile >> 14), static_cast<unsigned long long>(c0) + c1);
      } else {
        unsigned long long c = 0;
#pragma unroll
        for (int w = 0; w < kSThreads / 32; w++) c += warp_counts[w];
        if (c) atomicAdd(count, c);
      }
    }
  }
}

// ---- copy between different 16-byte phases ----------------------------------
// SURVEY.md §7 "arbitrary char16_t* alignment": when `out` and `in` differ mod
// 16 bytes, unit a (in-aligned coordinates) lands at out-aligned coordinate
// a + delta, delta = out phase - in phase. With s = delta mod 8 (1..7) and
// q = (delta - s) / 8, out vector vi + q holds the last s units of repaired
// vector vi-1 followed by the first 8-s units of repaired vector vi. In the
// rolling layout vector vi-1 sits in the previous lane (lane 31 of the
// previous k for lane 0), so each output vector is two register shuffles and
// a compile-time funnel combine away; only the two vectors that straddle a
// tile boundary are written unit by unit (half by each tile). Edge tiles (the
// first and last of a job) write every unit individually.
template <int S>
__device__ __forceinline__ uint4 combine_units(const uint4& P, const uint4& C) {
  const uint32_t W[8] = {P.x, P.y, P.z, P.w, C.x, C.y, C.z, C.w};
  uint32_t o[4];
#pragma unroll
  for (int w = 0; w < 4; w++) {
    const int i = 8 - S + 2 * w;  // first halfword of output word w in P ++ C
    o[w] = (i & 1) ? __funnelshift_r(W[i >> 1], W[(i >> 1) + 1], 16) : W[i >> 1];
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

__device__ __forceinline__ uint4 shfl4(const uint4& v, int src, bool up) {
  uint4 r;
  if (up) {
    r.x = __shfl_up_sync(kFull, v.x, 1), r.y = __shfl_up_sync(kFull, v.y, 1);
    r.z = __shfl_up_sync(kFull, v.z, 1), r.w = __shfl_up_sync(kFull, v.w, 1);
  } else {
    r.x = __shfl_sync(kFull, v.x, src), r.y = __shfl_sync(kFull, v.y, src);
    r.z = __shfl_sync(kFull, v.z, src), r.w = __shfl_sync(kFull, v.w, src);
  }
  return r;
}

// kBE / kCount: the codec-fused forms (u16m_fix_utf16_bytes into an output at
// another phase): big-endian units, rewritten units added to *count.
template <int S, bool kBE = false, bool kCount = false>
__global__ void __launch_bounds__(kSThreads, 4) stream_shift_kernel(Span s, int64_t q, unsigned long long* count) {
  const int lane = threadIdx.x & 31;
  const uint32_t lane_off = threadIdx.x / 32 * kSWarpVecs + lane;
  const uint64_t vbeg = s.lo / 8;
  const uint64_t vend = (s.hi + 7) / 8;
  const uint64_t ntiles = (vend - vbeg + kSCtaVecs - 1) / kSCtaVecs;
  uint64_t tile = blockIdx.x == 0 ? ntiles - 1 : blockIdx.x - 1;  // last (ragged) tile first
  if (s.tile_sel == kTilesEdges) tile = blockIdx.x == 0 ? 0 : ntiles - 1;
  if (s.tile_sel == kTilesInterior) tile = blockIdx.x + 1;
  if (tile >= ntiles) return;
  const uint64_t tv0 = vbeg + tile * kSCtaVecs;
  const bool interior = tv0 * 8 > s.lo && (tv0 + kSCtaVecs) * 8 < s.hi;
  const uint64_t v0 = tv0 + lane_off;

  uint4 v[kSV];
  uint32_t halo = 0;
  uint32_t counted = 0;
  if (interior) {
    const uint4* src = s.in + v0;
#pragma unroll
    for (int k = 0; k < kSV; k++) v[k] = ld_stream(src + k * 32);
    const uint16_t* src16 = reinterpret_cast<const uint16_t*>(src);
    if (lane == 0) halo = to_mem<kBE>(src16[-1]);
    if (lane == 31) halo = to_mem<kBE>(src16[(kSV - 1) * 32 * 8 + 8]);
  } else {
#pragma unroll
    for (int k = 0; k < kSV; k++) {
      const uint64_t vi = v0 + k * 32;
      v[k] = vi < vend ? ld_stream(s.in + vi) : make_uint4(0, 0, 0, 0);
    }
    // unit_at returns unit values for halos but raw memory words in range.
    const uint64_t warp_v0 = v0 - lane;
    if (lane == 0) {
      const int64_t a = static_cast<int64_t>(warp_v0 * 8) - 1;
      halo = unit_at(s, a);
      if (a >= static_cast<int64_t>(s.lo)) halo = to_mem<kBE>(halo);
    }
    if (lane == 31) {
      const int64_t a = static_cast<int64_t>((warp_v0 + kSWarpVecs) * 8);
      halo = unit_at(s, a);
      if (a < static_cast<int64_t>(s.hi)) halo = to_mem<kBE>(halo);
    }
#pragma unroll
    for (int k = 0; k < kSV; k++) {
      const uint64_t vi = v0 + k * 32;
      if (vi * 8 < s.lo || vi * 8 + 8 > s.hi) patch_edges<kBE>(s, vi, v[k]);
    }
  }

  Flags cur = classify8<kBE>(v[0]);
  uint32_t hp_carry = hflag_hi(halo);
  const uint32_t halo_l = lflag_lo(halo);
  uint4 carry = make_uint4(0, 0, 0, 0);  // lane 31's repaired vector k-1 (for lane 0)
#pragma unroll
  for (int k = 0; k < kSV; k++) {
    Flags nxt;
    if (k + 1 < kSV) nxt = classify8<kBE>(v[k + 1]);
    const uint32_t up = __shfl_sync(kFull, cur.H1, (lane + 31) & 31);
    const uint32_t dn = __shfl_sync(kFull, cur.L0, (lane + 1) & 31);
    uint32_t ln = dn;
    if (k + 1 < kSV) {
      const uint32_t dn_next = __shfl_sync(kFull, nxt.L0, (lane + 1) & 31);
      if (lane == 31) ln = dn_next;
    } else if (lane == 31) {
      ln = halo_l;
    }
    const uint32_t hp = lane ? up : hp_carry;
    hp_carry = up;
    uint32_t B0, B1;
    bad8(cur, hp, ln, B0, B1);
    const uint4 r = blend<kBE>(v[k], B0, B1);
    const uint64_t vi = v0 + k * 32;
    if constexpr (kCount) {
      if (interior) {
        counted += __popc(B0) + __popc(B1);
      } else {
        uint32_t c0 = B0, c1 = B1;
        mask_outside(s, vi, c0, c1);
        if (vi < vend) counted += __popc(c0) + __popc(c1);
      }
    }
    if (interior) {
      uint4 prev = shfl4(r, 0, true);
      if (lane == 0) prev = carry;
      carry = shfl4(r, 31, false);
      if (k == 0 && lane == 0) {
        // head of a vector straddling the tile start: the previous tile writes the tail
#pragma unroll
        for (int j = 0; j < 8 - S; j++) s.out_units[vi * 8 + j - s.lo] = static_cast<uint16_t>(get_unit(r, j));
      } else {
        st_stream(s.out + static_cast<int64_t>(vi) + q, combine_units<S>(prev, r));
      }
      if (k == kSV - 1 && lane == 31) {
#pragma unroll
        for (int j = 8 - S; j < 8; j++) s.out_units[vi * 8 + j - s.lo] = static_cast<uint16_t>(get_unit(r, j));
      }
    } else if (vi < vend) {
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const uint64_t a = vi * 8 + j;
        if (a >= s.lo && a < s.hi) s.out_units[a - s.lo] = static_cast<uint16_t>(get_unit(r, j));
      }
    }
    if (k + 1 < kSV) cur = nxt;
  }
  if constexpr (kCount) cta_count_add(counted, count);
}

// ---- batched form, non-persistent (buffer length known) ----------------------
// Persistent grids measured 15-20 % slower than one-tile-per-CTA grids for
// register-staged streaming (U16M_PERSIST), so the batched form also runs one
// 16384-unit tile per CTA. The grid is sized from the caller's buffer length
// (tiles past offsets[S] exit). A pre-pass records, for every warp tile
// (2048 units) that holds a string start, the index of its first string; a
// warp finds its strings with two dependent loads (that entry, then a
// 32-entry window of offsets) issued after — and overlapping — its 8 data
// loads. The table is first memset to kNoStart and the pre-pass writes only
// the tiles that hold a start, so a string spanning many tiles costs it
// nothing (a serial per-string fill made one 2^28-unit string 7x slower
// than the plain repair); a warp on a start-less tile only checks whether
// the next tile's first string starts exactly at its end.
constexpr int kFirstPerThread = 4;
constexpr uint64_t kNoStart = ~0ull;

// The strings' extent [A, B) clamped to the caller's buffer [0, n_units):
// offsets outside it are a contract error and must never turn into
// out-of-bounds accesses (negative, past the end, or B < A -> empty).
__device__ __forceinline__ void clamped_extent(const int64_t* offsets, uint64_t count, int64_t n_units, int64_t& A,
                                               int64_t& B) {
  A = __ldg(offsets);
  B = __ldg(offsets + count - 1);
  B = B < 0 ? 0 : (B < n_units ? B : n_units);
  A = A < 0 ? 0 : (A < B ? A : B);
}

// The table's "no start" fill, as the primary of a programmatic dependent
// launch chain fill -> tile_first_kernel -> batched_tile_kernel (a
// cudaMemsetAsync cannot start its successor early).
__global__ void table_fill_kernel(uint4* __restrict__ t, uint64_t n16) {
  asm volatile("griddepcontrol.launch_dependents;");
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n16;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    t[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
}

__global__ void tile_first_kernel(const int64_t* __restrict__ offsets, uint64_t count, uint32_t phase,
                                  uint64_t* __restrict__ tile_first, uint64_t nwt, int64_t n_units) {
  // Programmatic dependent launch: let the repair grid start now; its CTAs
  // issue their data loads and wait (griddepcontrol.wait) only before they
  // read this table.
  asm volatile("griddepcontrol.launch_dependents;");
  const uint64_t s0 = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) * kFirstPerThread;
  if (s0 >= count) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  int64_t A, B;
  clamped_extent(offsets, count, n_units, A, B);
  const int64_t base = ((A + phase) / 8) * 8 - phase;  // key of warp tile 0
  constexpr int64_t kTileUnits = kSWarpVecs * 8;        // one warp tile
  // Offsets outside the buffer are a contract error: clamp, never write out of bounds.
  auto tile_of = [&](int64_t p) -> uint64_t {
    const uint64_t t = p < base ? 0 : static_cast<uint64_t>(p - base) / kTileUnits;
    return t < nwt ? t : nwt - 1;
  };
  int64_t p[kFirstPerThread + 1];
  p[0] = s0 ? __ldg(offsets + s0 - 1) : 0;
#pragma unroll
  for (int j = 0; j < kFirstPerThread; j++) p[j + 1] = s0 + j < count ? __ldg(offsets + s0 + j) : 0;
  // the "no start" fill (the primary grid) is complete and visible from here
  asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
  for (int j = 0; j < kFirstPerThread; j++) {
    const uint64_t si = s0 + j;
    if (si >= count) break;
    const uint64_t t = tile_of(p[j + 1]);
    if (si == 0 || tile_of(p[j]) != t) tile_first[t] = si;
  }
}

// String starts of one warp tile [A0, A1): bit 8k+j of lane l's M marks
// unit A0 + 256k + 8l + j; `after`: a string starts exactly at A1.
struct StartScan {
  uint64_t M;
  bool after;
};

// Folds one 32-entry window of offsets (this lane's entry p) into st.
__device__ __forceinline__ void scan_window(int64_t p, int64_t A0, int64_t A1, int lane, StartScan& st) {
  uint32_t inr = __ballot_sync(kFull, p >= A0 && p < A1);
  st.after |= __ballot_sync(kFull, p == A1) != 0;
  while (inr) {
    const int j = __ffs(inr) - 1;
    inr &= inr - 1;
    const uint32_t r = static_cast<uint32_t>(__shfl_sync(kFull, p, j) - A0);
    if (lane == static_cast<int>((r >> 3) & 31)) st.M |= 1ull << (((r >> 8) << 3) | (r & 7));
  }
}

// kShift > 0 (copy only): `out` has a different 16-byte phase than `in`;
// s.out is out's 16-byte-aligned base, s.out_units the caller's out pointer,
// and vectors are stored shifted as in stream_shift_kernel (q: vector offset).
// The tile table is written by tile_first_kernel WHILE this grid is already
// running (programmatic dependent launch), so it must not be read through the
// read-only path: with `const __restrict__` the compiler emits
// LDG.CONSTANT and may hoist it above griddepcontrol.wait (a build that did
// read stale entries). It is read with ld.global.cg in inline asm that is
// ordered after the wait.
__device__ __forceinline__ uint64_t ld_table(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <bool kInPlace, int kGran, int kShift = 0>
__global__ void __launch_bounds__(kSThreads, 4) batched_tile_kernel(Span s, const int64_t* __restrict__ offsets,
                                                                    uint64_t count, uint32_t phase,
                                                                    const uint64_t* tile_first,
                                                                    uint64_t nwt, int64_t n_units, int64_t q) {
  static_assert(kShift == 0 || !kInPlace, "in place is always the same phase");
  const int lane = threadIdx.x & 31;
  {
    int64_t A, B;
    clamped_extent(offsets, count, n_units, A, B);
    s.lo = static_cast<uint64_t>(A) + phase;
    s.hi = static_cast<uint64_t>(B) + phase;
    s.out_units = kShift ? s.out_units + A : reinterpret_cast<uint16_t*>(s.out) + s.lo;
  }
  if (s.hi <= s.lo) return;
  const uint64_t vbeg = s.lo / 8;
  const uint64_t vend = (s.hi + 7) / 8;
  const uint64_t ntiles = (vend - vbeg + kSCtaVecs - 1) / kSCtaVecs;
  // the last (ragged, edge-path) tile first, as in stream_kernel
  const uint64_t tile = blockIdx.x == 0 ? ntiles - 1 : blockIdx.x - 1;
  if (blockIdx.x != 0 && tile >= ntiles - 1) return;
  const uint64_t tv0 = vbeg + tile * kSCtaVecs;
  const uint64_t wv0 = tv0 + threadIdx.x / 32 * kSWarpVecs;
  if (wv0 >= vend) return;  // warp tile past the job (no table entry either)
  const uint64_t v0 = wv0 + lane;
  const bool interior = tv0 * 8 > s.lo && (tv0 + kSCtaVecs) * 8 < s.hi;

  uint4 v[kSV];
  uint32_t halo = 0;
  if (interior) {
    const uint4* src = s.in + v0;
#pragma unroll
    for (int k = 0; k < kSV; k++) v[k] = ld_stream(src + k * 32);
    const uint16_t* src16 = reinterpret_cast<const uint16_t*>(src);
    if (lane == 0) halo = src16[-1];
    if (lane == 31) halo = src16[(kSV - 1) * 32 * 8 + 8];
  } else {
#pragma unroll
    for (int k = 0; k < kSV; k++) {
      const uint64_t vi = v0 + k * 32;
      v[k] = vi < vend ? ld_stream(s.in + vi) : make_uint4(0, 0, 0, 0);
    }
    if (lane == 0) halo = unit_at(s, static_cast<int64_t>(wv0 * 8) - 1);
    if (lane == 31) halo = unit_at(s, static_cast<int64_t>((wv0 + kSWarpVecs) * 8));
  }

  // String starts in this warp tile [A0, A1) and whether one starts at A1.
  const int64_t A0 = static_cast<int64_t>(wv0 * 8) - phase;
  const int64_t A1 = A0 + kSWarpVecs * 8;
  // Scan the offsets from this tile's first string; a tile without a start
  // (kNoStart: inside a long string) scans from the next tile's first string
  // instead, which only finds whether one starts exactly at A1.
  const uint64_t wt = (wv0 - vbeg) / kSWarpVecs;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the tile table is complete and visible
  const uint64_t c0 = ld_table(tile_first + wt);
  const uint64_t c1 = wt + 1 < nwt ? ld_table(tile_first + wt + 1) : kNoStart;
  const uint64_t first = c0 != kNoStart ? c0 : (c1 < count ? c1 : count);
  StartScan st{0, false};
  for (uint64_t scan = first;;) {
    const uint64_t idx = scan + lane;
    const int64_t p = idx < count ? __ldg(offsets + idx) : INT64_MAX;
    scan_window(p, A0, A1, lane, st);
    if (__ballot_sync(kFull, p <= A1) != kFull) break;
    scan = next_offsets_window(offsets, count, scan, p, lane);  // skips runs of empty strings
  }
  const uint64_t M = st.M;
  const bool start_after = st.after;
  if (!interior) {
#pragma unroll
    for (int k = 0; k < kSV; k++) {
      const uint64_t vi = v0 + k * 32;
      if (vi * 8 < s.lo || vi * 8 + 8 > s.hi) patch_edges(s, vi, v[k]);
    }
  }
  uint32_t F = 0;
#pragma unroll
  for (int k = 0; k < kSV; k++) F |= static_cast<uint32_t>((M >> (8 * k)) & 1u) << k;
  const uint32_t Fd = __shfl_sync(kFull, F, (lane + 1) & 31);
  const uint32_t after = lane == 31 ? ((Fd >> 1) | (start_after ? (1u << (kSV - 1)) : 0u)) : Fd;
  // Vectors k of this warp that hold a string start (or precede one): one
  // warp reduction up front instead of a vote per vector.
  uint32_t need = after;
#pragma unroll
  for (int k = 0; k < kSV; k++) need |= (static_cast<uint32_t>(M >> (8 * k)) & 0xFFu) ? (1u << k) : 0u;
  need = __reduce_or_sync(kFull, need);

  uint4 shift_carry = make_uint4(0, 0, 0, 0);  // kShift: lane 31's repaired vector k-1
  Flags cur = classify8(v[0]);
  uint32_t hp_carry = hflag_hi(halo);
  const uint32_t halo_l = lflag_lo(halo);
#pragma unroll
  for (int k = 0; k < kSV; k++) {
    Flags nxt;
    if (k + 1 < kSV) nxt = classify8(v[k + 1]);
    const uint32_t up = __shfl_sync(kFull, cur.H1, (lane + 31) & 31);
    const uint32_t dn = __shfl_sync(kFull, cur.L0, (lane + 1) & 31);
    uint32_t ln = dn;
    if (k + 1 < kSV) {
      const uint32_t dn_next = __shfl_sync(kFull, nxt.L0, (lane + 1) & 31);
      if (lane == 31) ln = dn_next;
    } else if (lane == 31) {
      ln = halo_l;
    }
    const uint32_t hp = lane ? up : hp_carry;
    hp_carry = up;
    const uint32_t bits = static_cast<uint32_t>(M >> (8 * k)) & 0xFFu;
    uint32_t B0, B1;
    const uint32_t aft = (after >> k) & 1u;
    // Most vectors of a warp hold no string start: skip the start-flag
    // algebra when no lane needs it (warp-uniform branch).
    if ((need >> k) & 1u)
      bad8(cur, hp, ln, B0, B1, spread4(bits), spread4(bits >> 4), aft << 7);
    else
      bad8(cur, hp, ln, B0, B1);
    const bool store = kInPlace ? group_dirty<kGran>((B0 | B1) != 0, lane) : true;
    const uint64_t vi = v0 + k * 32;
    if constexpr (kShift > 0) {
      const uint4 r = blend(v[k], B0, B1);
      if (interior) {
        uint4 prev = shfl4(r, 0, true);
        if (lane == 0) prev = shift_carry;
        shift_carry = shfl4(r, 31, false);
        if (k == 0 && lane == 0) {  // head of the vector straddling the warp tile start
#pragma unroll
          for (int j = 0; j < 8 - kShift; j++) s.out_units[vi * 8 + j - s.lo] = static_cast<uint16_t>(get_unit(r, j));
        } else {
          st_stream(s.out + static_cast<int64_t>(vi) + q, combine_units<kShift>(prev, r));
        }
        if (k == kSV - 1 && lane == 31) {
#pragma unroll
          for (int j = 8 - kShift; j < 8; j++) s.out_units[vi * 8 + j - s.lo] = static_cast<uint16_t>(get_unit(r, j));
        }
      } else if (vi < vend) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
          const uint64_t a = vi * 8 + j;
          if (a >= s.lo && a < s.hi) s.out_units[a - s.lo] = static_cast<uint16_t>(get_unit(r, j));
        }
      }
    } else if (interior || (vi * 8 >= s.lo && vi * 8 + 8 <= s.hi)) {
      if (store) st_stream(s.out + vi, blend(v[k], B0, B1));
    } else if (store && vi < vend) {
      const uint4 r = blend(v[k], B0, B1);
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const uint64_t a = vi * 8 + j;
        if (a >= s.lo && a < s.hi) {
          const uint32_t u = get_unit(r, j);
          if (!kInPlace || u != get_unit(v[k], j)) s.out_units[a - s.lo] = static_cast<uint16_t>(u);
        }
      }
    }
    if (k + 1 < kSV) cur = nxt;
  }
}

// Stream-ordered workspace comes from the device's default memory pool; keep
// freed blocks cached in the pool (release threshold = max) so per-call
// cudaMallocAsync/FreeAsync never go back to the driver.
void keep_pool_memory() {
  static std::once_flag once[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::call_once(once[dev], [dev] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
  });
}

static bool batched_pdl() {  // U16M_BATCHED_PDL=0: plain stream order (A/B)
  static const bool v = [] {
    const char* e = std::getenv("U16M_BATCHED_PDL");
    return !(e && std::strcmp(e, "0") == 0);
  }();
  return v;
}

cudaError_t launch_batched_tiles(const uint16_t* in, size_t n_units, const int64_t* offsets, size_t num_strings,
                                 uint16_t* out, cudaStream_t stream, size_t grid_units) {
  const uintptr_t ia = reinterpret_cast<uintptr_t>(in);
  const uintptr_t oa = reinterpret_cast<uintptr_t>(out);
  const uint32_t ph = static_cast<uint32_t>((ia & 15u) / 2);
  Span s;
  s.in = reinterpret_cast<const uint4*>(ia - 2 * ph);
  s.out = reinterpret_cast<uint4*>(oa - 2 * ph);
  s.out_units = nullptr;
  s.lo = s.hi = 0;
  s.left = s.right = -1;
  s.left_ptr = s.right_ptr = nullptr;
  s.tile_sel = kTilesAll;
  s.prefetch_tiles = 0;
  constexpr uint64_t kTileUnits = kSCtaVecs * 8;
  const uint64_t count = static_cast<uint64_t>(num_strings) + 1;
  const uint64_t ntiles_max = (static_cast<uint64_t>(grid_units ? grid_units : n_units) + 16) / kTileUnits + 2;
  const uint64_t nwtiles_max = ntiles_max * (kSThreads / 32);  // even
  uint64_t* table = nullptr;  // first string starting in or after each warp tile
  keep_pool_memory();
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&table), nwtiles_max * sizeof(uint64_t), stream);
  if (e != cudaSuccess) return e;
  // kNoStart fill (nwtiles_max is even: 16-byte stores) -> pre-pass -> repair,
  // each a programmatic dependent of the previous: a grid is scheduled while
  // its predecessor still runs and waits only where it reads its results.
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = batched_pdl() ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const uint64_t n16 = nwtiles_max / 2;
  table_fill_kernel<<<static_cast<unsigned>(std::min<uint64_t>((n16 + 255) / 256, 148 * 8)), 256, 0, stream>>>(
      reinterpret_cast<uint4*>(table), n16);
  note_launch();
  const uint64_t pthreads = (count + kFirstPerThread - 1) / kFirstPerThread;
  cfg.gridDim = dim3(static_cast<unsigned>((pthreads + 255) / 256));
  e = cudaLaunchKernelEx(&cfg, tile_first_kernel, offsets, count, ph, static_cast<uint64_t*>(table), nwtiles_max,
                         static_cast<int64_t>(n_units));
  if (e != cudaSuccess) return e;
  note_launch();
  const unsigned g = static_cast<unsigned>(ntiles_max);
  const int64_t nn = static_cast<int64_t>(n_units);
  // The repair grid: a programmatic dependent of tile_first_kernel.
  cfg.gridDim = dim3(g);
  cfg.blockDim = dim3(kSThreads);
  const uint64_t cnt = count, nwt = nwtiles_max;
  const uint64_t* tab = table;
  const int64_t q0 = 0;
  const int64_t po = static_cast<int64_t>((oa & 15u) / 2);
  const int64_t delta = po - static_cast<int64_t>(ph);
  const int sh = static_cast<int>(((delta % 8) + 8) % 8);
  if (sh != 0) {
    // out at a different 16-byte phase: shifted vector stores (copy only)
    Span t = s;
    t.out = reinterpret_cast<uint4*>(oa - 2 * po);
    t.out_units = out;
    const int64_t q = (delta - sh) / 8;
    switch (sh) {
      case 1: e = cudaLaunchKernelEx(&cfg, batched_tile_kernel<false, 1, 1>, t, offsets, cnt, ph, tab, nwt, nn, q); break;
      case 2: e = cudaLaunchKernelEx(&cfg, batched_tile_kernel<false, 1, 2>, t, offsets, cnt, ph, tab, nwt, nn, q); break;
      case 3: e = cudaLaunchKernelEx(&cfg, batched_tile_kernel<false, 1, 3>, t, offsets, cnt, ph, tab, nwt, nn, q); break;
      case 4: e = cudaLaunchKernelEx(&cfg, batched_tile_kernel<false, 1, 4>, t, offsets, cnt, ph, tab, nwt, nn, q); break;
      case 5: e = cudaLaunchKernelEx(&cfg, batched_tile_kernel<false, 1, 5>, t, offsets, cnt, ph, tab, nwt, nn, q); break;
      case 6: e = cudaLaunchKernelEx(&cfg, batched_tile_kernel<false, 1, 6>, t, offsets, cnt, ph, tab, nwt, nn, q); break;
      default: e = cudaLaunchKernelEx(&cfg, batched_tile_kernel<false, 1, 7>, t, offsets, cnt, ph, tab, nwt, nn, q); break;
    }
  } else if (in != out) {
    e = cudaLaunchKernelEx(&cfg, batched_tile_kernel<false, 1>, s, offsets, cnt, ph, tab, nwt, nn, q0);
  } else {
    e = cudaLaunchKernelEx(&cfg, batched_tile_kernel<true, kDefaultInplaceGran>, s, offsets, cnt, ph, tab, nwt, nn,
                           q0);
  }
  if (e != cudaSuccess) return e;
  note_launch();
  e = cudaGetLastError();
  const cudaError_t f = cudaFreeAsync(table, stream);
  return e != cudaSuccess ? e : f;
}


static int prefetch_setting() {
  static const int v = [] {
    const char* e = std::getenv("U16M_PREFETCH");
    return e ? std::atoi(e) : -1;  // -1: auto (one resident wave ahead)
  }();
  return v;
}

template <int kV, int kMB>
static cudaError_t launch_stream_v(Span s, int part, cudaStream_t stream) {
  constexpr int kCtaVecs = (kSThreads / 32) * 32 * kV;
  const uint64_t vbeg = s.lo / 8, vend = (s.hi + 7) / 8;
  const uint64_t ntiles = (vend - vbeg + kCtaVecs - 1) / kCtaVecs;
  uint64_t grid = ntiles;
  if (part == kTilesEdges) grid = ntiles < 2 ? ntiles : 2;
  if (part == kTilesInterior) grid = ntiles > 2 ? ntiles - 2 : 0;
  s.tile_sel = part;
  if (grid == 0) return cudaSuccess;
  {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int pf = prefetch_setting();
    // auto: one resident wave ahead, and only for jobs of more than two waves
    // (measured: +3% on config 1, a small loss on the 2-wave config 0).
    s.prefetch_tiles = pf >= 0 ? pf : (ntiles > static_cast<uint64_t>(2 * sms * kMB) ? sms * kMB : 0);
  }
  const unsigned g = static_cast<unsigned>(grid);
  if (s.in != s.out) {
    stream_kernel<false, 1, kV, kMB><<<g, kSThreads, 0, stream>>>(s, nullptr, nullptr);
  } else {
    stream_kernel<true, kDefaultInplaceGran, kV, kMB><<<g, kSThreads, 0, stream>>>(s, nullptr, nullptr);
  }
  note_launch();
  return cudaGetLastError();
}

// Byte-order-aware repair with a replacement count (codec fusion, §8(f-3)).
template <bool kInPlace, bool kBE>
static void launch_codec_t(const Span& s, unsigned g, unsigned long long* count, cudaStream_t stream) {
  if (count)
    stream_kernel<kInPlace, 2, 8, 4, kBE, true><<<g, kSThreads, 0, stream>>>(s, count, nullptr);
  else
    stream_kernel<kInPlace, 2, 8, 4, kBE, false><<<g, kSThreads, 0, stream>>>(s, nullptr, nullptr);
}

cudaError_t launch_stream_codec(const Span& s, bool big_endian, unsigned long long* count, cudaStream_t stream) {
  constexpr int kCtaVecs = (kSThreads / 32) * 32 * 8;
  const uint64_t vbeg = s.lo / 8, vend = (s.hi + 7) / 8;
  const uint64_t ntiles = (vend - vbeg + kCtaVecs - 1) / kCtaVecs;
  if (ntiles == 0) return cudaSuccess;
  Span t = s;
  t.tile_sel = kTilesAll;
  const unsigned g = static_cast<unsigned>(ntiles);
  const bool ip = s.in == s.out;
  if (ip && big_endian) launch_codec_t<true, true>(t, g, count, stream);
  else if (ip) launch_codec_t<true, false>(t, g, count, stream);
  else if (big_endian) launch_codec_t<false, true>(t, g, count, stream);
  else launch_codec_t<false, false>(t, g, count, stream);
  note_launch();
  return cudaGetLastError();
}

// Validation (§8(f-1)): the stream kernel with the count and no stores —
// 2 B/unit read-only, one tile per CTA. With half_tile_counts set it writes
// the rewrite count of every 8192-unit half tile instead of the total
// (2 * ceil(n_vectors / 2048) entries), and `count` (if set) is an array of
// totals per chunk of 32768 half tiles (zeroed by the caller).
cudaError_t launch_stream_count(const uint16_t* in, size_t n, unsigned long long* count, cudaStream_t stream,
                                uint32_t* half_tile_counts, int32_t left, int32_t right) {
  if (n == 0) return cudaSuccess;
  const uintptr_t ia = reinterpret_cast<uintptr_t>(in);
  const uint32_t ph = static_cast<uint32_t>((ia & 15u) / 2);
  Span s;
  s.in = reinterpret_cast<const uint4*>(ia - 2 * ph);
  s.out = nullptr;
  s.out_units = nullptr;
  s.lo = ph;
  s.hi = ph + n;
  s.left = left;
  s.right = right;
  s.left_ptr = s.right_ptr = nullptr;
  s.tile_sel = kTilesAll;
  const uint64_t ntiles = ((s.hi + 7) / 8 - s.lo / 8 + kSCtaVecs - 1) / kSCtaVecs;
  {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int pf = prefetch_setting();
    s.prefetch_tiles = pf >= 0 ? pf : (ntiles > static_cast<uint64_t>(2 * sms * 5) ? sms * 5 : 0);
  }
  // 5 resident CTAs per SM (48 registers, 16-20 bytes of spills): without
  // stores the extra CTA's loads in flight win (C1 98.3 -> 96.3 us, C4 1378 ->
  // 1344 us, profiles/r02/count_probe.txt); 6 spill 2 KB and 4 is slower.
  stream_kernel<false, 1, 8, 5, false, true, true>
      <<<static_cast<unsigned>(ntiles), kSThreads, 0, stream>>>(s, count, half_tile_counts);
  note_launch();
  return cudaGetLastError();
}

// ---- small offsets scans: one launch ----------------------------------------
// unpaired_surrogate_offsets / is_well_formed on a short buffer (a Python
// string, a small file: n <= kSmallScanUnits) is all launch latency: the
// count -> prefix -> emit chain is three launches plus a workspace
// allocation. Here ONE CTA walks the buffer in 16384-unit tiles (8 x 128-bit
// loads in flight per thread, the stream kernel's layout), ranks each tile's
// rewrites behind a running total and writes the ascending offsets and
// min(total, limit) itself; it stops at the tile that completes the limit.
// Every tile takes the guarded (edge) path: at this size the range tests cost
// nothing measurable.
__global__ void __launch_bounds__(kSThreads, 1) small_scan_kernel(Span s, unsigned long long limit,
                                                                  unsigned long long* offsets_out,
                                                                  unsigned long long* count_out) {
  __shared__ uint32_t warp_tot[kSThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t vbeg = s.lo / 8;
  const uint64_t vend = (s.hi + 7) / 8;
  const uint64_t ntiles = (vend - vbeg + kSCtaVecs - 1) / kSCtaVecs;
  unsigned long long base = 0;  // rewrites in the tiles before this one (CTA-uniform)
  for (uint64_t tile = 0; tile < ntiles && base < limit; tile++) {
    const uint64_t wv0 = vbeg + tile * kSCtaVecs + static_cast<uint64_t>(warp) * kSWarpVecs;
    const uint64_t v0 = wv0 + lane;
    uint4 v[kSV];
#pragma unroll
    for (int k = 0; k < kSV; k++) {
      const uint64_t vi = v0 + k * 32;
      v[k] = vi < vend ? ld_stream(s.in + vi) : make_uint4(0, 0, 0, 0);
    }
    uint32_t halo = 0;
    if (lane == 0) halo = unit_at(s, static_cast<int64_t>(wv0 * 8) - 1);
    if (lane == 31) halo = unit_at(s, static_cast<int64_t>((wv0 + kSWarpVecs) * 8));
#pragma unroll
    for (int k = 0; k < kSV; k++) {
      const uint64_t vi = v0 + k * 32;
      if (vi * 8 < s.lo || vi * 8 + 8 > s.hi) patch_edges(s, vi, v[k]);
    }
    uint32_t B0[kSV], B1[kSV];
    {
      Flags cur = classify8(v[0]);
      uint32_t hp_carry = hflag_hi(halo);
      const uint32_t halo_l = lflag_lo(halo);
      const int up_lane = (lane + 31) & 31, dn_lane = (lane + 1) & 31;
#pragma unroll
      for (int k = 0; k < kSV; k++) {
        Flags nxt;
        if (k + 1 < kSV) nxt = classify8(v[k + 1]);
        const uint32_t up = __shfl_sync(kFull, cur.H1, up_lane);
        const uint32_t dn = __shfl_sync(kFull, cur.L0, dn_lane);
        uint32_t ln = dn;
        if (k + 1 < kSV) {
          const uint32_t dn_next = __shfl_sync(kFull, nxt.L0, dn_lane);
          if (lane == 31) ln = dn_next;
        } else if (lane == 31) {
          ln = halo_l;
        }
        const uint32_t hp = lane ? up : hp_carry;
        hp_carry = up;
        bad8(cur, hp, ln, B0[k], B1[k]);
        if (k + 1 < kSV) cur = nxt;
      }
    }
#pragma unroll
    for (int k = 0; k < kSV; k++) {
      const uint64_t vi = v0 + k * 32;
      if (vi * 8 < s.lo || vi * 8 + 8 > s.hi) mask_outside(s, vi, B0[k], B1[k]);
    }
    uint32_t mine = 0;
#pragma unroll
    for (int k = 0; k < kSV; k++) mine += __popc(B0[k]) + __popc(B1[k]);
    const uint32_t warp_count = __reduce_add_sync(kFull, mine);
    __syncthreads();  // the previous tile's readers of warp_tot are done
    if (lane == 0) warp_tot[warp] = warp_count;
    __syncthreads();
    uint32_t total = 0, before = 0;
#pragma unroll
    for (int w = 0; w < kSThreads / 32; w++) {
      total += warp_tot[w];
      if (w < warp) before += warp_tot[w];
    }
    if (warp_count != 0 && base + before < limit) {
      // ranks follow unit order: warp, then row k, then lane
      uint32_t run = 0;
#pragma unroll
      for (int k = 0; k < kSV; k++) {
        const uint32_t c = __popc(B0[k]) + __popc(B1[k]);
        uint32_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, x, o);
          if (lane >= o) x += y;
        }
        unsigned long long r = base + before + run + x - c;
        run += __shfl_sync(kFull, x, 31);
        const uint64_t a0 = (v0 + k * 32) * 8 - s.lo;
        uint64_t bits = static_cast<uint64_t>(B0[k]) | (static_cast<uint64_t>(B1[k]) << 32);
        while (bits && r < limit) {
          const int bit = __ffsll(static_cast<long long>(bits)) - 1;
          bits &= bits - 1;
          offsets_out[r++] = a0 + (bit >> 3);
        }
      }
    }
    base += total;
  }
  if (threadIdx.x == 0) *count_out = base < limit ? base : limit;
}

// n in (0, kSmallScanUnits], limit > 0.
cudaError_t launch_small_scan(const uint16_t* in, size_t n, size_t limit, unsigned long long* offsets_out,
                              unsigned long long* count_out, cudaStream_t stream, int32_t left, int32_t right) {
  const uintptr_t ia = reinterpret_cast<uintptr_t>(in);
  const uint32_t ph = static_cast<uint32_t>((ia & 15u) / 2);
  Span s;
  s.in = reinterpret_cast<const uint4*>(ia - 2 * ph);
  s.out = nullptr;
  s.out_units = nullptr;
  s.lo = ph;
  s.hi = ph + n;
  s.left = left;
  s.right = right;
  s.left_ptr = s.right_ptr = nullptr;
  s.tile_sel = kTilesAll;
  s.prefetch_tiles = 0;
  small_scan_kernel<<<1, kSThreads, 0, stream>>>(s, static_cast<unsigned long long>(limit), offsets_out, count_out);
  note_launch();
  return cudaGetLastError();
}

// Copy with out at a different 16-byte phase than in (see stream_shift_kernel).
template <bool kBE, bool kCount>
static cudaError_t launch_shift_t(Span s, uint16_t* out, int part, unsigned long long* count, cudaStream_t stream) {
  const uintptr_t oa = reinterpret_cast<uintptr_t>(out);
  const int64_t pi = static_cast<int64_t>(s.lo);  // in phase (units); s.lo == phase for a plain job
  const int64_t po = static_cast<int64_t>((oa & 15u) / 2);
  const int64_t delta = po - pi;
  const int sh = static_cast<int>(((delta % 8) + 8) % 8);
  const int64_t q = (delta - sh) / 8;
  s.out = reinterpret_cast<uint4*>(oa - 2 * po);
  s.out_units = out;
  const uint64_t vbeg = s.lo / 8, vend = (s.hi + 7) / 8;
  const uint64_t ntiles = (vend - vbeg + kSCtaVecs - 1) / kSCtaVecs;
  uint64_t grid = ntiles;
  if (part == kTilesEdges) grid = ntiles < 2 ? ntiles : 2;
  if (part == kTilesInterior) grid = ntiles > 2 ? ntiles - 2 : 0;
  s.tile_sel = part;
  if (grid == 0) return cudaSuccess;
  const unsigned g = static_cast<unsigned>(grid);
  switch (sh) {
    case 1: stream_shift_kernel<1, kBE, kCount><<<g, kSThreads, 0, stream>>>(s, q, count); break;
    case 2: stream_shift_kernel<2, kBE, kCount><<<g, kSThreads, 0, stream>>>(s, q, count); break;
    case 3: stream_shift_kernel<3, kBE, kCount><<<g, kSThreads, 0, stream>>>(s, q, count); break;
    case 4: stream_shift_kernel<4, kBE, kCount><<<g, kSThreads, 0, stream>>>(s, q, count); break;
    case 5: stream_shift_kernel<5, kBE, kCount><<<g, kSThreads, 0, stream>>>(s, q, count); break;
    case 6: stream_shift_kernel<6, kBE, kCount><<<g, kSThreads, 0, stream>>>(s, q, count); break;
    case 7: stream_shift_kernel<7, kBE, kCount><<<g, kSThreads, 0, stream>>>(s, q, count); break;
    default: return cudaErrorInvalidValue;  // same phase: launch_stream
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_stream_shift(Span s, uint16_t* out, int part, cudaStream_t stream) {
  return launch_shift_t<false, false>(s, out, part, nullptr, stream);
}

// Codec-fused copy into an output at another 16-byte phase (byte order folded
// into the gather, replacement count): one pass with shifted stores.
cudaError_t launch_stream_shift_codec(const Span& s, uint16_t* out, bool big_endian, unsigned long long* count,
                                      cudaStream_t stream) {
  if (big_endian)
    return count ? launch_shift_t<true, true>(s, out, kTilesAll, count, stream)
                 : launch_shift_t<true, false>(s, out, kTilesAll, nullptr, stream);
  return count ? launch_shift_t<false, true>(s, out, kTilesAll, count, stream)
               : launch_shift_t<false, false>(s, out, kTilesAll, nullptr, stream);
}

// Byte swap of n units in place (p 16-byte aligned): the big-endian form of
// the host validation scan swaps each chunk on the device after its H2D copy
// (HBM-speed, hidden under the PCIe transfer of the next chunk) instead of on
// one host thread.
__global__ void byteswap_kernel(uint4* __restrict__ p, uint64_t nvec, uint16_t* __restrict__ tail, uint32_t ntail) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < nvec) {
    uint4 v = p[i];
    v.x = prmt(v.x, 0, 0x2301);
    v.y = prmt(v.y, 0, 0x2301);
    v.z = prmt(v.z, 0, 0x2301);
    v.w = prmt(v.w, 0, 0x2301);
    p[i] = v;
  } else if (i - nvec < ntail) {
    const uint32_t u = tail[i - nvec];
    tail[i - nvec] = static_cast<uint16_t>((u >> 8) | (u << 8));
  }
}

// *dst = *src, dst in mapped pinned host memory: how the host pipelines read a
// device counter between chunks without a copy-engine transfer (an 8-byte
// cudaMemcpyAsync queues behind the 64 MiB chunk copies on the same engine and
// stalled the kernels behind it: -4 % on error-dense input).
// (no system fence: the host reads after synchronising on an event recorded
// behind this kernel, which orders the posted write before the completion)
__global__ void store_u64_kernel(unsigned long long* dst, const unsigned long long* src) { *dst = *src; }

cudaError_t launch_store_u64(unsigned long long* dst_mapped, const unsigned long long* src, cudaStream_t stream) {
  store_u64_kernel<<<1, 1, 0, stream>>>(dst_mapped, src);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_byteswap(uint16_t* p, size_t n, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const uint64_t nvec = n / 8;
  const uint32_t ntail = static_cast<uint32_t>(n % 8);
  const uint64_t total = nvec + ntail;
  byteswap_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, stream>>>(reinterpret_cast<uint4*>(p), nvec,
                                                                                   p + nvec * 8, ntail);
  note_launch();
  return cudaGetLastError();
}

// Small copy jobs (config 0: 32 MiB = 1.73 waves of 32 KiB tiles) keep the
// same tiles: 16 KiB tiles (3.5 waves), 28 KiB tiles (1.98 waves), 8 CTAs/SM
// with 8 KiB tiles and an earlier L2 prefetch all measured slower (14.5 us
// vs 15.8-18.5 us, profiles/README.md).
cudaError_t launch_stream(const Span& s, int part, cudaStream_t stream) {
  return launch_stream_v<kSV, 4>(s, part, stream);
}

}  // namespace u16m
