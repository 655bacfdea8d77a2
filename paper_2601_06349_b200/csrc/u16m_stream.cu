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

#include <cstdint>

#include "u16m_internal.h"
#include "u16m_repair.cuh"

namespace u16m {

constexpr int kSV = 8;                        // vectors per thread
constexpr int kSThreads = 256;
constexpr int kSWarpVecs = 32 * kSV;          // 256 vectors = 4 KiB per warp
constexpr int kSCtaVecs = (kSThreads / 32) * kSWarpVecs;  // 2048 vectors = 32 KiB per CTA

template <bool kInPlace, int kGran>
__global__ void __launch_bounds__(kSThreads, 4) stream_kernel(Span s) {
  const int lane = threadIdx.x & 31;
  const uint32_t lane_off = threadIdx.x / 32 * kSWarpVecs + lane;
  const uint64_t vbeg = s.lo / 8;
  const uint64_t vend = (s.hi + 7) / 8;
  const uint64_t ntiles = (vend - vbeg + kSCtaVecs - 1) / kSCtaVecs;
  uint64_t tile = blockIdx.x;
  if (s.tile_sel == kTilesEdges) tile = blockIdx.x == 0 ? 0 : ntiles - 1;
  if (s.tile_sel == kTilesInterior) tile = blockIdx.x + 1;
  const uint64_t tv0 = vbeg + tile * kSCtaVecs;
  const bool interior = tv0 * 8 > s.lo && (tv0 + kSCtaVecs) * 8 < s.hi;
  const uint64_t v0 = tv0 + lane_off;  // this lane's vector k sits at v0 + 32k

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
    const uint64_t warp_v0 = v0 - lane;
    if (lane == 0) halo = unit_at(s, static_cast<int64_t>(warp_v0 * 8) - 1);
    if (lane == 31) halo = unit_at(s, static_cast<int64_t>((warp_v0 + kSWarpVecs) * 8));
#pragma unroll
    for (int k = 0; k < kSV; k++) {
      const uint64_t vi = v0 + k * 32;
      if (vi * 8 < s.lo || vi * 8 + 8 > s.hi) patch_edges(s, vi, v[k]);
    }
  }

  // Rolling pipeline over k: flags of vector k (cur) and k+1 (nxt) live.
  Flags cur = classify8(v[0]);
  uint32_t hp_carry = hflag_hi(halo);  // lane 0: H flags of the unit before vector 0
  const uint32_t halo_l = lflag_lo(halo);
  uint4* dst = s.out + v0;
#pragma unroll
  for (int k = 0; k < kSV; k++) {
    Flags nxt;
    if (k + 1 < kSV) nxt = classify8(v[k + 1]);
    const uint32_t up = __shfl_sync(kFull, cur.H1, (lane + 31) & 31);  // lane 0 gets lane 31's (vector k)
    const uint32_t dn = __shfl_sync(kFull, cur.L0, (lane + 1) & 31);
    uint32_t ln = dn;
    if (k + 1 < kSV) {
      const uint32_t dn_next = __shfl_sync(kFull, nxt.L0, (lane + 1) & 31);  // lane 31 gets lane 0's (vector k+1)
      if (lane == 31) ln = dn_next;
    } else if (lane == 31) {
      ln = halo_l;
    }
    const uint32_t hp = lane ? up : hp_carry;
    hp_carry = up;  // lane 0: lane 31's H flags of vector k precede vector k+1
    uint32_t B0, B1;
    bad8(cur, hp, ln, B0, B1);
    const bool store = kInPlace ? group_dirty<kGran>((B0 | B1) != 0, lane) : true;
    const uint64_t vi = v0 + k * 32;
    if (interior || (vi * 8 >= s.lo && vi * 8 + 8 <= s.hi)) {
      if (store) st_stream(dst + k * 32, blend(v[k], B0, B1));
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

cudaError_t launch_stream(const Span& s0, int part, cudaStream_t stream) {
  Span s = s0;
  const uint64_t vbeg = s.lo / 8, vend = (s.hi + 7) / 8;
  const uint64_t ntiles = (vend - vbeg + kSCtaVecs - 1) / kSCtaVecs;
  uint64_t grid = ntiles;
  if (part == kTilesEdges) grid = ntiles < 2 ? ntiles : 2;
  if (part == kTilesInterior) grid = ntiles > 2 ? ntiles - 2 : 0;
  s.tile_sel = part;
  if (grid == 0) return cudaSuccess;
  const unsigned g = static_cast<unsigned>(grid);
  const bool in_place = s.in == s.out;
  if (!in_place) {
    stream_kernel<false, 1><<<g, kSThreads, 0, stream>>>(s);
  } else {
    switch (inplace_granularity()) {
      case 1: stream_kernel<true, 1><<<g, kSThreads, 0, stream>>>(s); break;
      case 4: stream_kernel<true, 4><<<g, kSThreads, 0, stream>>>(s); break;
      case 8: stream_kernel<true, 8><<<g, kSThreads, 0, stream>>>(s); break;
      default: stream_kernel<true, 2><<<g, kSThreads, 0, stream>>>(s); break;
    }
  }
  note_launch();
  return cudaGetLastError();
}

}  // namespace u16m
