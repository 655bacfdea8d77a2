// sm_100a repair kernels: stream (copy / in-place / count) and batched CSR.
//
// One kernel template covers every form of the path. A CTA tile is 8 warps ×
// 32 lanes × kVecs 16-byte vectors = 8192 contiguous units (16 KiB); each warp
// owns 2 KiB of it. Per tile:
//   1. every lane issues its kVecs 128-bit loads up front (64 B in flight per
//      thread; at 2048 resident threads per SM that is 128 KiB per SM, well
//      above the ~45 KiB/SM Little's-law requirement at 6.4 TB/s);
//   2. lanes 0 and 31 load the 2-byte halo unit on each side of the warp tile
//      (a line the neighbouring warp streams anyway, so it is an L2 hit);
//   3. classification + warp-shuffle halo + blend entirely in registers
//      (u16m_repair.cuh);
//   4. one 128-bit streaming store per vector (copy), or a store only for
//      vectors that contain a rewrite (in-place: clean vectors cost no write).
//
// In-place race: a neighbouring warp may read a halo
// unit after its owner rewrote it to FFFD. A unit is only rewritten when no
// neighbour pairs with it, so the reader's decision is the same for the old
// and the new value; the 16-bit unit is read atomically either way.
//
// Batched form: units are the flat concatenation [offsets[0], offsets[S]);
// per tile, warp 0 finds the first string start inside the tile with a
// 32-ary warp-cooperative search over `offsets` (4 dependent rounds for 2^20
// strings) and marks every string start in a shared-memory bitmap; the
// stencil then treats a start as "no predecessor" and the unit before it as
// "no successor". The search runs while the tile's data loads are in flight.

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "u16m_internal.h"
#include "u16m_repair.cuh"

namespace u16m {

enum Mode : int {
  kCopy = 0,       // out = repair(in)
  kInPlace = 1,    // buf = repair(buf), stores only vectors with a rewrite
  // 2 was a count mode; counting now runs on the stream kernel (u16m_stream.cu)
  // 3 was a per-tile count mode; tile counts now come from the stream kernel
  kEmit = 4        // write ascending rewrite offsets (< limit) using tile prefixes
};

struct BatchArgs {
  const int64_t* offsets;  // device, num_strings + 1 entries
  uint64_t count;          // num_strings + 1
  uint32_t phase;          // (in & 15) / 2
};

struct ScanArgs {
  unsigned long long* count_out;    // kEmit: number written
  const unsigned long long* tile_prefix;  // kEmit input (exclusive prefix per tile)
  const uint32_t* tile_counts;      // kEmit input (rewrites per tile)
  unsigned long long* offsets_out;  // kEmit output
  unsigned long long limit;         // kEmit cap
};

// Marks every string start of this CTA tile in `starts` (bit i = aligned unit
// cta_v0*8 + i). Warp 0 searches; the CTA synchronises around it.
__device__ __forceinline__ void mark_string_starts(const BatchArgs& b, uint64_t cta_v0, uint32_t* starts,
                                                   int warp, int lane) {
  __syncthreads();  // previous tile's readers are done with `starts`
  if (warp == 0) {
    for (int i = lane; i < kCtaUnits / 32 + 2; i += 32) starts[i] = 0;
    __syncwarp();
    const int64_t key_lo = static_cast<int64_t>(cta_v0 * 8) - static_cast<int64_t>(b.phase);
    const int64_t key_hi = key_lo + kCtaUnits;
    uint64_t sidx = warp_lower_bound(b.offsets, 0, b.count, key_lo, lane);
    for (;;) {
      const uint64_t idx = sidx + lane;
      const int64_t p = idx < b.count ? __ldg(b.offsets + idx) : INT64_MAX;
      const bool inside = p <= key_hi;
      if (inside) {
        const uint64_t bit = static_cast<uint64_t>(p - key_lo);
        atomicOr(&starts[bit >> 5], 1u << (bit & 31));
      }
      if (__ballot_sync(kFull, inside) != kFull) break;
      sidx = next_offsets_window(b.offsets, b.count, sidx, p, lane);  // skips runs of empty strings
    }
  }
  __syncthreads();
}

// Bad-unit flags of the kVecs vectors of this lane, given their classified
// flags and the warp tile's halo unit (lane 0: unit before the tile; lane 31:
// unit after it).
template <bool kBatched>
__device__ __forceinline__ void tile_bad(const Flags (&f)[kVecs], uint32_t halo, int lane,
                                         const uint32_t* starts, uint32_t a_base,
                                         uint32_t (&B0)[kVecs], uint32_t (&B1)[kVecs]) {
  const uint32_t halo_h = hflag_hi(halo);
  const uint32_t halo_l = lflag_lo(halo);
  uint32_t up[kVecs], dn[kVecs];
#pragma unroll
  for (int k = 0; k < kVecs; k++) {
    up[k] = __shfl_sync(kFull, f[k].H1, (lane + 31) & 31);
    dn[k] = __shfl_sync(kFull, f[k].L0, (lane + 1) & 31);
  }
#pragma unroll
  for (int k = 0; k < kVecs; k++) {
    const uint32_t hp = lane ? up[k] : (k ? up[k - 1] : halo_h);
    const uint32_t ln = lane != 31 ? dn[k] : (k + 1 < kVecs ? dn[k + 1] : halo_l);
    if constexpr (kBatched) {
      const uint32_t a0 = a_base + static_cast<uint32_t>(k * 32 + lane) * 8;
      const uint64_t pair = static_cast<uint64_t>(starts[a0 >> 5]) |
                            (static_cast<uint64_t>(starts[(a0 >> 5) + 1]) << 32);
      const uint32_t bits = static_cast<uint32_t>(pair >> (a0 & 31));
      bad8(f[k], hp, ln, B0[k], B1[k], spread4(bits), spread4(bits >> 4), ((bits >> 8) & 1u) << 7);
    } else {
      bad8(f[k], hp, ln, B0[k], B1[k]);
    }
  }
}

template <int kMode, bool kSamePhase, bool kBatched, int kGran = 1>
__global__ void __launch_bounds__(kThreads) repair_kernel(Span s, BatchArgs b, ScanArgs sc) {
  constexpr bool kScanMode = kMode == kEmit;
  __shared__ uint32_t starts[kBatched ? (kCtaUnits / 32 + 2) : 1];
  __shared__ unsigned long long warp_sums[kScanMode ? kWarps : 1];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;

  if constexpr (kBatched) {
    // Range of the batch, read on the device (no host sync in the API).
    // Negative or decreasing ends are a contract error: clamp to an empty or
    // non-negative range so they never address units before the buffer (the
    // length-less form cannot check the far end; the caller guarantees it).
    int64_t A = __ldg(b.offsets), B = __ldg(b.offsets + b.count - 1);
    A = A < 0 ? 0 : A;
    B = B < A ? A : B;
    s.lo = static_cast<uint64_t>(A) + b.phase;
    s.hi = static_cast<uint64_t>(B) + b.phase;
    s.out_units = reinterpret_cast<uint16_t*>(s.out) + s.lo;
  }
  if (s.hi <= s.lo) return;
  const uint64_t vbeg = s.lo / 8;
  const uint64_t vend = (s.hi + 7) / 8;
  const uint64_t ntiles = (vend - vbeg + kCtaVecs - 1) / kCtaVecs;
  const uint32_t lane_off = static_cast<uint32_t>(warp * kWarpVecs + lane);  // vector offset in tile
  // Tile selection: all tiles, only the two edge tiles, or only the interior
  // tiles (the last two let a caller overlap a halo exchange with the body).
  uint64_t nwork = ntiles, tbase = 0;
  if (s.tile_sel == kTilesEdges) nwork = ntiles < 2 ? ntiles : 2;
  if (s.tile_sel == kTilesInterior) {
    nwork = ntiles > 2 ? ntiles - 2 : 0;
    tbase = 1;
  }

  // kEmit: min(limit, total rewrites), written by tile_prefix_kernel; a tile
  // whose prefix reaches it holds nothing to emit, nor does any later tile.
  unsigned long long emit_stop = 0;
  if constexpr (kMode == kEmit) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // launched as a dependent of tile_prefix_kernel
    emit_stop = *sc.count_out;
  }
  for (uint64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    const uint64_t tile = s.tile_sel == kTilesEdges && w == 1 ? ntiles - 1 : tbase + w;
    if constexpr (kMode == kEmit) {
      // Tile prefixes are non-decreasing, so once a tile's rewrites all rank
      // past the limit (or there are none left) the same holds for every later
      // tile: stop before touching data (the CLI asks for 10 offsets; the grid
      // is persistent).
      if (sc.tile_prefix[tile] >= emit_stop) break;
      if (sc.tile_counts[tile] == 0) continue;  // nothing to emit: skip the data
    }
    const uint64_t cta_v0 = vbeg + tile * kCtaVecs;
    const uint64_t warp_v0 = cta_v0 + static_cast<uint64_t>(warp) * kWarpVecs;
    // Interior tile: every vector full and both warp-tile halos in range.
    const bool interior = cta_v0 * 8 > s.lo && (cta_v0 + kCtaVecs) * 8 < s.hi;

    if (interior && (kMode == kCopy || kMode == kInPlace)) {
      // ---- fast path: no range checks, one 64-bit base per lane ----
      const uint4* src = s.in + cta_v0 + lane_off;
      uint4 v[kVecs];
#pragma unroll
      for (int k = 0; k < kVecs; k++) v[k] = ld_stream(src + k * 32);
      uint32_t halo = 0;
      const uint16_t* src16 = reinterpret_cast<const uint16_t*>(src);
      if (lane == 0) halo = src16[-1];
      if (lane == 31) halo = src16[(kVecs - 1) * 32 * 8 + 8];
      if constexpr (kBatched) mark_string_starts(b, cta_v0, starts, warp, lane);
      Flags f[kVecs];
#pragma unroll
      for (int k = 0; k < kVecs; k++) f[k] = classify8(v[k]);
      uint32_t B0[kVecs], B1[kVecs];
      tile_bad<kBatched>(f, halo, lane, starts, (lane_off - lane) * 8, B0, B1);
      if constexpr (kSamePhase) {
        uint4* dst = s.out + cta_v0 + lane_off;
#pragma unroll
        for (int k = 0; k < kVecs; k++) {
          if (kMode == kInPlace && !group_dirty<kGran>((B0[k] | B1[k]) != 0, lane)) continue;
          st_stream(dst + k * 32, blend(v[k], B0[k], B1[k]));
        }
      } else {
        uint16_t* dst = s.out_units + ((cta_v0 + lane_off) * 8 - s.lo);
#pragma unroll
        for (int k = 0; k < kVecs; k++) {
          const uint4 r = blend(v[k], B0[k], B1[k]);
#pragma unroll
          for (int j = 0; j < 8; j++) dst[k * 256 + j] = static_cast<uint16_t>(get_unit(r, j));
        }
      }
      continue;
    }

    // ---- general path: edge tiles, and the count / scan modes ----
    uint4 v[kVecs];
#pragma unroll
    for (int k = 0; k < kVecs; k++) {
      const uint64_t vi = warp_v0 + k * 32 + lane;
      v[k] = vi < vend ? ld_stream(s.in + vi) : make_uint4(0, 0, 0, 0);
    }
    uint32_t halo = 0;
    if (lane == 0) halo = unit_at(s, static_cast<int64_t>(warp_v0 * 8) - 1);
    if (lane == 31) halo = unit_at(s, static_cast<int64_t>((warp_v0 + kWarpVecs) * 8));
    if constexpr (kBatched) mark_string_starts(b, cta_v0, starts, warp, lane);

    Flags f[kVecs];
    bool edge[kVecs];
#pragma unroll
    for (int k = 0; k < kVecs; k++) {
      const uint64_t vi = warp_v0 + k * 32 + lane;
      edge[k] = vi * 8 < s.lo || vi * 8 + 8 > s.hi;
      if (edge[k]) patch_edges(s, vi, v[k]);
      f[k] = classify8(v[k]);
    }
    uint32_t B0[kVecs], B1[kVecs];
    tile_bad<kBatched>(f, halo, lane, starts, (lane_off - lane) * 8, B0, B1);
    if constexpr (kMode == kEmit) {
#pragma unroll
      for (int k = 0; k < kVecs; k++)
        if (edge[k]) mask_outside(s, warp_v0 + k * 32 + lane, B0[k], B1[k]);
    }

    if constexpr (kMode == kCopy || kMode == kInPlace) {
#pragma unroll
      for (int k = 0; k < kVecs; k++) {
        const uint64_t vi = warp_v0 + k * 32 + lane;
        if (vi >= vend) continue;
        const bool dirty = (B0[k] | B1[k]) != 0;
        if (kMode == kInPlace && !dirty) continue;
        const uint4 r = blend(v[k], B0[k], B1[k]);
        if (kSamePhase && !edge[k]) {
          st_stream(s.out + vi, r);
        } else {
#pragma unroll
          for (int j = 0; j < 8; j++) {
            const uint64_t a = vi * 8 + j;
            if (a >= s.lo && a < s.hi) {
              const uint32_t u = get_unit(r, j);
              if (kMode == kCopy || u != get_unit(v[k], j))
                s.out_units[a - s.lo] = static_cast<uint16_t>(u);
            }
          }
        }
      }
    } else {
      // Rank of each vector's rewrites inside the tile, in unit order
      // (warp-major, then k, then lane).
      uint32_t c[kVecs], pre[kVecs];
      uint32_t warp_total = 0;
#pragma unroll
      for (int k = 0; k < kVecs; k++) {
        c[k] = __popc(B0[k]) + __popc(B1[k]);
        uint32_t x = c[k];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(kFull, x, o);
          if (lane >= o) x += y;
        }
        pre[k] = warp_total + x - c[k];
        warp_total += __shfl_sync(kFull, x, 31);
      }
      __syncthreads();  // previous tile's readers of warp_sums are done
      if (lane == 0) warp_sums[warp] = warp_total;
      __syncthreads();
      unsigned long long before = 0;
#pragma unroll
      for (int w = 0; w < kWarps; w++)
        if (w < warp) before += warp_sums[w];
      const unsigned long long base = sc.tile_prefix[tile] + before;
      if (base < sc.limit) {
#pragma unroll
        for (int k = 0; k < kVecs; k++) {
          unsigned long long r = base + pre[k];
          const uint64_t vi = warp_v0 + k * 32 + lane;
          uint64_t bits = static_cast<uint64_t>(B0[k]) | (static_cast<uint64_t>(B1[k]) << 32);
          while (bits && r < sc.limit) {
            const int bit = __ffsll(static_cast<long long>(bits)) - 1;
            bits &= bits - 1;
            const uint64_t a = vi * 8 + (bit >> 3);
            sc.offsets_out[r++] = a - s.lo;
          }
        }
      }
    }
  }

}

// ---- host launchers --------------------------------------------------------

namespace {
std::atomic<unsigned long long> g_launches{0};

int sm_count_for_current_device() {
  static std::mutex mu;
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::lock_guard<std::mutex> lock(mu);
  if (cached[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

template <int kMode, bool kSamePhase, bool kBatched, int kGran = 1>
cudaError_t launch(const Span& s, const BatchArgs& b, const ScanArgs& sc, uint64_t grid,
                   cudaStream_t stream) {
  if (grid == 0) return cudaSuccess;
  if (grid > 0x7FFFFFFFull) grid = 0x7FFFFFFFull;
  repair_kernel<kMode, kSamePhase, kBatched, kGran>
      <<<static_cast<unsigned>(grid), kThreads, 0, stream>>>(s, b, sc);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

constexpr BatchArgs kNoBatch{nullptr, 0, 0};
constexpr ScanArgs kNoScan{nullptr, nullptr, nullptr, nullptr, 0};

Span make_span(const uint16_t* in, size_t n, uint16_t* out, int32_t left, int32_t right,
               const uint16_t* left_ptr, const uint16_t* right_ptr, bool* same_phase) {
  const uintptr_t ia = reinterpret_cast<uintptr_t>(in);
  const uintptr_t oa = reinterpret_cast<uintptr_t>(out);
  const uint32_t ph = static_cast<uint32_t>((ia & 15u) / 2);
  Span s;
  s.in = reinterpret_cast<const uint4*>(ia - 2 * ph);
  s.out = reinterpret_cast<uint4*>(oa - 2 * ph);  // aligned only when same phase
  s.out_units = out;
  s.lo = ph;
  s.hi = ph + n;
  s.left = left;
  s.right = right;
  s.left_ptr = left_ptr;
  s.right_ptr = right_ptr;
  s.tile_sel = kTilesAll;
  s.prefetch_tiles = 0;
  *same_phase = out != nullptr && ((ia & 15u) == (oa & 15u));
  return s;
}

uint64_t tiles_for(const Span& s) {
  const uint64_t vbeg = s.lo / 8, vend = (s.hi + 7) / 8;
  return (vend - vbeg + kCtaVecs - 1) / kCtaVecs;
}
}  // namespace

unsigned long long launch_count() { return g_launches.load(std::memory_order_relaxed); }
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Kernel family selection. Copy / in-place run the rolling register-pipeline
// stream kernel (u16m_stream.cu; measured best: 6.9 TB/s copy, config 1 in
// 131 us); the batched form runs the batched tile kernel (u16m_stream.cu)
// whenever the buffer can be bounded, else the TMA-pipelined kernel (its
// producer warp walks the offsets off the consumers' critical path; a
// persistent grid needs no length).
// The other families are A/B material only and are compiled in only with
// -DU16M_AB_VARIANTS (libu16m_ab.so, `_build.py --ab`; the product library
// holds the default path alone). There, U16M_KERNEL selects: "tma"
// (TMA-pipelined for everything), "ldg" (register-staged everywhere; the
// length-less batched entry then uses the general kernel), "general" (the
// 4-vector general kernel for everything). profiles/README.md has the numbers.
enum KernelChoice { kChoiceAuto = 0, kChoiceTma = 1, kChoiceGeneral = 2, kChoiceLdg = 3 };
#ifdef U16M_AB_VARIANTS
// (kChoiceGeneral and kChoiceAuto share the register-staged kernel for plain
// streams; they differ for the batched form.)
static int kernel_choice() {
  static const int choice = [] {
    const char* e = std::getenv("U16M_KERNEL");
    if (e && std::strcmp(e, "tma") == 0) return int(kChoiceTma);
    if (e && std::strcmp(e, "general") == 0) return int(kChoiceGeneral);
    if (e && std::strcmp(e, "ldg") == 0) return int(kChoiceLdg);
    return int(kChoiceAuto);
  }();
  return choice;
}

template <int kGran>
static cudaError_t launch_inplace(const Span& s, uint64_t grid, cudaStream_t stream) {
  return launch<kInPlace, true, false, kGran>(s, kNoBatch, kNoScan, grid, stream);
}
#else
static constexpr int kernel_choice() { return kChoiceAuto; }
#endif

cudaError_t launch_repair_part(const uint16_t* in, size_t n, uint16_t* out, int32_t left, int32_t right,
                               const uint16_t* left_ptr, const uint16_t* right_ptr, int part,
                               cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  bool same = false;
  Span s = make_span(in, n, out, left, right, left_ptr, right_ptr, &same);
#ifdef U16M_AB_VARIANTS
  const uint64_t ntiles = tiles_for(s);
  const int choice = kernel_choice();
  if ((in == out || same) && choice == kChoiceTma && n >= kTmaMinUnits) {
    // The TMA kernel has no tile selection: it does the whole job as "edges".
    if (part == kTilesInterior) return cudaSuccess;
    return launch_repair_tma(in, n, out, left, right, left_ptr, right_ptr, stream);
  }
  if (choice == kChoiceGeneral) {
    s.tile_sel = part;
    const uint64_t grid = part == kTilesAll ? ntiles
                          : part == kTilesEdges ? (ntiles < 2 ? ntiles : 2)
                                                : (ntiles > 2 ? ntiles - 2 : 0);
    if (in == out) return launch_inplace<kDefaultInplaceGran>(s, grid, stream);
    if (same) return launch<kCopy, true, false>(s, kNoBatch, kNoScan, grid, stream);
    return launch<kCopy, false, false>(s, kNoBatch, kNoScan, grid, stream);
  }
#endif
  if (in == out || same) return launch_stream(s, part, stream);
  return launch_stream_shift(s, out, part, stream);
}

cudaError_t launch_fix_bytes(const void* in, size_t n, void* out, bool big_endian, unsigned long long* count,
                             cudaStream_t stream, int32_t left, int32_t right) {
  if (n == 0) return cudaSuccess;
  bool same = false;
  const auto* i16 = static_cast<const uint16_t*>(in);
  auto* o16 = static_cast<uint16_t*>(out);
  const Span s = make_span(i16, n, o16, left, right, nullptr, nullptr, &same);
  if (!(i16 == o16 || same)) return launch_stream_shift_codec(s, o16, big_endian, count, stream);
  return launch_stream_codec(s, big_endian, count, stream);
}

cudaError_t launch_repair(const uint16_t* in, size_t n, uint16_t* out, int32_t left, int32_t right,
                          const uint16_t* left_ptr, const uint16_t* right_ptr, cudaStream_t stream) {
  return launch_repair_part(in, n, out, left, right, left_ptr, right_ptr, kTilesAll, stream);
}

cudaError_t launch_count_unpaired(const uint16_t* in, size_t n, unsigned long long* count_out,
                                  cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(count_out, 0, sizeof(unsigned long long), stream);
  if (e != cudaSuccess || n == 0) return e;
  return launch_stream_count(in, n, count_out, stream);
}

// Exclusive prefix over per-tile counts, one CTA per chunk of 32768 tiles:
// every thread loads its 32 consecutive counts with 8 independent 128-bit
// loads (the whole round in flight at once), scans them in registers, and a
// warp-shuffle + shared-memory block scan over the thread totals gives each
// thread its offset; prefixes are written back as 128-bit stores. `counts`
// and `prefix` are 16-byte aligned. Also writes *count_out = min(total,
// limit), the number of offsets the emit pass writes.
constexpr int kPrefixPer = 32;
__global__ void __launch_bounds__(1024) tile_prefix_kernel(const uint32_t* counts, uint64_t n,
                                                           unsigned long long* prefix, unsigned long long limit,
                                                           unsigned long long* count_out,
                                                           const unsigned long long* chunk_totals) {
  __shared__ unsigned long long warp_tot[32];
  // PDL: the emit grid may launch now; this kernel waits for the counts
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // One CTA per chunk of 32768 counts; the chunks before this one are summed
  // from the count pass's chunk totals (a single CTA walking 524 288 counts,
  // config 4's size, took 245 us of a 1.4 ms scan).
  unsigned long long carry = 0;
  for (uint32_t c = 0; c < blockIdx.x; c++) carry += chunk_totals[c];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long total = 0;
    for (uint32_t c = 0; c < gridDim.x; c++) total += chunk_totals[c];
    *count_out = total < limit ? total : limit;
  }
  {
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * (1024 * kPrefixPer);
    const uint64_t i0 = base + static_cast<uint64_t>(threadIdx.x) * kPrefixPer;
    uint32_t c[kPrefixPer];
    if (i0 + kPrefixPer <= n) {
      const uint4* src = reinterpret_cast<const uint4*>(counts + i0);
#pragma unroll
      for (int q = 0; q < kPrefixPer / 4; q++) {
        const uint4 v = src[q];
        c[4 * q] = v.x, c[4 * q + 1] = v.y, c[4 * q + 2] = v.z, c[4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < kPrefixPer; j++) c[j] = i0 + j < n ? counts[i0 + j] : 0u;
    }
    unsigned long long sum = 0;
#pragma unroll
    for (int j = 0; j < kPrefixPer; j++) sum += c[j];
    unsigned long long x = sum;  // inclusive scan of the thread sums within the warp
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    unsigned long long run = carry + x - sum;
    for (int w = 0; w < warp; w++) run += warp_tot[w];
    if (i0 + kPrefixPer <= n) {
      ulonglong2* dst = reinterpret_cast<ulonglong2*>(prefix + i0);
#pragma unroll
      for (int q = 0; q < kPrefixPer / 2; q++) {
        ulonglong2 w2;
        w2.x = run;
        run += c[2 * q];
        w2.y = run;
        run += c[2 * q + 1];
        dst[q] = w2;
      }
    } else {
#pragma unroll
      for (int j = 0; j < kPrefixPer; j++) {
        if (i0 + j < n) prefix[i0 + j] = run;
        run += c[j];
      }
    }
  }
}

cudaError_t launch_unpaired_offsets(const uint16_t* in, size_t n, size_t limit,
                                    unsigned long long* offsets_out, unsigned long long* count_out,
                                    cudaStream_t stream, int32_t left, int32_t right) {
  // (*count_out is always written by tile_prefix_kernel's first CTA)
  if (n == 0 || limit == 0) return cudaMemsetAsync(count_out, 0, sizeof(unsigned long long), stream);
  if (n <= kSmallScanUnits) return launch_small_scan(in, n, limit, offsets_out, count_out, stream, left, right);
  cudaError_t e = cudaSuccess;
  bool same = false;
  const Span s = make_span(in, n, nullptr, left, right, nullptr, nullptr, &same);
  const uint64_t tiles = tiles_for(s);  // 8192-unit tiles of the emit pass
  const uint64_t halves = 2 * (((s.hi + 7) / 8 - s.lo / 8 + 2 * kCtaVecs - 1) / (2 * kCtaVecs));
  void* ws = nullptr;
  keep_pool_memory();
  const size_t counts_bytes = (halves * sizeof(uint32_t) + 15) / 16 * 16;
  const uint64_t chunks = (halves + 1024 * kPrefixPer - 1) / (1024 * kPrefixPer);  // 32768 half tiles each
  const size_t prefix_bytes = (tiles * sizeof(unsigned long long) + 15) / 16 * 16;
  e = cudaMallocAsync(&ws, counts_bytes + prefix_bytes + chunks * sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  auto* counts = static_cast<uint32_t*>(ws);  // both 16-byte aligned (tile_prefix_kernel)
  auto* prefix = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + counts_bytes);
  auto* chunk_totals = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + counts_bytes + prefix_bytes);
  e = cudaMemsetAsync(chunk_totals, 0, chunks * sizeof(unsigned long long), stream);
  if (e != cudaSuccess) {
    cudaFreeAsync(ws, stream);
    return e;
  }
  // 1) rewrites per 8192-unit tile: the read-only stream kernel (8 vectors in
  //    flight per thread) writes one count per half of its 16384-unit tile;
  // 2) exclusive prefix + the total; 3) emit on a persistent grid that stops
  //    at the first tile ranked past the limit.
  e = launch_stream_count(in, n, chunk_totals, stream, counts, left, right);
  // (2) and (3) are programmatic dependent launches (PDL): each grid is
  // scheduled while its predecessor runs and waits (griddepcontrol.wait) only
  // for the predecessor's results.
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  if (e == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>((tiles + 1024 * kPrefixPer - 1) / (1024 * kPrefixPer)));
    cfg.blockDim = dim3(1024);
    cfg.stream = stream;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, tile_prefix_kernel, static_cast<const uint32_t*>(counts), tiles, prefix,
                           static_cast<unsigned long long>(limit), count_out,
                           static_cast<const unsigned long long*>(chunk_totals));
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  if (e == cudaSuccess) {
    ScanArgs sc = kNoScan;
    sc.count_out = count_out;
    sc.tile_prefix = prefix;
    sc.tile_counts = counts;
    sc.offsets_out = offsets_out;
    sc.limit = limit;
    const uint64_t grid = std::min<uint64_t>(tiles, static_cast<uint64_t>(sm_count_for_current_device()) * 8);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kThreads);
    cfg.stream = stream;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, repair_kernel<kEmit, true, false>, s, kNoBatch, sc);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  const cudaError_t f = cudaFreeAsync(ws, stream);
  return e != cudaSuccess ? e : f;
}

// The length-aware batched form runs the tile kernel unless an A/B choice
// pins another family ("tma" / "general").
bool batched_tiles_enabled() {
  const int c = kernel_choice();
  return c == kChoiceAuto || c == kChoiceLdg;
}

cudaError_t launch_batched(const uint16_t* in, const int64_t* offsets, size_t num_strings,
                           uint16_t* out, cudaStream_t stream) {
  const bool same16 = ((reinterpret_cast<uintptr_t>(in) ^ reinterpret_cast<uintptr_t>(out)) & 15u) == 0;
  if ((kernel_choice() == kChoiceTma || kernel_choice() == kChoiceAuto) && same16)
    return launch_batched_tma(in, offsets, num_strings, out, stream);
  const uintptr_t ia = reinterpret_cast<uintptr_t>(in);
  const uintptr_t oa = reinterpret_cast<uintptr_t>(out);
  const uint32_t ph = static_cast<uint32_t>((ia & 15u) / 2);
  Span s;
  s.in = reinterpret_cast<const uint4*>(ia - 2 * ph);
  s.out = reinterpret_cast<uint4*>(oa - 2 * ph);
  s.out_units = nullptr;  // set on the device from offsets[0]
  s.lo = s.hi = 0;
  s.left = s.right = -1;
  s.left_ptr = s.right_ptr = nullptr;
  s.tile_sel = kTilesAll;
  s.prefetch_tiles = 0;
  const BatchArgs b{offsets, static_cast<uint64_t>(num_strings) + 1, ph};
  // Persistent grid: the range is only known on the device.
  const uint64_t grid = static_cast<uint64_t>(sm_count_for_current_device()) * 8;
#ifdef U16M_AB_VARIANTS
  const bool same = (ia & 15u) == (oa & 15u);
  if (in == out) return launch<kInPlace, true, true>(s, b, kNoScan, grid, stream);
  if (same) return launch<kCopy, true, true>(s, b, kNoScan, grid, stream);
#endif
  return launch<kCopy, false, true>(s, b, kNoScan, grid, stream);  // out at another 16-byte phase
}

}  // namespace u16m
