// Device-side building blocks of the sm_100a repair kernels.
//
// The reference repairs 32-unit blocks with AVX-512 mask registers
// (proj/src/bitmask_kernel_avx512.cpp:30-61): lookback/XOR detection, a
// masked FFFD blend, and an end-aligned overlapping tail. On the B200 the same
// 3-point stencil is evaluated without blocks-with-
// lookback at all:
//   * each thread owns 16-byte vectors (8 units) loaded with 128-bit
//     coalesced accesses; a warp owns a contiguous tile of kVecs*512 bytes;
//   * per-unit classification is SWAR in registers: one PRMT gathers the high
//     bytes of 4 units into a word, and the surrogate / high / low tests are
//     byte-lane bit tricks (flag = bit 7 of each byte lane);
//   * the one-unit look-behind / look-ahead halo moves between lanes with two
//     warp shuffles per vector (H flags up, L flags down); only the two ends
//     of a warp tile load a 2-byte halo unit from global memory;
//   * the FFFD blend is one PRMT (sign-replicating byte select -> 16-bit
//     lane masks) plus one LOP3 per 32-bit word.
#pragma once

#include <cstdint>

namespace u16m {

constexpr int kThreads = 256;                   // threads per CTA
constexpr int kWarps = kThreads / 32;           // warps per CTA
constexpr int kVecs = 4;                        // 16 B vectors per thread per tile
constexpr int kWarpVecs = 32 * kVecs;           // vectors per warp tile
constexpr int kCtaVecs = kWarps * kWarpVecs;    // vectors per CTA tile
constexpr int kCtaUnits = kCtaVecs * 8;         // 8192 units = 16 KiB per CTA tile
constexpr uint32_t kFull = 0xFFFFFFFFu;

// Aligned-coordinate view of a logical range. Unit `a` (aligned coordinate)
// lives at ((const uint16_t*)base)[a]; the logical units are [lo, hi).
// Units outside the range read as their halo: a == lo-1 -> left neighbour,
// a == hi -> right neighbour, anything else -> 0 (a non-surrogate: "outside").
struct Span {
  const uint4* in;         // 16-byte aligned
  uint4* out;              // 16-byte aligned, same phase as in (fast path)
  uint16_t* out_units;     // out for the other-phase path: out_units[a - lo]
  uint64_t lo, hi;         // logical range in aligned units
  int32_t left, right;     // halo unit values, -1 = outside the logical buffer
  const uint16_t* left_ptr;   // device-side halo (overrides left/right if set)
  const uint16_t* right_ptr;
  int tile_sel;            // kTilesAll / kTilesEdges / kTilesInterior
  int prefetch_tiles;      // stream kernel: L2 bulk-prefetch distance in tiles (0 = off)
};

enum TileSel : int { kTilesAll = 0, kTilesEdges = 1, kTilesInterior = 2 };

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void st_stream(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// High/low-surrogate flags for the 4 units in words (wa, wb): bit 7 of byte
// lane j is set iff unit j is a high (H) / low (L) surrogate.
__device__ __forceinline__ void classify4(uint32_t wa, uint32_t wb, uint32_t& H, uint32_t& L) {
  const uint32_t hb = prmt(wa, wb, 0x7531);           // high bytes of units 0..3
  const uint32_t s = (hb & 0xF8F8F8F8u) ^ 0xD8D8D8D8u;  // 0 in lane j <=> surrogate
  const uint32_t t = (s >> 1) + 0x7C7C7C7Cu;           // bit 7 <=> lane nonzero (no carries)
  const uint32_t sur = ~t & 0x80808080u;
  const uint32_t b10 = hb << 5;                        // unit bit 10 -> lane bit 7
  H = sur & ~b10;
  L = sur & b10;
}

// Big-endian byte order (§8(f-3) codec fusion): the high byte of each unit
// is the FIRST byte in memory, so only the byte-gather selector changes; the
// vector stays in memory order end to end.
__device__ __forceinline__ void classify4_be(uint32_t wa, uint32_t wb, uint32_t& H, uint32_t& L) {
  const uint32_t hb = prmt(wa, wb, 0x6420);
  const uint32_t s = (hb & 0xF8F8F8F8u) ^ 0xD8D8D8D8u;
  const uint32_t t = (s >> 1) + 0x7C7C7C7Cu;
  const uint32_t sur = ~t & 0x80808080u;
  const uint32_t b10 = hb << 5;
  H = sur & ~b10;
  L = sur & b10;
}

// Flags of one vector: units 0-3 in (H0,L0), units 4-7 in (H1,L1).
struct Flags {
  uint32_t H0, L0, H1, L1;
};

template <bool kBE = false>
__device__ __forceinline__ Flags classify8(const uint4& v) {
  Flags f;
  if constexpr (kBE) {
    classify4_be(v.x, v.y, f.H0, f.L0);
    classify4_be(v.z, v.w, f.H1, f.L1);
  } else {
    classify4(v.x, v.y, f.H0, f.L0);
    classify4(v.z, v.w, f.H1, f.L1);
  }
  return f;
}

// Unit value <-> its 16-bit memory word in the given byte order.
template <bool kBE>
__device__ __forceinline__ uint32_t to_mem(uint32_t u) {
  return kBE ? (((u & 0xFFu) << 8) | ((u >> 8) & 0xFFu)) : u;
}

// Bad-unit flags. hp: byte lane 3 holds H(unit before unit 0); ln: byte lane
// 0 holds L(unit after unit 7). S0/S1/S2: optional string-start flags for
// units 0-3, 4-7 and the unit after unit 7 (batched form): a string start has
// no predecessor, and the unit before it has no successor.
__device__ __forceinline__ void bad8(const Flags& f, uint32_t hp, uint32_t ln, uint32_t& B0,
                                     uint32_t& B1, uint32_t S0 = 0, uint32_t S1 = 0,
                                     uint32_t S2 = 0) {
  uint32_t hprev0 = __funnelshift_l(hp, f.H0, 8);
  uint32_t hprev1 = __funnelshift_l(f.H0, f.H1, 8);
  uint32_t lnext0 = __funnelshift_r(f.L0, f.L1, 8);
  uint32_t lnext1 = __funnelshift_r(f.L1, ln, 8);
  hprev0 &= ~S0;
  hprev1 &= ~S1;
  lnext0 &= ~__funnelshift_r(S0, S1, 8);
  lnext1 &= ~__funnelshift_r(S1, S2, 8);
  B0 = (f.H0 & ~lnext0) | (f.L0 & ~hprev0);
  B1 = (f.H1 & ~lnext1) | (f.L1 & ~hprev1);
}

// Replace every flagged unit with U+FFFD. prmt selector nibbles 8..B copy
// byte 0..3 with its sign bit replicated -> 0xFF / 0x00 byte masks. U+FFFD in
// memory order is FD FF (LE) or FF FD (BE).
template <bool kBE = false>
__device__ __forceinline__ uint4 blend(uint4 v, uint32_t B0, uint32_t B1) {
  constexpr uint32_t R = kBE ? 0xFDFFFDFFu : 0xFFFDFFFDu;
  uint32_t m;
  m = prmt(B0, 0, 0x9988);
  v.x = (v.x & ~m) | (R & m);
  m = prmt(B0, 0, 0xBBAA);
  v.y = (v.y & ~m) | (R & m);
  m = prmt(B1, 0, 0x9988);
  v.z = (v.z & ~m) | (R & m);
  m = prmt(B1, 0, 0xBBAA);
  v.w = (v.w & ~m) | (R & m);
  return v;
}

__device__ __forceinline__ uint32_t halo_value(const Span& s, bool left_side) {
  if (left_side) {
    if (s.left_ptr) return *s.left_ptr;
    return s.left >= 0 ? static_cast<uint32_t>(s.left) : 0u;
  }
  if (s.right_ptr) return *s.right_ptr;
  return s.right >= 0 ? static_cast<uint32_t>(s.right) : 0u;
}

// Unit at aligned coordinate a (may be -1), honouring the range and halos.
__device__ __forceinline__ uint32_t unit_at(const Span& s, int64_t a) {
  if (a < static_cast<int64_t>(s.lo)) return a == static_cast<int64_t>(s.lo) - 1 ? halo_value(s, true) : 0u;
  if (a >= static_cast<int64_t>(s.hi)) return a == static_cast<int64_t>(s.hi) ? halo_value(s, false) : 0u;
  return reinterpret_cast<const uint16_t*>(s.in)[a];
}

__device__ __forceinline__ uint32_t get_unit(const uint4& v, int j) {
  const uint32_t w = j < 4 ? (j < 2 ? v.x : v.y) : (j < 6 ? v.z : v.w);
  return (j & 1) ? (w >> 16) : (w & 0xFFFFu);
}

__device__ __forceinline__ void set_unit(uint4& v, int j, uint32_t u) {
  uint32_t* w = j < 4 ? (j < 2 ? &v.x : &v.y) : (j < 6 ? &v.z : &v.w);
  *w = (j & 1) ? ((*w & 0x0000FFFFu) | (u << 16)) : ((*w & 0xFFFF0000u) | (u & 0xFFFFu));
}

// Vector vi straddles or lies outside [lo, hi): substitute out-of-range units
// (halo values are unit values; the vector is in memory byte order).
template <bool kBE = false>
__device__ __forceinline__ void patch_edges(const Span& s, uint64_t vi, uint4& v) {
  for (int j = 0; j < 8; j++) {
    const uint64_t a = vi * 8 + j;
    if (a < s.lo || a >= s.hi) set_unit(v, j, to_mem<kBE>(unit_at(s, static_cast<int64_t>(a))));
  }
}

// Clear the flags of units outside [lo, hi) (edge vectors; counting).
__device__ __forceinline__ void mask_outside(const Span& s, uint64_t vi, uint32_t& B0, uint32_t& B1) {
#pragma unroll
  for (int j = 0; j < 8; j++) {
    const uint64_t a = vi * 8 + j;
    if (a < s.lo || a >= s.hi) {
      if (j < 4) B0 &= ~(0x80u << (8 * j));
      else B1 &= ~(0x80u << (8 * (j - 4)));
    }
  }
}

__device__ __forceinline__ uint32_t hflag_hi(uint32_t u) {  // H(u) in byte lane 3
  return ((u & 0xFC00u) == 0xD800u) ? 0x80000000u : 0u;
}
__device__ __forceinline__ uint32_t lflag_lo(uint32_t u) {  // L(u) in byte lane 0
  return ((u & 0xFC00u) == 0xDC00u) ? 0x80u : 0u;
}

// In-place store policy: a lane writes its vector back when any lane of its
// aligned group of kGran lanes (kGran*16 contiguous bytes) holds a rewrite.
// kGran = 1 writes only dirty 16-byte vectors; larger groups trade extra
// bytes for whole-burst DRAM writes instead of scattered partial sectors.
// All 32 lanes must call it (warp ballot).
template <int kGran>
__device__ __forceinline__ bool group_dirty(bool dirty, int lane) {
  if constexpr (kGran == 1) {
    return dirty;
  } else {
    const uint32_t m = __ballot_sync(kFull, dirty);
    const uint32_t g = (kGran >= 32 ? 0xFFFFFFFFu : ((1u << kGran) - 1u)) << (lane & ~(kGran - 1));
    return (m & g) != 0;
  }
}

// ---- CSR offsets searches (warp-cooperative, warp-uniform results) ----------
// First index in [lo, hi) with off[idx] >= key, or hi: a 32-ary search, one
// dependent round of 32 loads per factor of 32.
__device__ __forceinline__ uint64_t warp_lower_bound(const int64_t* off, uint64_t lo, uint64_t hi, int64_t key,
                                                     int lane) {
  while (hi - lo > 32) {
    const uint64_t step = (hi - lo + 31) / 32;
    const uint64_t idx = lo + static_cast<uint64_t>(lane) * step;
    const bool pred = idx < hi ? (__ldg(off + idx) >= key) : true;
    const uint32_t m = __ballot_sync(kFull, pred);
    if (m == 0) {
      lo = lo + 31 * step + 1;
    } else {
      const int f = __ffs(m) - 1;
      if (f == 0) {
        hi = lo;
      } else {
        const uint64_t nlo = lo + static_cast<uint64_t>(f - 1) * step + 1;
        const uint64_t cand = lo + static_cast<uint64_t>(f) * step;
        hi = cand < hi ? cand : hi;
        lo = nlo;
      }
    }
  }
  const uint64_t idx = lo + lane;
  const bool pred = idx < hi ? (__ldg(off + idx) >= key) : true;
  const uint32_t m = __ballot_sync(kFull, pred);
  return m ? lo + (__ffs(m) - 1) : hi;
}

// First index >= lo with off[idx] > v, or count. Galloping (lane k probes
// lo + 2^k - 1), then a 32-ary search of the bracket: O(log run) rounds, so a
// run of a million equal offsets (empty strings) costs a few loads, not a
// million-entry walk.
// Out of line: it runs only on runs of empty strings, and inlining it into
// the tile kernels' scan loops measurably slowed the common path (C3 -1.5 %).
static __device__ __noinline__ uint64_t skip_equal_offsets(const int64_t* off, uint64_t count, uint64_t lo, int64_t v,
                                                       int lane) {
  for (;;) {
    if (lo >= count) return count;
    const uint64_t idx = lo + ((1ull << lane) - 1);
    const bool gt = idx >= count || __ldg(off + idx) > v;
    const uint32_t m = __ballot_sync(kFull, gt);
    if (m == 0) {  // 2^31 equal entries: keep galloping
      lo += 1ull << 31;
      continue;
    }
    const int k = __ffs(m) - 1;
    const uint64_t blo = k == 0 ? lo : lo + (1ull << (k - 1));
    uint64_t bhi = lo + (1ull << k) - 1;
    if (bhi > count) bhi = count;
    return warp_lower_bound(off, blo, bhi, v + 1, lane);
  }
}

// Start of the next 32-entry window of a forward offsets scan whose current
// window (this lane's entry p) starts at `scan`: scan + 32, or past the whole
// run when the window holds one repeated value.
__device__ __forceinline__ uint64_t next_offsets_window(const int64_t* off, uint64_t count, uint64_t scan,
                                                        int64_t p, int lane) {
  int same = 0;
  __match_all_sync(kFull, p, &same);
  return same ? skip_equal_offsets(off, count, scan + 32, p, lane) : scan + 32;
}

// 4 bits -> bit 7 of byte lanes 0..3.
__device__ __forceinline__ uint32_t spread4(uint32_t bits) {
  return (((bits & 0xFu) * 0x00204081u) & 0x01010101u) << 7;
}

}  // namespace u16m
