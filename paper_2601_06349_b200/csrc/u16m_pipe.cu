// Warp-pipelined streaming kernel: per-warp cp.async rings, persistent warps.
//
// Register-staged loads cap the bytes in flight at about half the register
// file (~128 KiB per SM at 8 x 16 B per thread), and config 1 (in place) is
// latency-bound at that depth (ncu: long-scoreboard stalls ~50%, DRAM ~66%).
// Here every warp streams one contiguous chain of 2 KiB stages through its
// own ring of kD stages in shared memory with 16-byte cp.async copies
// (LDGSTS, L1-bypassing): data in flight lives in shared memory, not in
// registers, so 24 warps x kD x 2 KiB = 192 KiB per SM are in flight while
// the registers hold only the stage being repaired.
//
// Each lane copies and later reads exactly its own 16-byte slots, so the
// ring needs no barriers at all: cp.async.wait_group per thread is the only
// synchronisation. Classification and the halo move through registers and
// shuffles as in the other kernels, rolling across stage boundaries: the
// last vector of a stage takes its look-ahead from the first vector of the
// next stage (already waited for), and the first vector takes its
// look-behind from the carried flags of the previous stage; only the two
// ends of a warp's chain read a 2-byte halo from global memory.

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "u16m_internal.h"
#include "u16m_repair.cuh"

namespace u16m {
namespace pipe {

constexpr int kPV = 4;                         // vectors per lane per stage
constexpr int kStageVecs = 32 * kPV;           // 128 vectors = 2 KiB per warp stage
constexpr int kD = 4;                          // ring depth (stages in flight per warp)
constexpr int kPWarps = 8;
constexpr int kPThreads = kPWarps * 32;
constexpr int kSmemPerWarp = kD * kStageVecs * 16;       // 8 KiB
constexpr int kSmemBytes = kPWarps * kSmemPerWarp;       // 64 KiB per CTA
constexpr int kCtasPerSm = 3;

__device__ __forceinline__ void cp_async16(uint32_t smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

template <bool kInPlace, int kGran, bool kInterleave>
__global__ void __launch_bounds__(kPThreads, kCtasPerSm) pipe_kernel(Span s) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const uint64_t vbeg = s.lo / 8;
  const uint64_t vend = (s.hi + 7) / 8;
  const uint64_t nstages = (vend - vbeg + kStageVecs - 1) / kStageVecs;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kPWarps + warp;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kPWarps;
  // Work items i = c0 .. c1-1 map to stages stage_of(i): a contiguous chain
  // per warp, or (kInterleave) stages gw, gw + nw, gw + 2nw, ... so that the
  // whole grid streams one neighbourhood of DRAM at a time.
  uint64_t c0, c1;
  if (kInterleave) {
    c0 = 0;
    c1 = gw < nstages ? (nstages - gw + nw - 1) / nw : 0;
  } else {
    c0 = nstages * gw / nw;
    c1 = nstages * (gw + 1) / nw;
  }
  if (c0 >= c1) return;
  auto stage_of = [&](uint64_t i) { return kInterleave ? gw + i * nw : i; };
  const uint32_t ring = static_cast<uint32_t>(__cvta_generic_to_shared(smem)) + warp * kSmemPerWarp + lane * 16;

  auto issue = [&](uint64_t i) {  // copy this lane's kPV vectors of item i
    if (i < c1) {
      const uint32_t slot = ring + static_cast<uint32_t>(i % kD) * (kStageVecs * 16);
      const uint64_t v0 = vbeg + stage_of(i) * kStageVecs + lane;
#pragma unroll
      for (int k = 0; k < kPV; k++)
        if (v0 + k * 32 < vend) cp_async16(slot + k * 512, s.in + v0 + k * 32);
    }
    cp_commit();  // one group per stage, empty groups keep the count uniform
  };
  auto fetch = [&](uint64_t i, uint4 (&v)[kPV]) {
    const uint64_t st = stage_of(i);
    const uint32_t slot = ring + static_cast<uint32_t>(i % kD) * (kStageVecs * 16);
#pragma unroll
    for (int k = 0; k < kPV; k++) v[k] = lds128(slot + k * 512);
    const uint64_t v0 = vbeg + st * kStageVecs + lane;
    if ((vbeg + st * kStageVecs) * 8 < s.lo || (vbeg + (st + 1) * kStageVecs) * 8 > s.hi) {
#pragma unroll
      for (int k = 0; k < kPV; k++) {
        const uint64_t vi = v0 + k * 32;
        if (vi * 8 < s.lo || vi * 8 + 8 > s.hi) patch_edges(s, vi, v[k]);
      }
    }
  };

#pragma unroll
  for (int d = 0; d < kD; d++) issue(c0 + d);

  // Look-behind of the chain's first unit (lane 0) — a global 2-byte read.
  uint32_t hp_carry = 0;
  if (lane == 0) hp_carry = hflag_hi(unit_at(s, static_cast<int64_t>((vbeg + stage_of(c0) * kStageVecs) * 8) - 1));

  uint4 v[kPV];
  cp_wait<kD - 1>();
  fetch(c0, v);
  Flags cur = classify8(v[0]);

  for (uint64_t i = c0; i < c1; i++) {
    const uint64_t st = stage_of(i);
    // Flags of the next stage's first vector (look-ahead for lane 31's last).
    uint4 vn[kPV];
    Flags first_next;
    const bool has_next = i + 1 < c1;
    if (has_next) {
      cp_wait<kD - 2>();
      fetch(i + 1, vn);
      first_next = classify8(vn[0]);
    }
    uint32_t ln_tail;
    {
      const uint32_t dn_first = __shfl_sync(kFull, has_next ? first_next.L0 : 0u, (lane + 1) & 31);
      ln_tail = dn_first;
      if ((kInterleave || !has_next) && lane == 31)
        ln_tail = lflag_lo(unit_at(s, static_cast<int64_t>((vbeg + (st + 1) * kStageVecs) * 8)));
    }
    if (kInterleave && lane == 0 && i > c0)
      hp_carry = hflag_hi(unit_at(s, static_cast<int64_t>((vbeg + st * kStageVecs) * 8) - 1));
    const uint64_t v0 = vbeg + st * kStageVecs + lane;
    const bool stage_interior =
        (vbeg + st * kStageVecs) * 8 >= s.lo && (vbeg + (st + 1) * kStageVecs) * 8 <= s.hi;
#pragma unroll
    for (int k = 0; k < kPV; k++) {
      Flags nxt;
      if (k + 1 < kPV) nxt = classify8(v[k + 1]);
      const uint32_t up = __shfl_sync(kFull, cur.H1, (lane + 31) & 31);
      const uint32_t dn = __shfl_sync(kFull, cur.L0, (lane + 1) & 31);
      uint32_t ln = dn;
      if (k + 1 < kPV) {
        const uint32_t dn_next = __shfl_sync(kFull, nxt.L0, (lane + 1) & 31);
        if (lane == 31) ln = dn_next;
      } else if (lane == 31) {
        ln = ln_tail;
      }
      const uint32_t hp = lane ? up : hp_carry;
      hp_carry = up;
      uint32_t B0, B1;
      bad8(cur, hp, ln, B0, B1);
      const bool store = kInPlace ? group_dirty<kGran>((B0 | B1) != 0, lane) : true;
      const uint64_t vi = v0 + k * 32;
      if (stage_interior || (vi * 8 >= s.lo && vi * 8 + 8 <= s.hi)) {
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
      if (k + 1 < kPV) cur = nxt;
    }
    issue(i + kD);  // item i's slot is free: every v[k] has been consumed
    if (has_next) {
#pragma unroll
      for (int k = 0; k < kPV; k++) v[k] = vn[k];
      cur = first_next;
    }
  }
  cp_wait<0>();
}

std::mutex g_mu;
int g_sms[64] = {0};
bool g_ready[64][2][9][2] = {};

static bool interleave() {
  static const bool v = [] {
    const char* e = std::getenv("U16M_PIPE_CHAIN");
    return !(e && e[0] == '1');
  }();
  return v;
}

template <bool kInPlace, int kGran, bool kIL>
cudaError_t launch_t(const Span& s, cudaStream_t stream) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 64) dev = 63;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    if (!g_ready[dev][kInPlace][kGran][kIL]) {
      e = cudaFuncSetAttribute(pipe_kernel<kInPlace, kGran, kIL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kSmemBytes);
      if (e != cudaSuccess) return e;
      int n = 0;
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
      g_sms[dev] = n > 0 ? n : 148;
      g_ready[dev][kInPlace][kGran][kIL] = true;
    }
  }
  const uint64_t vbeg = s.lo / 8, vend = (s.hi + 7) / 8;
  const uint64_t nstages = (vend - vbeg + kStageVecs - 1) / kStageVecs;
  uint64_t grid = static_cast<uint64_t>(g_sms[dev]) * kCtasPerSm;
  const uint64_t need = (nstages + kPWarps - 1) / kPWarps;  // at least one stage per warp
  if (need < grid) grid = need;
  pipe_kernel<kInPlace, kGran, kIL><<<static_cast<unsigned>(grid), kPThreads, kSmemBytes, stream>>>(s);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pipe

template <bool kIL>
static cudaError_t launch_pipe_il(const Span& s, cudaStream_t stream) {
  if (s.in != s.out) return pipe::launch_t<false, 1, kIL>(s, stream);
  switch (inplace_granularity()) {
    case 1: return pipe::launch_t<true, 1, kIL>(s, stream);
    case 4: return pipe::launch_t<true, 4, kIL>(s, stream);
    default: return pipe::launch_t<true, 2, kIL>(s, stream);
  }
}

cudaError_t launch_pipe(const Span& s, cudaStream_t stream) {
  return pipe::interleave() ? launch_pipe_il<true>(s, stream) : launch_pipe_il<false>(s, stream);
}

}  // namespace u16m
