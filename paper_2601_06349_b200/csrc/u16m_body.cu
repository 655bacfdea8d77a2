// Lean body kernel: the interior tiles of a copy / in-place repair.
//
// Every tile this kernel sees is "interior": all of its 16-byte vectors are
// inside the logical range and so are the units just before and after it.
// That removes every range check from the hot loop; the (at most two) edge
// tiles of a job go to the general kernel in u16m_kernels.cu, launched
// alongside this one (programmatic dependent launch lets the two grids run
// concurrently — they write disjoint units, and the only cross-reads are
// the benign in-place halo reads).
//
// Per thread: 4 x 128-bit streaming loads issued back to back (64 B in
// flight), lanes 0 / 31 load the warp tile's 2-byte halo units, SWAR
// classification + shuffle halo + blend (u16m_repair.cuh), 128-bit
// streaming stores (in place: only vectors holding a rewrite).
// Index math is one 64-bit base per tile; everything else is 32-bit.

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "u16m_internal.h"
#include "u16m_repair.cuh"

namespace u16m {

// In-place write-back granularity in lanes of 16 B (U16M_GRAN: 1, 2, 4, 8).
int inplace_granularity() {
  static const int g = [] {
    const char* e = std::getenv("U16M_GRAN");
    const int v = e ? std::atoi(e) : kDefaultInplaceGran;
    return (v == 1 || v == 2 || v == 4 || v == 8) ? v : kDefaultInplaceGran;
  }();
  return g;
}

template <bool kInPlace, int kGran>
__global__ void __launch_bounds__(kThreads) body_kernel(const uint4* __restrict__ in, uint4* out,
                                                        uint64_t first_vec) {
  const int lane = threadIdx.x & 31;
  const uint32_t lane_off = threadIdx.x / 32 * kWarpVecs + lane;
  const uint64_t v0 = first_vec + static_cast<uint64_t>(blockIdx.x) * kCtaVecs + lane_off;
  const uint4* src = in + v0;

  uint4 v[kVecs];
#pragma unroll
  for (int k = 0; k < kVecs; k++) v[k] = ld_stream(src + k * 32);
  const uint16_t* src16 = reinterpret_cast<const uint16_t*>(src);
  uint32_t halo = 0;
  if (lane == 0) halo = src16[-1];
  if (lane == 31) halo = src16[(kVecs - 1) * 32 * 8 + 8];

  Flags f[kVecs];
#pragma unroll
  for (int k = 0; k < kVecs; k++) f[k] = classify8(v[k]);
  uint32_t up[kVecs], dn[kVecs];
#pragma unroll
  for (int k = 0; k < kVecs; k++) {
    up[k] = __shfl_sync(kFull, f[k].H1, (lane + 31) & 31);
    dn[k] = __shfl_sync(kFull, f[k].L0, (lane + 1) & 31);
  }
  const uint32_t halo_h = hflag_hi(halo);
  const uint32_t halo_l = lflag_lo(halo);
  uint4* dst = out + v0;
#pragma unroll
  for (int k = 0; k < kVecs; k++) {
    const uint32_t hp = lane ? up[k] : (k ? up[k - 1] : halo_h);
    const uint32_t ln = lane != 31 ? dn[k] : (k + 1 < kVecs ? dn[k + 1] : halo_l);
    uint32_t B0, B1;
    bad8(f[k], hp, ln, B0, B1);
    if (kInPlace) {
      if (group_dirty<kGran>((B0 | B1) != 0, lane)) st_stream(dst + k * 32, blend(v[k], B0, B1));
    } else {
      st_stream(dst + k * 32, blend(v[k], B0, B1));
    }
  }
}

cudaError_t launch_body(const uint4* in, uint4* out, uint64_t first_vec, uint64_t ntiles, bool in_place,
                        cudaStream_t stream) {
  if (ntiles == 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(ntiles));
  cfg.blockDim = dim3(kThreads);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (!in_place) {
    e = cudaLaunchKernelEx(&cfg, body_kernel<false, 1>, in, out, first_vec);
  } else {
    switch (inplace_granularity()) {
      case 1: e = cudaLaunchKernelEx(&cfg, body_kernel<true, 1>, in, out, first_vec); break;
      case 2: e = cudaLaunchKernelEx(&cfg, body_kernel<true, 2>, in, out, first_vec); break;
      case 8: e = cudaLaunchKernelEx(&cfg, body_kernel<true, 8>, in, out, first_vec); break;
      default: e = cudaLaunchKernelEx(&cfg, body_kernel<true, 4>, in, out, first_vec); break;
    }
  }
  note_launch();
  return e;
}

}  // namespace u16m
