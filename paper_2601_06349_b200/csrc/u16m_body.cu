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

// kV vectors per thread; a CTA always covers one 1024-vector tile, so the
// block has 1024/kV threads (U16M_BODY_VECS selects 2, 4 or 8 for A/B runs).
template <bool kInPlace, int kGran, int kV>
__global__ void __launch_bounds__(kCtaVecs / kV) body_kernel(const uint4* __restrict__ in, uint4* out,
                                                             uint64_t first_vec) {
  constexpr int kWV = 32 * kV;  // vectors per warp tile
  const int lane = threadIdx.x & 31;
  const uint32_t lane_off = threadIdx.x / 32 * kWV + lane;
  const uint64_t v0 = first_vec + static_cast<uint64_t>(blockIdx.x) * kCtaVecs + lane_off;
  const uint4* src = in + v0;

  uint4 v[kV];
#pragma unroll
  for (int k = 0; k < kV; k++) v[k] = ld_stream(src + k * 32);
  const uint16_t* src16 = reinterpret_cast<const uint16_t*>(src);
  uint32_t halo = 0;
  if (lane == 0) halo = src16[-1];
  if (lane == 31) halo = src16[(kV - 1) * 32 * 8 + 8];

  Flags f[kV];
#pragma unroll
  for (int k = 0; k < kV; k++) f[k] = classify8(v[k]);
  uint32_t up[kV], dn[kV];
#pragma unroll
  for (int k = 0; k < kV; k++) {
    up[k] = __shfl_sync(kFull, f[k].H1, (lane + 31) & 31);
    dn[k] = __shfl_sync(kFull, f[k].L0, (lane + 1) & 31);
  }
  const uint32_t halo_h = hflag_hi(halo);
  const uint32_t halo_l = lflag_lo(halo);
  uint4* dst = out + v0;
#pragma unroll
  for (int k = 0; k < kV; k++) {
    const uint32_t hp = lane ? up[k] : (k ? up[k - 1] : halo_h);
    const uint32_t ln = lane != 31 ? dn[k] : (k + 1 < kV ? dn[k + 1] : halo_l);
    uint32_t B0, B1;
    bad8(f[k], hp, ln, B0, B1);
    if (kInPlace) {
      if (group_dirty<kGran>((B0 | B1) != 0, lane)) st_stream(dst + k * 32, blend(v[k], B0, B1));
    } else {
      st_stream(dst + k * 32, blend(v[k], B0, B1));
    }
  }
}

static int body_vecs() {
  static const int v = [] {
    const char* e = std::getenv("U16M_BODY_VECS");
    const int x = e ? std::atoi(e) : 4;
    return (x == 2 || x == 4 || x == 8) ? x : 4;
  }();
  return v;
}

template <int kV>
static cudaError_t launch_body_v(cudaLaunchConfig_t& cfg, const uint4* in, uint4* out, uint64_t first_vec,
                                 bool in_place) {
  cfg.blockDim = dim3(kCtaVecs / kV);
  if (!in_place) return cudaLaunchKernelEx(&cfg, body_kernel<false, 1, kV>, in, out, first_vec);
  switch (inplace_granularity()) {
    case 1: return cudaLaunchKernelEx(&cfg, body_kernel<true, 1, kV>, in, out, first_vec);
    case 4: return cudaLaunchKernelEx(&cfg, body_kernel<true, 4, kV>, in, out, first_vec);
    case 8: return cudaLaunchKernelEx(&cfg, body_kernel<true, 8, kV>, in, out, first_vec);
    default: return cudaLaunchKernelEx(&cfg, body_kernel<true, 2, kV>, in, out, first_vec);
  }
}

cudaError_t launch_body(const uint4* in, uint4* out, uint64_t first_vec, uint64_t ntiles, bool in_place,
                        cudaStream_t stream) {
  if (ntiles == 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(ntiles));
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  switch (body_vecs()) {
    case 2: e = launch_body_v<2>(cfg, in, out, first_vec, in_place); break;
    case 8: e = launch_body_v<8>(cfg, in, out, first_vec, in_place); break;
    default: e = launch_body_v<4>(cfg, in, out, first_vec, in_place); break;
  }
  note_launch();
  return e;
}

}  // namespace u16m
