// TMA-pipelined repair kernel (sm_100a): the streaming form of the path.
//
// The register-staged kernel (u16m_kernels.cu) keeps only one 16 KiB tile per
// CTA in flight and stalls its loads while it computes. Here a persistent CTA
// per SM slot runs a producer warp that streams tiles global -> shared memory
// with 1-D bulk async copies (cp.async.bulk, SASS UBLKCP) into a ring of
// kStages stages, each completed on an mbarrier by transaction bytes. Eight
// consumer warps take tiles off the ring, classify + repair in registers
// (u16m_repair.cuh) and store straight to global with 128-bit streaming
// stores; an "empty" mbarrier hands the stage back to the producer as soon as
// every consumer warp has pulled its vectors into registers. Loads therefore
// never wait on compute: up to kStages*16 KiB per CTA are in flight.
//
// Every stage holds the tile plus one 16-byte vector on each side, so the
// one-unit look-behind / look-ahead halos of all warps come from shared
// memory; inside a warp they move with shuffles.
//
// Batched (CSR) form: the producer warp also builds the tile's string-start
// bitmap in the stage (32-ary warp search over offsets + shared atomics)
// after it has issued the tile's bulk copy, and only then arrives on the
// stage's full barrier — the search latency is hidden behind the copies in
// flight and never sits on the consumer path.

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "u16m_internal.h"
#include "u16m_repair.cuh"

namespace u16m {
namespace tma {

constexpr int kConsumerWarps = kWarps;             // 8 warps x 32 lanes x kVecs vectors
constexpr int kThreadsTma = (kConsumerWarps + 1) * 32;
constexpr int kStages = 4;
constexpr int kTmaCtasPerSm = 3;
constexpr int kTileBytes = kCtaVecs * 16;          // 16 KiB
constexpr int kBitmapWords = kCtaUnits / 32 + 2;   // string starts of one tile (+1 unit)
constexpr int kStageBytes = 16 + kTileBytes + 16 + kBitmapWords * 4 + 8;  // pre | tile | post | bitmap
constexpr int kStageStride = (kStageBytes + 127) / 128 * 128;
constexpr int kSmemBytes = kStages * kStageStride + 2 * kStages * 8 + 128;

struct BatchArgsT {
  const int64_t* offsets;
  uint64_t count;  // num_strings + 1
  uint32_t phase;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}

__device__ __forceinline__ uint32_t lds16(uint32_t addr) {
  unsigned short u;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(u) : "r"(addr));
  return u;
}

// Range of the job (device-side for the batched form).
__device__ __forceinline__ void job_range(Span& s, const BatchArgsT& b, bool batched) {
  if (batched) {
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
}

template <int kInPlace, bool kBatched, int kGran>
__global__ void __launch_bounds__(kThreadsTma, kTmaCtasPerSm) repair_tma_kernel(Span s, BatchArgsT b) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageStride);
  uint64_t* empty = full + kStages;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  job_range(s, b, kBatched);
  if (s.hi <= s.lo) return;
  const uint64_t vbeg = s.lo / 8;
  const uint64_t vend = (s.hi + 7) / 8;
  const uint64_t ntiles = (vend - vbeg + kCtaVecs - 1) / kCtaVecs;
  const uint64_t t_begin = ntiles * blockIdx.x / gridDim.x;
  const uint64_t t_end = ntiles * (blockIdx.x + 1) / gridDim.x;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; i++) {
      mbar_init(smem_u32(&full[i]), kBatched ? 2 : 1);
      mbar_init(smem_u32(&empty[i]), kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ------------------------------ producer ------------------------------
    // This CTA owns the contiguous tiles [t_begin, t_end); the batched form
    // searches `offsets` once and then walks it forward tile by tile, with
    // the next tile's 32-entry window prefetched while the ring is full.
    uint32_t it = 0;
    uint64_t sidx = 0;
    int64_t win = INT64_MAX;
    if constexpr (kBatched) {
      if (t_begin < t_end) {
        const int64_t key0 = static_cast<int64_t>((vbeg + t_begin * kCtaVecs) * 8) - static_cast<int64_t>(b.phase);
        sidx = warp_lower_bound(b.offsets, 0, b.count, key0, lane);
        win = sidx + lane < b.count ? __ldg(b.offsets + sidx + lane) : INT64_MAX;
      }
    }
    for (uint64_t tile = t_begin; tile < t_end; tile++, it++) {
      const int st = it % kStages;
      const uint32_t phase = (it / kStages) & 1u;
      unsigned char* stage = smem + st * kStageStride;
      const uint32_t fbar = smem_u32(&full[st]);
      if (it >= kStages) mbar_wait(smem_u32(&empty[st]), phase ^ 1u);
      const uint64_t tv0 = vbeg + tile * kCtaVecs;
      const uint64_t a = tv0 > vbeg ? tv0 - 1 : tv0;                    // with the pre-halo vector
      const uint64_t e = tv0 + kCtaVecs + 1 < vend ? tv0 + kCtaVecs + 1 : vend;  // and the post-halo
      const uint32_t bytes = static_cast<uint32_t>((e - a) * 16);
      if (lane == 0) {
        mbar_arrive_expect_tx(fbar, bytes);
        bulk_g2s(smem_u32(stage + 16 + static_cast<int64_t>(a - tv0) * 16), s.in + a, bytes, fbar);
      }
      if constexpr (kBatched) {
        uint32_t* bits = reinterpret_cast<uint32_t*>(stage + 32 + kTileBytes);
        for (int i = lane; i < kBitmapWords; i += 32) bits[i] = 0;
        __syncwarp();
        const int64_t key_lo = static_cast<int64_t>(tv0 * 8) - static_cast<int64_t>(b.phase);
        const int64_t key_hi = key_lo + kCtaUnits;
        uint64_t scan = sidx, next = sidx;
        int64_t p = win;
        for (;;) {
          const bool inside = p <= key_hi;
          if (inside) {
            const uint64_t bit = static_cast<uint64_t>(p - key_lo);
            atomicOr(&bits[bit >> 5], 1u << (bit & 31));
          }
          next += __popc(__ballot_sync(kFull, p < key_hi));
          if (__ballot_sync(kFull, inside) != kFull) break;
          const int64_t p0 = __shfl_sync(kFull, p, 0), p31 = __shfl_sync(kFull, p, 31);
          if (p0 == p31) {  // a run of equal offsets (empty strings): skip it
            const uint64_t to = skip_equal_offsets(b.offsets, b.count, scan + 32, p31, lane);
            if (p31 < key_hi) next += to - (scan + 32);
            scan = to;
          } else {
            scan += 32;
          }
          p = scan + lane < b.count ? __ldg(b.offsets + scan + lane) : INT64_MAX;
        }
        sidx = next;  // first string starting at or after the next tile's first unit
        win = sidx + lane < b.count ? __ldg(b.offsets + sidx + lane) : INT64_MAX;  // prefetch
        __syncwarp();
        if (lane == 0) mbar_arrive(fbar);  // release: bitmap visible to the consumers
      }
    }
    return;
  }

  // ------------------------------ consumers -------------------------------
  const uint32_t lane_off = static_cast<uint32_t>(warp * kWarpVecs + lane);
  uint32_t it = 0;
  for (uint64_t tile = t_begin; tile < t_end; tile++, it++) {
    const int st = it % kStages;
    const uint32_t phase = (it / kStages) & 1u;
    unsigned char* stage = smem + st * kStageStride;
    const uint32_t sbase = smem_u32(stage + 16);   // vector tv0 of the tile
    const uint64_t tv0 = vbeg + tile * kCtaVecs;
    const bool interior = tv0 * 8 > s.lo && (tv0 + kCtaVecs) * 8 < s.hi;

    mbar_wait(smem_u32(&full[st]), phase);
    uint4 v[kVecs];
#pragma unroll
    for (int k = 0; k < kVecs; k++) v[k] = lds128(sbase + (lane_off + k * 32) * 16);
    uint32_t halo = 0;
    if (lane == 0) halo = lds16(sbase + (lane_off * 16) - 2);
    if (lane == 31) halo = lds16(sbase + (lane_off + (kVecs - 1) * 32 + 1) * 16);
    uint32_t starts_w[kVecs][2];
    if constexpr (kBatched) {
      const uint32_t* bits = reinterpret_cast<const uint32_t*>(stage + 32 + kTileBytes);
#pragma unroll
      for (int k = 0; k < kVecs; k++) {
        const uint32_t a0 = (lane_off + k * 32) * 8;
        starts_w[k][0] = bits[a0 >> 5];
        starts_w[k][1] = bits[(a0 >> 5) + 1];
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&empty[st]));  // stage may be refilled

    bool edge[kVecs];
#pragma unroll
    for (int k = 0; k < kVecs; k++) edge[k] = false;
    if (!interior) {
      // Edge tile of the job: units outside [lo, hi) and halos outside the
      // loaded range follow the range rules (unit_at).
      const uint64_t warp_v0 = tv0 + static_cast<uint64_t>(warp) * kWarpVecs;
      if (lane == 0) halo = unit_at(s, static_cast<int64_t>(warp_v0 * 8) - 1);
      if (lane == 31) halo = unit_at(s, static_cast<int64_t>((warp_v0 + kWarpVecs) * 8));
#pragma unroll
      for (int k = 0; k < kVecs; k++) {
        const uint64_t vi = tv0 + lane_off + k * 32;
        edge[k] = vi * 8 < s.lo || vi * 8 + 8 > s.hi;
        if (edge[k]) patch_edges(s, vi, v[k]);
      }
    }

    Flags f[kVecs];
#pragma unroll
    for (int k = 0; k < kVecs; k++) f[k] = classify8(v[k]);
    const uint32_t halo_h = hflag_hi(halo);
    const uint32_t halo_l = lflag_lo(halo);
    uint32_t up[kVecs], dn[kVecs];
#pragma unroll
    for (int k = 0; k < kVecs; k++) {
      up[k] = __shfl_sync(kFull, f[k].H1, (lane + 31) & 31);
      dn[k] = __shfl_sync(kFull, f[k].L0, (lane + 1) & 31);
    }
    uint4* dst = s.out + tv0 + lane_off;
#pragma unroll
    for (int k = 0; k < kVecs; k++) {
      const uint32_t hp = lane ? up[k] : (k ? up[k - 1] : halo_h);
      const uint32_t ln = lane != 31 ? dn[k] : (k + 1 < kVecs ? dn[k + 1] : halo_l);
      uint32_t B0, B1;
      if constexpr (kBatched) {
        const uint32_t a0 = (lane_off + k * 32) * 8;
        const uint64_t pair = static_cast<uint64_t>(starts_w[k][0]) | (static_cast<uint64_t>(starts_w[k][1]) << 32);
        const uint32_t bits = static_cast<uint32_t>(pair >> (a0 & 31));
        bad8(f[k], hp, ln, B0, B1, spread4(bits), spread4(bits >> 4), ((bits >> 8) & 1u) << 7);
      } else {
        bad8(f[k], hp, ln, B0, B1);
      }
      if (kInPlace && !group_dirty<kGran>((B0 | B1) != 0, lane)) continue;
      const uint4 r = blend(v[k], B0, B1);
      if (!edge[k]) {
        if (interior || tv0 + lane_off + k * 32 < vend) st_stream(dst + k * 32, r);
      } else {
        const uint64_t vi = tv0 + lane_off + k * 32;
        if (vi >= vend) continue;
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
}

std::mutex g_mu;
int g_sms[64] = {0};
bool g_attr_set[4][64][9] = {};

template <int kInPlace, bool kBatched, int kGran>
cudaError_t launch_tma(const Span& s, const BatchArgsT& b, uint64_t ntiles_hint, cudaStream_t stream) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    const int idx = kInPlace * 2 + (kBatched ? 1 : 0);
    if (dev < 64 && !g_attr_set[idx][dev][kGran]) {
      e = cudaFuncSetAttribute(repair_tma_kernel<kInPlace, kBatched, kGran>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
      if (e != cudaSuccess) return e;
      int n = 0;
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
      g_sms[dev] = n > 0 ? n : 148;
      g_attr_set[idx][dev][kGran] = true;
    }
  }
  uint64_t grid = static_cast<uint64_t>(dev < 64 ? g_sms[dev] : 148) * kTmaCtasPerSm;
  if (ntiles_hint > 0 && ntiles_hint < grid) grid = ntiles_hint;
  repair_tma_kernel<kInPlace, kBatched, kGran><<<static_cast<unsigned>(grid), kThreadsTma, kSmemBytes, stream>>>(s, b);
  note_launch();
  return cudaGetLastError();
}

}  // namespace tma

#ifdef U16M_AB_VARIANTS  // plain (non-batched) streams through the TMA ring: A/B only
cudaError_t launch_repair_tma(const uint16_t* in, size_t n, uint16_t* out, int32_t left, int32_t right,
                              const uint16_t* left_ptr, const uint16_t* right_ptr, cudaStream_t stream) {
  const uintptr_t ia = reinterpret_cast<uintptr_t>(in);
  const uintptr_t oa = reinterpret_cast<uintptr_t>(out);
  const uint32_t ph = static_cast<uint32_t>((ia & 15u) / 2);
  Span s;
  s.in = reinterpret_cast<const uint4*>(ia - 2 * ph);
  s.out = reinterpret_cast<uint4*>(oa - 2 * ph);
  s.out_units = out;
  s.lo = ph;
  s.hi = ph + n;
  s.left = left;
  s.right = right;
  s.left_ptr = left_ptr;
  s.right_ptr = right_ptr;
  s.tile_sel = kTilesAll;
  s.prefetch_tiles = 0;
  const uint64_t ntiles = ((s.hi + 7) / 8 - s.lo / 8 + kCtaVecs - 1) / kCtaVecs;
  const tma::BatchArgsT b{nullptr, 0, 0};
  if (in != out) return tma::launch_tma<0, false, 1>(s, b, ntiles, stream);
  return tma::launch_tma<1, false, kDefaultInplaceGran>(s, b, ntiles, stream);
}
#endif

cudaError_t launch_batched_tma(const uint16_t* in, const int64_t* offsets, size_t num_strings, uint16_t* out,
                               cudaStream_t stream) {
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
  const tma::BatchArgsT b{offsets, static_cast<uint64_t>(num_strings) + 1, ph};
  if (in == out) return tma::launch_tma<1, true, 1>(s, b, 0, stream);
  return tma::launch_tma<0, true, 1>(s, b, 0, stream);
}

}  // namespace u16m
