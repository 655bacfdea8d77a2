// On-device generators for BASELINE.json configs 0-4 (harness, not the repair
// path). Independent CUDA implementation of the spec in DESIGN.md §Inputs;
// tests/test_gpu_parity.py checks it bit-exact against the CPU oracle's
// or_gen_config / or_gen_c3_* (oracle/oracle.c).

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/u16m_datagen.h"
#include "u16m_internal.h"

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint32_t kChunk = 4096;
constexpr uint32_t kC2Tile = 256;
constexpr uint32_t kC4Region = 1u << 20;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t key(uint64_t seed, uint64_t stream, uint64_t index) {
  return mix64(seed * kGolden + stream * 0xD1B54A32D192ED03ull + index * 0x8CB92BA72F3D8DD7ull);
}
struct Rng {
  uint64_t s;
  __device__ uint64_t next() {
    s += kGolden;
    return mix64(s);
  }
  __device__ uint32_t below(uint32_t bound) {
    return static_cast<uint32_t>(__umul64hi(next(), static_cast<uint64_t>(bound)));
  }
};

__device__ __forceinline__ uint16_t bmp80(Rng& r) {
  const uint32_t x = r.below(0xD780u + 0x2000u);
  return static_cast<uint16_t>(x < 0xD780u ? 0x80u + x : 0xE000u + (x - 0xD780u));
}
__device__ __forceinline__ uint16_t bmp20(Rng& r) {
  const uint32_t x = r.below(0xD7E0u + 0x2000u);
  return static_cast<uint16_t>(x < 0xD7E0u ? 0x20u + x : 0xE000u + (x - 0xD7E0u));
}

// Config-0 character; returns units written (1 or 2).
__device__ int c0_char(Rng& r, uint16_t* d, uint64_t room, bool allow_lone) {
  const uint32_t x = r.below(allow_lone ? 1000u : 990u);
  if (x < 700u) { d[0] = static_cast<uint16_t>(0x20u + r.below(95u)); return 1; }
  if (x < 940u) { d[0] = bmp80(r); return 1; }
  if (x < 990u) {
    if (room >= 2) {
      d[0] = static_cast<uint16_t>(0xD800u + r.below(1024u));
      d[1] = static_cast<uint16_t>(0xDC00u + r.below(1024u));
      return 2;
    }
    d[0] = bmp80(r);
    return 1;
  }
  if (x < 995u) { d[0] = static_cast<uint16_t>(0xD800u + r.below(1024u)); return 1; }
  d[0] = static_cast<uint16_t>(0xDC00u + r.below(1024u));
  return 1;
}

__device__ int c2_char(Rng& r, uint16_t* d, uint64_t room) {
  const uint32_t x = r.below(100000u);
  if (x < 5u) { d[0] = static_cast<uint16_t>(0xD800u + r.below(1024u)); return 1; }
  if (x < 10u) { d[0] = static_cast<uint16_t>(0xDC00u + r.below(1024u)); return 1; }
  if (x < 50005u && room >= 2) {
    const uint32_t cp = 0x1F300u + r.below(0x800u) - 0x10000u;
    d[0] = static_cast<uint16_t>(0xD800u + (cp >> 10));
    d[1] = static_cast<uint16_t>(0xDC00u + (cp & 0x3FFu));
    return 2;
  }
  d[0] = bmp20(r);
  return 1;
}

// One thread per 4096-unit chunk of the logical buffer; writes the part of the
// chunk inside [first, first+count).
__global__ void gen_base_kernel(int cfg, uint64_t seed, uint64_t total, uint64_t first,
                                uint64_t count, uint64_t c0, uint64_t nchunks, uint16_t* out) {
  const uint64_t ci = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (ci >= nchunks) return;
  const uint64_t c = c0 + ci;
  const uint64_t a = c * kChunk;
  const uint64_t len = total - a < kChunk ? total - a : kChunk;
  const uint64_t end = first + count;
  Rng r{key(seed, 1, c)};
  uint16_t tmp[2];
  uint64_t k = 0;
  auto put = [&](uint64_t pos, uint16_t u) {
    if (pos >= first && pos < end) out[pos - first] = u;
  };
  if (cfg == 1) {
    while (k < len) {
      const uint64_t v = r.next();
      for (int j = 0; j < 4 && k < len; j++, k++) put(a + k, static_cast<uint16_t>(v >> (16 * j)));
    }
    return;
  }
  while (k < len) {
    const int m = cfg == 2 ? c2_char(r, tmp, len - k) : c0_char(r, tmp, len - k, true);
    for (int j = 0; j < m; j++) put(a + k + j, tmp[j]);
    k += m;
  }
}

__device__ int boundary_pattern(uint64_t seed, uint64_t stream, uint64_t tag, int kind,
                                uint16_t* val) {
  Rng r{key(seed, stream, tag)};
  const uint16_t h = static_cast<uint16_t>(0xD800u + r.below(1024u));
  const uint16_t l = static_cast<uint16_t>(0xDC00u + r.below(1024u));
  const uint16_t h2 = static_cast<uint16_t>(0xD800u + r.below(1024u));
  const uint16_t l2 = static_cast<uint16_t>(0xDC00u + r.below(1024u));
  switch (kind) {
    case 0: val[0] = h; val[1] = l; return 2;
    case 1: val[0] = h; val[1] = 0x0041; return 2;
    case 2: val[0] = 0x0042; val[1] = l; return 2;
    case 3: val[0] = h; val[1] = h2; val[2] = l; return 3;
    default: val[0] = l; val[1] = l2; return 2;
  }
}

// Boundary b = t * spacing for t in [t0, t0 + nt); pattern t % 5; writes b-1, b, b+1.
__global__ void gen_boundary_kernel(uint64_t seed, uint64_t stream, uint64_t spacing, uint64_t t0,
                                    uint64_t nt, uint64_t total, uint64_t first, uint64_t count,
                                    uint16_t* out) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= nt) return;
  const uint64_t t = t0 + i;
  const uint64_t b = t * spacing;
  uint16_t val[3];
  const int m = boundary_pattern(seed, stream, t, static_cast<int>(t % 5), val);
  for (int j = 0; j < m; j++) {
    const uint64_t p = b - 1 + j;
    if (p >= first && p < first + count && p < total) out[p - first] = val[j];
  }
}

// One CTA per 1 Mi-unit region of config 4; 10% of regions carry a run.
__global__ void gen_c4_runs_kernel(uint64_t seed, uint64_t total, uint64_t first, uint64_t count,
                                   uint64_t r0, uint16_t* out) {
  const uint64_t r = r0 + blockIdx.x;
  Rng g{key(seed, 5, r)};
  const uint32_t d = g.below(100u);
  if (d < 90u) return;
  const uint64_t ra = r * kC4Region;
  const uint64_t rlen = total - ra < kC4Region ? total - ra : kC4Region;
  const uint64_t len = 1u + g.below(static_cast<uint32_t>(rlen));
  const uint64_t st = ra + g.below(static_cast<uint32_t>(rlen - len + 1));
  const uint32_t phase = g.below(2u);
  const uint64_t end = first + count;
  const uint64_t lo = st > first ? st : first;
  const uint64_t hi = st + len < end ? st + len : end;
  for (uint64_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
    uint16_t v = 0xD800;
    if (d >= 95u) v = ((p - st + phase) & 1u) ? 0xDC00 : 0xD800;
    out[p - first] = v;
  }
}

__global__ void c3_lengths_kernel(uint64_t seed, uint64_t S, int64_t* offsets) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i == 0) offsets[0] = 0;
  if (i >= S) return;
  Rng r{key(seed, 3, i)};
  const uint32_t e = r.below(12u);
  offsets[i + 1] = static_cast<int64_t>((1u << e) + r.below(1u << e));
}

// Inclusive scan of offsets[1..S] in place, one CTA of 1024 threads.
__global__ void __launch_bounds__(1024) c3_scan_kernel(int64_t* offsets, uint64_t S) {
  __shared__ long long warp_tot[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t base = 0; base < S; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const long long c = i < S ? offsets[i + 1] : 0;
    long long x = c;
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    long long before = carry;
    for (int w = 0; w < warp; w++) before += warp_tot[w];
    if (i < S) offsets[i + 1] = before + x;
    __syncthreads();
    if (threadIdx.x == 1023) carry = before + x;
    __syncthreads();
  }
}

__global__ void c3_content_kernel(uint64_t seed, uint64_t S, const int64_t* offsets, uint16_t* out) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= S) return;
  uint16_t* x = out + offsets[i];
  const uint64_t len = static_cast<uint64_t>(offsets[i + 1] - offsets[i]);
  Rng r{key(seed, 4, i)};
  const bool has_err = r.below(100u) < 20u;
  uint64_t k = 0;
  uint16_t tmp[2];
  while (k < len) {
    const int m = c0_char(r, tmp, len - k, false);
    for (int j = 0; j < m; j++) x[k + j] = tmp[j];
    k += m;
  }
  if (has_err) {
    const uint32_t m = 1u + r.below(8u);
    for (uint32_t j = 0; j < m; j++) {
      const uint64_t p = r.below(static_cast<uint32_t>(len));
      const uint32_t hl = r.below(2u);
      x[p] = static_cast<uint16_t>((hl ? 0xD800u : 0xDC00u) + r.below(1024u));
    }
  }
  if (r.below(100u) < 3u) x[0] = static_cast<uint16_t>(0xDC00u + r.below(1024u));
  if (r.below(100u) < 3u) x[len - 1] = static_cast<uint16_t>(0xD800u + r.below(1024u));
}

__global__ void l2_flush_kernel(const uint4* p, size_t n16, unsigned* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n16;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u && sink) *sink = acc;  // keep the loads alive
}

thread_local std::string t_err;

u16m_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return U16M_OK;
  t_err = cudaGetErrorString(e);
  return U16M_ERR_CUDA;
}

unsigned grid_for(uint64_t n, unsigned block) { return static_cast<unsigned>((n + block - 1) / block); }

}  // namespace

extern "C" {

u16m_status u16m_gen_config(int cfg, uint64_t seed, uint64_t total, uint64_t shard_len,
                            uint64_t first, uint64_t count, uint16_t* out, void* stream_v) {
  if ((cfg != 0 && cfg != 1 && cfg != 2 && cfg != 4) || first + count > total || (count && !out))
    return U16M_ERR_INVALID_ARGUMENT;
  if (count == 0) return U16M_OK;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  const uint64_t end = first + count;
  const uint64_t c0 = first / kChunk, c1 = (end + kChunk - 1) / kChunk;
  gen_base_kernel<<<grid_for(c1 - c0, 128), 128, 0, stream>>>(cfg, seed, total, first, count, c0,
                                                              c1 - c0, out);
  u16m::note_launch();
  if (cfg == 2) {
    const uint64_t t0 = first / kC2Tile < 1 ? 1 : first / kC2Tile;
    const uint64_t t1 = end / kC2Tile;  // inclusive
    if (t1 >= t0) {
      gen_boundary_kernel<<<grid_for(t1 - t0 + 1, 256), 256, 0, stream>>>(
          seed, 2, kC2Tile, t0, t1 - t0 + 1, total, first, count, out);
      u16m::note_launch();
    }
  }
  if (cfg == 4) {
    const uint64_t r0 = first / kC4Region, r1 = (end + kC4Region - 1) / kC4Region;
    gen_c4_runs_kernel<<<static_cast<unsigned>(r1 - r0), 256, 0, stream>>>(seed, total, first, count,
                                                                          r0, out);
    u16m::note_launch();
    if (shard_len > 0 && total > shard_len) {
      const uint64_t nb = (total - 1) / shard_len;  // k = 1 .. nb
      gen_boundary_kernel<<<grid_for(nb, 256), 256, 0, stream>>>(seed, 6, shard_len, 1, nb, total,
                                                                 first, count, out);
      u16m::note_launch();
    }
  }
  return cuda_status(cudaGetLastError());
}

u16m_status u16m_gen_c3_offsets(uint64_t seed, size_t num_strings, int64_t* offsets,
                                uint64_t* total_units) {
  if (!offsets) return U16M_ERR_INVALID_ARGUMENT;
  c3_lengths_kernel<<<grid_for(num_strings > 0 ? num_strings : 1, 256), 256>>>(seed, num_strings,
                                                                               offsets);
  c3_scan_kernel<<<1, 1024>>>(offsets, num_strings);
  u16m::note_launch();
  u16m::note_launch();
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) {
    int64_t t = 0;
    e = cudaMemcpy(&t, offsets + num_strings, sizeof(t), cudaMemcpyDeviceToHost);
    if (total_units) *total_units = static_cast<uint64_t>(t);
  }
  return cuda_status(e);
}

u16m_status u16m_gen_c3_content(uint64_t seed, size_t num_strings, const int64_t* offsets,
                                uint16_t* out, void* stream_v) {
  if (!offsets || !out) return U16M_ERR_INVALID_ARGUMENT;
  if (num_strings == 0) return U16M_OK;
  c3_content_kernel<<<grid_for(num_strings, 128), 128, 0, static_cast<cudaStream_t>(stream_v)>>>(
      seed, num_strings, offsets, out);
  u16m::note_launch();
  return cuda_status(cudaGetLastError());
}

u16m_status u16m_l2_flush(const void* buf, size_t bytes, void* stream_v) {
  if (!buf) return U16M_ERR_INVALID_ARGUMENT;
  l2_flush_kernel<<<148 * 8, 256, 0, static_cast<cudaStream_t>(stream_v)>>>(
      static_cast<const uint4*>(buf), bytes / 16, nullptr);
  u16m::note_launch();
  return cuda_status(cudaGetLastError());
}

}  // extern "C"
