// Probe (not product): does any load / store cache policy move the in-place
// access pattern — read every 16-byte vector, write back only the 32-byte
// sectors that hold a surrogate — faster than ld.global.cs + st.global.cs?
// Same tile structure as the stream kernel (8 vectors per thread, 4 CTAs/SM,
// one tile per CTA, L2 bulk prefetch one resident wave ahead), no repair
// arithmetic. Two inputs: config-1-like (uniform 16-bit units, 2^28 units) and
// config-4-like (1 % surrogates + 5 % of 1 Mi-unit regions all D800, 2^32 units).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/stpol_probe.cu -o scripts/stpol_probe
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);    \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

enum LdPol { LD_CS = 0, LD_DEF, LD_CG, LD_NOALLOC, LD_EF, LD_EL, LD_N };
enum StPol { ST_CS = 0, ST_WB, ST_WT, ST_CG, ST_EF, ST_EL, ST_EU, ST_EN, ST_N };
static const char* kLdName[] = {"ld.cs", "ld", "ld.cg", "ld.L1::no_allocate", "ld+L2::evict_first", "ld+L2::evict_last"};
static const char* kStName[] = {"st.cs", "st.wb", "st.wt", "st.cg", "st+L2::evict_first", "st+L2::evict_last",
                                "st+L2::evict_unchanged", "st+L2::evict_normal"};

template <int P>
__device__ __forceinline__ uint4 ld(const uint4* p, uint64_t pol) {
  uint4 v;
  if constexpr (P == LD_CS)
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if constexpr (P == LD_DEF)
    asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if constexpr (P == LD_CG)
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if constexpr (P == LD_NOALLOC)
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
  else
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
  return v;
}

template <int P>
__device__ __forceinline__ void st(uint4* p, uint4 v, uint64_t pol) {
  if constexpr (P == ST_CS)
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else if constexpr (P == ST_WB)
    asm volatile("st.global.wb.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else if constexpr (P == ST_WT)
    asm volatile("st.global.wt.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else if constexpr (P == ST_CG)
    asm volatile("st.global.cg.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else
    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w), "l"(pol)
                 : "memory");
}

template <int P>
__device__ __forceinline__ uint64_t make_ld_policy() {
  uint64_t pol = 0;
  if constexpr (P == LD_EF) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if constexpr (P == LD_EL) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
template <int P>
__device__ __forceinline__ uint64_t make_st_policy() {
  uint64_t pol = 0;
  if constexpr (P == ST_EF) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if constexpr (P == ST_EL) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  if constexpr (P == ST_EU) asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
  if constexpr (P == ST_EN) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ bool has_sur(uint4 v) {
  uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    uint32_t a = (w[i] & 0xF800F800u) ^ 0xD800D800u;
    r |= ((a & 0xFFFFu) == 0) | ((a >> 16) == 0);
  }
  return r;
}
__device__ __forceinline__ bool sector_dirty(bool d, int lane) {
  const uint32_t m = __ballot_sync(0xFFFFFFFFu, d);
  return (m >> (lane & ~1)) & 3u;
}

constexpr int U = 8;
// kMode 0: write dirty sectors; 1: read only; 2: write every vector (in-place full rewrite)
template <int LP, int SP, int kMode>
__global__ void __launch_bounds__(256, 4) tile_kernel(uint4* buf, size_t nvec, int pf, unsigned* sink) {
  const int lane = threadIdx.x & 31;
  const size_t tv0 = (size_t)blockIdx.x * 256 * U;
  const size_t v0 = tv0 + (threadIdx.x / 32) * 32 * U + lane;
  if (pf > 0 && threadIdx.x == 0) {
    const size_t pv = tv0 + (size_t)pf * 256 * U;
    if (pv + 256 * U <= nvec)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(buf + pv), "r"(256 * U * 16) : "memory");
  }
  const uint64_t lpol = make_ld_policy<LP>();
  const uint64_t spol = make_st_policy<SP>();
  uint4 v[U];
#pragma unroll
  for (int k = 0; k < U; k++) v[k] = ld<LP>(buf + v0 + 32 * k, lpol);
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < U; k++) {
    const bool d = sector_dirty(has_sur(v[k]), lane);
    if (kMode == 0) {
      if (d) st<SP>(buf + v0 + 32 * k, v[k], spol);
    } else if (kMode == 2) {
      st<SP>(buf + v0 + 32 * k, v[k], spol);
    } else {
      acc ^= v[k].x ^ v[k].w ^ (uint32_t)d;
    }
  }
  if (kMode == 1 && acc == 0x7777777u) *sink = acc;
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// pattern 1: uniform 16-bit; pattern 4: 1 % surrogates, 5 % of 1 Mi-unit regions all D800
__global__ void fill_kernel(uint16_t* buf, size_t n, int pattern) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix64(i * 0x9E3779B97F4A7C15ull + 12345);
    uint16_t u;
    if (pattern == 1) {
      u = (uint16_t)h;
    } else {
      const uint64_t r = mix64((i >> 20) * 0xD1B54A32D192ED03ull + 99);
      if (r % 100 < 5) u = 0xD800;
      else u = (h % 100 == 0) ? (uint16_t)(0xD800 + ((h >> 20) & 0x7FF)) : (uint16_t)(0x20 + ((h >> 8) % 95));
    }
    buf[i] = u;
  }
}
__global__ void flush_kernel(const uint4* p, size_t n, unsigned* sink) {
  uint32_t a = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = p[i];
    a ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (a == 0x1234567u) *sink = a;
}

struct Ctx {
  uint4* buf;
  size_t nvec;
  uint4* fl;
  size_t flvec;
  unsigned* sink;
  int pf;
};

template <int LP, int SP, int kMode>
static float run(const Ctx& c, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a), cudaEventCreate(&b);
  std::vector<float> ms;
  const unsigned grid = (unsigned)(c.nvec / (256 * U));
  for (int r = 0; r < reps + 2; r++) {
    flush_kernel<<<148 * 8, 256>>>(c.fl, c.flvec, c.sink);
    cudaEventRecord(a);
    tile_kernel<LP, SP, kMode><<<grid, 256>>>(c.buf, c.nvec, c.pf, c.sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t;
    cudaEventElapsedTime(&t, a, b);
    if (r >= 2) ms.push_back(t);
  }
  cudaEventDestroy(a), cudaEventDestroy(b);
  std::sort(ms.begin(), ms.end());
  return ms[ms.size() / 2] * 1e3f;
}

static int g_mode = 0;  // 0: dirty sectors only (in place); 2: every vector rewritten (copy-like traffic)
template <int LP, int SP>
static void row(const Ctx& c, int reps, const char* tag) {
  const float t = g_mode == 2 ? run<LP, SP, 2>(c, reps) : run<LP, SP, 0>(c, reps);
  printf("%-6s %-22s %-24s %10.1f us  %7.1f GB/s input\n", tag, kLdName[LP], kStName[SP], t,
         c.nvec * 16.0 / (t * 1e-6) / 1e9);
  fflush(stdout);
}

template <int LP>
static void ld_rows(const Ctx& c, int reps, const char* tag) {
  row<LP, ST_CS>(c, reps, tag);
  row<LP, ST_WB>(c, reps, tag);
  row<LP, ST_WT>(c, reps, tag);
  row<LP, ST_CG>(c, reps, tag);
  row<LP, ST_EF>(c, reps, tag);
  row<LP, ST_EL>(c, reps, tag);
  row<LP, ST_EU>(c, reps, tag);
  row<LP, ST_EN>(c, reps, tag);
}

static int sweep(const Ctx& c, int reps, const char* tag) {
  printf("%s: %zu units; read-only %.1f us; full rewrite %.1f us\n", tag, c.nvec * 8,
         run<LD_CS, ST_CS, 1>(c, reps), run<LD_CS, ST_CS, 2>(c, reps));
  ld_rows<LD_CS>(c, reps, tag);
  ld_rows<LD_DEF>(c, reps, tag);
  ld_rows<LD_NOALLOC>(c, reps, tag);
  ld_rows<LD_EF>(c, reps, tag);
  ld_rows<LD_EL>(c, reps, tag);
  row<LD_CG, ST_CS>(c, reps, tag);
  // repeat the baseline at the end (drift check)
  row<LD_CS, ST_CS>(c, reps, tag);
  return 0;
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 9;
  g_mode = argc > 2 ? atoi(argv[2]) : 0;
  Ctx c;
  c.flvec = (512u << 20) / 16;
  CK(cudaMalloc(&c.fl, c.flvec * 16));
  CK(cudaMemset(c.fl, 1, c.flvec * 16));
  CK(cudaMalloc(&c.sink, 4));
  c.pf = 148 * 4;
  const size_t n1 = 1ull << 28, n4 = 1ull << 32;
  uint16_t* b;
  CK(cudaMalloc(&b, n4 * 2));
  c.buf = reinterpret_cast<uint4*>(b);
  fill_kernel<<<148 * 16, 256>>>(b, n1, 1);
  CK(cudaDeviceSynchronize());
  c.nvec = n1 / 8;
  sweep(c, reps, "C1");
  fill_kernel<<<148 * 16, 256>>>(b, n4, 4);
  CK(cudaDeviceSynchronize());
  c.nvec = n4 / 8;
  sweep(c, std::max(3, reps / 2), "C4");
  CK(cudaDeviceSynchronize());
  return 0;
}
