// Probe (not product): raw read bandwidth of 1-D bulk-async (TMA) streaming
// vs 128-bit LDG streaming on this B200, for the repair kernel's design.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/tma_probe.cu -o tma_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES, int TILE, int CONS_WARPS>
__global__ void tma_read(const uint4* in, size_t nvec, unsigned* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * TILE);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const size_t ntiles = nvec * 16 / TILE;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; i++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[i])), "r"(CONS_WARPS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == CONS_WARPS) {
    if (lane) return;
    uint32_t it = 0;
    for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, it++) {
      int st = it % STAGES;
      uint32_t ph = (it / STAGES) & 1;
      if (it >= STAGES) {
        uint32_t done;
        do {
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(done) : "r"(smem_u32(&empty[st])), "r"(ph ^ 1) : "memory");
        } while (!done);
      }
      uint32_t fb = smem_u32(&full[st]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(TILE) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(smem + st * TILE)), "l"((const char*)in + t * TILE), "r"(TILE), "r"(fb) : "memory");
    }
    return;
  }
  uint32_t acc = 0, it = 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, it++) {
    int st = it % STAGES;
    uint32_t ph = (it / STAGES) & 1;
    uint32_t done;
    do {
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(done) : "r"(smem_u32(&full[st])), "r"(ph) : "memory");
    } while (!done);
    const uint4* s = reinterpret_cast<const uint4*>(smem + st * TILE);
    for (int i = threadIdx.x; i < TILE / 16; i += CONS_WARPS * 32) { uint4 v = s[i]; acc ^= v.x ^ v.w; }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
  }
  if (acc == 0x1234567) *sink = acc;
}

// TMA load -> smem -> st.global (each consumer thread stores its vectors).
template <int STAGES, int TILE, int CONS_WARPS, bool BULK_STORE>
__global__ void tma_copy(const uint4* in, uint4* out, size_t nvec) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * TILE);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const size_t ntiles = nvec * 16 / TILE;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; i++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[i])), "r"(BULK_STORE ? 1 : CONS_WARPS));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == CONS_WARPS) {
    if (lane) return;
    uint32_t it = 0;
    for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, it++) {
      int st = it % STAGES;
      uint32_t ph = (it / STAGES) & 1;
      if (it >= STAGES) {
        uint32_t done;
        do {
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(done) : "r"(smem_u32(&empty[st])), "r"(ph ^ 1) : "memory");
        } while (!done);
      }
      uint32_t fb = smem_u32(&full[st]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(TILE) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(smem + st * TILE)), "l"((const char*)in + t * TILE), "r"(TILE), "r"(fb) : "memory");
    }
    return;
  }
  uint32_t it = 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x, it++) {
    int st = it % STAGES;
    uint32_t ph = (it / STAGES) & 1;
    uint32_t done;
    do {
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(done) : "r"(smem_u32(&full[st])), "r"(ph) : "memory");
    } while (!done);
    uint4* s = reinterpret_cast<uint4*>(smem + st * TILE);
    if (BULK_STORE) {
      for (int i = threadIdx.x; i < TILE / 16; i += CONS_WARPS * 32) { uint4 v = s[i]; v.x ^= 1; s[i] = v; }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, %0;" ::"r"(CONS_WARPS * 32));
      if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((char*)out + t * TILE),
                     "r"(smem_u32(s)), "r"(TILE) : "memory");
        asm volatile("cp.async.bulk.commit_group;");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
      }
    } else {
      uint4 v[TILE / 16 / (CONS_WARPS * 32)];
      for (int i = 0; i < TILE / 16 / (CONS_WARPS * 32); i++) v[i] = s[threadIdx.x + i * CONS_WARPS * 32];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
      for (int i = 0; i < TILE / 16 / (CONS_WARPS * 32); i++) {
        v[i].x ^= 1;
        asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(out + t * (TILE / 16) + threadIdx.x + i * CONS_WARPS * 32),
                     "r"(v[i].x), "r"(v[i].y), "r"(v[i].z), "r"(v[i].w) : "memory");
      }
    }
  }
}

template <int U>
__global__ void ldg_copy(const uint4* in, uint4* out, size_t nvec) {
  size_t base = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x;
  uint4 v[U];
#pragma unroll
  for (int k = 0; k < U; k++)
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                 : "l"(in + base + k * blockDim.x));
#pragma unroll
  for (int k = 0; k < U; k++) {
    v[k].x ^= 1;
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(out + base + k * blockDim.x), "r"(v[k].x), "r"(v[k].y),
                 "r"(v[k].z), "r"(v[k].w) : "memory");
  }
}

template <int U>
__global__ void ldg_read(const uint4* in, size_t nvec, unsigned* sink) {
  uint32_t acc = 0;
  size_t tile = (size_t)blockDim.x * U;
  for (size_t base = (size_t)blockIdx.x * tile; base < nvec; base += (size_t)gridDim.x * tile) {
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; k++) {
      asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                   : "l"(in + base + k * blockDim.x + threadIdx.x));
    }
#pragma unroll
    for (int k = 0; k < U; k++) acc ^= v[k].x ^ v[k].w;
  }
  if (acc == 0x1234567) *sink = acc;
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  for (int i = 0; i < 5; i++) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

template <int STAGES, int TILE, int CW, int CTAS>
void run_tma(const uint4* d, size_t nvec, unsigned* sink, int sms) {
  size_t smem = STAGES * TILE + 2 * STAGES * 8;
  cudaFuncSetAttribute(tma_read<STAGES, TILE, CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  float ms = timeit([&] { tma_read<STAGES, TILE, CW><<<sms * CTAS, (CW + 1) * 32, smem>>>(d, nvec, sink); });
  printf("tma stages=%2d tile=%6d cons_warps=%d ctas/sm=%d : %7.1f GB/s %s\n", STAGES, TILE, CW, CTAS,
         nvec * 16 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  size_t bytes = size_t(1) << 30;
  uint4* d; unsigned* sink;
  cudaMalloc(&d, bytes); cudaMalloc(&sink, 4);
  cudaMemset(d, 1, bytes);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t nvec = bytes / 16;
  for (int b : {256, 512}) {
    float ms = timeit([&] { ldg_read<4><<<sms * (2048 / b), b>>>(d, nvec, sink); });
    printf("ldg U=4 block=%d persistent: %7.1f GB/s\n", b, nvec * 16 / ms / 1e6);
    ms = timeit([&] { ldg_read<8><<<sms * (2048 / b), b>>>(d, nvec, sink); });
    printf("ldg U=8 block=%d persistent: %7.1f GB/s\n", b, nvec * 16 / ms / 1e6);
  }
  float ms = timeit([&] { ldg_read<4><<<nvec / (256 * 4), 256>>>(d, nvec, sink); });
  printf("ldg U=4 non-persistent: %7.1f GB/s\n", nvec * 16 / ms / 1e6);
  {
    uint4* o; cudaMalloc(&o, bytes);
    float m1 = timeit([&] { ldg_copy<4><<<nvec / 1024, 256>>>(d, o, nvec); });
    printf("ldg copy U=4: %7.1f GB/s (r+w)\n", 2 * nvec * 16 / m1 / 1e6);
    m1 = timeit([&] { ldg_copy<8><<<nvec / 1024, 128>>>(d, o, nvec); });
    printf("ldg copy U=8 128thr: %7.1f GB/s (r+w)\n", 2 * nvec * 16 / m1 / 1e6);
    m1 = timeit([&] { cudaMemcpyAsync(o, d, bytes, cudaMemcpyDeviceToDevice); });
    printf("cudaMemcpy D2D: %7.1f GB/s (r+w)\n", 2 * nvec * 16 / m1 / 1e6);
    size_t smem = 6 * 16384 + 2 * 6 * 8;
    cudaFuncSetAttribute(tma_copy<6, 16384, 8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(tma_copy<6, 16384, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    m1 = timeit([&] { tma_copy<6, 16384, 8, false><<<sms * 2, 288, smem>>>(d, o, nvec); });
    printf("tma load + stg: %7.1f GB/s (r+w) %s\n", 2 * nvec * 16 / m1 / 1e6, cudaGetErrorString(cudaGetLastError()));
    m1 = timeit([&] { tma_copy<6, 16384, 8, true><<<sms * 2, 288, smem>>>(d, o, nvec); });
    printf("tma load + bulk store: %7.1f GB/s (r+w) %s\n", 2 * nvec * 16 / m1 / 1e6, cudaGetErrorString(cudaGetLastError()));
    size_t smem2 = 4 * 16384 + 2 * 4 * 8;
    cudaFuncSetAttribute(tma_copy<4, 16384, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
    m1 = timeit([&] { tma_copy<4, 16384, 8, true><<<sms * 3, 288, smem2>>>(d, o, nvec); });
    printf("tma load + bulk store 4st x3: %7.1f GB/s (r+w) %s\n", 2 * nvec * 16 / m1 / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  run_tma<6, 16384, 8, 2>(d, nvec, sink, sms);
  run_tma<12, 16384, 8, 1>(d, nvec, sink, sms);
  run_tma<4, 16384, 8, 3>(d, nvec, sink, sms);
  run_tma<8, 8192, 8, 2>(d, nvec, sink, sms);
  run_tma<12, 8192, 4, 2>(d, nvec, sink, sms);
  run_tma<6, 32768, 8, 1>(d, nvec, sink, sms);
  run_tma<3, 32768, 8, 2>(d, nvec, sink, sms);
  run_tma<16, 4096, 4, 3>(d, nvec, sink, sms);
  run_tma<24, 4096, 4, 2>(d, nvec, sink, sms);
  return 0;
}
