// C ABI (include/u16m.h), device-memory entry points: argument validation,
// stream plumbing and the single-process multi-GPU shard driver. The
// host-memory entry points live in u16m_host.cu. All compute goes through the
// sm_100a kernels — there is no CPU fallback.
//
// Error behaviour mirrors the reference boundary (proj/src/driver.cpp:135-142):
// a length/argument problem is U16M_ERR_INVALID_ARGUMENT (the reference
// throws std::invalid_argument), a partial in/out overlap is U16M_ERR_ALIAS
// (the reference asserts), and hardware problems are U16M_ERR_CUDA /
// U16M_ERR_NO_DEVICE (the reference throws std::runtime_error when a native
// backend is missing, proj/src/bitmask_kernel.cpp:102-104).

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/u16m.h"
#include "u16m_abi.h"
#include "u16m_internal.h"

namespace u16m::abi {

thread_local std::string t_last_error;

u16m_status fail(u16m_status st, const std::string& detail) {
  t_last_error = detail;
  return st;
}

u16m_status cuda_fail(cudaError_t e, const char* what) {
  std::string d = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return fail(U16M_ERR_CUDA, d);
}

u16m_status check_device_present() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(U16M_ERR_NO_DEVICE, "no CUDA device visible (u16m has no CPU fallback)");
  }
  return U16M_OK;
}

u16m_status check_device_ptr(const void* p, const char* name) {
  cudaPointerAttributes a;
  const cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(U16M_ERR_NOT_DEVICE_MEMORY, std::string(name) + " is not a CUDA-visible pointer");
  }
  if (a.type == cudaMemoryTypeDevice) {
    // Memory of another GPU than the current one is only usable over peer
    // access; without it the kernel would fault (a sticky error that ends the
    // CUDA context), so refuse it here with a readable message.
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && a.device != cur) {
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, cur, a.device) != cudaSuccess || !can) {
        cudaGetLastError();
        return fail(U16M_ERR_NOT_DEVICE_MEMORY, std::string(name) + " is memory of cuda:" + std::to_string(a.device) +
                                                    ", the current device is cuda:" + std::to_string(cur) +
                                                    " and has no peer access to it (cudaSetDevice first)");
      }
      const cudaError_t pe = cudaDeviceEnablePeerAccess(a.device, 0);  // idempotent (NVLink peer loads)
      if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled)
        return cuda_fail(pe, "enabling peer access");
      cudaGetLastError();
    }
    return U16M_OK;
  }
  if (a.type == cudaMemoryTypeManaged) return U16M_OK;
  if (a.type == cudaMemoryTypeHost && a.devicePointer != nullptr) return U16M_OK;
  return fail(U16M_ERR_NOT_DEVICE_MEMORY,
              std::string(name) + " is host memory; use u16m_to_well_formed_host or the C++ API");
}

u16m_status check_pair(const uint16_t* in, size_t n, const uint16_t* out) {
  if (n == 0) return U16M_OK;
  if (in == nullptr || out == nullptr) return fail(U16M_ERR_INVALID_ARGUMENT, "null buffer with n > 0");
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 1u)
    return fail(U16M_ERR_MISALIGNED, "UTF-16 buffers must be 2-byte aligned");
  if (in != out && in < out + n && out < in + n)
    return fail(U16M_ERR_ALIAS, "in and out overlap partially (must be equal or disjoint)");
  return U16M_OK;
}

}  // namespace u16m::abi

namespace u16m {

// Units from `p` to the end of the device allocation holding it (driver
// cuMemGetAddressRange through the runtime's entry-point query, so the
// library needs no libcuda link), 0 when unknown. Memory mapped through the
// virtual memory management API (cuMemCreate + cuMemMap: e.g. PyTorch's
// expandable segments) is "unknown": there the range is one physical mapping
// (a 20 MiB page), not the buffer, and a tensor spans many of them
// (scripts/addr_range_probe.py: 2.9 M wrong units before this check).
// cuMemRetainAllocationHandle succeeds exactly for such mappings (it fails
// for cudaMalloc and stream-ordered pool allocations, whose range is the
// whole allocation).
size_t allocation_units_after(const void* p) {
  using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  using RetainFn = CUresult (*)(CUmemGenericAllocationHandle*, void*);
  using ReleaseFn = CUresult (*)(CUmemGenericAllocationHandle);
  auto entry = [](const char* name) -> void* {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return f;
  };
  static RangeFn range = reinterpret_cast<RangeFn>(entry("cuMemGetAddressRange"));
  static RetainFn retain = reinterpret_cast<RetainFn>(entry("cuMemRetainAllocationHandle"));
  static ReleaseFn release = reinterpret_cast<ReleaseFn>(entry("cuMemRelease"));
  if (range == nullptr || retain == nullptr || release == nullptr || p == nullptr) return 0;
  CUmemGenericAllocationHandle h = 0;
  if (retain(&h, const_cast<void*>(p)) == CUDA_SUCCESS) {
    release(h);
    return 0;  // VMM mapping: the range is not a bound of the buffer
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS) return 0;
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  if (a < base || a >= base + size) return 0;
  return (base + size - a) / sizeof(uint16_t);
}

}  // namespace u16m

using namespace u16m::abi;

namespace {

// ---- shard driver state ------------------------------------------------------
std::mutex g_peer_mu;
std::vector<std::pair<int, int>> g_peer_enabled;

bool ensure_peer(int from, int to) {
  if (from == to) return true;
  std::lock_guard<std::mutex> lock(g_peer_mu);
  for (auto& pr : g_peer_enabled)
    if (pr.first == from && pr.second == to) return true;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, from, to) != cudaSuccess || !can) {
    cudaGetLastError();
    return false;
  }
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(from);
  cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) e = cudaSuccess;
  cudaGetLastError();
  cudaSetDevice(prev);
  if (e != cudaSuccess) return false;
  g_peer_enabled.emplace_back(from, to);
  return true;
}

// Non-blocking streams for the shard driver, created once per (device, slot)
// and kept for the process: shards on distinct devices run concurrently, and
// up to kShardSlots shards on one device (virtual shards) too. A call no
// longer creates and destroys a stream per shard.
constexpr int kShardSlots = 8;
std::mutex g_stream_mu;
std::vector<std::pair<int, cudaStream_t>> g_streams;  // (device * kShardSlots + slot, stream)

cudaError_t cached_stream(int dev, int k, cudaStream_t* out) {
  const int key = dev * kShardSlots + (k % kShardSlots);
  std::lock_guard<std::mutex> lock(g_stream_mu);
  for (auto& e : g_streams)
    if (e.first == key) {
      *out = e.second;
      return cudaSuccess;
    }
  const cudaError_t e = cudaStreamCreateWithFlags(out, cudaStreamNonBlocking);  // on the current device (dev)
  if (e == cudaSuccess) g_streams.emplace_back(key, *out);
  return e;
}

}  // namespace

extern "C" {

const char* u16m_status_string(u16m_status status) {
  switch (status) {
    case U16M_OK: return "ok";
    case U16M_ERR_INVALID_ARGUMENT: return "invalid argument";
    case U16M_ERR_ALIAS: return "in and out overlap partially";
    case U16M_ERR_NOT_DEVICE_MEMORY: return "pointer is not device-accessible memory";
    case U16M_ERR_CUDA: return "CUDA error";
    case U16M_ERR_MISALIGNED: return "pointer is not 2-byte aligned";
    case U16M_ERR_NO_DEVICE: return "no CUDA device";
  }
  return "unknown status";
}

const char* u16m_last_error(void) { return t_last_error.c_str(); }
int u16m_api_version(void) { return U16M_API_VERSION; }
unsigned long long u16m_launch_count(void) { return u16m::launch_count(); }

u16m_status u16m_to_well_formed_halo_ptr(const uint16_t* in, size_t n, uint16_t* out,
                                         const uint16_t* left_ptr, const uint16_t* right_ptr,
                                         void* stream) {
  U16M_TRY(check_pair(in, n, out));
  if (n == 0) return U16M_OK;
  U16M_TRY(check_device_present());
  U16M_TRY(check_device_ptr(in, "in"));
  if (out != in) U16M_TRY(check_device_ptr(out, "out"));
  const cudaError_t e = u16m::launch_repair(in, n, out, -1, -1, left_ptr, right_ptr, as_stream(stream));
  return e == cudaSuccess ? U16M_OK : cuda_fail(e, "repair kernel launch");
}

u16m_status u16m_to_well_formed_part(const uint16_t* in, size_t n, uint16_t* out,
                                     const uint16_t* left_ptr, const uint16_t* right_ptr, int part,
                                     void* stream) {
  if (part != U16M_PART_ALL && part != U16M_PART_EDGES && part != U16M_PART_INTERIOR)
    return fail(U16M_ERR_INVALID_ARGUMENT, "part must be U16M_PART_ALL, _EDGES or _INTERIOR");
  U16M_TRY(check_pair(in, n, out));
  if (n == 0) return U16M_OK;
  U16M_TRY(check_device_present());
  U16M_TRY(check_device_ptr(in, "in"));
  if (out != in) U16M_TRY(check_device_ptr(out, "out"));
  const cudaError_t e =
      u16m::launch_repair_part(in, n, out, -1, -1, left_ptr, right_ptr, part, as_stream(stream));
  return e == cudaSuccess ? U16M_OK : cuda_fail(e, "repair kernel launch");
}

u16m_status u16m_to_well_formed_halo(const uint16_t* in, size_t n, uint16_t* out, int32_t left,
                                     int32_t right, void* stream) {
  if (left > 0xFFFF || right > 0xFFFF || left < -1 || right < -1)
    return fail(U16M_ERR_INVALID_ARGUMENT, "halo values must be a code unit or -1");
  U16M_TRY(check_pair(in, n, out));
  if (n == 0) return U16M_OK;
  U16M_TRY(check_device_present());
  U16M_TRY(check_device_ptr(in, "in"));
  if (out != in) U16M_TRY(check_device_ptr(out, "out"));
  const cudaError_t e = u16m::launch_repair(in, n, out, left, right, nullptr, nullptr, as_stream(stream));
  return e == cudaSuccess ? U16M_OK : cuda_fail(e, "repair kernel launch");
}

u16m_status u16m_to_well_formed(const uint16_t* in, size_t n, uint16_t* out, void* stream) {
  return u16m_to_well_formed_halo(in, n, out, -1, -1, stream);
}

u16m_status u16m_to_well_formed_in_place(uint16_t* buf, size_t n, void* stream) {
  return u16m_to_well_formed_halo(buf, n, buf, -1, -1, stream);
}

u16m_status u16m_to_well_formed_batched(const uint16_t* in, const int64_t* offsets,
                                        size_t num_strings, uint16_t* out, void* stream) {
  if (offsets == nullptr) return fail(U16M_ERR_INVALID_ARGUMENT, "offsets is null");
  if (num_strings == 0) return U16M_OK;
  if (in == nullptr || out == nullptr) return fail(U16M_ERR_INVALID_ARGUMENT, "null buffer");
  if ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 1u)
    return fail(U16M_ERR_MISALIGNED, "UTF-16 buffers must be 2-byte aligned");
  if (reinterpret_cast<uintptr_t>(offsets) & 7u)
    return fail(U16M_ERR_MISALIGNED, "offsets must be 8-byte aligned");
  U16M_TRY(check_device_present());
  U16M_TRY(check_device_ptr(in, "in"));
  if (out != in) U16M_TRY(check_device_ptr(out, "out"));
  U16M_TRY(check_device_ptr(offsets, "offsets"));
  // The caller gave no buffer length, and reading offsets[S] back would cost
  // a host sync. The allocations holding `in` and `out` bound it instead
  // (cuMemGetAddressRange): the register-staged tile kernel of the
  // length-aware form runs with its grid sized from that bound (CTAs past
  // offsets[S] exit at once). When the bound is unknown (not a cudaMalloc'd or
  // pool range, e.g. VMM-mapped pages) or loose enough that idle CTAs could
  // cost more than the tile form saves (> 4 GiB past `in`), the persistent TMA
  // kernel runs instead: its grid is the SM count and it reads the range on
  // the device, so it needs no bound at all.
  const size_t bound = std::min(u16m::allocation_units_after(in), u16m::allocation_units_after(out));
  cudaError_t e;
  if (bound > 0 && bound <= (size_t(1) << 31) && u16m::batched_tiles_enabled())
    e = u16m::launch_batched_tiles(in, bound, offsets, num_strings, out, as_stream(stream));
  else
    e = u16m::launch_batched(in, offsets, num_strings, out, as_stream(stream));
  return e == cudaSuccess ? U16M_OK : cuda_fail(e, "batched repair kernel launch");
}

u16m_status u16m_fix_utf16_bytes(const void* in, size_t n_units, void* out, int byte_order,
                                 unsigned long long* replacements, void* stream) {
  if (byte_order != U16M_LITTLE_ENDIAN && byte_order != U16M_BIG_ENDIAN)
    return fail(U16M_ERR_INVALID_ARGUMENT, "byte_order must be U16M_LITTLE_ENDIAN or U16M_BIG_ENDIAN");
  const auto* i = static_cast<const uint16_t*>(in);
  auto* o = static_cast<uint16_t*>(out);
  U16M_TRY(check_pair(i, n_units, o));
  if (n_units == 0) return U16M_OK;
  U16M_TRY(check_device_present());
  U16M_TRY(check_device_ptr(in, "in"));
  if (o != i) U16M_TRY(check_device_ptr(out, "out"));
  if (replacements) U16M_TRY(check_device_ptr(replacements, "replacements"));
  const bool be = byte_order == U16M_BIG_ENDIAN;
  // (an out at another 16-byte phase runs the shifted-store form: one pass)
  const cudaError_t e = u16m::launch_fix_bytes(in, n_units, out, be, replacements, as_stream(stream), -1, -1);
  return e == cudaSuccess ? U16M_OK : cuda_fail(e, "codec repair kernel launch");
}

u16m_status u16m_to_well_formed_batched_n(const uint16_t* in, size_t n_units, const int64_t* offsets,
                                          size_t num_strings, uint16_t* out, void* stream) {
  if (offsets == nullptr) return fail(U16M_ERR_INVALID_ARGUMENT, "offsets is null");
  if (num_strings == 0 || n_units == 0) return U16M_OK;
  U16M_TRY(check_pair(in, n_units, out));
  if (reinterpret_cast<uintptr_t>(offsets) & 7u) return fail(U16M_ERR_MISALIGNED, "offsets must be 8-byte aligned");
  U16M_TRY(check_device_present());
  U16M_TRY(check_device_ptr(in, "in"));
  if (out != in) U16M_TRY(check_device_ptr(out, "out"));
  U16M_TRY(check_device_ptr(offsets, "offsets"));
  const cudaError_t e = u16m::batched_tiles_enabled()  // any in/out phase (shifted stores when they differ)
                            ? u16m::launch_batched_tiles(in, n_units, offsets, num_strings, out, as_stream(stream))
                            : u16m::launch_batched(in, offsets, num_strings, out, as_stream(stream));
  return e == cudaSuccess ? U16M_OK : cuda_fail(e, "batched repair kernel launch");
}

u16m_status u16m_count_unpaired(const uint16_t* in, size_t n, unsigned long long* count_out,
                                void* stream) {
  if (count_out == nullptr) return fail(U16M_ERR_INVALID_ARGUMENT, "count_out is null");
  if (n > 0 && in == nullptr) return fail(U16M_ERR_INVALID_ARGUMENT, "null buffer with n > 0");
  if (reinterpret_cast<uintptr_t>(in) & 1u) return fail(U16M_ERR_MISALIGNED, "in not 2-byte aligned");
  U16M_TRY(check_device_present());
  U16M_TRY(check_device_ptr(count_out, "count_out"));
  if (n > 0) U16M_TRY(check_device_ptr(in, "in"));
  const cudaError_t e = u16m::launch_count_unpaired(in, n, count_out, as_stream(stream));
  return e == cudaSuccess ? U16M_OK : cuda_fail(e, "count kernel launch");
}

u16m_status u16m_unpaired_offsets(const uint16_t* in, size_t n, size_t limit,
                                  unsigned long long* offsets_out, unsigned long long* count_out,
                                  void* stream) {
  if (count_out == nullptr || (limit > 0 && offsets_out == nullptr))
    return fail(U16M_ERR_INVALID_ARGUMENT, "null output");
  if (n > 0 && in == nullptr) return fail(U16M_ERR_INVALID_ARGUMENT, "null buffer with n > 0");
  if (reinterpret_cast<uintptr_t>(in) & 1u) return fail(U16M_ERR_MISALIGNED, "in not 2-byte aligned");
  U16M_TRY(check_device_present());
  U16M_TRY(check_device_ptr(count_out, "count_out"));
  if (limit > 0) U16M_TRY(check_device_ptr(offsets_out, "offsets_out"));
  if (n > 0) U16M_TRY(check_device_ptr(in, "in"));
  const cudaError_t e =
      u16m::launch_unpaired_offsets(in, n, limit, offsets_out, count_out, as_stream(stream));
  return e == cudaSuccess ? U16M_OK : cuda_fail(e, "offsets kernels");
}


u16m_status u16m_to_well_formed_sharded(int num_shards, const int* device_ids,
                                        const uint16_t* const* shard_in, const size_t* shard_len,
                                        uint16_t* const* shard_out) {
  if (num_shards < 0 || (num_shards > 0 && (!device_ids || !shard_in || !shard_len || !shard_out)))
    return fail(U16M_ERR_INVALID_ARGUMENT, "null shard table");
  if (num_shards == 0) return U16M_OK;
  U16M_TRY(check_device_present());
  int prev = 0;
  cudaGetDevice(&prev);
  for (int g = 0; g < num_shards; g++) {
    U16M_TRY(check_pair(shard_in[g], shard_len[g], shard_out[g]));
    if (shard_len[g] == 0) continue;
    if (cudaSetDevice(device_ids[g]) != cudaSuccess) {
      cudaGetLastError();
      return fail(U16M_ERR_INVALID_ARGUMENT, "bad device id");
    }
    U16M_TRY(check_device_ptr(shard_in[g], "shard_in"));
    if (shard_out[g] != shard_in[g]) U16M_TRY(check_device_ptr(shard_out[g], "shard_out"));
  }
  // Halo pointers: the last unit of the previous non-empty shard and the first
  // unit of the next one, read by the kernel directly (same device, or a peer
  // over NVLink). Without peer access the two units are copied peer-to-peer,
  // stream-ordered, into a small scratch on the shard's device first.
  std::vector<cudaStream_t> streams(num_shards, nullptr);
  std::vector<uint16_t*> scratch(num_shards, nullptr);
  u16m_status st = U16M_OK;
  for (int g = 0; g < num_shards && st == U16M_OK; g++) {
    if (shard_len[g] == 0) continue;
    const int dev = device_ids[g];
    int k = 0;
    for (int h = 0; h < g; h++) k += (streams[h] != nullptr && device_ids[h] == dev);
    int lk = g - 1, rk = g + 1;
    while (lk >= 0 && shard_len[lk] == 0) lk--;
    while (rk < num_shards && shard_len[rk] == 0) rk++;
    const uint16_t* lp = lk >= 0 ? shard_in[lk] + shard_len[lk] - 1 : nullptr;
    const uint16_t* rp = rk < num_shards ? shard_in[rk] : nullptr;
    const bool lpeer = !lp || ensure_peer(dev, device_ids[lk]);
    const bool rpeer = !rp || ensure_peer(dev, device_ids[rk]);
    cudaSetDevice(dev);
    cudaError_t e = cached_stream(dev, k, &streams[g]);
    if (e != cudaSuccess) { st = cuda_fail(e, "shard stream"); break; }
    if (!lpeer || !rpeer) {
      u16m::keep_pool_memory();
      e = cudaMallocAsync(reinterpret_cast<void**>(&scratch[g]), 4, streams[g]);
      if (e == cudaSuccess && !lpeer)
        e = cudaMemcpyPeerAsync(scratch[g], dev, lp, device_ids[lk], 2, streams[g]);
      if (e == cudaSuccess && !rpeer)
        e = cudaMemcpyPeerAsync(scratch[g] + 1, dev, rp, device_ids[rk], 2, streams[g]);
      if (e != cudaSuccess) { st = cuda_fail(e, "halo fetch"); break; }
      if (!lpeer) lp = scratch[g];
      if (!rpeer) rp = scratch[g] + 1;
    }
    e = u16m::launch_repair(shard_in[g], shard_len[g], shard_out[g], -1, -1, lp, rp, streams[g]);
    if (e != cudaSuccess) { st = cuda_fail(e, "shard kernel launch"); break; }
  }
  for (int g = 0; g < num_shards; g++) {
    if (!streams[g]) continue;
    cudaSetDevice(device_ids[g]);
    if (scratch[g]) cudaFreeAsync(scratch[g], streams[g]);
    const cudaError_t e = cudaStreamSynchronize(streams[g]);
    if (e != cudaSuccess && st == U16M_OK) st = cuda_fail(e, "shard sync");
  }
  cudaSetDevice(prev);
  return st;
}

}  // extern "C"
