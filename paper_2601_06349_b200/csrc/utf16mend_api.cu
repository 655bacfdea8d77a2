// Source-compatible C++ API (include/utf16mend/driver.hpp) over the C ABI.
// Every compute path below ends in a u16m_* call, i.e. on the GPU.

#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <string>

#include "../../include/u16m.h"
#include "../../include/utf16mend/driver.hpp"
#include "u16m_abi.h"
#include "u16m_internal.h"

namespace utf16mend {

namespace {

[[noreturn]] void raise(u16m_status st) {
  std::string msg = std::string("utf16mend: ") + u16m_status_string(st) + ": " + u16m_last_error();
  if (st == U16M_ERR_INVALID_ARGUMENT || st == U16M_ERR_ALIAS || st == U16M_ERR_MISALIGNED)
    throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

void check(u16m_status st) {
  if (st != U16M_OK) raise(st);
}

bool is_device(const void* p) {
  if (p == nullptr) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void sync_default() {
  const cudaError_t e = cudaStreamSynchronize(nullptr);
  if (e != cudaSuccess) throw std::runtime_error(std::string("utf16mend: ") + cudaGetErrorString(e));
}

// RAII device scratch for the small outputs of the device-span helpers:
// stream-ordered on the legacy default stream from the device's pool, whose
// freed blocks stay cached (no cudaMalloc/cudaFree per call).
struct DeviceBuf {
  void* p = nullptr;
  explicit DeviceBuf(size_t bytes) {
    u16m::keep_pool_memory();
    if (bytes && cudaMallocAsync(&p, bytes, nullptr) != cudaSuccess) {
      cudaGetLastError();
      throw std::runtime_error("utf16mend: device allocation failed");
    }
  }
  ~DeviceBuf() {
    if (p) cudaFreeAsync(p, nullptr);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

void copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  if (bytes == 0) return;
  const cudaError_t e = cudaMemcpy(dst, src, bytes, kind);
  if (e != cudaSuccess) throw std::runtime_error(std::string("utf16mend: ") + cudaGetErrorString(e));
}

}  // namespace

// ---- kernel selection: the reference's surface, value for value ------------
// (proj/src/driver.cpp:15-108). The ids select nothing here — every id runs
// the one sm_100a path — but they are listed, validated and chosen exactly as
// the reference does so code that inspects them behaves the same.

std::string to_string(const kernel_id& id) {
  switch (id.kind) {
    case kernel_kind::scalar: return "scalar";
    case kernel_kind::generic: return "generic" + std::to_string(id.lanes);
    case kernel_kind::bitmask: return id.emulated ? "bitmask-emulated" : "bitmask";
    case kernel_kind::bytesplit: return id.emulated ? "bytesplit-emulated" : "bytesplit";
  }
  return "?";
}

std::optional<kernel_id> parse_kernel_id(std::string_view name) {
  static constexpr struct {
    std::string_view name;
    kernel_kind kind;
    unsigned lanes;
    bool emulated;
  } kNames[] = {
      {"scalar", kernel_kind::scalar, 0, false},        {"generic", kernel_kind::generic, 8, false},
      {"generic4", kernel_kind::generic, 4, false},     {"generic8", kernel_kind::generic, 8, false},
      {"generic16", kernel_kind::generic, 16, false},   {"generic32", kernel_kind::generic, 32, false},
      {"bitmask", kernel_kind::bitmask, 0, false},      {"bitmask-emulated", kernel_kind::bitmask, 0, true},
      {"bytesplit", kernel_kind::bytesplit, 0, false},  {"bytesplit-emulated", kernel_kind::bytesplit, 0, true},
  };
  for (const auto& e : kNames)
    if (e.name == name) return kernel_id{e.kind, e.lanes, e.emulated};
  return std::nullopt;
}

cpu_features detect_cpu_features() {
  cpu_features f;
#if defined(__x86_64__) || defined(__i386__)
  f.wide_mask_registers = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw");
#elif defined(__aarch64__)
  f.byte_deinterleave = true;
#endif
  return f;
}

bool kernel_supported(const kernel_id& id, const cpu_features& features) {
  switch (id.kind) {
    case kernel_kind::scalar: return true;
    case kernel_kind::generic: return id.lanes == 4 || id.lanes == 8 || id.lanes == 16 || id.lanes == 32;
    case kernel_kind::bitmask: return id.emulated || features.wide_mask_registers;
    case kernel_kind::bytesplit: return id.emulated || features.byte_deinterleave;
  }
  return false;
}

std::vector<kernel_id> available_kernels(const cpu_features& features) {
  std::vector<kernel_id> ids{kernel_id::scalar()};
  for (unsigned lanes : {4u, 8u, 16u, 32u}) ids.push_back(kernel_id::generic(lanes));
  if (features.wide_mask_registers) ids.push_back(kernel_id::bitmask());
  ids.push_back(kernel_id::bitmask(true));
  if (features.byte_deinterleave) ids.push_back(kernel_id::bytesplit());
  ids.push_back(kernel_id::bytesplit(true));
  return ids;
}

std::vector<kernel_id> available_kernels() { return available_kernels(detect_cpu_features()); }

kernel_id select_kernel(const std::optional<kernel_id>& override_id, const cpu_features& features) {
  if (override_id) {
    if (kernel_supported(*override_id, features)) return *override_id;
    switch (override_id->kind) {
      case kernel_kind::bitmask:
        throw std::invalid_argument(
            "kernel 'bitmask' requires 512-bit vectors with mask registers (AVX-512F/BW), which this host does "
            "not report");
      case kernel_kind::bytesplit:
        throw std::invalid_argument(
            "kernel 'bytesplit' requires NEON deinterleaving loads, which this host does not report");
      default:
        throw std::invalid_argument("generic kernel lane count must be 4, 8, 16, or 32");
    }
  }
  if (features.wide_mask_registers) return kernel_id::bitmask();
  if (features.byte_deinterleave) return kernel_id::bytesplit();
  return kernel_id::generic(8);
}

kernel_id select_kernel(const std::optional<kernel_id>& override_id) {
  static const cpu_features host = detect_cpu_features();
  if (override_id) return select_kernel(override_id, host);
  static const kernel_id chosen = [] {
    if (const char* env = std::getenv("UTF16MEND_KERNEL")) {
      const auto id = parse_kernel_id(env);
      if (id && kernel_supported(*id, host)) return *id;
      std::fprintf(stderr, "utf16mend: ignoring UTF16MEND_KERNEL=%s (%s); using default\n", env,
                   id ? "unsupported on this host" : "unknown kernel name");
    }
    return select_kernel(std::nullopt, host);
  }();
  return chosen;
}

std::string backend_name() { return "cuda-sm100a"; }

void to_well_formed(std::span<const char16_t> in, std::span<char16_t> out,
                    const std::optional<kernel_id>& kernel) {
  if (in.size() != out.size())
    throw std::invalid_argument("to_well_formed: input and output lengths differ");
  (void)select_kernel(kernel);  // the reference's validation (and UTF16MEND_KERNEL warning)
  const auto* i = reinterpret_cast<const uint16_t*>(in.data());
  auto* o = reinterpret_cast<uint16_t*>(out.data());
  if (in.empty()) return;
  const bool di = is_device(i), dout = is_device(o);
  if (di && dout) {
    check(u16m_to_well_formed(i, in.size(), o, nullptr));
    sync_default();
  } else if (!di && !dout) {
    // every visible GPU, each over its own PCIe link (one device for jobs
    // under 64 Mi units)
    check(u16m_to_well_formed_host_multi(i, in.size(), o, 0, nullptr));
  } else {
    throw std::invalid_argument("to_well_formed: in and out must both be host or both be device memory");
  }
}

void to_well_formed_in_place(std::span<char16_t> buffer, const std::optional<kernel_id>& kernel) {
  to_well_formed(buffer, buffer, kernel);
}

void to_well_formed_batched(std::span<const char16_t> in, std::span<const std::int64_t> offsets,
                            std::span<char16_t> out) {
  if (in.size() != out.size())
    throw std::invalid_argument("to_well_formed_batched: input and output lengths differ");
  if (offsets.empty()) throw std::invalid_argument("to_well_formed_batched: offsets is empty");
  const size_t S = offsets.size() - 1;
  const auto* i = reinterpret_cast<const uint16_t*>(in.data());
  auto* o = reinterpret_cast<uint16_t*>(out.data());
  const bool di = is_device(i), dout = is_device(o), doff = is_device(offsets.data());
  if (in.empty() && !di && !doff) {
    check(u16m_to_well_formed_batched_host(i, 0, offsets.data(), S, o));  // validates offsets
    return;
  }
  if (di != dout) throw std::invalid_argument("to_well_formed_batched: in and out must both be host or both be device memory");
  if (!di) {
    if (doff) throw std::invalid_argument("to_well_formed_batched: offsets are device memory but the strings are host memory");
    check(u16m_to_well_formed_batched_host(i, in.size(), offsets.data(), S, o));
    return;
  }
  // Device strings. Host offsets are validated and moved to the device; the
  // units outside [offsets[0], offsets[S]) are copied, as the host form does.
  std::int64_t ends[2] = {0, 0};
  const std::int64_t* d_off = offsets.data();
  std::optional<DeviceBuf> staged;
  if (!doff) {
    for (size_t s = 0; s < S; s++)
      if (offsets[s] < 0 || offsets[s + 1] < offsets[s] || static_cast<size_t>(offsets[s + 1]) > in.size())
        throw std::invalid_argument("to_well_formed_batched: offsets must be non-decreasing within the buffer");
    if (offsets[0] < 0 || static_cast<size_t>(offsets[0]) > in.size())
      throw std::invalid_argument("to_well_formed_batched: offsets must be non-decreasing within the buffer");
    staged.emplace(offsets.size_bytes());
    copy(staged->p, offsets.data(), offsets.size_bytes(), cudaMemcpyHostToDevice);
    d_off = staged->as<std::int64_t>();
    ends[0] = offsets.front();
    ends[1] = offsets.back();
  } else {
    copy(&ends[0], offsets.data(), sizeof(std::int64_t), cudaMemcpyDeviceToHost);
    copy(&ends[1], offsets.data() + S, sizeof(std::int64_t), cudaMemcpyDeviceToHost);
    if (ends[0] < 0 || ends[1] < ends[0] || static_cast<size_t>(ends[1]) > in.size())
      throw std::invalid_argument("to_well_formed_batched: offsets must be non-decreasing within the buffer");
  }
  check(u16m_to_well_formed_batched_n(i, in.size(), d_off, S, o, nullptr));
  if (o != i) {
    copy(o, i, static_cast<size_t>(ends[0]) * 2, cudaMemcpyDeviceToDevice);
    copy(o + ends[1], i + ends[1], (in.size() - static_cast<size_t>(ends[1])) * 2, cudaMemcpyDeviceToDevice);
  }
  sync_default();
}

void fix_scalar(std::span<const char16_t> in, std::span<char16_t> out) { to_well_formed(in, out); }

void fix_scalar(char16_t* out, const char16_t* in, std::size_t n) {
  to_well_formed(std::span<const char16_t>(in, n), std::span<char16_t>(out, n));
}

bool is_well_formed(std::span<const char16_t> in) {
  if (in.empty()) return true;
  const auto* i = reinterpret_cast<const uint16_t*>(in.data());
  if (is_device(i)) {
    DeviceBuf cnt(sizeof(unsigned long long));
    check(u16m_count_unpaired(i, in.size(), cnt.as<unsigned long long>(), nullptr));
    unsigned long long c = 0;
    copy(&c, cnt.p, sizeof(c), cudaMemcpyDeviceToHost);
    return c == 0;
  }
  // Host memory: chunked scan that stops at the first unpaired surrogate.
  unsigned long long first = 0;
  size_t found = 0;
  check(u16m_unpaired_offsets_host(i, in.size(), 1, &first, &found));
  return found == 0;
}

std::vector<std::size_t> unpaired_surrogate_offsets(std::span<const char16_t> in, std::size_t limit) {
  std::vector<std::size_t> result;
  if (in.empty() || limit == 0) return result;
  const size_t cap = limit < in.size() ? limit : in.size();
  const auto* i = reinterpret_cast<const uint16_t*>(in.data());
  std::vector<unsigned long long> tmp;
  if (is_device(i)) {
    DeviceBuf cnt(sizeof(unsigned long long)), offs(cap * sizeof(unsigned long long));
    check(u16m_unpaired_offsets(i, in.size(), cap, offs.as<unsigned long long>(), cnt.as<unsigned long long>(),
                                nullptr));
    sync_default();
    unsigned long long c = 0;
    copy(&c, cnt.p, sizeof(c), cudaMemcpyDeviceToHost);
    tmp.resize(c);
    copy(tmp.data(), offs.p, c * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  } else {
    tmp.resize(cap);
    size_t c = 0;
    check(u16m_unpaired_offsets_host(i, in.size(), cap, tmp.data(), &c));
    tmp.resize(c);
  }
  result.assign(tmp.begin(), tmp.end());
  return result;
}

}  // namespace utf16mend

// ---- kernel names for the C ABI / Python mirror -----------------------------
namespace {
int copy_out(const std::string& s, char* buf, size_t cap) {
  if (buf && cap) {
    const size_t k = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(buf, s.data(), k);
    buf[k] = '\0';
  }
  return static_cast<int>(s.size());
}
}  // namespace

extern "C" int u16m_kernel_names(char* buf, size_t cap) {
  std::string s;
  for (const auto& id : utf16mend::available_kernels()) s += (s.empty() ? "" : ",") + utf16mend::to_string(id);
  return copy_out(s, buf, cap);
}

extern "C" int u16m_default_kernel_name(char* buf, size_t cap) {
  return copy_out(utf16mend::to_string(utf16mend::select_kernel()), buf, cap);
}

extern "C" u16m_status u16m_select_kernel(const char* name, char* buf, size_t cap) {
  std::optional<utf16mend::kernel_id> id;
  if (name) {
    id = utf16mend::parse_kernel_id(name);
    if (!id) return u16m::abi::fail(U16M_ERR_INVALID_ARGUMENT, std::string("unknown kernel '") + name + "'");
  }
  try {
    copy_out(utf16mend::to_string(utf16mend::select_kernel(id)), buf, cap);
  } catch (const std::invalid_argument& e) {
    return u16m::abi::fail(U16M_ERR_INVALID_ARGUMENT, e.what());
  }
  return U16M_OK;
}

// ---- generate_utf16le (reference datagen contract) --------------------------
#include <random>

#include "../../include/u16m_datagen.h"

extern "C" u16m_status u16m_generate_reference_mix(size_t units, double pair_pct, double mismatch_pct,
                                                   uint64_t seed, uint16_t* out) {
  if (pair_pct < 0.0 || pair_pct > 1.0 || mismatch_pct < 0.0 || mismatch_pct > 1.0)
    return U16M_ERR_INVALID_ARGUMENT;
  if (units > 0 && out == nullptr) return U16M_ERR_INVALID_ARGUMENT;
  std::mt19937_64 rng(seed);
  auto below = [&](uint32_t n) {
    return static_cast<uint32_t>((static_cast<unsigned __int128>(rng()) * n) >> 64);
  };
  auto chance = [&](double p) {
    if (p <= 0.0) return false;
    if (p >= 1.0) return true;
    return rng() < static_cast<uint64_t>(p * 18446744073709551616.0);
  };
  auto filler = [&]() {
    constexpr uint32_t low_span = 0xD7FF, high_span = 0xFFFD - 0xE000 + 1;
    const uint32_t r = below(low_span + high_span);
    return static_cast<uint16_t>(r < low_span ? 1 + r : 0xE000 + (r - low_span));
  };
  const double q = pair_pct / (2.0 - pair_pct);
  size_t k = 0;
  while (k < units) {
    if (chance(q)) {
      if (k + 2 <= units) {
        out[k++] = static_cast<uint16_t>(0xD800 + below(0x400));
        out[k++] = static_cast<uint16_t>(0xDC00 + below(0x400));
      } else {
        out[k++] = filler();
      }
    } else if (chance(mismatch_pct)) {
      const uint32_t base = chance(0.5) ? 0xD800 : 0xDC00;
      out[k++] = static_cast<uint16_t>(base + below(0x400));
    } else {
      out[k++] = filler();
    }
  }
  return U16M_OK;
}
