// Source-compatible C++ API (include/utf16mend/driver.hpp) over the C ABI.
// Every compute path below ends in a u16m_* call, i.e. on the GPU.

#include <cuda_runtime.h>

#include <cstdlib>
#include <stdexcept>
#include <string>

#include "../../include/u16m.h"
#include "../../include/utf16mend/driver.hpp"

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

// RAII device scratch for host-span helpers that are not on the hot path.
struct DeviceBuf {
  void* p = nullptr;
  explicit DeviceBuf(size_t bytes) {
    if (bytes && cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      throw std::runtime_error("utf16mend: device allocation failed");
    }
  }
  ~DeviceBuf() {
    if (p) cudaFree(p);
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

void validate(const std::optional<kernel_id>& kernel) {
  if (kernel && !kernel_supported(*kernel, detect_cpu_features()))
    throw std::invalid_argument("generic kernel lane count must be 4, 8, 16, or 32");
}

}  // namespace

std::string to_string(const kernel_id& id) {
  switch (id.kind) {
    case kernel_kind::scalar: return "scalar";
    case kernel_kind::generic: return "generic" + std::to_string(id.lanes);
    case kernel_kind::bitmask: return id.emulated ? "bitmask-emulated" : "bitmask";
    case kernel_kind::bytesplit: return id.emulated ? "bytesplit-emulated" : "bytesplit";
    case kernel_kind::cuda: return "cuda-sm100a";
  }
  return "?";
}

std::optional<kernel_id> parse_kernel_id(std::string_view name) {
  if (name == "cuda-sm100a" || name == "cuda") return kernel_id::cuda();
  if (name == "scalar") return kernel_id::scalar();
  if (name == "generic") return kernel_id::generic();
  if (name == "generic4") return kernel_id::generic(4);
  if (name == "generic8") return kernel_id::generic(8);
  if (name == "generic16") return kernel_id::generic(16);
  if (name == "generic32") return kernel_id::generic(32);
  if (name == "bitmask") return kernel_id::bitmask();
  if (name == "bitmask-emulated") return kernel_id::bitmask(true);
  if (name == "bytesplit") return kernel_id::bytesplit();
  if (name == "bytesplit-emulated") return kernel_id::bytesplit(true);
  return std::nullopt;
}

cpu_features detect_cpu_features() { return {}; }

bool kernel_supported(const kernel_id& id, const cpu_features&) {
  // Any reference kernel name is accepted (and served by the one GPU path).
  return id.kind != kernel_kind::generic ||
         (id.lanes == 4 || id.lanes == 8 || id.lanes == 16 || id.lanes == 32);
}

std::vector<kernel_id> available_kernels(const cpu_features&) { return {kernel_id::cuda()}; }
std::vector<kernel_id> available_kernels() { return {kernel_id::cuda()}; }

kernel_id select_kernel(const std::optional<kernel_id>& override_id, const cpu_features& f) {
  if (override_id && !kernel_supported(*override_id, f))
    throw std::invalid_argument("generic kernel lane count must be 4, 8, 16, or 32");
  return kernel_id::cuda();
}

kernel_id select_kernel(const std::optional<kernel_id>& override_id) {
  return select_kernel(override_id, detect_cpu_features());
}

void to_well_formed(std::span<const char16_t> in, std::span<char16_t> out,
                    const std::optional<kernel_id>& kernel) {
  if (in.size() != out.size())
    throw std::invalid_argument("to_well_formed: input and output lengths differ");
  validate(kernel);
  const auto* i = reinterpret_cast<const uint16_t*>(in.data());
  auto* o = reinterpret_cast<uint16_t*>(out.data());
  if (in.empty()) return;
  const bool di = is_device(i), dout = is_device(o);
  if (di && dout) {
    check(u16m_to_well_formed(i, in.size(), o, nullptr));
    sync_default();
  } else if (!di && !dout) {
    check(u16m_to_well_formed_host(i, in.size(), o));
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
  if (is_device(i)) {
    check(u16m_to_well_formed_batched_n(i, in.size(), offsets.data(), S, o, nullptr));
    sync_default();
    return;
  }
  check(u16m_to_well_formed_batched_host(i, in.size(), offsets.data(), S, o));
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
