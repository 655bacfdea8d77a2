// GPU twin of cpp_dropin.cpp: the source-compatible C++ API
// (include/utf16mend/driver.hpp) on every memory placement a caller can hand
// it, checked against an independent host-side stencil (the reference's
// per-unit rule, proj/tests/test_helpers.hpp:42-53, restated here).
//   * device spans (cudaMalloc): copy, in place, batched with device and
//     host offsets, and units outside [offsets.front(), offsets.back())
//   * host spans longer than two pipeline chunks (default 32 Mi-unit chunks:
//     70 Mi units), pageable and in place
//   * is_well_formed / unpaired_surrogate_offsets on device spans, repeated
//     (stream-ordered scratch, no per-call cudaMalloc)
//   * mixed host/device spans -> std::invalid_argument
// Exit 0 = all correct; 1 = wrong result; 2 = wrong/missing exception.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "u16m_datagen.h"
#include "utf16mend/driver.hpp"

using namespace utf16mend;

static std::vector<char16_t> stencil(const std::vector<char16_t>& x, size_t a, size_t b) {
  std::vector<char16_t> y = x;
  for (size_t i = a; i < b; i++) {
    const char16_t u = x[i];
    const bool hi = (u & 0xFC00) == 0xD800, lo = (u & 0xFC00) == 0xDC00;
    if (hi && !(i + 1 < b && (x[i + 1] & 0xFC00) == 0xDC00)) y[i] = 0xFFFD;
    if (lo && !(i > a && (x[i - 1] & 0xFC00) == 0xD800)) y[i] = 0xFFFD;
  }
  return y;
}

static std::vector<char16_t> random_units(size_t n, uint64_t seed) {
  std::vector<char16_t> v(n);
  if (u16m_generate_reference_mix(n, 0.05, 0.02, seed, reinterpret_cast<uint16_t*>(v.data())) != U16M_OK)
    throw std::runtime_error("generate failed");
  return v;
}

#define REQUIRE(c)                                                   \
  do {                                                               \
    if (!(c)) {                                                      \
      std::fprintf(stderr, "wrong result at line %d: %s\n", __LINE__, #c); \
      return 1;                                                      \
    }                                                                \
  } while (0)

template <class T>
struct Dev {
  T* p = nullptr;
  size_t n = 0;
  explicit Dev(size_t n_) : n(n_) {
    if (cudaMalloc(&p, (n ? n : 1) * sizeof(T)) != cudaSuccess) throw std::runtime_error("cudaMalloc");
  }
  ~Dev() { cudaFree(p); }
  void put(const std::vector<T>& v) { cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice); }
  std::vector<T> get() const {
    std::vector<T> v(n);
    cudaMemcpy(v.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost);
    return v;
  }
  std::span<T> span() { return {p, n}; }
};

int main() {
  try {
    // ---- device spans ----------------------------------------------------
    {
      const size_t n = 1000003;
      const auto x = random_units(n, 7);
      const auto e = stencil(x, 0, n);
      Dev<char16_t> din(n), dout(n);
      din.put(x);
      to_well_formed(std::span<const char16_t>(din.p, n), dout.span());
      REQUIRE(dout.get() == e);
      to_well_formed_in_place(din.span(), kernel_id::scalar());
      REQUIRE(din.get() == e);
      // validation on device spans, repeated
      din.put(x);
      for (int r = 0; r < 50; r++) {
        REQUIRE(!is_well_formed(std::span<const char16_t>(din.p, n)));
        REQUIRE(is_well_formed(std::span<const char16_t>(dout.p, n)));
      }
      std::vector<std::size_t> want;
      for (size_t i = 0; i < n && want.size() < 100; i++)
        if (e[i] != x[i]) want.push_back(i);
      REQUIRE(unpaired_surrogate_offsets(std::span<const char16_t>(din.p, n), 100) == want);
      // mixed placements are an argument error
      std::vector<char16_t> host(n);
      try {
        to_well_formed(std::span<const char16_t>(din.p, n), std::span<char16_t>(host));
        return 2;
      } catch (const std::invalid_argument&) {
      }
    }
    // ---- batched on device spans: device offsets, host offsets, outside units
    {
      const size_t n = 300000;
      const auto x = random_units(n, 11);
      std::vector<std::int64_t> offs{17};
      while (offs.back() < static_cast<std::int64_t>(n) - 500)
        offs.push_back(std::min<std::int64_t>(offs.back() + 1 + (offs.size() * 7919) % 3000, n - 100));
      std::vector<char16_t> e = x;  // units outside [offs.front(), offs.back()) unchanged
      for (size_t s = 0; s + 1 < offs.size(); s++) {
        const auto part = stencil(x, offs[s], offs[s + 1]);
        for (std::int64_t i = offs[s]; i < offs[s + 1]; i++) e[i] = part[i];
      }
      Dev<char16_t> din(n), dout(n);
      Dev<std::int64_t> doff(offs.size());
      din.put(x);
      doff.put(offs);
      cudaMemset(dout.p, 0x5A, n * 2);
      to_well_formed_batched(std::span<const char16_t>(din.p, n), std::span<const std::int64_t>(doff.p, offs.size()),
                             dout.span());
      REQUIRE(dout.get() == e);
      cudaMemset(dout.p, 0x5A, n * 2);
      to_well_formed_batched(std::span<const char16_t>(din.p, n), std::span<const std::int64_t>(offs), dout.span());
      REQUIRE(dout.get() == e);
      to_well_formed_batched(std::span<const char16_t>(din.p, n), std::span<const std::int64_t>(offs), din.span());
      REQUIRE(din.get() == e);
      // host data with device offsets is an argument error
      std::vector<char16_t> hout(n);
      try {
        to_well_formed_batched(x, std::span<const std::int64_t>(doff.p, offs.size()), hout);
        return 2;
      } catch (const std::invalid_argument&) {
      }
      // bad device offsets are an argument error, not an out-of-bounds access
      std::vector<std::int64_t> bad{-5, 10, static_cast<std::int64_t>(n) + 9};
      Dev<std::int64_t> dbad(bad.size());
      dbad.put(bad);
      try {
        to_well_formed_batched(std::span<const char16_t>(din.p, n), std::span<const std::int64_t>(dbad.p, 3),
                               dout.span());
        return 2;
      } catch (const std::invalid_argument&) {
      }
    }
    // ---- host spans longer than two pipeline chunks (pageable) ------------
    {
      const size_t n = (size_t(70) << 20) + 5;
      std::vector<char16_t> x = random_units(n, 3);
      // a straddling pair exactly on every 32 Mi-unit chunk edge
      for (size_t c = size_t(32) << 20; c < n; c += size_t(32) << 20) {
        x[c - 1] = 0xD83D;
        x[c] = 0xDE0A;
      }
      const auto e = stencil(x, 0, n);
      std::vector<char16_t> out(n);
      to_well_formed(x, out);
      REQUIRE(out == e);
      to_well_formed_in_place(x);
      REQUIRE(x == e);
    }
    std::printf("ok\n");
    return 0;
  } catch (const std::exception& ex) {
    std::printf("exception: %s\n", ex.what());
    return 3;
  }
}
