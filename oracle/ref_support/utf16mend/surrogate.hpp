// TEST INFRASTRUCTURE — restated header, used ONLY to compile the reference's
// own sources into oracle/_ref/ (the CPU baseline and a second oracle). It is
// never linked into the product library.
//
// The reference ships 13 files that include "utf16mend/surrogate.hpp" but not
// the header itself. This file restates it from the
// reference's module contract and the call
// sites that pin its signatures:
//   classify / surrogate_class        proj/tests/test_surrogate.cpp:11-21
//   is_{high,low}_surrogate, is_surrogate  proj/tests/test_surrogate.cpp:24-33
//   compose_code_point                proj/tests/test_surrogate.cpp:35-48
//   fix_scalar(out, in, n)            proj/src/bitmask_kernel_avx512.cpp:67
//   fix_scalar(span in, span out)     proj/src/driver.cpp:116
//   is_well_formed                    proj/tests/test_surrogate.cpp:69-75
//   unpaired_surrogate_offsets        proj/tests/test_surrogate.cpp:122-128,
//                                     proj/bindings/module.cpp:77
//   replacement_character             proj/tests/test_helpers.hpp:35
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <vector>

namespace utf16mend {

inline constexpr char16_t replacement_character = 0xFFFD;

enum class surrogate_class : std::uint8_t { non_surrogate, high_surrogate, low_surrogate };

constexpr bool is_high_surrogate(char16_t u) { return (u & 0xFC00) == 0xD800; }
constexpr bool is_low_surrogate(char16_t u) { return (u & 0xFC00) == 0xDC00; }
constexpr bool is_surrogate(char16_t u) { return (u & 0xF800) == 0xD800; }

constexpr surrogate_class classify(char16_t u) {
  return is_high_surrogate(u)  ? surrogate_class::high_surrogate
         : is_low_surrogate(u) ? surrogate_class::low_surrogate
                               : surrogate_class::non_surrogate;
}

// ((h - 0xD800) << 10) + (l - 0xDC00) + 0x10000.
constexpr char32_t compose_code_point(char16_t high, char16_t low) {
  return static_cast<char32_t>(((static_cast<std::uint32_t>(high) - 0xD800u) << 10) +
                               (static_cast<std::uint32_t>(low) - 0xDC00u) + 0x10000u);
}

// Sequential consuming scan (pair rule SPEC.md:99). `out` may
// alias `in` exactly: every unit is read before it (or a later one) is written.
inline void fix_scalar(char16_t* out, const char16_t* in, std::size_t n) {
  std::size_t i = 0;
  while (i < n) {
    const char16_t u = in[i];
    if (is_high_surrogate(u) && i + 1 < n && is_low_surrogate(in[i + 1])) {
      const char16_t l = in[i + 1];
      out[i] = u;
      out[i + 1] = l;
      i += 2;
      continue;
    }
    out[i] = is_surrogate(u) ? replacement_character : u;
    i += 1;
  }
}

inline void fix_scalar(std::span<const char16_t> in, std::span<char16_t> out) {
  fix_scalar(out.data(), in.data(), in.size());
}

inline std::vector<std::size_t> unpaired_surrogate_offsets(std::span<const char16_t> in,
                                                           std::size_t limit = SIZE_MAX) {
  std::vector<std::size_t> offsets;
  std::size_t i = 0;
  const std::size_t n = in.size();
  while (i < n && offsets.size() < limit) {
    if (is_high_surrogate(in[i]) && i + 1 < n && is_low_surrogate(in[i + 1])) {
      i += 2;
      continue;
    }
    if (is_surrogate(in[i])) offsets.push_back(i);
    i += 1;
  }
  return offsets;
}

inline bool is_well_formed(std::span<const char16_t> in) {
  return unpaired_surrogate_offsets(in, 1).empty();
}

}  // namespace utf16mend
