// Source-compatible replacement for the reference's utf16mend/surrogate.hpp —
// a header the reference includes from 13 files but does not ship (SURVEY.md
// §0 fact 1). Signatures follow its call sites:
//   classify / surrogate_class            proj/tests/test_surrogate.cpp:11-21
//   is_{high,low}_surrogate, is_surrogate proj/tests/test_surrogate.cpp:24-33
//   compose_code_point                    proj/tests/test_surrogate.cpp:35-48
//   fix_scalar(out, in, n)                proj/src/bitmask_kernel_avx512.cpp:67
//   fix_scalar(span in, span out)         proj/src/driver.cpp:116
//   is_well_formed                        proj/tests/test_surrogate.cpp:69-75
//   unpaired_surrogate_offsets            proj/tests/test_surrogate.cpp:122-128, proj/bindings/module.cpp:77
//   replacement_character                 proj/tests/test_helpers.hpp:35
// The per-unit predicates are constexpr header code (callers classify single
// units with them). Every function that repairs or scans a buffer is served
// by the GPU through the C ABI (include/u16m.h) — `fix_scalar` keeps its name
// only so callers compile; its result is the reference's and
// it may alias exactly, as the reference's may. There is no CPU repair path.
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

/// Code point of a valid pair.
constexpr char32_t compose_code_point(char16_t high, char16_t low) {
  return static_cast<char32_t>(((static_cast<std::uint32_t>(high) - 0xD800u) << 10) +
                               (static_cast<std::uint32_t>(low) - 0xDC00u) + 0x10000u);
}

/// Repair n units (note the reference's out, in, n order); out == in allowed.
void fix_scalar(char16_t* out, const char16_t* in, std::size_t n);
/// Repair `in` into `out` (equal length; equal or disjoint).
void fix_scalar(std::span<const char16_t> in, std::span<char16_t> out);

/// True iff the buffer contains no unpaired surrogate (GPU count).
bool is_well_formed(std::span<const char16_t> in);

/// Ascending offsets of the units repair would rewrite, at most `limit`.
std::vector<std::size_t> unpaired_surrogate_offsets(std::span<const char16_t> in,
                                                    std::size_t limit = SIZE_MAX);

}  // namespace utf16mend
