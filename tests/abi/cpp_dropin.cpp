// Source written against the REFERENCE's driver.hpp API (proj/include/
// utf16mend/driver.hpp:64-69) — compiled unchanged against include/utf16mend/
// driver.hpp and linked to libu16m.so. Exit codes: 0 = repaired correctly,
// 3 = std::runtime_error (no CUDA device: the path has no CPU fallback),
// 1 = wrong result, 2 = wrong exception.
#include <cstdint>
#include <cstdio>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "utf16mend/driver.hpp"
#include "utf16mend/surrogate.hpp"

// The per-unit predicates are constexpr, as the reference's call sites use
// them (proj/tests/test_surrogate.cpp:11-48).
static_assert(utf16mend::is_high_surrogate(0xDBFF) && !utf16mend::is_high_surrogate(0xDC00));
static_assert(utf16mend::is_low_surrogate(0xDC00) && utf16mend::is_surrogate(0xDFFF));
static_assert(utf16mend::classify(0x41) == utf16mend::surrogate_class::non_surrogate);
static_assert(utf16mend::compose_code_point(0xD83D, 0xDE0A) == 0x1F60A);

int main() {
  using namespace utf16mend;
  std::vector<char16_t> in;
  for (const char c : std::string("Hello, world!Hello, world!Hello")) in.push_back(static_cast<char16_t>(c));
  in[10] = 0xD800;
  in[21] = 0xDC00;
  in[29] = 0xD83D;
  in[30] = 0xDE0A;
  std::vector<char16_t> expected = in;
  expected[10] = expected[21] = 0xFFFD;
  std::vector<char16_t> out(in.size());
  // length mismatch is std::invalid_argument before any device work
  try {
    std::vector<char16_t> short_out(3);
    to_well_formed(in, short_out);
    return 2;
  } catch (const std::invalid_argument&) {
  }
  try {
    to_well_formed(in, out, kernel_id::bitmask());
    std::vector<char16_t> buf = in;
    to_well_formed_in_place(buf, parse_kernel_id("generic8"));
    if (out != expected || buf != expected) return 1;
    // surrogate.hpp entry points (reference out, in, n order; exact aliasing allowed)
    std::vector<char16_t> fs(in.size()), alias = in;
    fix_scalar(fs.data(), in.data(), in.size());
    fix_scalar(std::span<const char16_t>(alias), std::span<char16_t>(alias));
    if (fs != expected || alias != expected) return 1;
    if (is_well_formed(in) || !is_well_formed(expected)) return 1;
    if (unpaired_surrogate_offsets(in) != std::vector<std::size_t>{10, 21}) return 1;
    if (unpaired_surrogate_offsets(in, 1) != std::vector<std::size_t>{10}) return 1;
    // batched on host vectors: strings [0,11) [11,22) [22,31) — the lone units stay lone
    std::vector<char16_t> bo(in.size());
    const std::vector<std::int64_t> offs{0, 11, 22, 31};
    to_well_formed_batched(in, offs, bo);
    if (bo != expected) return 1;
    try {
      const std::vector<std::int64_t> bad{0, 20, 11, 31};
      to_well_formed_batched(in, bad, bo);
      return 2;
    } catch (const std::invalid_argument&) {
    }
    std::printf("repaired %s\n", to_string(select_kernel()).c_str());
    return 0;
  } catch (const std::runtime_error& e) {
    std::printf("runtime_error: %s\n", e.what());
    return 3;
  } catch (...) {
    return 2;
  }
}
