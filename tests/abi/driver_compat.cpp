// The reference's own driver tests (proj/tests/test_driver.cpp:12-113),
// assertion for assertion, compiled against include/utf16mend/driver.hpp and
// linked to libu16m.so. doctest is absent here, so each TEST_CASE is a block
// and CHECK counts failures. Modes:
//   driver_compat select            — the kernel-selection cases (no GPU)
//   driver_compat repair IN EXP     — the repair cases (need a GPU); IN/EXP are
//                                      the Fig. 4 mixed sample (hex units,
//                                      from tests/golden), since
//                                      testutil::mixed_sample_* are test-only
//                                      reference code
//   driver_compat env               — prints select_kernel() (UTF16MEND_KERNEL)
// Exit 0 = every check passed.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "u16m_datagen.h"
#include "utf16mend/driver.hpp"

using namespace utf16mend;

static int failures = 0;
#define CHECK(cond)                                                    \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::fprintf(stderr, "CHECK failed at line %d: %s\n", __LINE__, #cond); \
      failures++;                                                      \
    }                                                                  \
  } while (0)
#define CHECK_FALSE(cond) CHECK(!(cond))
#define CHECK_THROWS_AS(expr, exc)      \
  do {                                  \
    bool _thrown = false;               \
    try {                               \
      (void)(expr);                     \
    } catch (const exc&) {              \
      _thrown = true;                   \
    } catch (...) {                     \
    }                                   \
    CHECK(_thrown && #exc);             \
  } while (0)

static void select_cases() {
  {  // "kernel_id strings round-trip"
    const kernel_id ids[] = {
        kernel_id::scalar(),      kernel_id::generic(4),   kernel_id::generic(8),
        kernel_id::generic(16),   kernel_id::generic(32),  kernel_id::bitmask(),
        kernel_id::bitmask(true), kernel_id::bytesplit(), kernel_id::bytesplit(true),
    };
    for (const kernel_id& id : ids) CHECK(parse_kernel_id(to_string(id)) == id);
    CHECK(parse_kernel_id("generic") == kernel_id::generic(8));
    CHECK_FALSE(parse_kernel_id("turbo").has_value());
    CHECK_FALSE(parse_kernel_id("").has_value());
  }
  {  // default-constructed id is the reference's generic/8
    const kernel_id d{};
    CHECK(d == kernel_id::generic(8));
    CHECK(d.kind == kernel_kind::generic && d.lanes == 8 && !d.emulated);
  }
  {  // "select_kernel honours an explicit override"
    const cpu_features bare{};
    CHECK(select_kernel(kernel_id::scalar(), bare) == kernel_id::scalar());
    CHECK(select_kernel(kernel_id::generic(16), bare) == kernel_id::generic(16));
    CHECK(select_kernel(kernel_id::bitmask(true), bare) == kernel_id::bitmask(true));
    CHECK(select_kernel(kernel_id::bytesplit(true), bare) == kernel_id::bytesplit(true));
  }
  {  // "select_kernel rejects native overrides the host cannot run"
    const cpu_features bare{};
    CHECK_THROWS_AS(select_kernel(kernel_id::bitmask(), bare), std::invalid_argument);
    CHECK_THROWS_AS(select_kernel(kernel_id::bytesplit(), bare), std::invalid_argument);
    CHECK_THROWS_AS(select_kernel(kernel_id::generic(7), bare), std::invalid_argument);
    try {
      select_kernel(kernel_id::bitmask(), bare);
    } catch (const std::invalid_argument& e) {
      CHECK(std::string(e.what()).find("mask registers") != std::string::npos);
    }
  }
  {  // "select_kernel picks the widest native kernel, generic8 otherwise"
    CHECK(select_kernel({}, cpu_features{}) == kernel_id::generic(8));
    CHECK(select_kernel({}, cpu_features{.wide_mask_registers = true}) == kernel_id::bitmask());
    CHECK(select_kernel({}, cpu_features{.byte_deinterleave = true}) == kernel_id::bytesplit());
    CHECK(select_kernel({}, cpu_features{.wide_mask_registers = true, .byte_deinterleave = true}) ==
          kernel_id::bitmask());
  }
  {  // "select_kernel is deterministic within a process"
    const kernel_id first = select_kernel();
    for (int i = 0; i < 5; i++) CHECK(select_kernel() == first);
    CHECK(kernel_supported(first, detect_cpu_features()));
  }
  {  // "available_kernels lists emulated backends unconditionally"
    const auto bare = available_kernels(cpu_features{});
    CHECK(std::find(bare.begin(), bare.end(), kernel_id::bitmask(true)) != bare.end());
    CHECK(std::find(bare.begin(), bare.end(), kernel_id::bytesplit(true)) != bare.end());
    CHECK(std::find(bare.begin(), bare.end(), kernel_id::bitmask()) == bare.end());
    const auto full = available_kernels(cpu_features{.wide_mask_registers = true, .byte_deinterleave = true});
    CHECK(std::find(full.begin(), full.end(), kernel_id::bitmask()) != full.end());
    CHECK(std::find(full.begin(), full.end(), kernel_id::bytesplit()) != full.end());
  }
  {  // "to_well_formed rejects mismatched buffer lengths" (before any device work)
    const std::vector<char16_t> in(8, 0x0041);
    std::vector<char16_t> out(7);
    CHECK_THROWS_AS(to_well_formed(in, out), std::invalid_argument);
  }
  {  // an override the host cannot run is rejected by to_well_formed too
    const std::vector<char16_t> in(8, 0x0041);
    std::vector<char16_t> out(8);
    CHECK_THROWS_AS(to_well_formed(in, out, kernel_id::generic(7)), std::invalid_argument);
  }
  // exhaustive switch over the reference's four enumerators compiles warning-free
  for (const kernel_id& id : available_kernels()) {
    switch (id.kind) {
      case kernel_kind::scalar:
      case kernel_kind::generic:
      case kernel_kind::bitmask:
      case kernel_kind::bytesplit: break;
    }
  }
  CHECK(backend_name() == "cuda-sm100a");
}

static std::vector<char16_t> parse_units(const char* hex) {
  std::vector<char16_t> v;
  std::string s(hex);
  size_t i = 0;
  while (i < s.size()) {
    size_t j = s.find(',', i);
    if (j == std::string::npos) j = s.size();
    v.push_back(static_cast<char16_t>(std::stoul(s.substr(i, j - i), nullptr, 16)));
    i = j + 1;
  }
  return v;
}

static void repair_cases(const std::vector<char16_t>& in, const std::vector<char16_t>& expected) {
  {  // "every selectable kernel repairs the mixed sample in both modes"
    for (const kernel_id& id : available_kernels()) {
      std::vector<char16_t> out(in.size());
      to_well_formed(in, out, id);
      CHECK(out == expected);
      std::vector<char16_t> buffer = in;
      to_well_formed_in_place(buffer, id);
      CHECK(buffer == expected);
    }
  }
  {  // "all kernels produce identical output on random inputs" (generate() via
     // the library's restatement of proj/src/datagen.cpp, pinned by tests/golden)
    const auto kernels = available_kernels();
    for (std::uint64_t seed = 0; seed < 150; seed++) {
      const size_t n = (seed * 37) % 500;
      std::vector<char16_t> inr(n);
      if (u16m_generate_reference_mix(n, 0.08, 0.3, 40000 + seed, reinterpret_cast<uint16_t*>(inr.data())) != U16M_OK)
        CHECK(false);
      std::vector<char16_t> reference(n);
      to_well_formed(inr, reference, kernel_id::scalar());
      std::vector<char16_t> scalar_ref(n);
      fix_scalar(std::span<const char16_t>(inr), std::span<char16_t>(scalar_ref));
      CHECK(reference == scalar_ref);
      for (const kernel_id& id : kernels) {
        std::vector<char16_t> out(n);
        to_well_formed(inr, out, id);
        CHECK(out == reference);
      }
    }
  }
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "select";
  try {
    if (mode == "select") {
      select_cases();
    } else if (mode == "env") {
      std::printf("%s\n", to_string(select_kernel()).c_str());
      return 0;
    } else if (mode == "repair" && argc == 4) {
      repair_cases(parse_units(argv[2]), parse_units(argv[3]));
    } else {
      std::fprintf(stderr, "usage: driver_compat select | env | repair IN EXPECTED\n");
      return 2;
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "exception: %s\n", e.what());
    return 3;
  }
  if (failures) std::fprintf(stderr, "%d check(s) failed\n", failures);
  return failures ? 1 : 0;
}
