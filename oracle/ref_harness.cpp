// TEST INFRASTRUCTURE — C entry points over the reference's OWN compiled code
// (oracle/_ref/libutf16mend_ref.so). Used by tests/ (to pin the C oracle and
// generate golden vectors) and by bench.py's reference arm / cpu_baseline leg.
// Never linked into the product.
//
// Everything here calls the reference's public API unchanged:
//   to_well_formed / to_well_formed_in_place   proj/src/driver.cpp:135-147
//   select_kernel / available_kernels / parse  proj/src/driver.cpp:15-108
//   generate (mt19937_64 datagen)              proj/src/datagen.cpp:44-74
//   reference_fix, mixed_sample_*, alphabet    proj/tests/test_helpers.hpp:21-104
// The only added logic is the multi-threaded harness extension
// (ref_to_well_formed_mt): contiguous shards, each repaired by the reference
// on its own thread, then the 2 units on each side of every interior shard
// edge are recomputed from the saved original neighbourhood with the
// reference's per-unit stencil. This is labelled as a harness extension in
// the reference itself is single-threaded (bench.hpp:51).

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <optional>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "test_helpers.hpp"
#include "utf16mend/bench.hpp"
#include "utf16mend/datagen.hpp"
#include "utf16mend/driver.hpp"
#include "utf16mend/surrogate.hpp"

using namespace utf16mend;

namespace {

std::optional<kernel_id> kernel_from(const char* name) {
  if (name == nullptr || name[0] == '\0') return std::nullopt;
  return parse_kernel_id(name);
}

int copy_string(const std::string& s, char* buf, size_t cap) {
  if (cap == 0) return -1;
  const size_t k = std::min(cap - 1, s.size());
  std::memcpy(buf, s.data(), k);
  buf[k] = '\0';
  return static_cast<int>(s.size());
}

// Stencil value of unit i of `x` (length n), the reference's reference_fix rule
// (proj/tests/test_helpers.hpp:42-53) for a single position.
char16_t stencil_at(const char16_t* x, size_t n, size_t i) {
  const char16_t u = x[i];
  if (is_high_surrogate(u) && !(i + 1 < n && is_low_surrogate(x[i + 1])))
    return replacement_character;
  if (is_low_surrogate(u) && !(i >= 1 && is_high_surrogate(x[i - 1])))
    return replacement_character;
  return u;
}

}  // namespace

extern "C" {

int ref_to_well_formed(const uint16_t* in, size_t n, uint16_t* out, const char* kernel) {
  try {
    const auto id = kernel_from(kernel);
    if (kernel && kernel[0] && !id) return -2;
    to_well_formed(std::span<const char16_t>(reinterpret_cast<const char16_t*>(in), n),
                   std::span<char16_t>(reinterpret_cast<char16_t*>(out), n), id);
    return 0;
  } catch (...) {
    return -1;
  }
}

int ref_to_well_formed_in_place(uint16_t* buf, size_t n, const char* kernel) {
  try {
    const auto id = kernel_from(kernel);
    if (kernel && kernel[0] && !id) return -2;
    to_well_formed_in_place(std::span<char16_t>(reinterpret_cast<char16_t*>(buf), n), id);
    return 0;
  } catch (...) {
    return -1;
  }
}

// Harness extension: `threads` contiguous shards; `out == in` for in-place.
int ref_to_well_formed_mt(const uint16_t* in_u, size_t n, uint16_t* out_u, int threads,
                          const char* kernel) {
  try {
    const auto id = kernel_from(kernel);
    if (kernel && kernel[0] && !id) return -2;
    const auto* in = reinterpret_cast<const char16_t*>(in_u);
    auto* out = reinterpret_cast<char16_t*>(out_u);
    size_t t = threads < 1 ? 1 : static_cast<size_t>(threads);
    if (n < 64 * t) t = 1;
    std::vector<size_t> bounds(t + 1);
    for (size_t k = 0; k <= t; k++) bounds[k] = n * k / t;
    // Save x[p-2 .. p+1] around every interior edge p before anything runs.
    std::vector<std::array<char16_t, 4>> saved(t);
    for (size_t k = 1; k < t; k++) {
      const size_t p = bounds[k];
      for (int j = 0; j < 4; j++) saved[k][j] = in[p - 2 + j];
    }
    std::vector<std::thread> pool;
    for (size_t k = 0; k < t; k++) {
      pool.emplace_back([&, k] {
        const size_t a = bounds[k], b = bounds[k + 1];
        if (in == out)
          to_well_formed_in_place(std::span<char16_t>(out + a, b - a), id);
        else
          to_well_formed(std::span<const char16_t>(in + a, b - a),
                         std::span<char16_t>(out + a, b - a), id);
      });
    }
    for (auto& th : pool) th.join();
    for (size_t k = 1; k < t; k++) {
      const size_t p = bounds[k];
      // Window w = x[p-2], x[p-1], x[p], x[p+1]; global ends are respected.
      const char16_t* w = saved[k].data();
      const size_t lo = p - 2;  // n >= 64*t so 2 <= p and p+1 < n
      (void)lo;
      out[p - 1] = stencil_at(w, 4, 1);
      out[p] = stencil_at(w, 4, 2);
    }
    return 0;
  } catch (...) {
    return -1;
  }
}

int ref_reference_fix(const uint16_t* in, size_t n, uint16_t* out) {
  const auto r = testutil::reference_fix(
      std::span<const char16_t>(reinterpret_cast<const char16_t*>(in), n));
  std::memcpy(out, r.data(), n * sizeof(char16_t));
  return 0;
}

int ref_fix_scalar(const uint16_t* in, size_t n, uint16_t* out) {
  fix_scalar(reinterpret_cast<char16_t*>(out), reinterpret_cast<const char16_t*>(in), n);
  return 0;
}

int ref_generate(size_t n, double pair_pct, double mismatch_pct, uint64_t seed,
                 uint16_t* out) {
  const auto v = generate({.length_units = n,
                           .pair_pct = pair_pct,
                           .mismatch_pct = mismatch_pct,
                           .seed = seed});
  std::memcpy(out, v.data(), n * sizeof(char16_t));
  return 0;
}

int ref_mixed_sample(uint16_t* in31, uint16_t* expected31) {
  const auto a = testutil::mixed_sample_input();
  const auto b = testutil::mixed_sample_expected();
  std::memcpy(in31, a.data(), a.size() * 2);
  std::memcpy(expected31, b.data(), b.size() * 2);
  return static_cast<int>(a.size());
}

int ref_boundary_alphabet(uint16_t* out8) {
  for (int i = 0; i < 8; i++) out8[i] = testutil::boundary_alphabet[i];
  return 8;
}

size_t ref_unpaired_surrogate_offsets(const uint16_t* in, size_t n, size_t limit,
                                      uint64_t* out) {
  const auto v = unpaired_surrogate_offsets(
      std::span<const char16_t>(reinterpret_cast<const char16_t*>(in), n), limit);
  for (size_t i = 0; i < v.size(); i++) out[i] = v[i];
  return v.size();
}

// The reference's own CSV reader (proj/src/bench.cpp:172-203) over a file:
// one line per parsed point, "impl|input_units|bytes|best_ns|mean_ns|gbps|
// error_margin_pct" with %.17g (exact round trip). Returns the full length,
// -1 when the file cannot be opened, -2 when parse_csv throws.
int ref_parse_csv(const char* path, char* buf, size_t cap) {
  std::ifstream in(path);
  if (!in) return -1;
  try {
    const auto series = parse_csv(in);
    std::string s;
    char line[512];
    for (const auto& sr : series)
      for (const auto& p : sr.points) {
        const auto& r = p.result;
        std::snprintf(line, sizeof line, "%s|%zu|%zu|%llu|%.17g|%.17g|%.17g\n", r.impl_name.c_str(), r.input_units,
                      r.bytes_per_rep, static_cast<unsigned long long>(r.best_ns), r.mean_ns, r.throughput_gbps,
                      r.error_margin_pct);
        s += line;
      }
    return copy_string(s, buf, cap);
  } catch (...) {
    return -2;
  }
}

int ref_default_kernel(char* buf, size_t cap) { return copy_string(to_string(select_kernel()), buf, cap); }

int ref_available_kernels(char* buf, size_t cap) {
  std::string s;
  for (const auto& id : available_kernels()) {
    if (!s.empty()) s += ",";
    s += to_string(id);
  }
  return copy_string(s, buf, cap);
}

}  // extern "C"
