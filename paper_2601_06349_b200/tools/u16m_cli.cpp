// u16m — command-line front end over the C ABI (§8(f-3): codec fusion + `fix`).
//
// Mirrors the reference CLI's `fix`, `check` and `generate` subcommands
// (proj/tools/main.cpp:62-139, 199-281): same options, messages and exit codes
// (0 ok, 1 ill-formed for `check`, 2 usage / I/O / codec errors). Byte-order
// handling follows the reference codec contract (proj/include/utf16mend/
// codec.hpp:14-54 and its tests, proj/tests/test_codec.cpp): BOM detection
// when the order is "auto" (little-endian otherwise, with a warning), a BOM
// matching an explicit order is recognised, odd byte counts are rejected
// unless --pad-final turns the dangling byte into U+FFFD. The repair itself
// runs on the GPU in the file's own byte order (u16m_fix_utf16_bytes_host:
// no separate swap pass) and counts replacements on the device.
//
// The reference's `bench` subcommand (CPU throughput sweeps, CSV/SVG) is not
// mirrored; bench.py is this repo's harness.

#include <cerrno>
#include <cstdint>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <iterator>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "u16m.h"
#include "utf16mend/driver.hpp"
#include "u16m_datagen.h"

namespace {

struct usage_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

enum class order { little, big };

std::vector<uint8_t> read_file(const std::string& path) {
  // Block reads (a byte-wise istreambuf_iterator copy ran at well under 1 GB/s).
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw std::runtime_error(path + ": " + std::strerror(errno));
  std::vector<uint8_t> buf;
  if (std::fseek(f, 0, SEEK_END) == 0) {
    const long size = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    if (size > 0) {
      buf.resize(static_cast<size_t>(size));
      buf.resize(std::fread(buf.data(), 1, buf.size(), f));
    }
  }
  std::vector<uint8_t> blk(size_t(1) << 20);  // the rest (pipes, files that grew)
  for (size_t got; (got = std::fread(blk.data(), 1, blk.size(), f)) > 0;)
    buf.insert(buf.end(), blk.begin(), blk.begin() + static_cast<std::ptrdiff_t>(got));
  const bool err = std::ferror(f) != 0;
  std::fclose(f);
  if (err) throw std::runtime_error(path + ": read failed");
  return buf;
}

void write_file(const std::string& path, const std::vector<uint8_t>& bytes) {
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw std::runtime_error(path + ": " + std::strerror(errno));
  f.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
  if (!f) throw std::runtime_error(path + ": write failed");
}

std::optional<order> parse_order(const std::string& s) {
  if (s == "le") return order::little;
  if (s == "be") return order::big;
  if (s == "auto") return std::nullopt;
  throw usage_error("--endianness must be le, be or auto");
}

void check_status(u16m_status st) {
  if (st != U16M_OK) throw std::runtime_error(std::string(u16m_status_string(st)) + ": " + u16m_last_error());
}

// Where the units of a raw UTF-16 file lie (decode's contract without the copy).
struct layout {
  size_t start = 0;    // 2 when a BOM is consumed
  size_t n_units = 0;  // whole units after the BOM
  order byte_order = order::little;
  bool had_bom = false;
  bool padded = false;  // a dangling final byte (only with --pad-final)
};

layout locate(const std::vector<uint8_t>& in, std::optional<order> explicit_order, bool pad_final) {
  layout l;
  const bool le_bom = in.size() >= 2 && in[0] == 0xFF && in[1] == 0xFE;
  const bool be_bom = in.size() >= 2 && in[0] == 0xFE && in[1] == 0xFF;
  if (explicit_order) {
    l.byte_order = *explicit_order;
    l.had_bom = (*explicit_order == order::little && le_bom) || (*explicit_order == order::big && be_bom);
  } else {
    l.byte_order = be_bom ? order::big : order::little;
    l.had_bom = le_bom || be_bom;
  }
  l.start = l.had_bom ? 2 : 0;
  const size_t body = in.size() - l.start;
  if (body % 2 != 0) {
    if (!pad_final) throw std::runtime_error("truncated UTF-16: odd number of bytes (use --pad-final)");
    l.padded = true;
  }
  l.n_units = body / 2;
  return l;
}

void write_parts(const std::string& path, std::initializer_list<std::pair<const uint8_t*, size_t>> parts) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error(path + ": " + std::strerror(errno));
  bool ok = true;
  for (const auto& [p, n] : parts)
    if (n) ok = ok && std::fwrite(p, 1, n, f) == n;
  ok = std::fclose(f) == 0 && ok;
  if (!ok) throw std::runtime_error(path + ": write failed");
}

std::vector<uint8_t> encode(const std::vector<uint8_t>& unit_bytes, order o, bool with_bom) {
  std::vector<uint8_t> out;
  out.reserve(unit_bytes.size() + 2);
  if (with_bom) {
    if (o == order::little) out.insert(out.end(), {0xFF, 0xFE});
    else out.insert(out.end(), {0xFE, 0xFF});
  }
  out.insert(out.end(), unit_bytes.begin(), unit_bytes.end());
  return out;
}

void append_fffd(std::vector<uint8_t>& b, order o) {
  if (o == order::little) b.insert(b.end(), {0xFD, 0xFF});
  else b.insert(b.end(), {0xFF, 0xFD});
}

// Options -------------------------------------------------------------------
struct args {
  std::vector<std::string> pos;
  std::vector<std::pair<std::string, std::string>> opts;
  bool has(const std::string& k) const {
    for (auto& kv : opts)
      if (kv.first == k) return true;
    return false;
  }
  std::string get(const std::string& k, const std::string& def) const {
    for (auto& kv : opts)
      if (kv.first == k) return kv.second;
    return def;
  }
};

args parse(int argc, char** argv, int first, const std::vector<std::pair<std::string, std::string>>& with_value,
           const std::vector<std::pair<std::string, std::string>>& flags) {
  args a;
  for (int i = first; i < argc; i++) {
    std::string t = argv[i];
    bool matched = false;
    for (auto& [short_name, long_name] : with_value) {
      if (t == short_name || t == long_name) {
        if (i + 1 >= argc) throw usage_error(t + " needs a value");
        a.opts.emplace_back(long_name, argv[++i]);
        matched = true;
        break;
      }
      if (t.rfind(long_name + "=", 0) == 0) {
        a.opts.emplace_back(long_name, t.substr(long_name.size() + 1));
        matched = true;
        break;
      }
    }
    if (matched) continue;
    for (auto& [short_name, long_name] : flags) {
      if (t == short_name || t == long_name) {
        a.opts.emplace_back(long_name, "1");
        matched = true;
        break;
      }
    }
    if (matched) continue;
    if (!t.empty() && t[0] == '-' && t != "-") throw usage_error("unknown option " + t);
    a.pos.push_back(t);
  }
  return a;
}

// -k / UTF16MEND_KERNEL go through the library's reference-compatible
// selection (proj/tools/main.cpp:46-50,63-77 -> proj/src/driver.cpp:71-108):
// an unknown name is a usage error; an override the host does not support
// throws std::invalid_argument (exit 2); without -k a bad UTF16MEND_KERNEL
// warns and falls back. Every id runs the one GPU path.
std::optional<utf16mend::kernel_id> kernel_option(const args& a) {
  if (!a.has("--kernel")) return std::nullopt;
  const std::string name = a.get("--kernel", "");
  const auto id = utf16mend::parse_kernel_id(name);
  if (!id) throw usage_error("unknown kernel '" + name + "'");
  return id;
}

int cmd_fix(int argc, char** argv) {
  const args a = parse(argc, argv, 2,
                       {{"-o", "--output"}, {"-e", "--endianness"}, {"-k", "--kernel"}, {"--bom", "--bom"}},
                       {{"-i", "--in-place"}, {"--pad-final", "--pad-final"}});
  if (a.pos.size() != 1) throw usage_error("fix: exactly one input path");
  const std::string path = a.pos[0];
  const bool in_place = a.has("--in-place");
  if (in_place && a.has("--output")) throw usage_error("--output excludes --in-place");
  if (!in_place && !a.has("--output")) throw usage_error("fix: one of --in-place or --output");
  const std::string bom = a.get("--bom", "preserve");
  if (bom != "preserve" && bom != "strip" && bom != "require") throw usage_error("--bom must be preserve, strip or require");
  (void)utf16mend::select_kernel(kernel_option(a));
  const auto explicit_order = parse_order(a.get("--endianness", "auto"));

  // The units are repaired where they lie in the file buffer (no decode /
  // encode copies of the payload); the output is written as BOM + units
  // (+ U+FFFD for a dangling byte), exactly what decode -> fix -> encode gives.
  auto bytes = read_file(path);
  const layout d = locate(bytes, explicit_order, a.has("--pad-final"));
  if (!explicit_order && !d.had_bom)
    std::cerr << "utf16mend: " << path << ": no BOM found, assuming little-endian\n";
  if (bom == "require" && !d.had_bom) throw std::runtime_error(path + ": BOM required but not present");

  unsigned long long replacements = 0;
  uint8_t* units = bytes.data() + d.start;
  if (d.n_units > 0)
    check_status(u16m_fix_utf16_bytes_host(units, d.n_units, units,
                                           d.byte_order == order::big ? U16M_BIG_ENDIAN : U16M_LITTLE_ENDIAN,
                                           &replacements));
  std::vector<uint8_t> head, tail;
  if (d.had_bom && bom != "strip") head = encode({}, d.byte_order, true);  // the BOM alone
  if (d.padded) {
    append_fffd(tail, d.byte_order);  // a dangling byte decodes as U+FFFD (codec contract)
    replacements++;
  }
  write_parts(in_place ? path : a.get("--output", ""),
              {{head.data(), head.size()}, {units, 2 * d.n_units}, {tail.data(), tail.size()}});
  std::cout << replacements << (replacements == 1 ? " replacement\n" : " replacements\n");
  return 0;
}

int cmd_check(int argc, char** argv) {
  const args a = parse(argc, argv, 2, {{"-e", "--endianness"}}, {});
  if (a.pos.size() != 1) throw usage_error("check: exactly one input path");
  const std::string path = a.pos[0];
  const auto explicit_order = parse_order(a.get("--endianness", "auto"));
  const auto bytes = read_file(path);
  const layout d = locate(bytes, explicit_order, false);
  if (!explicit_order && !d.had_bom)
    std::cerr << "utf16mend: " << path << ": no BOM found, assuming little-endian\n";
  const size_t n = d.n_units;
  // The units are scanned where they lie in the file buffer, in the file's
  // byte order (big-endian chunks are swapped on the device).
  unsigned long long offs[10];
  size_t count = 0;
  check_status(u16m_unpaired_offsets_bytes_host(bytes.data() + d.start, n,
                                                d.byte_order == order::big ? U16M_BIG_ENDIAN : U16M_LITTLE_ENDIAN,
                                                10, offs, &count));
  if (count == 0) {
    std::cout << path << ": well-formed\n";
    return 0;
  }
  std::cout << path << ": ill-formed; first offending unit offsets:";
  for (size_t i = 0; i < count; i++) std::cout << ' ' << offs[i];
  std::cout << '\n';
  return 1;
}

int cmd_generate(int argc, char** argv) {
  const args a = parse(argc, argv, 2,
                       {{"-n", "--units"}, {"--pair-pct", "--pair-pct"}, {"--mismatch-pct", "--mismatch-pct"},
                        {"--seed", "--seed"}, {"-e", "--endianness"}, {"-o", "--output"}},
                       {{"--bom", "--bom"}});
  if (!a.has("--units")) throw usage_error("generate: --units is required");
  const size_t units = std::stoull(a.get("--units", "0"));
  const double pair = std::stod(a.get("--pair-pct", "0"));
  const double mis = std::stod(a.get("--mismatch-pct", "0"));
  if (pair < 0 || pair > 1 || mis < 0 || mis > 1) throw usage_error("rates must be within [0, 1]");
  const uint64_t seed = std::stoull(a.get("--seed", "0"));
  const std::string e = a.get("--endianness", "le");
  if (e != "le" && e != "be") throw usage_error("--endianness must be le or be");
  std::vector<uint16_t> u(units);
  if (units) check_status(u16m_generate_reference_mix(units, pair, mis, seed, u.data()));
  std::vector<uint8_t> raw(2 * units);
  for (size_t i = 0; i < units; i++) {
    raw[2 * i] = static_cast<uint8_t>(e == "le" ? (u[i] & 0xFF) : (u[i] >> 8));
    raw[2 * i + 1] = static_cast<uint8_t>(e == "le" ? (u[i] >> 8) : (u[i] & 0xFF));
  }
  const auto out = encode(raw, e == "le" ? order::little : order::big, a.has("--bom"));
  if (a.has("--output")) {
    write_file(a.get("--output", ""), out);
  } else {
    std::fwrite(out.data(), 1, out.size(), stdout);
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) throw usage_error("a subcommand is required: fix, check or generate");
    const std::string sub = argv[1];
    if (sub == "fix") return cmd_fix(argc, argv);
    if (sub == "check") return cmd_check(argc, argv);
    if (sub == "generate") return cmd_generate(argc, argv);
    if (sub == "-h" || sub == "--help") {
      std::cout << "u16m fix <path> (-o OUT | -i) [-e le|be|auto] [-k KERNEL] [--bom preserve|strip|require] "
                   "[--pad-final]\nu16m check <path> [-e le|be|auto]\nu16m generate -n UNITS [--pair-pct P] "
                   "[--mismatch-pct M] [--seed S] [-e le|be] [--bom] [-o OUT]\n";
      return 0;
    }
    throw usage_error("unknown subcommand " + sub);
  } catch (const usage_error& e) {
    std::cerr << "utf16mend: " << e.what() << '\n';
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "utf16mend: " << e.what() << '\n';
    return 2;
  }
}
