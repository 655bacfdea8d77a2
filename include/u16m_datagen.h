/* u16m datagen — on-device seeded synthetic inputs for BASELINE.json configs
 * 0-4 (bench/test harness, not part of the repair path).
 *
 * The generators are counter-based (splitmix64 keyed by (seed, stream,
 * index)) so any window of the logical buffer — in particular one GPU's shard
 * of the 64 GiB config 4 — is generated independently and bit-identically to
 * the CPU oracle's or_gen_config (oracle/oracle.c). Spec: DESIGN.md §Inputs.
 * Device pointers; asynchronous on `stream`.
 */
#ifndef U16M_DATAGEN_H
#define U16M_DATAGEN_H

#include <stddef.h>
#include <stdint.h>

#include "u16m.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Units [first, first+count) of the logical buffer of `total` units of config
 * cfg in {0,1,2,4}; shard_len (config 4) = per-GPU shard length whose edges
 * carry adversarial patterns (0 = none). */
u16m_status u16m_gen_config(int cfg, uint64_t seed, uint64_t total, uint64_t shard_len,
                            uint64_t first, uint64_t count, uint16_t* out, void* stream);

/* Config 3: offsets (num_strings+1 int64, device) from seeded log-uniform
 * lengths. Synchronous (returns the total unit count in *total_units). */
u16m_status u16m_gen_c3_offsets(uint64_t seed, size_t num_strings, int64_t* offsets,
                                uint64_t* total_units);

/* Config 3 string contents given device offsets. Asynchronous. */
u16m_status u16m_gen_c3_content(uint64_t seed, size_t num_strings, const int64_t* offsets,
                                uint16_t* out, void* stream);

/* The reference's own Python-facing generator, generate_utf16le
 * (proj/bindings/module.cpp:80-93 -> proj/src/datagen.cpp:44-74): seeded
 * std::mt19937_64 with the reference's bounded-draw mapping, on the host
 * (it is a sequential RNG stream; the RNG identity is the contract,
 * proj/include/utf16mend/datagen.hpp:21-22). Host output buffer. */
u16m_status u16m_generate_reference_mix(size_t units, double pair_pct, double mismatch_pct,
                                        uint64_t seed, uint16_t* out);

/* Streaming-read L2 flush helper for benchmarks: reads `bytes` of `buf`. */
u16m_status u16m_l2_flush(const void* buf, size_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif
