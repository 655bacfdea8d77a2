/* TEST INFRASTRUCTURE — the CPU oracle. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / reference legs may load it, and only as the
 * checker or the timed CPU baseline. The product (libu16m.so) never links it.
 *
 * A plain-C restatement of the reference's repair path and of the synthetic
 * input generators (see oracle.c for file:line citations). Parity pins:
 * tests/test_oracle.py checks every function here against the reference's own
 * compiled code (oracle/_ref) and against the committed golden fixtures in
 * tests/golden/.
 */
#ifndef U16M_ORACLE_H
#define U16M_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- repair (reference semantics) ---------------------------------------- */
void or_fix_scalar(uint16_t* out, const uint16_t* in, size_t n); /* out-first, like the ref */
void or_stencil(const uint16_t* in, size_t n, uint16_t* out);
/* Stencil with explicit neighbours: left/right are the units just outside
 * [0,n), or -1 for "outside the logical buffer". */
void or_stencil_halo(const uint16_t* in, size_t n, uint16_t* out, int32_t left, int32_t right);
/* Per-string fix_scalar over [offsets[s], offsets[s+1]); out may equal in. */
int or_fix_batched(const uint16_t* in, const int64_t* offsets, size_t num_strings, uint16_t* out);
size_t or_unpaired_offsets(const uint16_t* in, size_t n, size_t limit, uint64_t* out);
int or_is_well_formed(const uint16_t* in, size_t n);
/* Multi-threaded stencil (contiguous shards, exact halos): the fast checker
 * for large buffers. out must not alias in. */
void or_stencil_mt(const uint16_t* in, size_t n, uint16_t* out, int threads);

/* ---- the reference's mt19937_64 generator, restated --------------------- */
void or_ref_generate(size_t n, double pair_pct, double mismatch_pct, uint64_t seed,
                     uint16_t* out);

/* ---- counter-based config generators ----------------- */
uint64_t or_rng_key(uint64_t seed, uint64_t stream, uint64_t index);
uint64_t or_rng_next(uint64_t* state);
uint32_t or_rng_below(uint64_t* state, uint32_t bound);
/* Writes units [first, first+count) of the logical config buffer of
 * `total` units. cfg in {0,1,2,4}. For cfg 4, `shard_len` is the per-GPU
 * shard length (shard edges get adversarial patterns). */
int or_gen_config(int cfg, uint64_t seed, uint64_t total, uint64_t shard_len, uint64_t first,
                  uint64_t count, uint16_t* out);
/* Config 3: lengths -> offsets (num_strings+1 entries, offsets[0]=0). */
void or_gen_c3_offsets(uint64_t seed, size_t num_strings, int64_t* offsets);
void or_gen_c3_content(uint64_t seed, size_t num_strings, const int64_t* offsets, uint16_t* out);

#ifdef __cplusplus
}
#endif
#endif
