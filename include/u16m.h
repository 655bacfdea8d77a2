/* u16m — B200-native ill-formed UTF-16 repair, C ABI.
 *
 * Drop-in boundary for the reference's repair path (utf16mend). Every entry
 * point computes exactly the reference's to_well_formed semantics: a high
 * surrogate (D800-DBFF) not followed by a low surrogate, and a low surrogate
 * (DC00-DFFF) not preceded by a high surrogate, becomes U+FFFD; every other
 * unit is copied unchanged (reference SPEC.md:67-77).
 *
 * Conventions
 *   - uint16_t is layout-identical to the reference's char16_t.
 *   - Argument order is (in, n, out), the north-star order. The reference's
 *     lower-level pointer forms are out-first (fix_scalar(out,in,n),
 *     proj/src/bitmask_kernel_avx512.cpp:63); those are not exported.
 *   - `out` must equal `in` exactly or not overlap it at all
 *     (proj/src/driver.cpp:139-140); partial overlap -> U16M_ERR_ALIAS.
 *   - Device entry points take device-accessible pointers and a CUDA stream
 *     (cudaStream_t / CUstream passed as void*; NULL = legacy default stream).
 *     They are asynchronous and stream-ordered; nothing is allocated.
 *   - There is no CPU fallback: without a CUDA device every compute entry
 *     point returns U16M_ERR_NO_DEVICE.
 *   - Errors never throw across the ABI. u16m_last_error() returns a
 *     thread-local detail string for the most recent failure on this thread.
 */
#ifndef U16M_H
#define U16M_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define U16M_API_VERSION 1

typedef enum u16m_status {
  U16M_OK = 0,
  U16M_ERR_INVALID_ARGUMENT = 1, /* null pointer with n>0, bad offsets, ...     */
  U16M_ERR_ALIAS = 2,            /* in/out overlap partially                    */
  U16M_ERR_NOT_DEVICE_MEMORY = 3,/* device entry point got a host pointer      */
  U16M_ERR_CUDA = 4,             /* a CUDA runtime call or launch failed        */
  U16M_ERR_MISALIGNED = 5,       /* pointer not 2-byte aligned                  */
  U16M_ERR_NO_DEVICE = 6         /* no CUDA device visible                      */
} u16m_status;

/* Replaces: utf16mend::to_well_formed(span<const char16_t>, span<char16_t>,
 * optional<kernel_id>) — proj/include/utf16mend/driver.hpp:64-65,
 * proj/src/driver.cpp:135-142. Device pointers, async on `stream`. */
u16m_status u16m_to_well_formed(const uint16_t* in, size_t n, uint16_t* out, void* stream);

/* Replaces: utf16mend::to_well_formed_in_place(span<char16_t>, ...) —
 * proj/include/utf16mend/driver.hpp:68-69, proj/src/driver.cpp:144-147. */
u16m_status u16m_to_well_formed_in_place(uint16_t* buf, size_t n, void* stream);

/* NEW (north star item 4; no reference function): each string
 * [offsets[s], offsets[s+1]) for s < num_strings is repaired independently —
 * string edges are "outside", so no pairing across strings. `offsets` is a
 * DEVICE array of num_strings+1 non-decreasing int64 unit indices into
 * in/out (a negative offsets[0] is clamped to 0; offsets past the end of the
 * buffers are undefined behaviour — use the _n form to have them clamped);
 * units outside [offsets[0], offsets[num_strings]) are untouched.
 * out may equal in. No host synchronisation: the grid is sized from the
 * device allocations holding in/out (cuMemGetAddressRange). */
u16m_status u16m_to_well_formed_batched(const uint16_t* in, const int64_t* offsets,
                                        size_t num_strings, uint16_t* out, void* stream);

/* Same, with the length of the in/out buffers (units) known to the caller —
 * the form the C++, Python and CLI front ends use. The grid is sized from
 * n_units (no host sync), strings are located through a per-tile table built
 * by a pre-pass, and every CTA streams one tile (the fastest form measured).
 * Requires offsets[num_strings] <= n_units (units past n_units are never
 * touched). Allocates a small stream-ordered workspace (cudaMallocAsync). */
u16m_status u16m_to_well_formed_batched_n(const uint16_t* in, size_t n_units, const int64_t* offsets,
                                          size_t num_strings, uint16_t* out, void* stream);

/* One contiguous piece of a larger logical buffer (the per-shard primitive for
 * one-process-per-GPU callers). `left`/`right` are the units just outside
 * [0,n) in the logical buffer, or -1 where the logical buffer ends. Device
 * pointers, async. */
u16m_status u16m_to_well_formed_halo(const uint16_t* in, size_t n, uint16_t* out, int32_t left,
                                     int32_t right, void* stream);

/* Same, but the neighbour units are read on the device from `left_ptr` /
 * `right_ptr` (any device-accessible address: local, or a peer GPU's memory
 * over NVLink with peer access enabled); NULL = logical buffer ends there. */
u16m_status u16m_to_well_formed_halo_ptr(const uint16_t* in, size_t n, uint16_t* out,
                                         const uint16_t* left_ptr, const uint16_t* right_ptr,
                                         void* stream);

/* Split form of u16m_to_well_formed_halo_ptr for overlapping a halo exchange
 * with the bulk of the work. The job's 8192-unit tiles are cut into
 * U16M_PART_INTERIOR (every tile except the first and the last; reads no
 * halo) and U16M_PART_EDGES (the first and last tiles; the only part that
 * reads left_ptr / right_ptr). The two parts write disjoint units and may
 * run concurrently on different streams; INTERIOR + EDGES == ALL. */
#define U16M_PART_ALL 0
#define U16M_PART_EDGES 1
#define U16M_PART_INTERIOR 2
u16m_status u16m_to_well_formed_part(const uint16_t* in, size_t n, uint16_t* out,
                                     const uint16_t* left_ptr, const uint16_t* right_ptr, int part,
                                     void* stream);

/* NEW (north star item 5): one logical buffer split into contiguous shards
 * resident on (possibly) different GPUs of this process. Shard g lives on
 * device device_ids[g]; shard_out[g] == shard_in[g] for in-place. Halo units
 * cross shard edges as direct peer loads over NVLink when peer access is
 * available, else through a 2-byte peer copy. Synchronous: returns when every
 * shard is repaired. Runs on the library's own non-blocking streams, so work
 * that wrote the shards must be complete (synchronised) before the call.
 * Device ids may repeat (virtual shards on one GPU). */
u16m_status u16m_to_well_formed_sharded(int num_shards, const int* device_ids,
                                        const uint16_t* const* shard_in, const size_t* shard_len,
                                        uint16_t* const* shard_out);

/* Host-memory form behind the source-compatible C++ API: stages through the
 * current device in pipelined chunks (H2D / repair / D2H overlapped across
 * streams). Synchronous. Pinned host memory gets full-duplex DMA. */
u16m_status u16m_to_well_formed_host(const uint16_t* in, size_t n, uint16_t* out);

/* Host-memory form over several GPUs (north star item 5 for host-resident
 * data; behind utf16mend::to_well_formed on host spans, which replaces
 * proj/src/driver.cpp:135-147): the buffer is cut into contiguous ranges, one
 * per device, each streamed through that device's own pipeline and PCIe link
 * concurrently (one host thread per extra device); the halo unit at each
 * range edge is read from the caller's input. num_devices = 0 (device_ids
 * NULL) = every visible device. Ranges are at least 32 Mi units, so small
 * jobs use fewer devices. Ids may repeat. Synchronous; in == out or disjoint. */
u16m_status u16m_to_well_formed_host_multi(const uint16_t* in, size_t n, uint16_t* out, int num_devices,
                                           const int* device_ids);

/* §8(f) row 1 — validation. Device pointers. `count_out` (device, uint64) gets
 * the number of units repair would rewrite; is_well_formed <=> count == 0.
 * Async; the caller reads count_out after synchronising `stream`. */
u16m_status u16m_count_unpaired(const uint16_t* in, size_t n, unsigned long long* count_out,
                                void* stream);

/* Replaces: unpaired_surrogate_offsets(span, limit) (call sites
 * proj/bindings/module.cpp:72-78, proj/tools/main.cpp:104). Writes up to
 * `limit` ascending unit offsets to `offsets_out` (device) and the number
 * written to *count_out (device). Async. */
u16m_status u16m_unpaired_offsets(const uint16_t* in, size_t n, size_t limit,
                                  unsigned long long* offsets_out,
                                  unsigned long long* count_out, void* stream);

/* §8(f-3) codec fusion — replaces the decode -> to_well_formed -> replacement
 * count -> encode sequence of the CLI's `fix` (proj/tools/main.cpp:62-89,
 * codec.hpp:21-35): repairs n UTF-16 units stored as raw bytes in the given
 * byte order (U16M_LITTLE_ENDIAN / U16M_BIG_ENDIAN) without a separate swap
 * pass, writing the same byte order, and ADDS the number of replaced units to
 * *replacements (device uint64; NULL = don't count). in/out: device, equal
 * (in place) or disjoint, at any 2-byte alignment. Async. A BOM
 * (FEFF) is an ordinary non-surrogate unit and may stay in the buffer. */
#define U16M_LITTLE_ENDIAN 0
#define U16M_BIG_ENDIAN 1
u16m_status u16m_fix_utf16_bytes(const void* in, size_t n_units, void* out, int byte_order,
                                 unsigned long long* replacements, void* stream);

/* Host-memory forms (synchronous, staged through the GPU): the codec-fused
 * repair with the replacement count returned in *replacements (host, may be
 * NULL), and unpaired_surrogate_offsets for host buffers (units in host
 * order; up to `limit` offsets, number written in *count_out). */
u16m_status u16m_fix_utf16_bytes_host(const void* in, size_t n_units, void* out, int byte_order,
                                      unsigned long long* replacements);
/* The same spread over several GPUs as u16m_to_well_formed_host_multi
 * (u16m_fix_utf16_bytes_host = every visible device): contiguous ranges, one
 * per device and PCIe link, halo units read from the caller's input in its
 * byte order; *replacements is the sum over the ranges. */
u16m_status u16m_fix_utf16_bytes_host_multi(const void* in, size_t n_units, void* out, int byte_order,
                                            unsigned long long* replacements, int num_devices,
                                            const int* device_ids);
u16m_status u16m_unpaired_offsets_host(const uint16_t* in, size_t n, size_t limit,
                                       unsigned long long* offsets_out, size_t* count_out);
/* Same over raw UTF-16 bytes in the given byte order (CLI `check` of a
 * big-endian file, proj/tools/main.cpp:96-115): big-endian chunks are
 * byte-swapped on the device after their H2D copy. */
u16m_status u16m_unpaired_offsets_bytes_host(const void* in, size_t n_units, int byte_order, size_t limit,
                                             unsigned long long* offsets_out, size_t* count_out);
/* Batched form on host memory (behind the C++ to_well_formed_batched on host
 * spans): `in`/`out` hold n_units units (equal or disjoint), `offsets` (host)
 * num_strings + 1 non-decreasing entries within [0, n_units]. Synchronous. */
u16m_status u16m_to_well_formed_batched_host(const uint16_t* in, size_t n_units, const int64_t* offsets,
                                             size_t num_strings, uint16_t* out);

/* The reference's kernel-selection names (proj/src/driver.cpp:15-108):
 * available_kernels() comma-joined, and select_kernel() (honours
 * UTF16MEND_KERNEL, warning on bad values as the reference does). Every name
 * is served by the one sm_100a path. Writes a NUL-terminated string of at most
 * cap bytes; returns the full length. (Python available_kernels /
 * default_kernel, proj/bindings/module.cpp:93-104.) */
int u16m_kernel_names(char* buf, size_t cap);
int u16m_default_kernel_name(char* buf, size_t cap);
/* select_kernel(parse_kernel_id(name)) (name NULL = no override): writes the
 * chosen name; an unknown name or an override the host does not support
 * returns U16M_ERR_INVALID_ARGUMENT with the reference's message in
 * u16m_last_error() (proj/src/driver.cpp:71-86, proj/bindings/module.cpp:42-47). */
u16m_status u16m_select_kernel(const char* name, char* buf, size_t cap);

const char* u16m_status_string(u16m_status status);
const char* u16m_last_error(void);
int u16m_api_version(void);
/* Number of kernel launches this process has issued through the library
 * (bench evidence: the "gpu_launches" count). */
unsigned long long u16m_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* U16M_H */
