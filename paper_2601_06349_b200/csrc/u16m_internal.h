// Internal host-side declarations shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace u16m {

// Repair [0,n) of `in` into `out` (out == in: in place). left/right: halo
// unit values (-1 = outside); left_ptr/right_ptr: device-side halo units
// (override the values when non-null).
cudaError_t launch_repair(const uint16_t* in, size_t n, uint16_t* out, int32_t left, int32_t right,
                          const uint16_t* left_ptr, const uint16_t* right_ptr, cudaStream_t stream);

// TMA-pipelined forms (u16m_tma.cu); same 16-byte phase for in and out.
constexpr size_t kTmaMinUnits = size_t(1) << 15;
cudaError_t launch_repair_tma(const uint16_t* in, size_t n, uint16_t* out, int32_t left, int32_t right,
                              const uint16_t* left_ptr, const uint16_t* right_ptr, cudaStream_t stream);
cudaError_t launch_batched_tma(const uint16_t* in, const int64_t* offsets, size_t num_strings, uint16_t* out,
                               cudaStream_t stream);

cudaError_t launch_batched(const uint16_t* in, const int64_t* offsets, size_t num_strings,
                           uint16_t* out, cudaStream_t stream);

// In-place write-back granularity in lanes of 16 B: 2 = one 32-byte DRAM
// sector (measured best of 16/32/64/128 B; the former U16M_GRAN A/B knob,
// profiles/README.md — scripts/ab_lib.sh rebuilds an older commit to rerun it).
constexpr int kDefaultInplaceGran = 2;

// Part of a job: part = 0 all tiles, 1 only the two edge tiles (the only
// ones that read the halos), 2 only the interior tiles. Edges + interior ==
// all; the two parts write disjoint units and may run concurrently.
cudaError_t launch_repair_part(const uint16_t* in, size_t n, uint16_t* out, int32_t left, int32_t right,
                               const uint16_t* left_ptr, const uint16_t* right_ptr, int part,
                               cudaStream_t stream);

// Rolling-pipeline streaming kernel (u16m_stream.cu) for same-phase copy and
// in-place jobs; `s` from make_span, part as in launch_repair_part.
struct Span;
cudaError_t launch_stream(const Span& s, int part, cudaStream_t stream);
// Copy into an `out` whose 16-byte phase differs from in's (s from make_span).
cudaError_t launch_stream_shift(Span s, uint16_t* out, int part, cudaStream_t stream);
cudaError_t launch_stream_shift_codec(const Span& s, uint16_t* out, bool big_endian, unsigned long long* count,
                                      cudaStream_t stream);
// Codec-fused form (u16m_stream.cu): same-phase buffers in little- or
// big-endian byte order, optional device replacement counter (accumulated).
cudaError_t launch_stream_codec(const Span& s, bool big_endian, unsigned long long* count, cudaStream_t stream);
// Keep the device default mempool's freed blocks cached (stream-ordered
// per-call workspaces stay cheap).
void keep_pool_memory();
// Count of units repair would rewrite, read-only stream kernel (adds to *count).
cudaError_t launch_stream_count(const uint16_t* in, size_t n, unsigned long long* count, cudaStream_t stream,
                                uint32_t* half_tile_counts = nullptr, int32_t left = -1, int32_t right = -1);
// Batched form with the buffer length known: tile table pre-pass + one tile
// per CTA (u16m_stream.cu). offsets[S] <= n_units.
bool batched_tiles_enabled();
// grid_units: size the grid and the tile table for this many units instead
// of n_units (a job whose strings lie in a window of a larger coordinate
// range, e.g. one chunk of the host pipeline addressed with absolute offsets).
cudaError_t launch_batched_tiles(const uint16_t* in, size_t n_units, const int64_t* offsets, size_t num_strings,
                                 uint16_t* out, cudaStream_t stream, size_t grid_units = 0);


// §8(f-3): byte-order-aware repair + replacement count (same 16-byte phase).
// left/right: halo UNIT values (byte order already resolved), -1 = outside.
cudaError_t launch_fix_bytes(const void* in, size_t n, void* out, bool big_endian, unsigned long long* count,
                             cudaStream_t stream, int32_t left, int32_t right);

cudaError_t launch_count_unpaired(const uint16_t* in, size_t n, unsigned long long* count_out,
                                  cudaStream_t stream);

// left/right: halo units around [in, in+n) (-1 = outside the buffer), so a
// caller can scan a long host buffer chunk by chunk.
cudaError_t launch_unpaired_offsets(const uint16_t* in, size_t n, size_t limit,
                                    unsigned long long* offsets_out, unsigned long long* count_out,
                                    cudaStream_t stream, int32_t left = -1, int32_t right = -1);

// Short buffers (0 < n <= kSmallScanUnits, limit > 0): the whole offsets scan
// in one single-CTA launch (u16m_stream.cu).
constexpr size_t kSmallScanUnits = size_t(64) << 10;
cudaError_t launch_small_scan(const uint16_t* in, size_t n, size_t limit, unsigned long long* offsets_out,
                              unsigned long long* count_out, cudaStream_t stream, int32_t left, int32_t right);

// *dst_mapped (mapped pinned host memory, device address) = *src (device), stream-ordered, no copy engine.
cudaError_t launch_store_u64(unsigned long long* dst_mapped, const unsigned long long* src, cudaStream_t stream);

// In-place byte swap of n units (p 16-byte aligned).
cudaError_t launch_byteswap(uint16_t* p, size_t n, cudaStream_t stream);

// Units from p to the end of its device allocation (0 = unknown).
size_t allocation_units_after(const void* p);

unsigned long long launch_count();
void note_launch();

}  // namespace u16m
