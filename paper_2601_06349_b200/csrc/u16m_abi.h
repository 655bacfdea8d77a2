// Internal helpers shared by the C ABI translation units (u16m_capi.cu:
// device entry points and the shard driver; u16m_host.cu: host-memory entry
// points): argument checks, the thread-local error string, status mapping.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>

#include "../../include/u16m.h"

namespace u16m::abi {

u16m_status fail(u16m_status st, const std::string& detail);
u16m_status cuda_fail(cudaError_t e, const char* what);
u16m_status check_device_present();
// Device-accessible: device or managed memory, or pinned host memory mapped
// into the device address space.
u16m_status check_device_ptr(const void* p, const char* name);
u16m_status check_pair(const uint16_t* in, size_t n, const uint16_t* out);
inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace u16m::abi

#define U16M_TRY(expr)                 \
  do {                                 \
    const u16m_status _st = (expr);    \
    if (_st != U16M_OK) return _st;    \
  } while (0)
