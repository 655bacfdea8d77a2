// C ABI, host-memory entry points (include/u16m.h): the staged copy-engine
// pipeline for host buffers (pinned: direct DMA; pageable: pinned bounce
// buffers filled by a host copy pool), the chunked validation scan, and the
// batched form on host memory. All repair and scan work runs on the GPU.

#include <cuda_runtime.h>
#include <immintrin.h>
#include <unistd.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/u16m.h"
#include "u16m_abi.h"
#include "u16m_internal.h"

using namespace u16m::abi;

namespace {

// ---- host staging pipeline -------------------------------------------------
// Three streams (H2D copy engine, compute, D2H copy engine) over a ring of
// device chunk buffers, ordered by events: chunk c's H2D waits only for the
// D2H that last used its buffer, so the host->device and device->host copy
// engines both stay busy (PCIe full duplex) while the kernel runs between
// them.
constexpr int kRing = 8;
constexpr size_t kChunkUnits = size_t(32) << 20;  // largest chunk: 64 MiB

bool pipe_chunk_override() {
  static const bool o = std::getenv("U16M_PIPE_CHUNK_KIB") != nullptr;
  return o;
}

// Pipeline chunk in units (U16M_PIPE_CHUNK_KIB overrides; at most kChunkUnits).
size_t pipe_chunk_units() {
  static const size_t c = [] {
    const char* e = std::getenv("U16M_PIPE_CHUNK_KIB");
    size_t kib = e ? static_cast<size_t>(std::atoll(e)) : 32768;
    size_t u = kib * 512;
    if (u < 4096) u = 4096;
    return u > kChunkUnits ? kChunkUnits : u;
  }();
  return c;
}

// Chunk of a plain / byte-order-fused host job over `units` units. Pinned
// buffers of 2 GiB and more stream in 64 MiB chunks: the DMA engines idle for
// the kernel + event latency between a chunk's H2D and its D2H, and with the
// two directions sharing ~96 GB/s every idle microsecond costs 0.4; fewer,
// larger chunks halve that (8 GiB: 48.1 -> 48.6 GB/s; 128 MiB the same, 256 MiB
// 47.7). Smaller jobs keep 32 MiB (512 MiB: 46.1 against 44.8 at 64 MiB — the
// unoverlapped first H2D and last D2H weigh more), pageable jobs too (their
// bounce buffers are pinned memory: 4 x chunk).
size_t job_chunk_units(size_t units, bool pinned) {
  if (pipe_chunk_override() || !pinned) return pipe_chunk_units();
  return units >= (size_t(1) << 30) ? kChunkUnits : pipe_chunk_units();
}

// Device ring slots hold the largest chunk a job may use.
size_t ring_slot_units() { return pipe_chunk_override() ? pipe_chunk_units() : kChunkUnits; }

constexpr int kStage = 4;  // pinned bounce buffers for pageable host jobs

struct HostPipe {
  int device = -1;
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  unsigned long long* counter = nullptr;  // device replacement counter (codec jobs)
  uint16_t* dbuf[kRing] = {};
  cudaEvent_t loaded[kRing] = {}, repaired[kRing] = {}, drained[kRing] = {};
  cudaEvent_t counted[kRing] = {};        // pinned in-place jobs: the chunk's counter snapshot has landed
  uint16_t* stage[kStage] = {};           // pinned, allocated on the first pageable job
  cudaEvent_t staged[kStage] = {};
  unsigned long long* stage_total = nullptr;  // pinned [kStage]: the counter after each staged chunk's kernel
  unsigned long long* ring_total = nullptr;   // pinned [kRing]: the same for pinned in-place jobs
  uint16_t* small = nullptr;              // pinned + mapped, small jobs (kSmallUnits), lazily
  unsigned long long* small_count = nullptr;  // pinned, the small path's count read-back
  unsigned long long* small_offs = nullptr;   // pinned, small scans' offsets read-back (kSmallOffs)
  unsigned long long* small_dev = nullptr;    // device, small scans' offsets + count
  std::mutex mu;                          // one job per device pipeline at a time
};

// Jobs up to this many units skip the copy-engine pipeline: the kernel reads
// and writes host memory directly over PCIe (pinned memory is mapped into the
// device's address space), so a call is one launch + one synchronisation
// instead of two DMAs, four events and three synchronisations.
constexpr size_t kSmallUnits = size_t(64) << 10;
constexpr size_t kSmallOffs = 4096;  // offsets read back with the count in one synchronisation

// Streaming (non-temporal) copy for the staging copies: the destination is
// written once and read next by a DMA engine or not at all, so bypassing the
// caches saves the read-for-ownership of every destination line.
__attribute__((target("avx512f"))) void copy_stream_avx512(char* dst, const char* src, size_t n) {
  size_t head = (64 - (reinterpret_cast<uintptr_t>(dst) & 63)) & 63;
  head = std::min(head, n);
  std::memcpy(dst, src, head);
  dst += head, src += head, n -= head;
  for (; n >= 256; n -= 256, dst += 256, src += 256) {
    const __m512i a = _mm512_loadu_si512(src), b = _mm512_loadu_si512(src + 64);
    const __m512i c = _mm512_loadu_si512(src + 128), d = _mm512_loadu_si512(src + 192);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(dst), a);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + 64), b);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + 128), c);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + 192), d);
  }
  std::memcpy(dst, src, n);
  _mm_sfence();  // streaming stores globally visible before the copy is reported done
}

void copy_piece(char* dst, const char* src, size_t n) {
  static const bool nt = [] {
    const char* e = std::getenv("U16M_HOST_NT");
    return __builtin_cpu_supports("avx512f") && !(e && std::strcmp(e, "0") == 0);
  }();
  if (nt) copy_stream_avx512(dst, src, n);
  else std::memcpy(dst, src, n);
}

// Parallel host memcpy for the pageable-memory staging of the host pipeline:
// the driver stages pageable copies through its own small bounce buffers on
// one thread (7 GB/s measured for a 512 MiB job), so large pageable jobs are
// copied into / out of pinned buffers by this pool instead. Worker threads
// live for the process (the pool is never destroyed: no join at exit).
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* pool = new CopyPool;
    return *pool;
  }
  void copy(void* dst, const void* src, size_t bytes) {
    if (bytes < (size_t(1) << 20)) {
      std::memcpy(dst, src, bytes);
      return;
    }
    std::lock_guard<std::mutex> job(job_mu_);  // device threads of a multi-GPU job share the pool
    if (getpid() != pid_) respawn();  // forked child: the workers did not survive the fork
    if (workers_ == 0) {
      std::memcpy(dst, src, bytes);
      return;
    }
    const size_t parts = static_cast<size_t>(workers_) + 1;
    {
      std::lock_guard<std::mutex> l(mu_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      bytes_ = bytes;
      piece_ = (bytes / parts + 4095) & ~size_t(4095);
      pending_ = workers_;
      ++gen_;
    }
    cv_.notify_all();
    piece(workers_);  // the caller copies the last piece
    std::unique_lock<std::mutex> l(mu_);
    done_.wait(l, [this] { return pending_ == 0; });
  }

 private:
  CopyPool() { respawn(); }
  void respawn() {
    pid_ = getpid();
    pending_ = 0;
    const char* e = std::getenv("U16M_HOST_THREADS");
    int t = e ? std::atoi(e) : static_cast<int>(std::thread::hardware_concurrency());
    t = std::max(1, std::min(t, 16));
    workers_ = t - 1;
    const unsigned long long g = gen_;
    for (int i = 0; i < workers_; i++) std::thread([this, i, g] { run(i, g); }).detach();
  }
  void piece(int i) {
    const size_t a = std::min(bytes_, static_cast<size_t>(i) * piece_);
    const size_t b = i == workers_ ? bytes_ : std::min(bytes_, a + piece_);
    if (b > a) copy_piece(dst_ + a, src_ + a, b - a);
  }
  void run(int i, unsigned long long seen) {
    for (;;) {
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return gen_ != seen; });
        seen = gen_;
      }
      piece(i);
      std::lock_guard<std::mutex> l(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_;
  int workers_ = 0, pending_ = 0;
  pid_t pid_ = 0;
  unsigned long long gen_ = 0;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0, piece_ = 0;
};

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

std::mutex g_pipes_mu;
std::vector<HostPipe*> g_pipes;  // one per device, created lazily, never freed

// The device's pipeline (created on first use on the calling thread, which
// must have made `device` current). Jobs lock HostPipe::mu.
HostPipe* pipe_for(int device, u16m_status* st) {
  std::lock_guard<std::mutex> lock(g_pipes_mu);
  for (HostPipe* p : g_pipes)
    if (p->device == device) return p;
  auto* p = new HostPipe;
  p->device = device;
  cudaError_t e = cudaStreamCreateWithFlags(&p->h2d, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->comp, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&p->counter, sizeof(unsigned long long));
  for (int i = 0; i < kRing && e == cudaSuccess; i++) {
    e = cudaEventCreateWithFlags(&p->loaded[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->repaired[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->drained[i], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    *st = cuda_fail(e, "host pipeline setup");
    for (int i = 0; i < kRing; i++) {  // release what was created (null handles are skipped)
      if (p->dbuf[i]) cudaFree(p->dbuf[i]);
      if (p->loaded[i]) cudaEventDestroy(p->loaded[i]);
      if (p->repaired[i]) cudaEventDestroy(p->repaired[i]);
      if (p->drained[i]) cudaEventDestroy(p->drained[i]);
    }
    if (p->counter) cudaFree(p->counter);
    if (p->h2d) cudaStreamDestroy(p->h2d);
    if (p->comp) cudaStreamDestroy(p->comp);
    if (p->d2h) cudaStreamDestroy(p->d2h);
    delete p;
    cudaGetLastError();
    return nullptr;
  }
  g_pipes.push_back(p);
  return p;
}

// Device ring slot k / pinned bounce buffer k, allocated on first use at the
// full chunk size (a one-chunk job never pays for the other slots: cudaHostAlloc
// of 32 MiB alone takes tens of ms).
cudaError_t ensure_dbuf(HostPipe* p, int k) {
  if (p->dbuf[k]) return cudaSuccess;
  return cudaMalloc(&p->dbuf[k], ring_slot_units() * sizeof(uint16_t));
}

cudaError_t ensure_stage(HostPipe* p, int k) {
  if (p->stage[k]) return cudaSuccess;
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&p->stage[k]), pipe_chunk_units() * sizeof(uint16_t),
                                cudaHostAllocDefault);
  if (e == cudaSuccess && !p->staged[k]) e = cudaEventCreateWithFlags(&p->staged[k], cudaEventDisableTiming);
  if (e != cudaSuccess && p->stage[k]) {
    cudaFreeHost(p->stage[k]);
    p->stage[k] = nullptr;
  }
  return e;
}

// Whole-buffer copies between host memory and a device buffer for the host
// entry points that need the data resident at once (batched). Pinned host
// memory is copied directly; pageable memory goes through two pinned bounce
// buffers, the CopyPool filling (draining) one while the copy engine moves
// the other. Synchronous.
cudaError_t h2d_staged(HostPipe* p, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  if (is_pinned(src)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, p->h2d) == cudaSuccess
                                 ? cudaStreamSynchronize(p->h2d) : cudaGetLastError();
  const size_t cb = pipe_chunk_units() * sizeof(uint16_t);
  cudaError_t e = cudaSuccess;
  size_t i = 0;
  for (size_t off = 0; off < bytes && e == cudaSuccess; off += cb, i++) {
    const int k = static_cast<int>(i % 2);
    const size_t len = std::min(cb, bytes - off);
    e = ensure_stage(p, k);
    if (e == cudaSuccess && i >= 2) e = cudaEventSynchronize(p->staged[k]);  // its previous DMA is done
    if (e != cudaSuccess) break;
    CopyPool::get().copy(p->stage[k], static_cast<const char*>(src) + off, len);
    e = cudaMemcpyAsync(static_cast<char*>(dst) + off, p->stage[k], len, cudaMemcpyHostToDevice, p->h2d);
    if (e == cudaSuccess) e = cudaEventRecord(p->staged[k], p->h2d);
  }
  const cudaError_t f = cudaStreamSynchronize(p->h2d);
  return e != cudaSuccess ? e : f;
}

cudaError_t d2h_staged(HostPipe* p, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  if (is_pinned(dst)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, p->d2h) == cudaSuccess
                                 ? cudaStreamSynchronize(p->d2h) : cudaGetLastError();
  const size_t cb = pipe_chunk_units() * sizeof(uint16_t);
  const size_t nchunks = (bytes + cb - 1) / cb;
  cudaError_t e = cudaSuccess;
  auto issue = [&](size_t i) {  // DMA chunk i into bounce buffer i % 2
    const int k = static_cast<int>(i % 2);
    const size_t off = i * cb, len = std::min(cb, bytes - off);
    cudaError_t r = ensure_stage(p, k);
    if (r == cudaSuccess)
      r = cudaMemcpyAsync(p->stage[k], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, p->d2h);
    if (r == cudaSuccess) r = cudaEventRecord(p->staged[k], p->d2h);
    return r;
  };
  e = issue(0);
  for (size_t i = 0; i < nchunks && e == cudaSuccess; i++) {
    const int k = static_cast<int>(i % 2);
    if (i + 1 < nchunks) e = issue(i + 1);  // the other buffer was drained in the previous iteration
    if (e == cudaSuccess) e = cudaEventSynchronize(p->staged[k]);
    if (e != cudaSuccess) break;
    const size_t off = i * cb, len = std::min(cb, bytes - off);
    CopyPool::get().copy(static_cast<char*>(dst) + off, p->stage[k], len);
  }
  const cudaError_t f = cudaStreamSynchronize(p->d2h);
  return e != cudaSuccess ? e : f;
}

// Host jobs run the staged copy-engine pipeline: H2D copy -> repair kernel ->
// D2H copy on 3 streams over a ring of device chunks. Measured on the B200
// box and dropped (round 1, scripts/e2e_probe.py, 512 MiB in place / copy,
// input GB/s; full-duplex PCIe tops out at 46-50 each way): the kernel
// storing only rewritten 32-byte groups straight into mapped host memory
// (36.0 / -), and the kernel reading and writing mapped host buffers directly
// (36.4 / 38.5) — small posted PCIe writes from SMs cost more than a
// full-duplex DMA copy. Also dropped: write-back at 64-512-byte groups
// (36.7-40.8), chunks of 4-64 MiB (34-40 in place; ~20 us fixed cost per
// chunk), a geometric ramp of the end chunks (no change).

// Pinned in-place jobs whose kernels add their rewrites to p->counter: the
// device-to-host copy of a chunk WITHOUT rewrites is skipped (the caller's
// buffer already holds it), so clean text moves at the one-way H2D rate
// instead of the full-duplex rate. Whether chunk j is clean is known only
// after its kernel: the running counter is copied to pinned memory after
// every kernel, and chunk j's D2H is decided one iteration later (chunk j+1's
// H2D is queued first, so the H2D engine never waits for the host). Checking
// costs a host wake-up per chunk, so after a dirty chunk the next 7 (then 15,
// 31, 63 while checks keep finding rewrites) are copied back unchecked; on
// error-dense data the sequence of DMAs is the one of the plain pipeline
// (8 GiB of config 4 in place: 48.1 -> 47.9 GB/s; clean text 46 -> 55 GB/s).
template <class Compute>
u16m_status pipeline_pinned_inplace(HostPipe* p, uint16_t* buf, const std::vector<std::pair<size_t, size_t>>& chunks,
                                    Compute compute) {
  cudaError_t e = cudaSuccess;
  if (p->ring_total == nullptr) {
    e = cudaHostAlloc(reinterpret_cast<void**>(&p->ring_total), kRing * sizeof(unsigned long long),
                      cudaHostAllocMapped);
    if (e != cudaSuccess) return cuda_fail(e, "pipeline counters");
  }
  void* ring_total_dev = nullptr;  // the device's view of ring_total
  e = cudaHostGetDevicePointer(&ring_total_dev, p->ring_total, 0);
  for (int i = 0; i < kRing && e == cudaSuccess; i++)
    if (!p->counted[i]) e = cudaEventCreateWithFlags(&p->counted[i], cudaEventDisableTiming);
  if (e != cudaSuccess) return cuda_fail(e, "pipeline counters");
  bool d2h_issued[kRing] = {};
  bool checking = true;
  int unchecked_left = 0, backoff = 7;
  auto decide = [&](size_t j) -> cudaError_t {
    const int k = static_cast<int>(j % kRing);
    bool dirty = true;
    if (checking) {
      const cudaError_t r = cudaEventSynchronize(p->counted[k]);  // chunk j's kernel ran and its count has landed
      if (r != cudaSuccess) return r;
      const unsigned long long before = j ? p->ring_total[(j - 1) % kRing] : 0ull;
      dirty = p->ring_total[k] != before;
      if (dirty) {  // copy the next chunks back unchecked: 7, then 15, 31, 63 while checks keep finding rewrites
        checking = false;
        unchecked_left = backoff;
        backoff = std::min(2 * backoff + 1, 63);
      } else {
        backoff = 7;
      }
    } else if (--unchecked_left == 0) {
      checking = true;
    }
    d2h_issued[k] = dirty;
    if (!dirty) return cudaSuccess;
    cudaStreamWaitEvent(p->d2h, p->repaired[k], 0);
    const cudaError_t r =
        cudaMemcpyAsync(buf + chunks[j].first, p->dbuf[k], chunks[j].second * 2, cudaMemcpyDeviceToHost, p->d2h);
    if (r != cudaSuccess) return r;
    return cudaEventRecord(p->drained[k], p->d2h);
  };
  for (size_t c = 0; c < chunks.size(); c++) {
    const size_t c0 = chunks[c].first, len = chunks[c].second;
    const int k = static_cast<int>(c % kRing);
    if (c >= static_cast<size_t>(kRing)) {  // the slot's last user (chunk c - kRing, decided long ago) is finished
      e = cudaStreamWaitEvent(p->h2d, d2h_issued[k] ? p->drained[k] : p->repaired[k], 0);
      if (e != cudaSuccess) return cuda_fail(e, "pipeline wait");
    }
    e = ensure_dbuf(p, k);
    if (e != cudaSuccess) return cuda_fail(e, "device chunk buffer");
    e = cudaMemcpyAsync(p->dbuf[k], buf + c0, len * 2, cudaMemcpyHostToDevice, p->h2d);
    if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
    cudaEventRecord(p->loaded[k], p->h2d);
    cudaStreamWaitEvent(p->comp, p->loaded[k], 0);
    e = compute(p->dbuf[k], c0, len);
    if (e != cudaSuccess) return cuda_fail(e, "repair kernel launch");
    // The D2H copy waits for the kernel alone: the counter snapshot (a store
    // into host memory, slow to retire while the link is saturated) runs beside
    // it — behind `repaired` it delayed every D2H by ~25 us, 1.8 % of the job.
    cudaEventRecord(p->repaired[k], p->comp);
    e = u16m::launch_store_u64(static_cast<unsigned long long*>(ring_total_dev) + k, p->counter, p->comp);
    if (e != cudaSuccess) return cuda_fail(e, "chunk rewrite count");
    cudaEventRecord(p->counted[k], p->comp);
    if (c >= 1) {
      e = decide(c - 1);
      if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
    }
  }
  if (!chunks.empty()) {
    e = decide(chunks.size() - 1);
    if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
  }
  e = cudaStreamSynchronize(p->d2h);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->comp);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->h2d);
  if (e != cudaSuccess) return cuda_fail(e, "host pipeline sync");
  return U16M_OK;
}

// The staged copy-engine pipeline over a list of unit ranges of the caller's
// buffers: per chunk H2D -> compute(dbuf, c0, len) on p->comp -> D2H. The
// chunks may have any lengths up to ring_slot_units() (pageable buffers: up to
// pipe_chunk_units(), the size of the bounce buffers). The calling thread
// must have made p->device current and hold p->mu.
// track_clean (pageable in-place jobs whose kernels add their rewrites to
// p->counter, reset by the caller): a chunk without rewrites is not copied
// back — `out` is `in` and already holds it — which halves the host copy
// work, the limit of pageable jobs, on clean text.
template <class Compute>
u16m_status pipeline_chunks(HostPipe* p, const uint16_t* in, uint16_t* out,
                            const std::vector<std::pair<size_t, size_t>>& chunks, Compute compute,
                            bool track_clean = false) {
  cudaError_t e = cudaSuccess;
  // Pageable host memory: the copy engines cannot DMA it directly, so every
  // chunk is copied (by the CopyPool threads) into a pinned bounce buffer,
  // moved H2D, repaired, moved D2H back into the same bounce buffer and
  // copied out. The host copies of chunk c+1 (in) and c+1-kStage (out)
  // overlap the GPU work of chunk c. This replaces the driver's own
  // single-threaded staging of pageable copies (7 GB/s on a 512 MiB job).
  if (!is_pinned(in) || !is_pinned(out)) {
    CopyPool& pool = CopyPool::get();
    const size_t nchunks = chunks.size();
    const bool skip_clean = track_clean && in == out;
    if (skip_clean && p->stage_total == nullptr) {
      e = cudaHostAlloc(reinterpret_cast<void**>(&p->stage_total), kStage * sizeof(unsigned long long),
                        cudaHostAllocMapped);
      if (e != cudaSuccess) return cuda_fail(e, "staging buffers");
    }
    void* stage_total_dev = nullptr;  // the device's view of stage_total
    if (skip_clean) {
      e = cudaHostGetDevicePointer(&stage_total_dev, p->stage_total, 0);
      if (e != cudaSuccess) return cuda_fail(e, "staging buffers");
    }
    unsigned long long seen_total = 0;  // p->counter after the last chunk copied out (chunks drain in order)
    auto copy_out = [&](size_t c) -> cudaError_t {
      const int k = static_cast<int>(c % kStage);
      const cudaError_t r = cudaEventSynchronize(p->staged[k]);
      if (r != cudaSuccess) return r;
      if (skip_clean) {
        const unsigned long long total = p->stage_total[k];
        const bool clean = total == seen_total;
        seen_total = total;
        if (clean) return cudaSuccess;  // nothing was rewritten: the caller's buffer already holds this chunk
      }
      pool.copy(out + chunks[c].first, p->stage[k], chunks[c].second * sizeof(uint16_t));
      return cudaSuccess;
    };
    for (size_t c = 0; c < nchunks; c++) {
      const int k = static_cast<int>(c % kStage);  // bounce buffer and device buffer slot
      if (c >= static_cast<size_t>(kStage)) {
        e = copy_out(c - kStage);  // frees slot k (its D2H is complete)
        if (e != cudaSuccess) return cuda_fail(e, "staged D2H");
      }
      e = ensure_stage(p, k);
      if (e == cudaSuccess) e = ensure_dbuf(p, k);
      if (e != cudaSuccess) return cuda_fail(e, "staging buffers");
      const size_t c0 = chunks[c].first, len = chunks[c].second;
      pool.copy(p->stage[k], in + c0, len * sizeof(uint16_t));
      e = cudaMemcpyAsync(p->dbuf[k], p->stage[k], len * 2, cudaMemcpyHostToDevice, p->h2d);
      if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
      cudaEventRecord(p->loaded[k], p->h2d);
      cudaStreamWaitEvent(p->comp, p->loaded[k], 0);
      e = compute(p->dbuf[k], c0, len);
      if (e != cudaSuccess) return cuda_fail(e, "repair kernel launch");
      if (skip_clean) {  // the running rewrite count after this chunk (complete before staged[k])
        e = u16m::launch_store_u64(static_cast<unsigned long long*>(stage_total_dev) + k, p->counter, p->comp);
        if (e != cudaSuccess) return cuda_fail(e, "chunk rewrite count");
      }
      cudaEventRecord(p->repaired[k], p->comp);
      cudaStreamWaitEvent(p->d2h, p->repaired[k], 0);
      e = cudaMemcpyAsync(p->stage[k], p->dbuf[k], len * 2, cudaMemcpyDeviceToHost, p->d2h);
      if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
      cudaEventRecord(p->staged[k], p->d2h);
    }
    for (size_t c = nchunks > static_cast<size_t>(kStage) ? nchunks - kStage : 0; c < nchunks; c++) {
      e = copy_out(c);
      if (e != cudaSuccess) return cuda_fail(e, "staged D2H");
    }
    e = cudaStreamSynchronize(p->comp);
    if (e != cudaSuccess) return cuda_fail(e, "host pipeline sync");
    return U16M_OK;
  }
  if (track_clean && in == out) return pipeline_pinned_inplace(p, out, chunks, compute);
  // Pinned: every chunk is DMA'd straight between the caller's buffer and a
  // device ring slot; chunk c's H2D waits only for the D2H that last used its
  // slot, so both copy engines stay busy while the kernel runs between them.
  for (size_t c = 0; c < chunks.size(); c++) {
    const size_t c0 = chunks[c].first, len = chunks[c].second;
    const int k = static_cast<int>(c % kRing);
    if (c >= static_cast<size_t>(kRing)) {
      e = cudaStreamWaitEvent(p->h2d, p->drained[k], 0);
      if (e != cudaSuccess) return cuda_fail(e, "pipeline wait");
    }
    e = ensure_dbuf(p, k);
    if (e != cudaSuccess) return cuda_fail(e, "device chunk buffer");
    e = cudaMemcpyAsync(p->dbuf[k], in + c0, len * 2, cudaMemcpyHostToDevice, p->h2d);
    if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
    cudaEventRecord(p->loaded[k], p->h2d);
    cudaStreamWaitEvent(p->comp, p->loaded[k], 0);
    e = compute(p->dbuf[k], c0, len);
    if (e != cudaSuccess) return cuda_fail(e, "repair kernel launch");
    cudaEventRecord(p->repaired[k], p->comp);
    cudaStreamWaitEvent(p->d2h, p->repaired[k], 0);
    e = cudaMemcpyAsync(out + c0, p->dbuf[k], len * 2, cudaMemcpyDeviceToHost, p->d2h);
    if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
    cudaEventRecord(p->drained[k], p->d2h);
  }
  e = cudaStreamSynchronize(p->d2h);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->comp);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->h2d);
  if (e != cudaSuccess) return cuda_fail(e, "host pipeline sync");
  return U16M_OK;
}

// One host job's share on one device: units [a, b) of the caller's buffers
// (`in`/`out` hold n units), halo units read from the caller's input at
// a-1 and b (-1 at the buffer's ends), in fixed-size chunks. Device
// replacement counts (codec jobs) accumulate in p->counter, which the caller
// reset.
u16m_status host_range(HostPipe* p, const uint16_t* in, size_t n, uint16_t* out, size_t a, size_t b,
                       int byte_order, bool count) {
  const bool be = byte_order == U16M_BIG_ENDIAN;
  auto unit = [&](size_t i) -> int32_t {  // unit value of in[i] in the job's byte order
    const uint32_t w = in[i];
    return static_cast<int32_t>(be ? (((w & 0xFFu) << 8) | (w >> 8)) : w);
  };
  auto repair = [&](uint16_t* d, size_t c0, size_t len) {
    // Halo units come from the caller's input at enqueue time. In place, a
    // neighbouring chunk (or another device's range) may already have been
    // written back; a rewritten neighbour is benign (a unit is only rewritten
    // when no neighbour pairs with it).
    const int32_t left = c0 > 0 ? unit(c0 - 1) : -1;
    const int32_t right = c0 + len < n ? unit(c0 + len) : -1;
    if (byte_order < 0 && !count)
      return u16m::launch_repair(d, len, d, left, right, nullptr, nullptr, p->comp);
    return u16m::launch_fix_bytes(d, len, d, be, count ? p->counter : nullptr, p->comp, left, right);
  };
  const size_t chunk = job_chunk_units(b - a, is_pinned(in) && is_pinned(out));
  std::vector<std::pair<size_t, size_t>> chunks;
  chunks.reserve((b - a + chunk - 1) / chunk);
  // (a ramp of smaller chunks at the head and tail — the only transfers nothing
  // overlaps — measured +0.1 %, within noise: profiles/r02/ab_host_chunk_size.txt)
  for (size_t c0 = a; c0 < b; c0 += chunk) chunks.emplace_back(c0, std::min(chunk, b - c0));
  return pipeline_chunks(p, in, out, chunks, repair, /*track_clean=*/count);
}

// Device-accessible address of pinned (page-locked, mapped) host memory, or
// nullptr for pageable memory.
void* mapped_view(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// A whole small job (n <= kSmallUnits) on one device: the repair kernel runs
// on the caller's pinned buffers through their mapped addresses, or — for
// pageable buffers — on the device's small pinned buffer after one host
// memcpy. Zero-copy PCIe traffic is fine at this size; what the call costs
// is API latency, and this path has one launch and one synchronisation.
// The small-job buffers of a device pipeline, allocated on first use.
cudaError_t ensure_small(HostPipe* p) {
  if (p->small) return cudaSuccess;
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&p->small), kSmallUnits * sizeof(uint16_t) + 64,
                                cudaHostAllocMapped);
  if (e == cudaSuccess)
    e = cudaHostAlloc(reinterpret_cast<void**>(&p->small_count), sizeof(unsigned long long), cudaHostAllocMapped);
  if (e == cudaSuccess)
    e = cudaHostAlloc(reinterpret_cast<void**>(&p->small_offs), kSmallOffs * sizeof(unsigned long long),
                      cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaMalloc(&p->small_dev, (kSmallUnits + 8) * sizeof(unsigned long long));
  if (e != cudaSuccess) {
    if (p->small) cudaFreeHost(p->small);
    if (p->small_count) cudaFreeHost(p->small_count);
    if (p->small_offs) cudaFreeHost(p->small_offs);
    p->small = nullptr;
    p->small_count = p->small_offs = nullptr;
    cudaGetLastError();
  }
  return e;
}

u16m_status host_small(HostPipe* p, const uint16_t* in, size_t n, uint16_t* out, int byte_order,
                       unsigned long long* replacements) {
  cudaError_t e = ensure_small(p);
  if (e != cudaSuccess) return cuda_fail(e, "small-job buffers");
  const uint16_t* din = static_cast<const uint16_t*>(mapped_view(in));
  uint16_t* dout = in == out ? const_cast<uint16_t*>(din) : static_cast<uint16_t*>(mapped_view(out));
  const bool direct = din != nullptr && dout != nullptr;
  if (!direct) {
    std::memcpy(p->small, in, n * sizeof(uint16_t));
    void* d = nullptr;
    e = cudaHostGetDevicePointer(&d, p->small, 0);
    if (e != cudaSuccess) return cuda_fail(e, "small-job buffer mapping");
    din = dout = static_cast<uint16_t*>(d);
  }
  const bool be = byte_order == U16M_BIG_ENDIAN;
  if (byte_order < 0) {
    e = u16m::launch_repair(din, n, dout, -1, -1, nullptr, nullptr, p->comp);
  } else {
    if (replacements) e = cudaMemsetAsync(p->counter, 0, sizeof(unsigned long long), p->comp);
    if (e == cudaSuccess)
      e = u16m::launch_fix_bytes(din, n, dout, be, replacements ? p->counter : nullptr, p->comp, -1, -1);
    if (e == cudaSuccess && replacements)
      e = cudaMemcpyAsync(p->small_count, p->counter, sizeof(unsigned long long), cudaMemcpyDeviceToHost, p->comp);
  }
  if (e != cudaSuccess) return cuda_fail(e, "small-job repair");
  e = cudaStreamSynchronize(p->comp);
  if (e != cudaSuccess) return cuda_fail(e, "small-job sync");
  if (!direct) std::memcpy(out, p->small, n * sizeof(uint16_t));
  if (replacements) *replacements = *p->small_count;
  return U16M_OK;
}

u16m_status host_device_job(int dev, const uint16_t* in, size_t n, uint16_t* out, size_t a, size_t b,
                            int byte_order, unsigned long long* replacements) {
  cudaError_t e = cudaSetDevice(dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  u16m_status st = U16M_OK;
  HostPipe* p = pipe_for(dev, &st);
  if (p == nullptr) return st;
  std::lock_guard<std::mutex> lock(p->mu);  // one staged job per device at a time
  if (a == 0 && b == n && n <= kSmallUnits) return host_small(p, in, n, out, byte_order, replacements);
  // In-place jobs count their rewrites even when the caller does not ask for
  // the count: chunks without any are not copied back (pipeline_chunks).
  const bool count = replacements != nullptr || in == out;
  if (count) {
    e = cudaMemsetAsync(p->counter, 0, sizeof(unsigned long long), p->comp);
    if (e != cudaSuccess) return cuda_fail(e, "counter reset");
  }
  st = host_range(p, in, n, out, a, b, byte_order, count);
  if (st == U16M_OK && replacements) {
    e = cudaMemcpy(replacements, p->counter, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "replacement count");
  }
  return st;
}

// Smallest share worth a device of its own (a 64 MiB share is ~1.4 ms of
// PCIe time; below that a thread + device switch costs more than it saves).
constexpr size_t kMinUnitsPerDevice = size_t(32) << 20;

// Shared body of the host-memory entry points. byte_order < 0: plain repair
// (units in host order); 0/1: codec-fused repair in LE/BE byte order with an
// optional replacement count (host pointer). `devs`: the devices to spread
// the job over in contiguous ranges (one host thread per extra device), or
// nullptr = the calling thread's current device.
u16m_status host_pipeline(const uint16_t* in, size_t n, uint16_t* out, int byte_order,
                          unsigned long long* replacements, const std::vector<int>* devs = nullptr) {
  U16M_TRY(check_pair(in, n, out));
  if (replacements) *replacements = 0;
  if (n == 0) return U16M_OK;
  U16M_TRY(check_device_present());
  int cur = 0;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  std::vector<int> use = devs ? *devs : std::vector<int>{cur};
  const size_t g = std::max<size_t>(1, std::min(use.size(), n / kMinUnitsPerDevice));
  use.resize(g);
  if (g == 1) {
    u16m_status st = host_device_job(use[0], in, n, out, 0, n, byte_order, replacements);
    cudaSetDevice(cur);
    return st;
  }
  // Contiguous ranges, 4096-unit aligned: each device streams its own range
  // over its own PCIe link. Ranges meet only through the halo units, read
  // from the caller's input (benign in place, see host_range).
  std::vector<size_t> bounds(g + 1);
  for (size_t k = 0; k <= g; k++) bounds[k] = k == g ? n : (n / g * k) & ~size_t(4095);
  std::vector<u16m_status> sts(g, U16M_OK);
  std::vector<unsigned long long> counts(g, 0);
  std::vector<std::string> errs(g);
  std::vector<std::thread> pool;
  for (size_t k = 1; k < g; k++)
    pool.emplace_back([&, k] {
      sts[k] = host_device_job(use[k], in, n, out, bounds[k], bounds[k + 1], byte_order,
                               replacements ? &counts[k] : nullptr);
      if (sts[k] != U16M_OK) errs[k] = u16m_last_error();
    });
  sts[0] = host_device_job(use[0], in, n, out, bounds[0], bounds[1], byte_order, replacements ? &counts[0] : nullptr);
  if (sts[0] != U16M_OK) errs[0] = u16m_last_error();
  for (auto& t : pool) t.join();
  cudaSetDevice(cur);
  for (size_t k = 0; k < g; k++)
    if (sts[k] != U16M_OK) return fail(sts[k], "device " + std::to_string(use[k]) + ": " + errs[k]);
  if (replacements)
    for (unsigned long long c : counts) *replacements += c;
  return U16M_OK;
}

u16m_status device_list(int num_devices, const int* device_ids, std::vector<int>* out) {
  int visible = 0;
  if (cudaGetDeviceCount(&visible) != cudaSuccess || visible == 0) {
    cudaGetLastError();
    return fail(U16M_ERR_NO_DEVICE, "no CUDA device visible (u16m has no CPU fallback)");
  }
  if (num_devices < 0) return fail(U16M_ERR_INVALID_ARGUMENT, "num_devices < 0");
  if (num_devices == 0) {
    for (int d = 0; d < visible; d++) out->push_back(d);
    return U16M_OK;
  }
  if (device_ids == nullptr) return fail(U16M_ERR_INVALID_ARGUMENT, "device_ids is null with num_devices > 0");
  for (int k = 0; k < num_devices; k++) {
    if (device_ids[k] < 0 || device_ids[k] >= visible)
      return fail(U16M_ERR_INVALID_ARGUMENT, "device id " + std::to_string(device_ids[k]) + " is not visible");
    out->push_back(device_ids[k]);
  }
  return U16M_OK;
}

}  // namespace

extern "C" {

u16m_status u16m_to_well_formed_host(const uint16_t* in, size_t n, uint16_t* out) {
  return host_pipeline(in, n, out, -1, nullptr);
}

u16m_status u16m_to_well_formed_host_multi(const uint16_t* in, size_t n, uint16_t* out, int num_devices,
                                           const int* device_ids) {
  U16M_TRY(check_pair(in, n, out));
  if (n == 0) return U16M_OK;
  std::vector<int> devs;
  U16M_TRY(device_list(num_devices, device_ids, &devs));
  return host_pipeline(in, n, out, -1, nullptr, &devs);
}

u16m_status u16m_fix_utf16_bytes_host_multi(const void* in, size_t n_units, void* out, int byte_order,
                                            unsigned long long* replacements, int num_devices,
                                            const int* device_ids) {
  if (byte_order != U16M_LITTLE_ENDIAN && byte_order != U16M_BIG_ENDIAN)
    return fail(U16M_ERR_INVALID_ARGUMENT, "byte_order must be U16M_LITTLE_ENDIAN or U16M_BIG_ENDIAN");
  const auto* i = static_cast<const uint16_t*>(in);
  auto* o = static_cast<uint16_t*>(out);
  U16M_TRY(check_pair(i, n_units, o));
  if (replacements) *replacements = 0;
  if (n_units == 0) return U16M_OK;
  std::vector<int> devs;
  U16M_TRY(device_list(num_devices, device_ids, &devs));
  return host_pipeline(i, n_units, o, byte_order, replacements, &devs);
}

u16m_status u16m_fix_utf16_bytes_host(const void* in, size_t n_units, void* out, int byte_order,
                                      unsigned long long* replacements) {
  // every visible GPU, each over its own PCIe link (one for jobs under 64 Mi units)
  return u16m_fix_utf16_bytes_host_multi(in, n_units, out, byte_order, replacements, 0, nullptr);
}

u16m_status u16m_to_well_formed_batched_host(const uint16_t* in, size_t n_units, const int64_t* offsets,
                                             size_t num_strings, uint16_t* out) {
  if (offsets == nullptr) return fail(U16M_ERR_INVALID_ARGUMENT, "offsets is null");
  U16M_TRY(check_pair(in, n_units, out));
  if (num_strings == 0 || n_units == 0) {
    if (out != in && n_units) std::memcpy(out, in, n_units * sizeof(uint16_t));
    return U16M_OK;
  }
  for (size_t s = 0; s < num_strings; s++)
    if (offsets[s] < 0 || offsets[s + 1] < offsets[s] || static_cast<size_t>(offsets[s + 1]) > n_units)
      return fail(U16M_ERR_INVALID_ARGUMENT, "offsets must be non-decreasing within the buffer");
  U16M_TRY(check_device_present());
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  u16m_status st = U16M_OK;
  HostPipe* p = pipe_for(dev, &st);
  if (p == nullptr) return st;
  std::lock_guard<std::mutex> lock(p->mu);
  u16m::keep_pool_memory();
  // The buffer streams through the copy-engine pipeline in fixed chunks, like
  // a plain host job; the offsets array goes H2D once. Per chunk [c0, c1):
  // the strings lying wholly inside run the batched tile kernel (addressed
  // with the absolute offsets), and a string cut by the chunk's start and/or
  // end is repaired on its in-chunk segment by the plain kernel with the real
  // neighbour unit (read from the caller's input) as the halo on the cut side
  // and "outside" on the string's own end — so strings of any length, even
  // longer than a chunk, and buffers larger than device memory stream
  // through. Units in no string pass through unchanged.
  const size_t S = num_strings;
  const size_t off_bytes = (S + 1) * sizeof(int64_t);
  int64_t* d_off = nullptr;
  e = cudaMallocAsync(reinterpret_cast<void**>(&d_off), off_bytes, p->comp);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->comp);
  if (e != cudaSuccess) return cuda_fail(e, "device offsets");
  e = h2d_staged(p, d_off, offsets, off_bytes);
  if (e != cudaSuccess) {
    cudaFreeAsync(d_off, p->comp);
    return cuda_fail(e, "offsets H2D");
  }
  const int64_t* o_end = offsets + S + 1;
  auto repair = [&](uint16_t* d, size_t c0, size_t len) -> cudaError_t {
    const size_t c1 = c0 + len;
    const int64_t a = static_cast<int64_t>(c0), b = static_cast<int64_t>(c1);
    // lo: first boundary >= c0; hi: first boundary > c1
    const size_t lo = static_cast<size_t>(std::lower_bound(offsets, o_end, a) - offsets);
    const size_t hi = static_cast<size_t>(std::upper_bound(offsets, o_end, b) - offsets);
    auto plain = [&](size_t u0, size_t u1, int32_t left, int32_t right) -> cudaError_t {
      if (u1 <= u0) return cudaSuccess;
      uint16_t* q = d + (u0 - c0);
      return u16m::launch_repair(q, u1 - u0, q, left, right, nullptr, nullptr, p->comp);
    };
    cudaError_t r = cudaSuccess;
    // a string that started before c0 and is still running at c0
    const bool head_cut = lo >= 1 && lo <= S && offsets[lo] > a;
    if (head_cut) {
      const size_t e0 = static_cast<size_t>(offsets[lo]);
      if (e0 > c1)  // the whole chunk is inside one string
        return plain(c0, c1, in[c0 - 1], in[c1]);
      r = plain(c0, e0, in[c0 - 1], -1);
      if (r != cudaSuccess) return r;
    }
    // strings wholly inside: [lo, hi - 1)
    if (hi >= 1 && hi - 1 > lo) {
      const size_t sa = lo, sb = hi - 1;
      r = u16m::launch_batched_tiles(d - c0, c1, d_off + sa, sb - sa, d - c0, p->comp, len);
      if (r != cudaSuccess) return r;
    }
    // a string that starts inside the chunk and runs past c1
    if (hi >= 1 && hi <= S && offsets[hi - 1] < b && offsets[hi - 1] >= a)
      r = plain(static_cast<size_t>(offsets[hi - 1]), c1, -1, in[c1]);
    return r;
  };
  const size_t chunk = pipe_chunk_units();
  std::vector<std::pair<size_t, size_t>> chunks;
  chunks.reserve((n_units + chunk - 1) / chunk);
  for (size_t c0 = 0; c0 < n_units; c0 += chunk) chunks.emplace_back(c0, std::min(chunk, n_units - c0));
  st = pipeline_chunks(p, in, out, chunks, repair);
  cudaFreeAsync(d_off, p->comp);
  cudaStreamSynchronize(p->comp);
  return st;
}

}  // extern "C"

namespace {

// Chunked host validation scan; byte_order < 0: units in host order, else the
// bytes' order (big-endian chunks are byte-swapped on the device after their
// H2D copy).
u16m_status unpaired_offsets_host(const uint16_t* in, size_t n, int byte_order, size_t limit,
                                  unsigned long long* offsets_out, size_t* count_out) {
  if (count_out == nullptr || (limit > 0 && offsets_out == nullptr))
    return fail(U16M_ERR_INVALID_ARGUMENT, "null output");
  *count_out = 0;
  if (n == 0 || limit == 0) return U16M_OK;
  if (in == nullptr) return fail(U16M_ERR_INVALID_ARGUMENT, "null buffer with n > 0");
  if (reinterpret_cast<uintptr_t>(in) & 1u) return fail(U16M_ERR_MISALIGNED, "in not 2-byte aligned");
  U16M_TRY(check_device_present());
  if (limit > n) limit = n;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  u16m_status st = U16M_OK;
  HostPipe* p = pipe_for(dev, &st);
  if (p == nullptr) return st;
  std::lock_guard<std::mutex> lock(p->mu);
  if (n <= kSmallUnits) {
    // Small buffer: the scan kernels read host memory directly (mapped pinned
    // memory: the caller's, or the small buffer after one memcpy — also for
    // big-endian bytes, swapped there on the device); count and offsets come
    // back with one synchronisation when limit <= kSmallOffs.
    e = ensure_small(p);
    if (e != cudaSuccess) return cuda_fail(e, "small-job buffers");
    const bool be_small = byte_order == U16M_BIG_ENDIAN;
    const uint16_t* din = be_small ? nullptr : static_cast<const uint16_t*>(mapped_view(in));
    if (din == nullptr) {
      std::memcpy(p->small, in, n * sizeof(uint16_t));
      void* d = nullptr;
      e = cudaHostGetDevicePointer(&d, p->small, 0);
      if (e == cudaSuccess && be_small) e = u16m::launch_byteswap(static_cast<uint16_t*>(d), n, p->comp);
      if (e != cudaSuccess) return cuda_fail(e, "small scan staging");
      din = static_cast<const uint16_t*>(d);
    }
    // limit <= kSmallOffs (is_well_formed asks for 1, the CLI for 10): the scan
    // kernel writes the count and the offsets straight into mapped pinned host
    // memory — one launch and one synchronisation, no device-to-host copies.
    const bool one_sync = limit <= kSmallOffs;
    unsigned long long* d_off = p->small_dev;
    unsigned long long* d_cnt = p->small_dev + kSmallUnits;
    if (one_sync) {
      void *mo = nullptr, *mc = nullptr;
      e = cudaHostGetDevicePointer(&mo, p->small_offs, 0);
      if (e == cudaSuccess) e = cudaHostGetDevicePointer(&mc, p->small_count, 0);
      if (e != cudaSuccess) return cuda_fail(e, "small scan output mapping");
      d_off = static_cast<unsigned long long*>(mo);
      d_cnt = static_cast<unsigned long long*>(mc);
    }
    e = u16m::launch_unpaired_offsets(din, n, limit, d_off, d_cnt, p->comp, -1, -1);
    if (e == cudaSuccess && !one_sync)
      e = cudaMemcpyAsync(p->small_count, d_cnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, p->comp);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->comp);
    if (e != cudaSuccess) return cuda_fail(e, "small scan");
    const size_t cnt = static_cast<size_t>(*p->small_count);
    if (one_sync) {
      std::memcpy(offsets_out, p->small_offs, cnt * sizeof(unsigned long long));
    } else if (cnt) {
      e = cudaMemcpy(offsets_out, d_off, cnt * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return cuda_fail(e, "small scan offsets");
    }
    *count_out = cnt;
    return U16M_OK;
  }
  // Chunked, read-only scan: chunk c+1 moves H2D (straight from pinned memory,
  // or through a pinned bounce buffer filled by the CopyPool) while chunk c
  // is scanned with its neighbours' units as halos; the scan stops at the
  // first chunk that completes `limit` offsets (the CLI check asks for 10,
  // is_well_formed for 1), so an ill-formed buffer is rarely read to its end.
  const bool pinned = is_pinned(in);
  const size_t chunk = pipe_chunk_units();
  const bool be = byte_order == U16M_BIG_ENDIAN;
  auto unit = [&](size_t i) -> int32_t {
    const uint32_t w = in[i];
    return static_cast<int32_t>(be ? (((w & 0xFFu) << 8) | (w >> 8)) : w);
  };

  const size_t cap = std::min(limit, chunk);
  void* ws = nullptr;
  u16m::keep_pool_memory();
  e = cudaMallocAsync(&ws, cap * sizeof(unsigned long long) + 64, p->comp);
  if (e != cudaSuccess) return cuda_fail(e, "workspace");
  auto* d_off = static_cast<unsigned long long*>(ws);
  auto* d_cnt = d_off + cap;
  const size_t nchunks = (n + chunk - 1) / chunk;
  auto load = [&](size_t c) -> cudaError_t {  // H2D of chunk c into device slot c % 2
    const int k = static_cast<int>(c % 2);
    cudaError_t r = ensure_dbuf(p, k);
    if (r == cudaSuccess && !pinned) r = ensure_stage(p, k);
    if (r != cudaSuccess) return r;
    const size_t c0 = c * chunk, len = std::min(chunk, n - c0);
    const uint16_t* src = in + c0;
    if (!pinned) {
      CopyPool::get().copy(p->stage[k], src, len * sizeof(uint16_t));
      src = p->stage[k];
    }
    r = cudaMemcpyAsync(p->dbuf[k], src, len * 2, cudaMemcpyHostToDevice, p->h2d);
    if (r == cudaSuccess && be) r = u16m::launch_byteswap(p->dbuf[k], len, p->h2d);
    if (r == cudaSuccess) cudaEventRecord(p->loaded[k], p->h2d);
    return r;
  };
  size_t found = 0;
  e = load(0);
  for (size_t c = 0; c < nchunks && e == cudaSuccess; c++) {
    const int k = static_cast<int>(c % 2);
    const size_t c0 = c * chunk, len = std::min(chunk, n - c0);
    // the next chunk's slot was last read by chunk c-1's scan, finished below
    if (c + 1 < nchunks) e = load(c + 1);
    if (e != cudaSuccess) break;
    cudaStreamWaitEvent(p->comp, p->loaded[k], 0);
    const int32_t left = c0 > 0 ? unit(c0 - 1) : -1;
    const int32_t right = c0 + len < n ? unit(c0 + len) : -1;
    e = u16m::launch_unpaired_offsets(p->dbuf[k], len, std::min(limit - found, cap), d_off, d_cnt, p->comp,
                                      left, right);
    if (e != cudaSuccess) break;
    unsigned long long cnt = 0;
    e = cudaMemcpyAsync(&cnt, d_cnt, sizeof(cnt), cudaMemcpyDeviceToHost, p->comp);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->comp);
    if (e == cudaSuccess && cnt) e = cudaMemcpy(offsets_out + found, d_off, cnt * 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) break;
    for (size_t i = 0; i < cnt; i++) offsets_out[found + i] += c0;  // chunk-relative -> buffer offsets
    found += cnt;
    if (found >= limit) break;
  }
  const cudaError_t f = cudaStreamSynchronize(p->h2d);  // a prefetched chunk may still read `in`
  cudaFreeAsync(ws, p->comp);
  cudaStreamSynchronize(p->comp);
  if (e != cudaSuccess) return cuda_fail(e, "unpaired offsets");
  if (f != cudaSuccess) return cuda_fail(f, "unpaired offsets");
  *count_out = found;
  return U16M_OK;
}

}  // namespace

extern "C" {

u16m_status u16m_unpaired_offsets_host(const uint16_t* in, size_t n, size_t limit,
                                       unsigned long long* offsets_out, size_t* count_out) {
  return unpaired_offsets_host(in, n, -1, limit, offsets_out, count_out);
}

u16m_status u16m_unpaired_offsets_bytes_host(const void* in, size_t n_units, int byte_order, size_t limit,
                                             unsigned long long* offsets_out, size_t* count_out) {
  if (byte_order != U16M_LITTLE_ENDIAN && byte_order != U16M_BIG_ENDIAN)
    return fail(U16M_ERR_INVALID_ARGUMENT, "byte_order must be U16M_LITTLE_ENDIAN or U16M_BIG_ENDIAN");
  return unpaired_offsets_host(static_cast<const uint16_t*>(in), n_units, byte_order, limit, offsets_out, count_out);
}

}  // extern "C"
