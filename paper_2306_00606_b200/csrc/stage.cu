// Host->device staging of PAGEABLE caller memory (efg_expected_force with a
// reference-style Graph: plain numpy arrays).  The driver copies pageable
// memory through its own pinned bounce buffer on one thread (~11 GB/s on the
// B200 boxes: 33 ms for R-MAT22's 370 MB); here host threads copy pieces of
// the input into a ring of library-owned pinned buffers in parallel, and the
// copy stream moves each piece to the device as soon as it is staged, so the
// PCIe copy, the host copies and the engine's per-chunk work overlap.
//
// Stream order: every piece is enqueued as
//     [host gate: piece staged] -> cudaMemcpyAsync(dst, ring[b]) -> event[p]
// on the copy stream.  The gate is a cudaLaunchHostFunc callback that blocks
// until a worker thread has filled the piece's ring buffer.  The workers run
// while the pieces are enqueued (a long input's gates, copies and events can
// fill the stream's queue, and then the enqueue waits for gates that only the
// workers open); worker t stages pieces t, t+T, ... in increasing order, each
// once it is on the stream (see work()).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "efg_internal.cuh"

namespace efg {

#ifndef EFG_STAGE_WAITVALUE
#define EFG_STAGE_WAITVALUE 1
#endif
constexpr bool kStageWaitValue = EFG_STAGE_WAITVALUE;

namespace {
void CUDART_CB gate_fn(void* arg) {
  auto* g = static_cast<HostStager::Gate*>(arg);
  HostStager* s = g->owner;
  std::unique_lock<std::mutex> lock(s->mu);
  s->cv.wait(lock, [&] { return s->ready[g->idx] != 0; });
}
}  // namespace

bool is_pageable(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at{};
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear: plain host memory on some driver versions
    return true;
  }
  return at.type == cudaMemoryTypeUnregistered;
}

void HostStager::begin(int threads) {
  for (auto& w : workers) w.join();  // (none: the previous call's finish() joined them)
  workers.clear();
  {
    std::lock_guard<std::mutex> lock(mu);
    pieces.clear();
    ready.clear();
    enqueued = 0;
    closed = false;
    failed = false;
  }
  gates.clear();
  if (flags_h && flags_used) std::memset(flags_h, 0, (size_t)flags_used * sizeof(uint32_t));  // last call's waits are done
  flags_used = 0;
  piece = kPiece;
  if (const char* e = getenv("EFG_STAGE_PIECE_KB"))  // smaller pieces (tests: many more stream operations)
    piece = std::max<size_t>(4096, std::min<size_t>(kPiece, (size_t)atoll(e) << 10));
  if (threads <= 0) return;  // nothing pageable in this call
  if (kStageWaitValue && !flags_h) {
    cudaDriverEntryPointQueryResult q{};
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && fn) {
      void* h = nullptr;
      if (cudaHostAlloc(&h, kFlags * sizeof(uint32_t), cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess) {
        std::memset(h, 0, kFlags * sizeof(uint32_t));
        void* d = nullptr;
        if (cudaHostGetDevicePointer(&d, h, 0) == cudaSuccess) {
          flags_h = static_cast<uint32_t*>(h);
          flags_d = d;
          wait_fn = fn;
        } else {
          cudaFreeHost(h);
        }
      }
    }
    cudaGetLastError();  // a failed probe leaves the host-function gates in place
  }
  if (bufs.empty()) {
    for (int b = 0; b < kRing; ++b) {
      void* p = nullptr;
      EFG_CUDA_CHECK(cudaHostAlloc(&p, kPiece, cudaHostAllocPortable));
      bufs.push_back(static_cast<char*>(p));
    }
  }
  // Workers run from the start: the stream's queue of gates, copies and events
  // may fill while add() enqueues (the enqueue then blocks until the stream
  // drains), and only staged pieces open the gates that drain it.
  const int T = std::max(1, std::min<int>(threads, kRing / 2));
  for (int t = 0; t < T; ++t) workers.emplace_back([this, t, T] { work(t, T); });
}

void HostStager::ensure(size_t npieces) {
  while (true) {
    {
      std::lock_guard<std::mutex> lock(mu);
      if (ev.size() >= npieces) return;
    }
    cudaEvent_t e;
    EFG_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    std::lock_guard<std::mutex> lock(mu);
    ev.push_back(e);
  }
}

void HostStager::add(cudaStream_t s, void* dst, const void* src, size_t bytes) {
  const char* from = static_cast<const char*>(src);
  char* to = static_cast<char*>(dst);
  size_t first, last;
  {
    std::lock_guard<std::mutex> lock(mu);
    first = pieces.size();
    for (size_t off = 0; off < bytes; off += piece)
      pieces.push_back({from + off, to + off, std::min(piece, bytes - off)});
    last = pieces.size();
    while (ready.size() < last) ready.push_back(0);
  }
  ensure(last);
  for (size_t p = first; p < last; ++p) gates.push_back({this, (int64_t)p});
  for (size_t p = first; p < last; ++p) {
    cudaEvent_t e;
    size_t nbytes;
    char* d;
    {
      std::lock_guard<std::mutex> lock(mu);
      e = ev[p];
      nbytes = pieces[p].bytes;
      d = pieces[p].dst;
    }
    if (wait_fn && (int64_t)p < kFlags) {
      using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
      const CUresult r = reinterpret_cast<WaitFn>(wait_fn)(
          (CUstream)s, (CUdeviceptr)(static_cast<char*>(flags_d) + p * sizeof(uint32_t)), 1u, CU_STREAM_WAIT_VALUE_GEQ);
      if (r != CUDA_SUCCESS) throw Error(EFG_CUDA, "cuStreamWaitValue32 failed");
      flags_used = (int64_t)p + 1;
    } else {
      EFG_CUDA_CHECK(cudaLaunchHostFunc(s, gate_fn, &gates[p]));
    }
    EFG_CUDA_CHECK(cudaMemcpyAsync(d, bufs[p % kRing], nbytes, cudaMemcpyHostToDevice, s));
    EFG_CUDA_CHECK(cudaEventRecord(e, s));
    {
      std::lock_guard<std::mutex> lock(mu);
      enqueued = (int64_t)p + 1;  // its ring buffer's previous copy event is recorded: a worker may stage it
    }
    cv.notify_all();
  }
}

void HostStager::close() {
  {
    std::lock_guard<std::mutex> lock(mu);
    closed = true;
  }
  cv.notify_all();
}

// Worker t stages pieces t, t+T, ... in increasing order, each once it is on
// the stream; before reusing ring buffer b it waits for event[p - kRing] (the
// device copy of the piece that used b last).  That copy depends only on gates
// <= p - kRing, all owned by pieces a worker reaches before p: no cycle.
void HostStager::work(int t, int T) {
  for (int64_t p = t;; p += T) {
    Piece pc;
    cudaEvent_t prev = nullptr;
    {
      std::unique_lock<std::mutex> lock(mu);
      cv.wait(lock, [&] { return p < enqueued || closed; });
      if (p >= enqueued) return;  // closed and no such piece
      pc = pieces[p];
      if (p >= kRing) prev = ev[p - kRing];
    }
    bool ok = true;
    if (prev && cudaEventSynchronize(prev) != cudaSuccess) ok = false;
    if (ok) std::memcpy(bufs[p % kRing], pc.src, pc.bytes);
    {
      std::lock_guard<std::mutex> lock(mu);
      if (!ok) failed = true;
      ready[p] = 1;  // even on failure: a gate must never block forever
    }
    if (flags_h && p < kFlags) {  // the device-side gate: the staged bytes are visible before the flag
      std::atomic_thread_fence(std::memory_order_seq_cst);
      __atomic_store_n(flags_h + p, 1u, __ATOMIC_RELEASE);
    }
    cv.notify_all();
  }
}

void HostStager::finish() {
  for (auto& w : workers) w.join();
  workers.clear();
  if (failed) throw Error(EFG_CUDA, "host staging: a device copy of the staged input failed");
}

HostStager::~HostStager() {
  close();
  for (auto& w : workers) w.join();
  if (flags_h) cudaFreeHost(flags_h);
  for (auto p : bufs) cudaFreeHost(p);
  for (auto e : ev) cudaEventDestroy(e);
}

}  // namespace efg
