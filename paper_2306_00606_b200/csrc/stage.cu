// Host->device staging of PAGEABLE caller memory (efg_expected_force with a
// reference-style Graph: plain numpy arrays).  The driver copies pageable
// memory through its own pinned bounce buffer on one thread (~11 GB/s on the
// B200 boxes: 33 ms for R-MAT22's 370 MB); here host threads copy pieces of
// the input into a ring of library-owned pinned buffers in parallel, and the
// copy stream moves each piece to the device as soon as it is staged, so the
// PCIe copy, the host copies and the engine's per-chunk work overlap.
//
// Stream order: every piece is enqueued up front (before the engine waits on
// the chunk events) as
//     [host gate: piece staged] -> cudaMemcpyAsync(dst, ring[b]) -> event[p]
// on the copy stream.  The gate is a cudaLaunchHostFunc callback that blocks
// until a worker thread has filled the piece's ring buffer.  Worker t stages
// pieces t, t+T, ... in increasing order; before reusing ring buffer b it
// waits for event[p - R] (the device copy of the piece that used b last).
// That copy depends only on gates <= p - R, all owned by pieces a worker
// reaches before p, so the waits cannot form a cycle.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <thread>

#include "efg_internal.cuh"

namespace efg {

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

void HostStager::begin() {
  pieces.clear();
  gates.clear();
  std::lock_guard<std::mutex> lock(mu);
  ready.clear();
  failed = false;
}

void HostStager::ensure(size_t npieces) {
  if (bufs.empty()) {
    for (int b = 0; b < kRing; ++b) {
      void* p = nullptr;
      EFG_CUDA_CHECK(cudaHostAlloc(&p, kPiece, cudaHostAllocPortable));
      bufs.push_back(static_cast<char*>(p));
    }
  }
  while (ev.size() < npieces) {
    cudaEvent_t e;
    EFG_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ev.push_back(e);
  }
}

void HostStager::add(cudaStream_t s, void* dst, const void* src, size_t bytes) {
  const char* from = static_cast<const char*>(src);
  char* to = static_cast<char*>(dst);
  for (size_t off = 0; off < bytes; off += kPiece) pieces.push_back({from + off, to + off, std::min(kPiece, bytes - off)});
  ensure(pieces.size());
  // enqueue only the new pieces (earlier add() calls queued theirs)
  const size_t first = gates.size();
  {
    std::lock_guard<std::mutex> lock(mu);  // gate callbacks of earlier pieces may be reading `ready`
    while (ready.size() < pieces.size()) ready.push_back(0);
  }
  for (size_t p = first; p < pieces.size(); ++p) gates.push_back({this, (int64_t)p});
  for (size_t p = first; p < pieces.size(); ++p) {
    EFG_CUDA_CHECK(cudaLaunchHostFunc(s, gate_fn, &gates[p]));
    EFG_CUDA_CHECK(cudaMemcpyAsync(pieces[p].dst, bufs[p % kRing], pieces[p].bytes, cudaMemcpyHostToDevice, s));
    EFG_CUDA_CHECK(cudaEventRecord(ev[p], s));
  }
}

void HostStager::start(int threads) {
  const int64_t np = (int64_t)pieces.size();
  if (np == 0) return;
  const int T = std::max(1, std::min<int>(threads, kRing / 2));
  for (int t = 0; t < T; ++t) {
    workers.emplace_back([this, t, T, np] {
      for (int64_t p = t; p < np; p += T) {
        bool ok = true;
        if (p >= kRing && cudaEventSynchronize(ev[p - kRing]) != cudaSuccess) ok = false;
        if (ok) std::memcpy(bufs[p % kRing], pieces[p].src, pieces[p].bytes);
        {
          std::lock_guard<std::mutex> lock(mu);
          if (!ok) failed = true;
          ready[p] = 1;  // even on failure: a gate must never block forever
        }
        cv.notify_all();
      }
    });
  }
}

void HostStager::finish() {
  for (auto& w : workers) w.join();
  workers.clear();
  if (failed) throw Error(EFG_CUDA, "host staging: a device copy of the staged input failed");
}

HostStager::~HostStager() {
  for (auto& w : workers) w.join();
  for (auto p : bufs) cudaFreeHost(p);
  for (auto e : ev) cudaEventDestroy(e);
}

}  // namespace efg
