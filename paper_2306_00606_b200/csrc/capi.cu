// C ABI of libefg.so (include/efg.h): status codes, thread-local last error,
// per-context serialisation, host<->device staging and timing.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "efg_internal.cuh"

namespace efg {
int check_line_factor();
int check_line_direct();
int check_line_prep();
int check_line_alg1();
thread_local int64_t g_launches = 0;
thread_local int64_t g_lib_calls = 0;
thread_local Profiler* g_prof = nullptr;

cudaEvent_t Profiler::take() {
  if (used == pool.size()) {
    cudaEvent_t e;
    EFG_CUDA_CHECK(cudaEventCreate(&e));
    pool.push_back(e);
  }
  return pool[used++];
}

void Profiler::resolve() {
  timeline.clear();
  for (auto& r : pending) {
    float ms = 0.f, t0 = 0.f;
    EFG_CUDA_CHECK(cudaEventElapsedTime(&ms, r.a, r.b));
    EFG_CUDA_CHECK(cudaEventElapsedTime(&t0, pending.front().a, r.a));
    auto& t = totals[r.name];
    t.first += ms;
    t.second += 1;
    timeline.push_back({r.name, t0, ms});
  }
  pending.clear();
  used = 0;
}

Profiler::~Profiler() {
  for (auto e : pool) cudaEventDestroy(e);
}

void prof_begin(Profiler* p, const char* name, cudaStream_t s) {
  Profiler::Rec r{name, p->take(), p->take()};
  EFG_CUDA_CHECK(cudaEventRecord(r.a, s));
  p->pending.push_back(r);
}

void prof_end(Profiler* p, cudaStream_t s) { EFG_CUDA_CHECK(cudaEventRecord(p->pending.back().b, s)); }

Context::~Context() {
  for (auto& kv : bufs) kv.second.release();
  csr.b_off.release();
  csr.b_nbr.release();
  csr.b_orig.release();
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : aux_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : chunk_ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : side_ev)
    if (e) cudaEventDestroy(e);
  if (copy_stream) cudaStreamDestroy(copy_stream);
  if (side_stream) cudaStreamDestroy(side_stream);
  if (own_stream && stream) cudaStreamDestroy(stream);
}
}  // namespace efg

using efg::Context;

struct efg_ctx {
  Context c;
};

namespace {
thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

template <class F>
int guarded(efg_ctx* ctx, F&& body) {
  if (!ctx) return fail(efg::EFG_INVALID, "null efg context");
  std::lock_guard<std::mutex> lock(ctx->c.mu);
  try {
    cudaError_t e = cudaSetDevice(ctx->c.device);
    if (e != cudaSuccess) return fail(efg::EFG_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    efg::g_prof = ctx->c.prof.on ? &ctx->c.prof : nullptr;
    body(ctx->c);
#ifdef EFG_BOUNDS_CHECK
    {  // bounds-checked build: any device index check that failed during the call
      EFG_CUDA_CHECK(cudaStreamSynchronize(ctx->c.stream));
      const int lf = efg::check_line_factor(), ld = efg::check_line_direct(), lp = efg::check_line_prep(),
                la = efg::check_line_alg1();
      if (lf || ld || lp || la)
        throw efg::Error(efg::EFG_CUDA, "device bounds check failed: ef_factor.cu:" + std::to_string(lf) +
                                            " ef_direct.cu:" + std::to_string(ld) + " prep.cu:" + std::to_string(lp) +
                                            " ef_alg1.cu:" + std::to_string(la));
    }
#endif
    if (efg::g_prof && !ctx->c.prof.pending.empty()) {
      EFG_CUDA_CHECK(cudaStreamSynchronize(ctx->c.stream));
      ctx->c.prof.resolve();
    }
    efg::g_prof = nullptr;
    g_last_error.clear();
    return efg::EFG_OK;
  } catch (const efg::Error& err) {
    efg::g_prof = nullptr;
    ctx->c.prof.pending.clear();
    ctx->c.prof.used = 0;
    return fail(err.code, err.what());
  } catch (const std::bad_alloc&) {
    return fail(efg::EFG_OOM, "host out of memory");
  } catch (const std::exception& err) {
    return fail(efg::EFG_CUDA, err.what());
  }
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  EFG_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

int resolve_engine(int mode, int engine) {
  if (engine == EFG_ENGINE_AUTO)
    return mode == EFG_MODE_VERTEX_CENTRIC ? EFG_ENGINE_DIRECT : EFG_ENGINE_FACTORIZED;
  return engine;
}

// Run one EF pass over device CSR `g` for seeds r; outputs device, index = seed - r.lo.
void run_engine(Context& c, const efg::CSRView& g, const efg::Staging& stg, efg::SeedRange r, int engine, double* ef,
                int64_t* tot, uint8_t* fl, int64_t* T, double* W, efg_stats* st) {
  EFG_REQUIRE(engine == EFG_ENGINE_FACTORIZED || engine == EFG_ENGINE_DIRECT || engine == EFG_ENGINE_ALG1,
              "unknown engine " + std::to_string(engine));
  cudaEvent_t* ev = c.ev;
  efg::PrepInfo info;
  if (engine == EFG_ENGINE_FACTORIZED) {
    // records ev[2] (start) and ev[3] (preparation done) itself
    info = efg::ef_factorized(c, g, stg, r, ef, tot, fl, T, W, st);
  } else {
    for (int k = 0; k < stg.nchunks; ++k)
      if (stg.ready[k]) EFG_CUDA_CHECK(cudaStreamWaitEvent(c.stream, stg.ready[k], 0));
    efg::Prepared P;
    if (st) EFG_CUDA_CHECK(cudaEventRecord(ev[2], c.stream));
    efg::prepare(c, g, false, P);
    if (st) EFG_CUDA_CHECK(cudaEventRecord(ev[3], c.stream));
    if (engine == EFG_ENGINE_ALG1)
      efg::ef_alg1(c, P, r, ef, tot, fl, T, W, st);
    else
      efg::ef_direct(c, P, r, ef, tot, fl, T, W, st);
    info.dmax = P.dmax;
    info.sum_c2 = P.sum_c2;
  }
  if (st) {
    EFG_CUDA_CHECK(cudaEventRecord(ev[4], c.stream));
    EFG_CUDA_CHECK(cudaEventSynchronize(ev[4]));
    st->ms_prepare = elapsed(ev[2], ev[3]);
    st->ms_enumerate = elapsed(ev[3], ev[4]);
    st->dmax = info.dmax;
    st->cluster_visits = 3 * info.sum_c2;
    st->clusters_processed = info.sum_c2;
    st->bytes_alg = 16 * info.sum_c2 + 32 * g.m2 + 33 * g.n;
    st->engine = engine;
  }
}

// A single chunk already resident on the device.
efg::Staging resident(const efg::CSRView& g) {
  efg::Staging s;
  s.nchunks = 1;
  s.row[1] = g.n;
  s.slot[1] = g.m2;
  return s;
}

template <class T>
T* stage(Context& c, const char* name, const T* host, int64_t count) {
  T* d = c.buf(name).as<T>(count > 0 ? count : 1);
  if (count > 0) EFG_CUDA_CHECK(cudaMemcpyAsync(d, host, count * sizeof(T), cudaMemcpyHostToDevice, c.stream));
  return d;
}

}  // namespace

extern "C" {

int efg_abi_version(void) { return EFG_ABI_VERSION; }

const char* efg_last_error(void) { return g_last_error.c_str(); }

int efg_create(int device, efg_ctx** out) {
  if (!out) return fail(efg::EFG_INVALID, "null output pointer");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return fail(efg::EFG_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(efg::EFG_INVALID, "device index out of range");
  efg_ctx* ctx = new (std::nothrow) efg_ctx;
  if (!ctx) return fail(efg::EFG_OOM, "host out of memory");
  ctx->c.device = device;
  int rc = guarded(ctx, [&](Context& c) {
    EFG_CUDA_CHECK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    c.own_stream = true;
    for (auto& x : c.ev) EFG_CUDA_CHECK(cudaEventCreate(&x));
    for (auto& x : c.chunk_ev) EFG_CUDA_CHECK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    for (auto& x : c.aux_ev) EFG_CUDA_CHECK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    EFG_CUDA_CHECK(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
    for (auto& x : c.side_ev) EFG_CUDA_CHECK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    EFG_CUDA_CHECK(cudaStreamCreateWithFlags(&c.side_stream, cudaStreamNonBlocking));
    EFG_CUDA_CHECK(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, device));
  });
  if (rc) {
    delete ctx;
    return rc;
  }
  *out = ctx;
  return 0;
}

int efg_destroy(efg_ctx* ctx) {
  if (!ctx) return 0;
  cudaSetDevice(ctx->c.device);
  if (ctx->c.stream) cudaStreamSynchronize(ctx->c.stream);
  delete ctx;
  return 0;
}

int efg_set_stream(efg_ctx* ctx, void* stream) {
  return guarded(ctx, [&](Context& c) {
    if (c.own_stream && c.stream) {
      EFG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
      EFG_CUDA_CHECK(cudaStreamDestroy(c.stream));
    }
    if (stream) {
      c.stream = static_cast<cudaStream_t>(stream);
      c.own_stream = false;
    } else {
      EFG_CUDA_CHECK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
      c.own_stream = true;
    }
  });
}

int efg_synchronize(efg_ctx* ctx) {
  return guarded(ctx, [&](Context& c) { EFG_CUDA_CHECK(cudaStreamSynchronize(c.stream)); });
}

int efg_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return fail(efg::EFG_INVALID, "bad host_alloc arguments");
  cudaError_t e = cudaHostAlloc(out, bytes > 0 ? (size_t)bytes : 1, cudaHostAllocPortable);
  if (e != cudaSuccess) return fail(efg::EFG_OOM, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
  return 0;
}

int efg_host_free(void* p) {
  if (p) cudaFreeHost(p);
  return 0;
}

int efg_format_ef_csv(const int64_t* orig_ids, const double* ef, const int64_t* cluster_total, int64_t n,
                      int32_t threads, char* buf, int64_t cap, int64_t* len_out) {
  constexpr int64_t kRowMax = 64;  // 20 + 1 + 24 (%.9g) + 1 + 20 + 1 < 64
  if (n < 0 || !len_out || (n > 0 && (!orig_ids || !ef || !cluster_total || !buf)) || cap < kRowMax * n)
    return fail(efg::EFG_INVALID, "bad efg_format_ef_csv arguments (cap must be >= 64 n)");
  try {
    const int T = (int)std::max<int64_t>(1, std::min<int64_t>(std::max(threads, 1), (n + 65535) / 65536));
    std::vector<std::string> part(T);
    auto work = [&](int t) {
      const int64_t lo = n * t / T, hi = n * (t + 1) / T;
      std::string& out = part[t];
      out.resize((size_t)((hi - lo) * kRowMax));
      char* p = &out[0];
      for (int64_t i = lo; i < hi; ++i)
        p += std::snprintf(p, kRowMax, "%lld,%.9g,%lld\n", (long long)orig_ids[i], ef[i], (long long)cluster_total[i]);
      out.resize((size_t)(p - &out[0]));
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    int64_t len = 0;
    for (auto& s : part) {
      std::memcpy(buf + len, s.data(), s.size());
      len += (int64_t)s.size();
    }
    *len_out = len;
    return 0;
  } catch (const std::exception& e) {
    return fail(efg::EFG_OOM, std::string("efg_format_ef_csv: ") + e.what());
  }
}

int efg_build_graph(efg_ctx* ctx, const int64_t* edges, int64_t k, int64_t* n_out, int64_t* m_out) {
  if (k < 0 || (k > 0 && !edges)) return fail(efg::EFG_INVALID, "bad edge array");
  return guarded(ctx, [&](Context& c) {
    const int64_t* d_edges = stage(c, "edges_in", edges, 2 * k);
    efg::build_csr_device(c, d_edges, k, c.csr);
    EFG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    if (n_out) *n_out = c.csr.n;
    if (m_out) *m_out = c.csr.m;
  });
}

int efg_rmat_build(efg_ctx* ctx, int32_t scale, int64_t avg_degree, const double* probs, const uint64_t* pcg_state,
                   const uint64_t* pcg_inc, int32_t* truncated, int64_t* n_out, int64_t* m_out) {
  if (!probs || !pcg_state || !pcg_inc) return fail(efg::EFG_INVALID, "null R-MAT argument");
  return guarded(ctx, [&](Context& c) {
    bool tr = false;
    efg::rmat_build_device(c, scale, avg_degree, probs, pcg_state, pcg_inc, tr, c.csr);
    EFG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    if (truncated) *truncated = tr ? 1 : 0;
    if (n_out) *n_out = c.csr.n;
    if (m_out) *m_out = c.csr.m;
  });
}

int efg_fetch_graph(efg_ctx* ctx, int64_t* offsets, int32_t* neighbors, int64_t* orig_ids) {
  return guarded(ctx, [&](Context& c) {
    const int64_t n = c.csr.n, m = c.csr.m;
    if (offsets) {
      if (n == 0) {
        offsets[0] = 0;
      } else {
        EFG_CUDA_CHECK(cudaMemcpyAsync(offsets, c.csr.offsets, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
      }
    }
    if (neighbors && m) EFG_CUDA_CHECK(cudaMemcpyAsync(neighbors, c.csr.nbr, 2 * m * sizeof(int32_t), cudaMemcpyDeviceToHost, c.stream));
    if (orig_ids && n) EFG_CUDA_CHECK(cudaMemcpyAsync(orig_ids, c.csr.orig_ids, n * sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    EFG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  });
}

int efg_graph_device(efg_ctx* ctx, const int64_t** d_offsets, const int32_t** d_neighbors, int64_t* n_out,
                     int64_t* m_out) {
  return guarded(ctx, [&](Context& c) {
    if (d_offsets) *d_offsets = c.csr.offsets;
    if (d_neighbors) *d_neighbors = c.csr.nbr;
    if (n_out) *n_out = c.csr.n;
    if (m_out) *m_out = c.csr.m;
  });
}

int efg_expected_force(efg_ctx* ctx, const int64_t* offsets, const int32_t* neighbors, int64_t n, int32_t mode,
                       int32_t engine, double* ef, int64_t* cluster_total, uint8_t* flags,
                       int64_t* clusters_processed, int64_t* T_out, double* W_out, efg_stats* stats) {
  if (n < 0 || !offsets) return fail(efg::EFG_INVALID, "bad offsets");
  if (mode != EFG_MODE_CLUSTER_CENTRIC && mode != EFG_MODE_VERTEX_CENTRIC)
    return fail(efg::EFG_INVALID, "unknown mode " + std::to_string(mode) + "; expected cluster_centric or vertex_centric");
  if (n > 0 && (!ef || !cluster_total || !flags)) return fail(efg::EFG_INVALID, "null output array");
  return guarded(ctx, [&](Context& c) {
    efg::g_launches = 0;
    efg_stats local{};
    efg_stats* st = stats ? stats : &local;
    std::memset(st, 0, sizeof *st);
    const int eng = resolve_engine(mode, engine);
    if (n == 0) {
      if (clusters_processed) *clusters_processed = 0;
      st->engine = eng;
      return;
    }
    const int64_t m2 = offsets[n] - offsets[0];
    EFG_REQUIRE(offsets[0] == 0 && m2 >= 0 && m2 % 2 == 0, "offsets must start at 0 and cover 2m entries");
    EFG_REQUIRE(n < (int64_t(1) << 31), "graph too large: n exceeds int32 id space");
    cudaEvent_t* ev = c.ev;
    EFG_CUDA_CHECK(cudaEventRecord(ev[0], c.stream));
    // Inputs on the copy stream: offsets, then the neighbours in row chunks of
    // about equal size; the engine starts on the offsets and takes up each
    // chunk's rows as it lands (efg::Staging).
    EFG_CUDA_CHECK(cudaStreamWaitEvent(c.copy_stream, ev[0], 0));
    efg::CSRView g;
    g.n = n;
    g.m2 = m2;
    int64_t* d_off = c.buf("h_offsets").as<int64_t>(n + 1);
    int32_t* d_nbr = c.buf("h_nbr").as<int32_t>(m2 > 0 ? m2 : 1);
    g.offsets = d_off;
    g.nbr = d_nbr;
    // pageable caller memory (a reference Graph's numpy arrays) goes through
    // the pinned staging ring (stage.cu); page-locked memory is copied directly
    const bool stage_off = efg::is_pageable(offsets), stage_nbr = efg::is_pageable(neighbors);
    int workers = (int)std::max(1u, std::thread::hardware_concurrency() / 2);
    if (const char* e = getenv("EFG_STAGE_WORKERS")) workers = std::max(1, atoi(e));  // tuning (tools/ab_env.sh)
    struct JoinGuard {  // never leave staging workers running past this call
      efg::HostStager& s;
      ~JoinGuard() {
        s.close();
        for (auto& w : s.workers) w.join();
        s.workers.clear();
      }
    } join_guard{c.stager};
    c.stager.begin(stage_off || stage_nbr ? workers : 0);
    auto h2d = [&](void* dst, const void* src, size_t bytes, bool staged) {
      if (staged)
        c.stager.add(c.copy_stream, dst, src, bytes);
      else
        EFG_REGION("h2d", c.copy_stream,
                   EFG_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c.copy_stream)));
    };
    h2d(d_off, offsets, (n + 1) * sizeof(int64_t), stage_off);
    EFG_CUDA_CHECK(cudaEventRecord(c.chunk_ev[0], c.copy_stream));
    efg::Staging stg;
    // Chunks growing from a small first one: the engine starts once it lands,
    // and the per-row work of each chunk (orientation, sorts, histograms,
    // tables, pushes: slower per slot than the copy) covers the next chunk's
    // copy.  Measured at R-MAT22 (pass 23.3 ms, H2D 6.7 ms), e2e pinned ms:
    // 1 chunk 29.9; 25 %: 28.3; 10/25/45: 26.9; 10/23/41/65: 27.0;
    // 12/28/50/79: 26.8; 15/30/55/80: 26.6; 20/40/65: 26.1; 18/38/62: 25.9;
    // 15/40/70: 26.0; 15/35/62: 25.85 (tools/ab_stage.sh, r02).
    // chunk k's slots end at split[k] % of 2m (cumulative; the last chunk ends at 100 %)
    // Smaller inputs (ER-1M, Chung-Lu 2^20: ~70 MB, 1.3 ms of copy) pay more in
    // per-chunk launches than they overlap: two chunks, the first 40 % (ER-1M e2e
    // ms: 1 chunk 3.28, 25 %: 3.20, 40 %: 3.06-3.11, 15/35/62: 3.59; Chung-Lu:
    // 5.91, 6.00, 6.11, 6.52).
    int split[efg::kMaxChunks] = {15, 35, 62};
    stg.nchunks = m2 >= (int64_t(1) << 25) ? 4 : m2 >= (int64_t(1) << 22) ? 2 : 1;
    if (stg.nchunks == 2) split[0] = 40;
    if (const char* e = getenv("EFG_STAGE_SPLITS")) {  // tuning override (tools/ab_stage.sh): "10,25,45" / "none"
      int k = 0;
      if (!strcmp(e, "none")) e = "";
      for (const char* q = e; *q && k < efg::kMaxChunks - 1; ++k) {
        split[k] = std::max(1, std::min(99, atoi(q)));
        while (*q && *q != ',') ++q;
        if (*q == ',') ++q;
      }
      stg.nchunks = k + 1;
    }
    for (int k = 0; k <= stg.nchunks; ++k) {
      const int64_t target = k == 0 ? 0 : k == stg.nchunks ? m2 : m2 * split[k - 1] / 100;
      stg.row[k] = k == stg.nchunks ? n : std::lower_bound(offsets, offsets + n + 1, target) - offsets;
      if (k > 0 && stg.row[k] < stg.row[k - 1]) stg.row[k] = stg.row[k - 1];
      stg.slot[k] = offsets[stg.row[k]];
    }
    for (int k = 0; k < stg.nchunks; ++k) {
      const int64_t e0 = stg.slot[k], e1 = stg.slot[k + 1];
      if (e1 > e0) h2d(d_nbr + e0, neighbors + e0, (e1 - e0) * sizeof(int32_t), stage_nbr);
      EFG_CUDA_CHECK(cudaEventRecord(c.chunk_ev[1 + k], c.copy_stream));
      stg.ready[k] = c.chunk_ev[1 + k];
    }
    EFG_CUDA_CHECK(cudaEventRecord(ev[1], c.copy_stream));  // all inputs resident
    c.stager.close();  // every piece is on the stream
    EFG_CUDA_CHECK(cudaStreamWaitEvent(c.stream, c.chunk_ev[0], 0));
    double* d_ef = c.buf("o_ef").as<double>(n);
    int64_t* d_tot = c.buf("o_tot").as<int64_t>(n);
    uint8_t* d_fl = c.buf("o_fl").as<uint8_t>(n);
    int64_t* d_T = T_out ? c.buf("o_T").as<int64_t>(n) : nullptr;
    double* d_W = W_out ? c.buf("o_W").as<double>(n) : nullptr;
    stg.total_host = cluster_total;
    c.total_sent = false;
    run_engine(c, g, stg, efg::SeedRange{0, n}, eng, d_ef, d_tot, d_fl, d_T, d_W, st);
    EFG_CUDA_CHECK(cudaEventRecord(ev[5], c.stream));
    EFG_REGION("d2h", c.stream, EFG_CUDA_CHECK(cudaMemcpyAsync(ef, d_ef, n * sizeof(double), cudaMemcpyDeviceToHost, c.stream)));
    if (c.total_sent)  // the engine already queued it on the copy stream
      EFG_CUDA_CHECK(cudaStreamWaitEvent(c.stream, c.aux_ev[1], 0));
    else
      EFG_CUDA_CHECK(cudaMemcpyAsync(cluster_total, d_tot, n * sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    EFG_CUDA_CHECK(cudaMemcpyAsync(flags, d_fl, n, cudaMemcpyDeviceToHost, c.stream));
    if (T_out) EFG_CUDA_CHECK(cudaMemcpyAsync(T_out, d_T, n * sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    if (W_out) EFG_CUDA_CHECK(cudaMemcpyAsync(W_out, d_W, n * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    EFG_CUDA_CHECK(cudaEventRecord(ev[6], c.stream));
    EFG_CUDA_CHECK(cudaEventSynchronize(ev[6]));
    c.stager.finish();
    st->ms_h2d = elapsed(ev[0], ev[1]);
    st->ms_d2h = elapsed(ev[5], ev[6]);
    st->ms_device = elapsed(ev[0], ev[6]);
    st->h2d_bytes = (n + 1) * 8 + m2 * 4;
    st->d2h_bytes = n * 17 + (T_out ? n * 8 : 0) + (W_out ? n * 8 : 0);
    if (mode == EFG_MODE_VERTEX_CENTRIC) st->clusters_processed = st->cluster_visits;
    if (clusters_processed) *clusters_processed = st->clusters_processed;
    st->launches = efg::g_launches;
  });
}

int efg_expected_force_device(efg_ctx* ctx, const int64_t* d_offsets, const int32_t* d_neighbors, int64_t n,
                              int64_t seed_lo, int64_t seed_hi, int32_t engine, double* d_ef,
                              int64_t* d_cluster_total, uint8_t* d_flags, int64_t* d_T, double* d_W,
                              efg_stats* stats) {
  if (n < 0 || seed_lo < 0 || seed_hi < seed_lo || seed_hi > n)
    return fail(efg::EFG_INVALID, "bad seed range");
  return guarded(ctx, [&](Context& c) {
    efg::g_launches = 0;
    if (stats) std::memset(stats, 0, sizeof *stats);
    const int eng = resolve_engine(EFG_MODE_CLUSTER_CENTRIC, engine);
    if (n == 0 || seed_hi == seed_lo) return;
    int64_t off_n = 0;
    EFG_CUDA_CHECK(cudaMemcpyAsync(&off_n, d_offsets + n, sizeof off_n, cudaMemcpyDeviceToHost, c.stream));
    EFG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    efg::CSRView g;
    g.n = n;
    g.m2 = off_n;
    g.offsets = d_offsets;
    g.nbr = d_neighbors;
    if (stats) EFG_CUDA_CHECK(cudaEventRecord(c.ev[0], c.stream));
    run_engine(c, g, resident(g), efg::SeedRange{seed_lo, seed_hi}, eng, d_ef, d_cluster_total, d_flags, d_T, d_W,
               stats);
    if (stats) {
      EFG_CUDA_CHECK(cudaEventRecord(c.ev[6], c.stream));
      EFG_CUDA_CHECK(cudaEventSynchronize(c.ev[6]));
      stats->ms_device = elapsed(c.ev[0], c.ev[6]);
      stats->launches = efg::g_launches;
    }
  });
}

namespace {
// One distributed part: validate, view the graph, run ef_factorized in `mode`.
int run_part(efg_ctx* ctx, const int64_t* d_offsets, const int32_t* d_neighbors, int64_t n, int32_t part,
             int32_t nparts, const int64_t* bounds, int mode, int32_t* d_adjp, int32_t* d_dplus, uint64_t* d_words,
             double* d_ws, efg_stats* stats) {
  if (n < 0 || nparts < 1 || part < 0 || part >= nparts) return fail(efg::EFG_INVALID, "bad part");
  if (n > 0 && (!d_words || !d_ws)) return fail(efg::EFG_INVALID, "null output array");
  if (mode != efg::kDistRepl && n > 0 && !bounds) return fail(efg::EFG_INVALID, "row-partitioned part needs bounds");
  if ((mode == efg::kDistRows || mode == efg::kDistList) && n > 0 && (!d_adjp || !d_dplus))
    return fail(efg::EFG_INVALID, "rows / listing parts need d_adjp and d_dplus");
  if (bounds) {
    if (bounds[0] != 0 || bounds[nparts] != n) return fail(efg::EFG_INVALID, "bounds must run from 0 to n");
    for (int p = 0; p < nparts; ++p)
      if (bounds[p + 1] < bounds[p]) return fail(efg::EFG_INVALID, "bounds must be non-decreasing");
  }
  static_assert(EFG_DIST_WORDS == efg::kDistWords, "word count");
  return guarded(ctx, [&](Context& c) {
    efg::g_launches = 0;
    if (stats) std::memset(stats, 0, sizeof *stats);
    if (n == 0) return;
    int64_t off_n = 0;
    EFG_CUDA_CHECK(cudaMemcpyAsync(&off_n, d_offsets + n, sizeof off_n, cudaMemcpyDeviceToHost, c.stream));
    EFG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    efg::CSRView g{n, off_n, d_offsets, d_neighbors};
    efg::DistPart dp;
    dp.part = part;
    dp.nparts = nparts;
    dp.mode = mode;
    if (bounds) {
      dp.node_lo = bounds[part];
      dp.node_hi = bounds[part + 1];
    } else {
      std::vector<int64_t> b(nparts + 1);
      efg::part_bounds(c, g, nparts, b.data());
      dp.node_lo = b[part];
      dp.node_hi = b[part + 1];
    }
    dp.words = reinterpret_cast<unsigned long long*>(d_words);
    dp.ws = d_ws;
    dp.adjp = d_adjp;
    dp.dplus = d_dplus;
    if (stats) EFG_CUDA_CHECK(cudaEventRecord(c.ev[0], c.stream));
    efg::ef_factorized(c, g, resident(g), efg::SeedRange{0, n}, nullptr, nullptr, nullptr, nullptr, nullptr, stats,
                       &dp);
    if (stats) {
      EFG_CUDA_CHECK(cudaEventRecord(c.ev[6], c.stream));
      EFG_CUDA_CHECK(cudaEventSynchronize(c.ev[6]));
      stats->ms_device = elapsed(c.ev[0], c.ev[6]);
      stats->launches = efg::g_launches;
      stats->engine = EFG_ENGINE_FACTORIZED;
    }
  });
}
}  // namespace

int efg_part_bounds(efg_ctx* ctx, const int64_t* d_offsets, const int32_t* d_neighbors, int64_t n, int32_t nparts,
                    int64_t* bounds_out) {
  if (n < 0 || nparts < 1 || !bounds_out) return fail(efg::EFG_INVALID, "bad part-bounds arguments");
  return guarded(ctx, [&](Context& c) {
    bounds_out[0] = 0;
    for (int p = 1; p <= nparts; ++p) bounds_out[p] = n;
    if (n == 0) return;
    int64_t off_n = 0;
    EFG_CUDA_CHECK(cudaMemcpyAsync(&off_n, d_offsets + n, sizeof off_n, cudaMemcpyDeviceToHost, c.stream));
    EFG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    efg::CSRView g{n, off_n, d_offsets, d_neighbors};
    efg::part_bounds(c, g, nparts, bounds_out);
  });
}

int efg_ef_partial(efg_ctx* ctx, const int64_t* d_offsets, const int32_t* d_neighbors, int64_t n, int32_t part,
                   int32_t nparts, uint64_t* d_words, double* d_ws, efg_stats* stats) {
  return run_part(ctx, d_offsets, d_neighbors, n, part, nparts, nullptr, efg::kDistRepl, nullptr, nullptr, d_words,
                  d_ws, stats);
}

int efg_ef_partial_rows(efg_ctx* ctx, const int64_t* d_offsets, const int32_t* d_neighbors, int64_t n, int32_t part,
                        int32_t nparts, const int64_t* bounds, int32_t* d_adjp, int32_t* d_dplus, uint64_t* d_words,
                        double* d_ws, efg_stats* stats) {
  return run_part(ctx, d_offsets, d_neighbors, n, part, nparts, bounds, efg::kDistRows, d_adjp, d_dplus, d_words,
                  d_ws, stats);
}

int efg_ef_partial_tables(efg_ctx* ctx, const int64_t* d_offsets, const int32_t* d_neighbors, int64_t n,
                          int32_t part, int32_t nparts, const int64_t* bounds, uint64_t* d_words, double* d_ws,
                          efg_stats* stats) {
  return run_part(ctx, d_offsets, d_neighbors, n, part, nparts, bounds, efg::kDistTables, nullptr, nullptr, d_words,
                  d_ws, stats);
}

int efg_ef_partial_list(efg_ctx* ctx, const int64_t* d_offsets, const int32_t* d_neighbors, int64_t n, int32_t part,
                        int32_t nparts, const int64_t* bounds, int32_t* d_adjp, int32_t* d_dplus, uint64_t* d_words,
                        double* d_ws, efg_stats* stats) {
  return run_part(ctx, d_offsets, d_neighbors, n, part, nparts, bounds, efg::kDistList, d_adjp, d_dplus, d_words,
                  d_ws, stats);
}

int efg_ef_finish(efg_ctx* ctx, const int64_t* d_offsets, const int32_t* d_neighbors, int64_t n, int64_t seed_lo,
                  int64_t seed_hi, const uint64_t* d_words, const double* d_ws, double* d_ef,
                  int64_t* d_cluster_total, uint8_t* d_flags, int64_t* d_T, double* d_W) {
  if (n < 0 || seed_lo < 0 || seed_hi < seed_lo || seed_hi > n) return fail(efg::EFG_INVALID, "bad seed range");
  return guarded(ctx, [&](Context& c) {
    if (n == 0 || seed_hi == seed_lo) return;
    int64_t off_n = 0;
    EFG_CUDA_CHECK(cudaMemcpyAsync(&off_n, d_offsets + n, sizeof off_n, cudaMemcpyDeviceToHost, c.stream));
    EFG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    efg::CSRView g;
    g.n = n;
    g.m2 = off_n;
    g.offsets = d_offsets;
    g.nbr = d_neighbors;
    efg::ef_finish(c, g, efg::SeedRange{seed_lo, seed_hi}, reinterpret_cast<const unsigned long long*>(d_words), d_ws,
                   d_ef, d_cluster_total, d_flags, d_T, d_W);
  });
}

int efg_shard_bounds(efg_ctx* ctx, const int64_t* d_offsets, const int32_t* d_neighbors, int64_t n, int32_t engine,
                     int32_t parts, int64_t* bounds_out) {
  if (parts < 1 || !bounds_out || n < 0) return fail(efg::EFG_INVALID, "bad shard arguments");
  return guarded(ctx, [&](Context& c) {
    const int eng = resolve_engine(EFG_MODE_CLUSTER_CENTRIC, engine);
    bounds_out[0] = 0;
    for (int p = 1; p <= parts; ++p) bounds_out[p] = n;
    if (n == 0) return;
    int64_t off_n = 0;
    EFG_CUDA_CHECK(cudaMemcpyAsync(&off_n, d_offsets + n, sizeof off_n, cudaMemcpyDeviceToHost, c.stream));
    EFG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    efg::CSRView g{n, off_n, d_offsets, d_neighbors};
    efg::Prepared P;
    efg::prepare(c, g, eng == EFG_ENGINE_FACTORIZED, P);
    int64_t* work = c.buf("k2_work").as<int64_t>(n);
    if (eng == EFG_ENGINE_FACTORIZED)
      efg::factorized_work(c, P, work);
    else
      efg::direct_work(c, P, work);
    std::vector<int64_t> h(n);
    EFG_CUDA_CHECK(cudaMemcpyAsync(h.data(), work, n * sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    EFG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    // inclusive prefix; cut at p * total / parts (first seed whose prefix reaches the target)
    long double total = 0;
    for (int64_t v = 0; v < n; ++v) total += h[v];
    long double acc = 0;
    int p = 1;
    for (int64_t v = 0; v < n && p < parts; ++v) {
      acc += h[v];
      while (p < parts && acc >= total * p / parts) bounds_out[p++] = v + 1;
    }
    for (; p < parts; ++p) bounds_out[p] = n;
    for (p = 1; p <= parts; ++p) bounds_out[p] = std::max(bounds_out[p], bounds_out[p - 1]);
  });
}

int efg_profile_enable(efg_ctx* ctx, int32_t on) {
  return guarded(ctx, [&](Context& c) { c.prof.on = on != 0; });
}

int efg_profile_reset(efg_ctx* ctx) {
  return guarded(ctx, [&](Context& c) { c.prof.totals.clear(); });
}

int efg_profile_report(efg_ctx* ctx, char* buf, int64_t cap) {
  if (!buf || cap < 3) return fail(efg::EFG_INVALID, "bad report buffer");
  return guarded(ctx, [&](Context& c) {
    std::string js = "{";
    bool first = true;
    for (auto& kv : c.prof.totals) {
      if (!first) js += ",";
      first = false;
      js += "\"" + kv.first + "\":[" + std::to_string(kv.second.first) + "," + std::to_string(kv.second.second) + "]";
    }
    js += "}";
    EFG_REQUIRE((int64_t)js.size() < cap, "report buffer too small");
    std::memcpy(buf, js.c_str(), js.size() + 1);
  });
}

int efg_profile_timeline(efg_ctx* ctx, char* buf, int64_t cap) {
  if (!buf || cap < 3) return fail(efg::EFG_INVALID, "bad timeline buffer");
  return guarded(ctx, [&](Context& c) {
    std::string js = "[";
    char item[256];
    for (size_t k = 0; k < c.prof.timeline.size(); ++k) {
      const auto& sp = c.prof.timeline[k];
      snprintf(item, sizeof item, "%s[\"%s\",%.4f,%.4f]", k ? "," : "", sp.name.c_str(), sp.start, sp.ms);
      js += item;
    }
    js += "]";
    EFG_REQUIRE((int64_t)js.size() < cap, "timeline buffer too small");
    std::memcpy(buf, js.c_str(), js.size() + 1);
  });
}

int efg_topk_device(efg_ctx* ctx, const double* d_ef, int64_t n, int64_t k, int64_t* ids_out) {
  if (n < 0 || k < 0 || (k > 0 && !ids_out)) return fail(efg::EFG_INVALID, "bad topk arguments");
  return guarded(ctx, [&](Context& c) {
    const int64_t kk = std::min(k, n);
    if (kk == 0) return;
    int64_t* d_ids = c.buf("t_out").as<int64_t>(kk);
    efg::topk_device(c, d_ef, n, kk, d_ids);
    EFG_CUDA_CHECK(cudaMemcpyAsync(ids_out, d_ids, kk * sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    EFG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  });
}

int efg_topk(efg_ctx* ctx, const double* ef, int64_t n, int64_t k, int64_t* ids_out) {
  if (n < 0 || k < 0 || (n > 0 && !ef) || (k > 0 && !ids_out)) return fail(efg::EFG_INVALID, "bad topk arguments");
  return guarded(ctx, [&](Context& c) {
    const int64_t kk = std::min(k, n);
    if (kk == 0) return;
    const double* d_ef = stage(c, "t_in", ef, n);
    int64_t* d_ids = c.buf("t_out").as<int64_t>(kk);
    efg::topk_device(c, d_ef, n, kk, d_ids);
    EFG_CUDA_CHECK(cudaMemcpyAsync(ids_out, d_ids, kk * sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    EFG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  });
}

int efg_rank_ascending(efg_ctx* ctx, const double* ef, int64_t n, int64_t* order_out) {
  if (n < 0 || (n > 0 && (!ef || !order_out))) return fail(efg::EFG_INVALID, "bad rank arguments");
  return guarded(ctx, [&](Context& c) {
    if (n == 0) return;
    const double* d_ef = stage(c, "t_in", ef, n);
    int64_t* d_order = c.buf("t_out").as<int64_t>(n);
    efg::rank_ascending_device(c, d_ef, n, d_order);
    EFG_CUDA_CHECK(cudaMemcpyAsync(order_out, d_order, n * sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
    EFG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  });
}

int efg_ef_bins(efg_ctx* ctx, const double* ef, int64_t n, int64_t k, double* target_out, int64_t* rep_out) {
  if (k < 1) return fail(efg::EFG_INVALID, "k must be >= 1");
  if (n < 0 || (n > 0 && !ef) || !target_out || !rep_out) return fail(efg::EFG_INVALID, "bad ef_bins arguments");
  return guarded(ctx, [&](Context& c) {
    int64_t distinct = 0;
    if (n > 0) {
      const double* d_ef = stage(c, "t_in", ef, n);
      double* d_t = c.buf("t_bin_t").as<double>(k);
      int64_t* d_r = c.buf("t_out").as<int64_t>(k);
      distinct = efg::ef_bins_device(c, d_ef, n, k, d_t, d_r);
      if (distinct >= k) {
        EFG_CUDA_CHECK(cudaMemcpyAsync(target_out, d_t, k * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        EFG_CUDA_CHECK(cudaMemcpyAsync(rep_out, d_r, k * sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
        EFG_CUDA_CHECK(cudaStreamSynchronize(c.stream));
      }
    }
    EFG_REQUIRE(distinct >= k, "only " + std::to_string(distinct) + " distinct EF values; choose k <= that");
  });
}

}  // extern "C"
