// Internal (C++) interfaces between the efg translation units.
#pragma once
#include <condition_variable>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "../../include/efg.h"

namespace efg {

// Device-resident CSR (Graph arrays of efgraph/graph.py:34-57).
struct DeviceCSR {
  int64_t n = 0, m = 0;
  int64_t* offsets = nullptr;   // [n+1]
  int32_t* nbr = nullptr;       // [2m], strictly ascending per row
  int64_t* orig_ids = nullptr;  // [n]
  DevBuf b_off, b_nbr, b_orig;
  void alloc(int64_t n_, int64_t m_) {
    offsets = b_off.as<int64_t>(n_ + 1);
    nbr = b_nbr.as<int32_t>(2 * m_ > 0 ? 2 * m_ : 1);
    orig_ids = b_orig.as<int64_t>(n_ > 0 ? n_ : 1);
  }
};

struct Profiler {
  struct Rec {
    std::string name;
    cudaEvent_t a, b;
  };
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<Rec> pending;
  std::map<std::string, std::pair<double, int64_t>> totals;  // name -> (ms, launches)
  struct Span {
    std::string name;
    float start, ms;  // start relative to the call's first recorded event
  };
  std::vector<Span> timeline;  // every record of the last resolved call (efg_profile_timeline)
  cudaEvent_t take();
  void resolve();  // after a stream sync
  ~Profiler();
};

// Pageable host -> device copies through a ring of pinned buffers filled by
// host worker threads (stage.cu).  begin(threads) starts the workers; add()
// enqueues a range's pieces on a stream (gate callback + copy + event each)
// and hands them to the workers as it goes; close() says no more pieces come;
// finish() joins the workers.
struct HostStager {
#ifndef EFG_STAGE_PIECE_MB
#define EFG_STAGE_PIECE_MB 8
#endif
#ifndef EFG_STAGE_RING
#define EFG_STAGE_RING 16
#endif
  static constexpr size_t kPiece = size_t(EFG_STAGE_PIECE_MB) << 20;
  static constexpr int kRing = EFG_STAGE_RING;
  struct Piece {
    const char* src;
    char* dst;
    size_t bytes;
  };
  struct Gate {
    HostStager* owner;
    int64_t idx;
  };
  std::vector<char*> bufs;        // kRing pinned buffers of kPiece bytes
  std::vector<cudaEvent_t> ev;    // per piece: its device copy done (guarded by mu)
  std::vector<Piece> pieces;      // guarded by mu
  std::deque<Gate> gates;         // stable addresses (callback arguments)
  std::deque<uint8_t> ready;      // guarded by mu
  size_t piece = kPiece;          // this call's piece size (<= kPiece; EFG_STAGE_PIECE_KB, tests)
  // device-side gates: the copy stream waits on a flag in mapped page-locked
  // memory (cuStreamWaitValue32) that the worker sets after staging the piece
  static constexpr int64_t kFlags = int64_t(1) << 20;
  uint32_t* flags_h = nullptr;    // [kFlags] host view
  void* flags_d = nullptr;        // device view
  void* wait_fn = nullptr;        // cuStreamWaitValue32 (driver entry point), or null: host-function gates
  int64_t flags_used = 0;         // flags set by the previous call (reset at begin)
  int64_t enqueued = 0;           // pieces whose gate / copy / event are on the stream (guarded by mu)
  bool closed = false;            // guarded by mu
  std::mutex mu;
  std::condition_variable cv;
  std::vector<std::thread> workers;
  bool failed = false;
  void begin(int threads);
  void add(cudaStream_t s, void* dst, const void* src, size_t bytes);
  void close();
  void finish();
  ~HostStager();

 private:
  void ensure(size_t npieces);
  void work(int t, int T);
};
bool is_pageable(const void* p);

// Read-only view of a CSR that some caller owns (device pointers).
struct CSRView {
  int64_t n = 0, m2 = 0;                 // m2 = 2m adjacency entries
  const int64_t* offsets = nullptr;
  const int32_t* nbr = nullptr;
};

// Per-call derived arrays (all device pointers into context scratch).
struct Prepared {
  CSRView g;
  int32_t dmax = 0;
  int64_t sum_c2 = 0;           // sum_v C(dv, 2) = cluster_count (graph.py:249-255)
  int32_t* deg = nullptr;       // [n]
  int32_t* nd = nullptr;        // [2m]  degree of each adjacency entry
  int64_t* s1 = nullptr;        // [n]   sum of neighbour degrees
  int64_t* s2 = nullptr;        // [n]   sum of squared neighbour degrees
  double* ftab = nullptr;       // [3*dmax+8]  F[d] = d ln d (0 for d = 0)
  double* gtab = nullptr;       // [3*dmax+8]  G[S] = F(S-6) - F(S-4)
  int64_t ftab_len = 0;
  // degree-ordered orientation: j in Adj+(i) iff (d_j, j) > (d_i, i)
  int32_t* dplus = nullptr;     // [n]   |Adj+(v)|
  int32_t* adjj = nullptr;      // [2m] Adj+ rows as rank labels, slot space: row v at [offsets[v], +dplus[v])
  int32_t* adjd = nullptr;      // [2m] degree of each Adj+ entry
  int32_t* rank_of = nullptr;   // [n]  position in descending (degree, id) order
  int32_t* deg_by_rank = nullptr;  // [n]
  int32_t* by_rank = nullptr;   // [n]  node of each rank label
  int32_t* pc = nullptr;        // [2m] per slot (v->i): |Adj+(i)|
};

struct Context {
  int device = 0;
  int num_sms = kNumSMs;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::map<std::string, DevBuf> bufs;
  std::mutex mu;
  cudaEvent_t ev[16] = {};
  cudaStream_t copy_stream = nullptr;   // host->device staging of efg_expected_force inputs
  cudaEvent_t chunk_ev[9] = {};         // offsets + neighbour chunks resident (kMaxChunks + 1)
  cudaEvent_t aux_ev[2] = {};           // early cluster-total read-back: totals written / copied
  cudaStream_t side_stream = nullptr;   // independent preparation kernels run beside the main stream
  cudaEvent_t side_ev[2] = {};          // fork / join of side_stream
  bool total_sent = false;              // set by the engine when it queued that read-back
  Profiler prof;
  // degrees, F/G tables and rank labels of the last distributed rows part,
  // reused by the listing part that follows on the same graph
  // (prepare_head invalidates it)
  struct {
    Prepared P;
    bool valid = false;
  } dist_head;
  HostStager stager;  // pageable inputs of efg_expected_force
  DeviceCSR csr;  // resident graph of efg_build_graph / efg_rmat_build
  DevBuf& buf(const std::string& name) { return bufs[name]; }
  ~Context();
};

struct SeedRange {
  int64_t lo = 0, hi = 0;
};

// csr_build.cu
void build_csr_device(Context& ctx, const int64_t* d_edges, int64_t k, DeviceCSR& out);

// rmat.cu -- device R-MAT sampler (bit-identical to the reference generator)
void rmat_build_device(Context& ctx, int scale, int64_t avg_degree, const double* probs, const uint64_t* state,
                       const uint64_t* inc, bool& truncated, DeviceCSR& out);

// prep.cu
void prepare(Context& ctx, const CSRView& g, bool need_orientation, Prepared& P);
void prepare_head(Context& ctx, const CSRView& g, bool need_orientation, Prepared& P);
void prepare_rows(Context& ctx, Prepared& P, int64_t r0, int64_t r1, int64_t e0, int64_t e1);
// need_slot_table: the per-slot |Adj+(i)| table P.pc (K2 work, per-seed
// triangle paths); whole-graph listing passes gather it from dplus instead
void prepare_tail(Context& ctx, Prepared& P, bool need_orientation, bool need_slot_table, int64_t r0 = 0,
                  int64_t r1 = -1);  // sorts the Adj+ rows of nodes [r0, r1) (r1 < 0: all)

// Host inputs arriving on a copy stream in row chunks (efg_expected_force):
// work on the rows of chunk k may start once ready[k] has fired (null event:
// already resident).  The offsets are resident before any of it.
constexpr int kMaxChunks = 8;
struct Staging {
  int nchunks = 1;
  int64_t row[kMaxChunks + 1] = {};   // row bounds
  int64_t slot[kMaxChunks + 1] = {};  // offsets[row[k]]
  cudaEvent_t ready[kMaxChunks] = {};
  // whole-graph pass from host inputs: cluster totals depend only on degrees
  // and S1, so they are read back to `total_host` on the copy stream while the
  // listing still runs (the epilogue then skips them)
  int64_t* total_host = nullptr;
};

// ef_factor.cu -- factorised cluster-centric engine
struct PrepInfo {
  int32_t dmax = 0;
  int64_t sum_c2 = 0;
};
// One part of a distributed whole-graph pass.  Part p owns the node range
// [node_lo, node_hi) (efg_part_bounds: contiguous, balanced by row work): its
// rows' neighbour degrees, S1/S2, label-sorted Adj+ rows, chain tables and
// pushes; and it lists the triangles of every nparts-th listing work unit.
// Integer words per node (planar): chain hi / lo / S1 sums [0, 3n), triangle
// hi / lo / count / pad [3n, 7n), S1 [7n, 8n), S2 [8n, 9n) (own rows only);
// the caller sums them over all parts (integer addition, disjoint supports:
// exact in any order) before ef_finish.  Modes:
//   kDistRepl -- efg_ef_partial: every rank prepares ALL rows' orientation
//                itself (no exchange), tables / pushes of its range only;
//   kDistRows -- efg_ef_partial_rows: its range's rows only (neighbour
//                degrees, S1/S2, label-sorted Adj+ rows into the caller's
//                slot-space buffer adjp, |Adj+| into dplus); the caller then
//                exchanges adjp / dplus (each part broadcasts its slot / node
//                range) so that every rank holds all rows;
//   kDistTables -- efg_ef_partial_tables: its range's histograms, chain
//                tables and pushes (runs while the exchange is in flight);
//   kDistList -- efg_ef_partial_list: the listing on the exchanged adjp /
//                dplus (the preceding kDistRows call cleared the words).
constexpr int kDistWords = 9;  // u64 words per node
enum DistMode { kDistRepl = 0, kDistRows = 1, kDistList = 2, kDistTables = 3 };
struct DistPart {
  int32_t part = 0, nparts = 1;
  int mode = kDistRepl;
  int64_t node_lo = 0, node_hi = 0;
  unsigned long long* words = nullptr;  // [kDistWords n]
  double* ws = nullptr;                 // [n]
  int32_t* adjp = nullptr;              // [2m] slot-space Adj+ rows (kDistRows out / kDistList in)
  int32_t* dplus = nullptr;             // [n] |Adj+(v)| (same)
};
// Balanced contiguous node ranges of the distributed pass (bounds[nparts+1], host).
void part_bounds(Context& ctx, const CSRView& g, int32_t nparts, int64_t* bounds);
PrepInfo ef_factorized(Context& ctx, const CSRView& g, const Staging& stg, SeedRange r, double* ef, int64_t* total,
                       uint8_t* flags, int64_t* T_out, double* W_out, efg_stats* st, const DistPart* dp = nullptr);
void ef_finish(Context& ctx, const CSRView& g, SeedRange r, const unsigned long long* words, const double* ws,
               double* ef, int64_t* total, uint8_t* flags, int64_t* T_out, double* W_out);

// ef_direct.cu -- direct per-seed enumeration (original formulation)
void ef_direct(Context& ctx, Prepared& P, SeedRange r, double* ef, int64_t* total, uint8_t* flags,
               int64_t* T_out, double* W_out, efg_stats* st);

// ef_alg1.cu -- Algorithm 1 of the paper (middle-triplet scatter), cross-check engine
void ef_alg1(Context& ctx, Prepared& P, SeedRange r, double* ef, int64_t* total, uint8_t* flags, int64_t* T_out,
             double* W_out, efg_stats* st);

// K2 -- per-seed work estimates (int64 [n]) used for balanced sharding
void factorized_work(Context& ctx, Prepared& P, int64_t* d_work);
void direct_work(Context& ctx, Prepared& P, int64_t* d_work);

// topk.cu -- K5
void topk_device(Context& ctx, const double* d_ef, int64_t n, int64_t k, int64_t* d_ids_out);
// ranking consumers: np.argsort(ef, kind="stable") and ef_bins (analysis.py:84-103, :240)
void rank_ascending_device(Context& ctx, const double* d_ef, int64_t n, int64_t* d_order);
// returns the number of distinct values; outputs are written only when it is >= k
int64_t ef_bins_device(Context& ctx, const double* d_ef, int64_t n, int64_t k, double* d_targets, int64_t* d_rep);

}  // namespace efg
