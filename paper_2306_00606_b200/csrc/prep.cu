// Per-call preparation of the arrays every EF engine reads.
//
// Reference counterparts: g.degrees() (graph.py:63-65), the key span / degree
// bound (expected_force.py:177-180: cluster degree < 3*dmax), and the
// internal-edge test structure (_und_edge_codes + _edge_mask,
// expected_force.py:183-197), which is replaced here by a degree-ordered
// orientation of the CSR: each undirected edge appears once, in the list of
// its lower-ranked endpoint, so every triangle is discovered exactly once per
// member seed.
#include <cub/cub.cuh>

#include "common.cuh"
#include "efg_internal.cuh"

namespace efg {

namespace {

__global__ void k_deg(const int64_t* __restrict__ offsets, int64_t n, int32_t* __restrict__ deg) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v < n) deg[v] = (int32_t)(offsets[v + 1] - offsets[v]);
}

// F[d] = d * ln d, the per-cluster term of W (expected_force.py:318-321 uses
// (c*d)*ln d per histogram row; per cluster c = 1).
__global__ void k_ftab(double* __restrict__ F, int64_t len) {
  int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d < len) F[d] = d > 0 ? (double)d * log((double)d) : 0.0;
}

// G[S] = F(S-6) - F(S-4): the W change of one triangle cluster unit (S = dv+di+dj >= 6).
__global__ void k_gtab(const double* __restrict__ F, double* __restrict__ G, int64_t len) {
  int64_t S = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (S < len) G[S] = S >= 6 ? F[S - 6] - F[S - 4] : 0.0;
}

__device__ __forceinline__ bool ranks_above(int32_t dj, int32_t j, int32_t di, int32_t i) {
  return dj > di || (dj == di && j > i);
}

// Warp per row: s1[v] = sum of neighbour degrees, s2[v] = sum of their
// squares, and (with the orientation) Adj+(v) = the neighbours ranking above
// v, compacted in order as rank labels + degrees into v's own slot range
// [offsets[v], offsets[v] + dplus[v]) -- slot space, so no scan is needed and
// the pass runs per row chunk while the rest of the graph is still copied.
constexpr int kRowUnroll = 4;
#ifndef EFG_ROW_THREADS
#define EFG_ROW_THREADS 256
#endif
constexpr int kRowThreads = EFG_ROW_THREADS;
#ifndef EFG_RANK_KEYS32
#define EFG_RANK_KEYS32 1
#endif
constexpr bool kRankKeys32 = EFG_RANK_KEYS32;
#ifndef EFG_SORT_LARGE_PER_SM
#define EFG_SORT_LARGE_PER_SM 8
#endif
#ifndef EFG_SORT_SMALL_PER_SM
#define EFG_SORT_SMALL_PER_SM 32  // k_sort_small ms (r02): 8: 0.46, 16: 0.41, 32: 0.38-0.39
#endif
// Rows longer than kRowBig (hubs) would be one warp's serial chain of
// dependent loads (the top R-MAT22 hub: 965 steps, ~1 ms); with the
// orientation they go to the first kRowBigBlocks CTAs of the same launch,
// which walk the ranks in descending degree order, a CTA per row.
constexpr int32_t kRowBig = 2048;
#ifndef EFG_ROW_BIG_BLOCKS
#define EFG_ROW_BIG_BLOCKS 296  // hub-row CTAs of k_row_sums (r02: 74: 1.33 ms, 148: 0.96, 296: 0.89, 592-888: 0.885)
#endif
constexpr int kRowBigBlocks = EFG_ROW_BIG_BLOCKS;

__device__ __forceinline__ void row_sums_big(const int64_t* __restrict__ offsets, const int32_t* __restrict__ nbr,
                                             int32_t* __restrict__ nd, const int32_t* __restrict__ deg,
                                             int64_t r0, int64_t r1,
                                             int64_t* __restrict__ s1, int64_t* __restrict__ s2,
                                             int32_t* __restrict__ dplus, const int32_t* __restrict__ rank_of,
                                             int32_t* __restrict__ adjj, int32_t* __restrict__ adjd,
                                             const int32_t* __restrict__ by_rank,
                                             const int32_t* __restrict__ deg_by_rank, int64_t n, int32_t nbig) {
  constexpr int T = kRowThreads, NW = T / 32, U = kRowUnroll;
  __shared__ int wc[U * NW];
  __shared__ int64_t ws[NW], wq[NW];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t r = blockIdx.x; r < n; r += nbig) {
    if (deg_by_rank[r] <= kRowBig) break;  // ranks are in descending degree order
    const int32_t v = by_rank[r];
    if (v < r0 || v >= r1) continue;
    const int64_t b = offsets[v], e = offsets[v + 1];
    const int32_t dv = (int32_t)(e - b);
    int64_t s = 0, q = 0, out = b;
    // tiles of T*U slots; slot order (k, thread) is kept by a scan of the
    // per-(k, warp) counts, so Adj+(v) comes out exactly as the warp path writes it
    for (int64_t p0 = b; p0 < e; p0 += T * U) {
      int32_t j[U], dj[U], lab[U];
      bool take[U];
      unsigned msk[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int64_t p = p0 + T * k + threadIdx.x;
        j[k] = p < e ? nbr[p] : 0;
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {  // neighbour degrees (written out as nd: k_nd fused here)
        const int64_t p = p0 + T * k + threadIdx.x;
        dj[k] = p < e ? __ldg(deg + j[k]) : 0;
        lab[k] = p < e ? __ldg(rank_of + j[k]) : 0;
        if (p < e) nd[p] = dj[k];
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        take[k] = false;
        if (p0 + T * k + threadIdx.x < e) {
          s += dj[k];
          q += (int64_t)dj[k] * dj[k];
          take[k] = ranks_above(dj[k], j[k], dv, v);
        }
        msk[k] = __ballot_sync(0xffffffffu, take[k]);
        if (lane == 0) wc[k * NW + w] = __popc(msk[k]);
      }
      __syncthreads();
      int64_t before[U];
      int total = 0;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        for (int x = 0; x < NW; ++x) {
          if (x == w) before[k] = total;
          total += wc[k * NW + x];
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k)
        if (take[k]) {
          const int64_t o = EFG_CLAMP(out + before[k] + __popc(msk[k] & ((1u << lane) - 1)), e);
          adjj[o] = lab[k];
          adjd[o] = dj[k];
        }
      out += total;
      __syncthreads();  // wc is rewritten by the next tile
    }
    for (int o = 16; o; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      q += __shfl_xor_sync(0xffffffffu, q, o);
    }
    if (lane == 0) {
      ws[w] = s;
      wq[w] = q;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t ts = 0, tq = 0;
      for (int x = 0; x < NW; ++x) {
        ts += ws[x];
        tq += wq[x];
      }
      s1[v] = ts;
      s2[v] = tq;
      dplus[v] = (int32_t)(out - b);
    }
    __syncthreads();
  }
}

// One row by the whole warp: neighbour degrees, S1 / S2, Adj+ (slot space).
__device__ __forceinline__ void row_sums_warp(const int64_t* __restrict__ offsets, const int32_t* __restrict__ nbr,
                                              int32_t* __restrict__ nd, const int32_t* __restrict__ deg, int64_t v,
                                              int64_t* __restrict__ s1, int64_t* __restrict__ s2,
                                              int32_t* __restrict__ dplus, const int32_t* __restrict__ rank_of,
                                              int32_t* __restrict__ adjj, int32_t* __restrict__ adjd, int lane) {
  int64_t b = offsets[v], e = offsets[v + 1];
  int32_t dv = (int32_t)(e - b);
  int64_t s = 0, q = 0;
  int64_t out = b;
  if (dv <= 32) {  // most rows: one group, no unrolled predicated tail
    const bool in = lane < dv;
    const int32_t j = in ? nbr[b + lane] : 0, dj = in ? __ldg(deg + j) : 0;
    const int32_t lab = in && adjj ? __ldg(rank_of + j) : 0;  // used only where taken
    if (in) nd[b + lane] = dj;
    const bool take = in && ranks_above(dj, j, dv, (int32_t)v);
    int32_t s32 = dj;  // dv <= 32 neighbours of degree < 2^31 each: s fits 64 bits, q per lane too
    int64_t q64 = (int64_t)dj * dj;
    const unsigned mask = __ballot_sync(0xffffffffu, take);
    if (take && adjj) {
      const int64_t o = b + __popc(mask & ((1u << lane) - 1));
      adjj[o] = lab;
      adjd[o] = dj;
    }
    s = s32;
    q = q64;
    out = b + __popc(mask);
  } else {
  // kRowUnroll groups of 32 per iteration: all loads of a group are in flight
  // together (hub rows are one warp's serial chain otherwise)
  constexpr int U = kRowUnroll;
  for (int64_t p0 = b; p0 < e; p0 += 32 * U) {
    int32_t j[U], dj[U], lab[U];
    bool take[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t p = p0 + 32 * k + lane;
      j[k] = p < e ? nbr[p] : 0;
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t p = p0 + 32 * k + lane;
      dj[k] = p < e ? __ldg(deg + j[k]) : 0;
      lab[k] = p < e && adjj ? __ldg(rank_of + j[k]) : 0;
      if (p < e) nd[p] = dj[k];
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      take[k] = false;
      if (p0 + 32 * k + lane < e) {
        s += dj[k];
        q += (int64_t)dj[k] * dj[k];
        take[k] = ranks_above(dj[k], j[k], dv, (int32_t)v);
      }
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const unsigned mask = __ballot_sync(0xffffffffu, take[k]);
      if (take[k] && adjj) {
        const int64_t o = EFG_CLAMP(out + __popc(mask & ((1u << lane) - 1)), e);
        adjj[o] = lab[k];
        adjd[o] = dj[k];
      }
      out += __popc(mask);
    }
  }
  }
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    q += __shfl_xor_sync(0xffffffffu, q, o);
  }
  if (lane == 0) {
    s1[v] = s;
    s2[v] = q;
    dplus[v] = (int32_t)(out - b);
  }
}

// Rows [r0, r1): four consecutive rows per warp.  A quad whose rows all have
// degree <= 8 (most rows of a skewed graph: 1.46 M of R-MAT22's 2.18 M) is
// done by 8-lane groups in one step; other quads take their rows one after
// another with the whole warp.  Rows of degree > kRowBig belong to the first
// nbig CTAs (row_sums_big).
__global__ void __launch_bounds__(kRowThreads) k_row_sums(
    const int64_t* __restrict__ offsets, const int32_t* __restrict__ nbr, int32_t* __restrict__ nd,
    const int32_t* __restrict__ deg, int64_t r0, int64_t r1, int64_t* __restrict__ s1, int64_t* __restrict__ s2, int32_t* __restrict__ dplus,
    const int32_t* __restrict__ rank_of, int32_t* __restrict__ adjj, int32_t* __restrict__ adjd,
    const int32_t* __restrict__ by_rank, const int32_t* __restrict__ deg_by_rank, int64_t n, int32_t nbig) {
  if ((int32_t)blockIdx.x < nbig) {
    row_sums_big(offsets, nbr, nd, deg, r0, r1, s1, s2, dplus, rank_of, adjj, adjd, by_rank, deg_by_rank, n, nbig);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int64_t v0 = r0 + 4 * (((blockIdx.x - nbig) * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (v0 >= r1) return;
  const int g = lane >> 3, t = lane & 7;
  const int64_t vg = v0 + g;
  const bool valid = vg < r1;
  const int64_t bg = valid ? offsets[vg] : 0;
  const int32_t dg = valid ? (int32_t)(offsets[vg + 1] - bg) : 0;
  if (__all_sync(0xffffffffu, dg <= 8)) {
    const bool in = t < dg;
    const int32_t j = in ? nbr[bg + t] : 0, dj = in ? __ldg(deg + j) : 0;
    const int32_t lab = in && adjj ? __ldg(rank_of + j) : 0;
    if (in) nd[bg + t] = dj;
    const bool take = in && ranks_above(dj, j, dg, (int32_t)vg);
    int64_t sg = dj, qg = (int64_t)dj * dj;
    for (int o = 4; o; o >>= 1) {  // within the 8-lane group
      sg += __shfl_xor_sync(0xffffffffu, sg, o);
      qg += __shfl_xor_sync(0xffffffffu, qg, o);
    }
    const unsigned gm = (__ballot_sync(0xffffffffu, take) >> (8 * g)) & 0xffu;
    if (take && adjj) {
      const int64_t o = EFG_CLAMP(bg + __popc(gm & ((1u << t) - 1)), bg + dg);
      adjj[o] = lab;
      adjd[o] = dj;
    }
    if (t == 0 && valid) {
      s1[vg] = sg;
      s2[vg] = qg;
      dplus[vg] = __popc(gm);
    }
    return;
  }
  if (__all_sync(0xffffffffu, dg <= 32)) {
    // all four rows fit one 32-lane step: lane e takes slot e of every row, the four
    // rows' loads and gathers issued together (one row after another was four
    // dependent load chains per warp)
    int64_t bk[4];
    int32_t dk[4], jk[4], djk[4], labk[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      bk[k] = __shfl_sync(0xffffffffu, bg, 8 * k);
      dk[k] = __shfl_sync(0xffffffffu, dg, 8 * k);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) jk[k] = lane < dk[k] ? nbr[bk[k] + lane] : 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool in = lane < dk[k];
      djk[k] = in ? __ldg(deg + jk[k]) : 0;
      labk[k] = in && adjj ? __ldg(rank_of + jk[k]) : 0;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t v = v0 + k;
      const bool in = lane < dk[k];
      if (in) nd[bk[k] + lane] = djk[k];
      const bool take = in && ranks_above(djk[k], jk[k], dk[k], (int32_t)v);
      const unsigned mask = __ballot_sync(0xffffffffu, take);
      if (take && adjj) {
        const int64_t o = EFG_CLAMP(bk[k] + __popc(mask & ((1u << lane) - 1)), bk[k] + dk[k]);
        adjj[o] = labk[k];
        adjd[o] = djk[k];
      }
      int64_t sv = djk[k], qv = (int64_t)djk[k] * djk[k];
      for (int o = 16; o; o >>= 1) {
        sv += __shfl_xor_sync(0xffffffffu, sv, o);
        qv += __shfl_xor_sync(0xffffffffu, qv, o);
      }
      if (lane == k && v < r1) {
        s1[v] = sv;
        s2[v] = qv;
        dplus[v] = __popc(mask);
      }
    }
    return;
  }
  for (int k = 0; k < 4 && v0 + k < r1; ++k) {
    const int64_t v = v0 + k;
    if (nbig > 0 && offsets[v + 1] - offsets[v] > kRowBig) continue;  // a hub: one of the first nbig CTAs has it
    row_sums_warp(offsets, nbr, nd, deg, v, s1, s2, dplus, rank_of, adjj, adjd, lane);
  }
}

// Per adjacency slot e = (v -> i): how long Adj+(i) is (it starts at offsets[i]: slot space).
__global__ void k_slot_plus(const int32_t* __restrict__ nbr, int64_t m2, const int32_t* __restrict__ dplus,
                            int32_t* __restrict__ pc) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m2) return;
  pc[e] = dplus[nbr[e]];
}

// Rank label of each node: its position in descending (degree, id) order, so
// j in Adj+(i) iff rank(j) < rank(i) and the frequent probe targets (high
// degree) get small labels.
__global__ void k_rank_keys(const int32_t* __restrict__ deg, int64_t n, int32_t dmax, uint64_t* __restrict__ key,
                            int32_t* __restrict__ val) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  key[v] = ((uint64_t)(uint32_t)(dmax - deg[v]) << 32) | (uint32_t)(n - 1 - v);
  val[v] = (int32_t)v;
}

// stable variant: position i holds node n-1-i (ids descending), the key is its
// degree's distance below dmax only -- an LSD radix sort keeps equal keys in
// that order, so a log2(dmax)-bit sort gives the (degree desc, id desc) order
__global__ void k_rank_keys32(const int32_t* __restrict__ deg, int64_t n, int32_t dmax, uint32_t* __restrict__ key,
                              int32_t* __restrict__ val) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t v = n - 1 - i;
  key[i] = (uint32_t)(dmax - deg[v]);
  val[i] = (int32_t)v;
}

__global__ void k_rank_scatter(const int32_t* __restrict__ by_rank, int64_t n, const int32_t* __restrict__ deg,
                               int32_t* __restrict__ rank_of, int32_t* __restrict__ deg_by_rank) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int32_t v = by_rank[r];
  rank_of[v] = (int32_t)r;
  deg_by_rank[r] = deg[v];
}

// ---- Adj+ rows sorted by label (ascending): the triangle listing stops a
// row scan at the first label >= rank(v).  Rows are short (|Adj+| <= sqrt(2m)),
// so one warp sorts a row in registers: a bitonic network over 32*I labels,
// I per lane in blocked order (within-lane stages are register min/max,
// cross-lane stages shuffles).  Degrees are re-gathered by label afterwards.
template <int I>
__device__ __forceinline__ void sort_row(int32_t* __restrict__ row, int32_t* __restrict__ rowd, int p, int lane,
                                         const int32_t* __restrict__ deg_by_rank) {
  uint32_t x[I];
#pragma unroll
  for (int i = 0; i < I; ++i) {  // any input arrangement: load coalesced
    const int t = i * 32 + lane;
    x[i] = t < p ? (uint32_t)row[t] : 0xffffffffu;
  }
  warp_bitonic<I>(x, lane);
#pragma unroll
  for (int i = 0; i < I; ++i) {  // sorted in blocked order
    const int t = lane * I + i;
    if (t < p) {
      row[t] = (int32_t)x[i];
      rowd[t] = __ldg(deg_by_rank + x[i]);
    }
  }
}

// Warp per row (register bitonic sort up to 1024 entries; longer rows, rare,
// rank by counting through a scratch row).  Two kernels keep the short-row
// kernel's registers low.
// Sort one Adj+ row (pv >= 2 entries) by label.
template <bool SMALL>
__device__ __forceinline__ void sort_one(int64_t b, int pv, int lane, const int32_t* __restrict__ deg_by_rank,
                                         int32_t* __restrict__ adjj, int32_t* __restrict__ adjd,
                                         int32_t* __restrict__ scratch) {
  int32_t* row = adjj + b;
  int32_t* rowd = adjd + b;
  if (SMALL) {
    if (pv <= 32) sort_row<1>(row, rowd, pv, lane, deg_by_rank);
    else if (pv <= 64) sort_row<2>(row, rowd, pv, lane, deg_by_rank);
    else if (pv <= 128) sort_row<4>(row, rowd, pv, lane, deg_by_rank);
    else sort_row<8>(row, rowd, pv, lane, deg_by_rank);
  } else if (pv <= 512) {
    sort_row<16>(row, rowd, pv, lane, deg_by_rank);
  } else if (pv <= 1024) {
    sort_row<32>(row, rowd, pv, lane, deg_by_rank);
  } else {
    for (int t = lane; t < pv; t += 32) {
      const int32_t key = row[t];
      int32_t rank = 0;
      for (int o = 0; o < pv; ++o) rank += row[o] < key;
      scratch[b + rank] = key;
    }
    __syncwarp();
    for (int t = lane; t < pv; t += 32) {
      row[t] = scratch[b + t];
      rowd[t] = __ldg(deg_by_rank + row[t]);
    }
  }
  __syncwarp();
}

// A row of 2..16 entries sorted by ONE thread in registers (a 16-input bitonic
// network, padding sorts last): most Adj+ rows are this short (low-degree
// nodes have few higher-ranked neighbours), and a warp-wide sort per such row
// left most lanes idle.
__device__ __forceinline__ void sort_row_thread16(int32_t* __restrict__ row, int32_t* __restrict__ rowd, int p,
                                                  const int32_t* __restrict__ deg_by_rank) {
  uint32_t x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = i < p ? (uint32_t)row[i] : 0xffffffffu;
#pragma unroll
  for (int k = 2; k <= 16; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const uint32_t lo = min(x[i], x[l]), hi = max(x[i], x[l]);
          const bool up = (i & k) == 0;
          x[i] = up ? lo : hi;
          x[l] = up ? hi : lo;
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 16; ++i)
    if (i < p) {
      row[i] = (int32_t)x[i];
      rowd[i] = __ldg(deg_by_rank + x[i]);
    }
}

// Rows of 2..256 entries of nodes [r0, r1): rows of <= 16 entries a thread each,
// the longer ones a warp each (per group of 32 nodes).
__global__ void k_sort_small(const int64_t* __restrict__ offsets, const int32_t* __restrict__ dplus, int64_t r0, int64_t r1,
                             const int32_t* __restrict__ deg_by_rank, int32_t* __restrict__ adjj,
                             int32_t* __restrict__ adjd, int32_t* __restrict__ scratch) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r0 + g * 32 < r1; g += nw) {
    const int64_t mine = r0 + g * 32 + lane;
    int p = 0;
    if (mine < r1) p = dplus[mine];
    if (p >= 2 && p <= 16) {
      const int64_t b = offsets[mine];
      sort_row_thread16(adjj + b, adjd + b, p, deg_by_rank);
    }
    unsigned todo = __ballot_sync(0xffffffffu, p > 16 && p <= 256);
    while (todo) {
      const int x = __ffs(todo) - 1;
      todo &= todo - 1;
      const int pv = __shfl_sync(0xffffffffu, p, x);
      sort_one<true>(offsets[r0 + g * 32 + x], pv, lane, deg_by_rank, adjj, adjd, scratch);
    }
  }
}

// Rows of more than 256 entries belong to nodes of degree > 256: a warp per
// node in rank (descending degree) order, so the long rows -- clustered at
// low ids in R-MAT graphs -- spread over all warps.
__global__ void k_sort_large(const int64_t* __restrict__ offsets, const int32_t* __restrict__ dplus, int64_t n,
                             const int32_t* __restrict__ by_rank, const int32_t* __restrict__ deg_by_rank,
                             int32_t* __restrict__ adjj, int32_t* __restrict__ adjd, int32_t* __restrict__ scratch,
                             int64_t r0, int64_t r1) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    if (deg_by_rank[r] <= 256) break;
    const int32_t v = by_rank[r];
    if (v < r0 || v >= r1) continue;  // another part's row
    const int pv = dplus[v];
    if (pv > 256) sort_one<false>(offsets[v], pv, lane, deg_by_rank, adjj, adjd, scratch);
  }
}

struct Choose2 {
  __host__ __device__ int64_t operator()(const int32_t& d) const { return (int64_t)d * (d - 1) / 2; }
};

}  // namespace

// Offsets-only part: degrees, dmax (the one host sync), the F/G tables and
// the rank labels.  Runs while the neighbour arrays may still be in flight.
void prepare_head(Context& ctx, const CSRView& g, bool need_orientation, Prepared& P) {
  ctx.dist_head.valid = false;  // its buffers are about to be rewritten
  cudaStream_t s = ctx.stream;
  const int B = 256;
  P.g = g;
  const int64_t n = g.n, m2 = g.m2;
  P.deg = ctx.buf("deg").as<int32_t>(n);
  P.nd = ctx.buf("nd").as<int32_t>(m2);
  P.s1 = ctx.buf("s1").as<int64_t>(n);
  P.s2 = ctx.buf("s2").as<int64_t>(n);
  EFG_LAUNCH(k_deg, ceil_div(n, B), B, 0, s, g.offsets, n, P.deg);
  // dmax -> F table length (cluster degree <= 3*dmax - 4)
  int32_t* dmax_d = ctx.buf("dmax").as<int32_t>(1);
  size_t tmp = 0;
  EFG_CUDA_CHECK(cub::DeviceReduce::Max(nullptr, tmp, P.deg, dmax_d, n, s));
  EFG_REGION("cub::DeviceReduce::Max", s, EFG_CUDA_CHECK(cub::DeviceReduce::Max(ctx.buf("cub").get(tmp), tmp, P.deg, dmax_d, n, s)));
  int32_t dmax = 0;
  EFG_CUDA_CHECK(cudaMemcpyAsync(&dmax, dmax_d, sizeof dmax, cudaMemcpyDeviceToHost, s));
  EFG_CUDA_CHECK(cudaStreamSynchronize(s));
  P.dmax = dmax;
  {
    cub::TransformInputIterator<int64_t, Choose2, const int32_t*> c2(P.deg, Choose2{});
    int64_t* sum_d = ctx.buf("sumc2").as<int64_t>(1);
    EFG_CUDA_CHECK(cub::DeviceReduce::Sum(nullptr, tmp, c2, sum_d, n, s));
    EFG_REGION("cub::DeviceReduce::Sum", s, EFG_CUDA_CHECK(cub::DeviceReduce::Sum(ctx.buf("cub").get(tmp), tmp, c2, sum_d, n, s)));
    EFG_CUDA_CHECK(cudaMemcpyAsync(&P.sum_c2, sum_d, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  }
  P.ftab_len = 3 * (int64_t)(dmax > 1 ? dmax : 1) + 8;
  P.ftab = ctx.buf("ftab").as<double>(P.ftab_len);
  EFG_LAUNCH(k_ftab, ceil_div(P.ftab_len, B), B, 0, s, P.ftab, P.ftab_len);
  P.gtab = ctx.buf("gtab").as<double>(P.ftab_len);
  EFG_LAUNCH(k_gtab, ceil_div(P.ftab_len, B), B, 0, s, P.ftab, P.gtab, P.ftab_len);
  if (!need_orientation) return;
  EFG_REQUIRE(m2 / 2 < (int64_t(1) << 31), "more than 2^31-1 edges: oriented adjacency index exceeds int32");
  int32_t* val = ctx.buf("rank_val").as<int32_t>(2 * n);
  if (kRankKeys32) {  // stable sort on the degree alone (3 passes at dmax ~ 1e5 instead of 7)
    uint32_t* key = ctx.buf("rank_key32").as<uint32_t>(2 * n);
    EFG_LAUNCH(k_rank_keys32, ceil_div(n, B), B, 0, s, P.deg, n, dmax, key, val);
    int bits = 1;
    while (bits < 32 && (uint64_t(1) << bits) <= (uint64_t)dmax) ++bits;
    EFG_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, key + n, val, val + n, n, 0, bits, s));
    EFG_REGION("cub::DeviceRadixSort::SortPairs", s,
               EFG_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(ctx.buf("cub").get(tmp), tmp, key, key + n, val, val + n,
                                                              n, 0, bits, s)));
  } else {
    uint64_t* key = ctx.buf("rank_key").as<uint64_t>(2 * n);
    EFG_LAUNCH(k_rank_keys, ceil_div(n, B), B, 0, s, P.deg, n, dmax, key, val);
    int bits = 32;
    while (bits < 64 && (uint64_t(1) << (bits - 32)) <= (uint64_t)dmax) ++bits;
    EFG_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, key + n, val, val + n, n, 0, bits, s));
    EFG_REGION("cub::DeviceRadixSort::SortPairs", s,
               EFG_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(ctx.buf("cub").get(tmp), tmp, key, key + n, val,
                                                              val + n, n, 0, bits, s)));
  }
  P.rank_of = ctx.buf("rank_of").as<int32_t>(n);
  P.deg_by_rank = ctx.buf("deg_by_rank").as<int32_t>(n);
  EFG_LAUNCH(k_rank_scatter, ceil_div(n, B), B, 0, s, val + n, n, P.deg, P.rank_of, P.deg_by_rank);
  P.by_rank = val + n;
  // Adj+ in slot space: row v at [offsets[v], offsets[v] + dplus[v])
  P.adjj = ctx.buf("adjj").as<int32_t>(m2 > 0 ? m2 : 1);
  P.adjd = ctx.buf("adjd").as<int32_t>(m2 > 0 ? m2 : 1);
}

// Rows [r0, r1) (slots [e0, e1)) whose neighbours are resident: neighbour
// degrees, S1, S2 and (with the orientation) Adj+ in slot space.
void prepare_rows(Context& ctx, Prepared& P, int64_t r0, int64_t r1, int64_t, int64_t) {
  cudaStream_t s = ctx.stream;
  if (!P.dplus) P.dplus = ctx.buf("dplus").as<int32_t>(P.g.n > 0 ? P.g.n : 1);  // (or the caller's buffer)
  const int32_t nbig = P.rank_of ? kRowBigBlocks : 0;  // hub CTAs need the rank order
  EFG_LAUNCH(k_row_sums, nbig + ceil_div(ceil_div(r1 - r0, 4) * 32, kRowThreads), kRowThreads, 0, s, P.g.offsets,
             P.g.nbr, P.nd,
             P.deg, r0, r1, P.s1, P.s2, P.dplus, P.rank_of, P.rank_of ? P.adjj : nullptr, P.adjd, P.by_rank, P.deg_by_rank,
             P.g.n, nbig);
}

// Everything that needs all neighbours: the label-sorted orientation.
void prepare_tail(Context& ctx, Prepared& P, bool need_orientation, bool need_slot_table, int64_t r0, int64_t r1) {
  if (!need_orientation) return;
  cudaStream_t s = ctx.stream;
  const int B = 256;
  const CSRView& g = P.g;
  const int64_t n = g.n, m2 = g.m2;
  {
    // rows sorted by label: a row scan for a higher-ranked v can stop at v (triangle listing)
    int32_t* scratch = ctx.buf("adjj_scratch").as<int32_t>(m2 > 0 ? m2 : 1);
    if (r1 < 0) r1 = n;
    const int64_t groups = ceil_div(r1 - r0, 32);
    // the few long rows (> 256 entries, a warp each for a long time) sort on
    // the side stream while the short rows and the slot table fill the GPU
    EFG_CUDA_CHECK(cudaEventRecord(ctx.side_ev[0], s));
    EFG_CUDA_CHECK(cudaStreamWaitEvent(ctx.side_stream, ctx.side_ev[0], 0));
    EFG_LAUNCH(k_sort_large, EFG_SORT_LARGE_PER_SM * ctx.num_sms, B, 0, ctx.side_stream, g.offsets, P.dplus, n, P.by_rank,
               P.deg_by_rank, P.adjj, P.adjd, scratch, r0, r1);
    EFG_CUDA_CHECK(cudaEventRecord(ctx.side_ev[1], ctx.side_stream));
    EFG_LAUNCH(k_sort_small, std::min<int64_t>(ceil_div(groups * 32, B), EFG_SORT_SMALL_PER_SM * ctx.num_sms), B, 0, s,
               g.offsets,
               P.dplus, r0, r1, P.deg_by_rank, P.adjj, P.adjd, scratch);
  }
  if (need_slot_table) {
    P.pc = ctx.buf("pc").as<int32_t>(m2);
    EFG_LAUNCH(k_slot_plus, ceil_div(m2, B), B, 0, s, g.nbr, m2, P.dplus, P.pc);
  }
  EFG_CUDA_CHECK(cudaStreamWaitEvent(s, ctx.side_ev[1], 0));  // join: rows sorted
}

void prepare(Context& ctx, const CSRView& g, bool need_orientation, Prepared& P) {
  prepare_head(ctx, g, need_orientation, P);
  prepare_rows(ctx, P, 0, g.n, 0, g.m2);
  prepare_tail(ctx, P, need_orientation, true);
}

EFG_CHECK_ACCESSOR(check_line_prep)

}  // namespace efg
