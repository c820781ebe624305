// K3 (factorised) -- per-seed Expected Force by degree-histogram factorisation.
//
// Replaces the reference's enumeration hot loop (expected_force.py:222-276
// `_chunk_histograms`, :212-216 `_cluster_keys`, :191-197 `_edge_mask`) and
// its entropy pass (:306-328 `_scores_from_histograms`).  For a seed v with
// A = Adj(v), dv = |A|, every size-3 cluster rooted at v is
//   star  {v,i,j}, i<j in A:          d = dv+di+dj-4-2[i~j], weight 2
//   chain v->i->k, k in Adj(i)\{v}:   d = dv+di+dk-4-2[k~v], weight 1
// (expected_force.py:375-390).  EF needs
//   T = sum w d (exact, int64), mass = sum w, W = sum w d ln d,
//   EF = ln T - W/T  (expected_force.py:322-324).
// The clusters are not visited one by one.  They are summed in classes:
//   * chains through i without the triangle term depend on v only through
//     dv, so C_i(y) = sum_x H_i(x) F(y+di-4+x) - F(2y+di-4) is tabulated
//     once per (i, distinct neighbour degree y) and looked up by each seed;
//   * stars without the triangle term depend on (di, dj) only: a
//     self-convolution of v's neighbour-degree histogram H_v, which equals
//     v's own chain table weighted by H_v:
//       2[sum_{a<b} h_a h_b F(dv-4+x_a+x_b) + sum_a C(h_a,2) F(dv-4+2x_a)]
//         = sum_b h_b C_v(x_b)                    (|D_v| terms, no pair loop);
//   * a cluster whose three nodes form a triangle has degree D-2 instead of
//     D = dv+di+dj-4; each triangle at v carries star weight 2 and two chains
//     (v->i->j, v->j->i), so the correction is 4 (F(D-2) - F(D)) per triangle,
//     found once per seed through the degree-ordered orientation Adj+.
// T and mass have closed forms given the triangle count t(v):
//   T    = 2C(dv,2)(dv-4) + 2(dv-1)S1(v) + sum_i [(di-1)(dv+di-4) + S1(i) - dv] - 8 t(v)
//   mass = dv(dv-1) + S1(v) - dv          (test_expected_force.py:139-147)
// All sums run in a fixed order per seed (no atomics on values), so results
// are bitwise reproducible and independent of sharding.
#include <cstdlib>

#include <cub/cub.cuh>

#include "common.cuh"
#include "efg_internal.cuh"

namespace efg {

namespace {

constexpr int kHashSlots = 8192;     // smem hash of Adj(v) for dv <= 4096
constexpr int kHashMaxDeg = kHashSlots / 2;

struct FArgs {
  const int64_t* offsets;
  const int32_t* nbr;
  const int32_t* nd;       // degree of each adjacency entry
  const int64_t* s1;
  const double* F;
  const double* G;         // G[S] = F(S-6) - F(S-4): triangle correction per unit weight
  const int64_t* PT;       // P[S] = rint(G[S] 2^40): triangle sums are exact integers (any order, any path)
  const uint64_t* PQ;      // Q = -P (the block listing's table)
  int64_t flen;            // F / G / PT table length (bounds-checked builds)
  const int32_t* pc;       // [2m] |Adj+(nbr[e])|
  const int32_t* adjj;     // oriented adjacency Adj+ as rank labels
  const int32_t* adjd;     // degree of each Adj+ entry
  const int32_t* deg;
  const int32_t* rank_of;      // node -> rank label
  const int32_t* deg_by_rank;  // rank label -> degree
  const int32_t* dcnt;     // |D_i|: H_i = hkey/hcnt[offsets[i], offsets[i] + dcnt[i])
  const int32_t* hkey;
  const int32_t* hcnt;
  const int4* rowhash;     // bucketed hash of Adj+(i) for |Adj+(i)| >= kRevMin, at bucket 2*offsets[i]
  // per node: pushed chain sums (see chain_push) and the stars term
  const int64_t* s2;
  const unsigned long long* cwh;
  const unsigned long long* cwl;
  const unsigned long long* cp2;
  const double* cws;
  double c0;
  int64_t seed_lo;
  // per-seed partials, index v - seed_lo
  int64_t* tri;
  int64_t* Wth;  // W_t in fixed point, two words: (sum of P >> 32, sum of P & (2^32 - 1)), P = rint(G 2^40)
  int64_t* Wtl;
};

// ---------------------------------------------------------------- H build
// H_i (the histogram of the degrees of Adj(i): distinct values ascending, with
// counts) is stored in adjacency-slot space: row i occupies hkey/hcnt
// [offsets[i], offsets[i] + dcnt[i]) (|D_i| <= d_i), so no scan/compaction pass
// is needed.  Size classes: d <= 32 a warp per row
// (bitonic sort, k_hist_warp), 32 < d <= 256 a warp per row (32x8 register
// bitonic sort, k_hist_warp8), 256 < d <= 2048 a CTA per row (radix sort,
// k_hist_block), d > 2048 windowed counting (k_hist_count).

// d <= 32: warp per row, 32-lane bitonic sort of the neighbour degrees.
__global__ void k_hist_warp(const int32_t* __restrict__ rows, int64_t count, const int64_t* __restrict__ offsets,
                            const int32_t* __restrict__ nd, int32_t* __restrict__ hkey, int32_t* __restrict__ hcnt,
                            int32_t* __restrict__ dcnt) {
  const int lane = threadIdx.x & 31;
  const int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (q >= count) return;
  const int32_t i = rows[q];
  const int64_t b = offsets[i];
  const int d = (int)(offsets[i + 1] - b);
  int32_t x = lane < d ? nd[b + lane] : 0x7fffffff;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int32_t y = __shfl_xor_sync(0xffffffffu, x, j);
      const bool up = (lane & k) == 0;          // ascending block
      const bool lower = (lane & j) == 0;
      x = (lower == up) ? min(x, y) : max(x, y);
    }
  }
  const int32_t prev = __shfl_up_sync(0xffffffffu, x, 1);
  const bool head = lane < d && (lane == 0 || x != prev);
  const unsigned heads = __ballot_sync(0xffffffffu, head);
  if (head) {
    const unsigned above = heads & ~((2u << lane) - 1);   // heads after this lane
    const int next = above ? __ffs(above) - 1 : d;
    const int r = __popc(heads & ((1u << lane) - 1));
    hkey[b + r] = x;
    hcnt[b + r] = next - lane;
  }
  if (lane == 0) dcnt[i] = __popc(heads);
}

// 32 < d <= 256: warp per row, the neighbour degrees sorted in registers
// (32x8 bitonic), run heads by comparison with the left neighbour, their
// positions compacted by a warp scan; counts = distance to the next head.
#ifndef EFG_HIST_W8_WARPS
#define EFG_HIST_W8_WARPS 8
#endif
constexpr int kHistW8Warps = EFG_HIST_W8_WARPS;
__global__ void __launch_bounds__(kHistW8Warps * 32)
k_hist_warp8(const int32_t* __restrict__ rows, int64_t count, const int64_t* __restrict__ offsets,
             const int32_t* __restrict__ nd, int32_t* __restrict__ hkey, int32_t* __restrict__ hcnt,
             int32_t* __restrict__ dcnt) {
  __shared__ int32_t hpos[kHistW8Warps][257];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (q >= count) return;
  const int32_t i = rows[q];
  const int64_t b = offsets[i];
  const int d = (int)(offsets[i + 1] - b);
  uint32_t x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int p = lane * 8 + u;
    x[u] = p < d ? (uint32_t)nd[b + p] : 0xffffffffu;
  }
  warp_bitonic<8>(x, lane);
  const uint32_t left = __shfl_up_sync(0xffffffffu, x[7], 1);
  bool hd[8];
  int nh = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int p = lane * 8 + u;
    const uint32_t prev = u == 0 ? left : x[u > 0 ? u - 1 : 0];
    hd[u] = p < d && (p == 0 || x[u] != prev);
    nh += hd[u];
  }
  int incl = nh;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  int rank = incl - nh;
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (hd[u]) {
      hpos[w][rank] = lane * 8 + u;
      hkey[b + rank] = (int32_t)x[u];
      ++rank;
    }
  if (lane == 0) hpos[w][total] = d;
  __syncwarp();
  for (int r = lane; r < total; r += 32) hcnt[b + r] = hpos[w][r + 1] - hpos[w][r];
  if (lane == 0) dcnt[i] = total;
}

#ifndef EFG_HIST_THREADS
#define EFG_HIST_THREADS 128  // k_hist_block (rows of 257..2048 slots) ms (r02): 128: 0.470, 256: 0.489, 512: 0.766
#endif
constexpr int kHistThreads = EFG_HIST_THREADS, kHistItems = 2048 / EFG_HIST_THREADS;  // rows of <= 2048 slots
// 256 < d <= THREADS*ITEMS (2048): CTA per row, radix sort in shared memory
// over the bits degrees actually use (keys < 2^bits; padding = 2^bits - 1
// sorts last).
template <int kHistThreads, int kHistItems>
__global__ void __launch_bounds__(kHistThreads)
k_hist_block(const int32_t* __restrict__ rows, int64_t count, const int64_t* __restrict__ offsets,
             const int32_t* __restrict__ nd, int32_t* __restrict__ hkey, int32_t* __restrict__ hcnt,
             int32_t* __restrict__ dcnt, int bits) {
  using Sort = cub::BlockRadixSort<uint32_t, kHistThreads, kHistItems>;
  using Scan = cub::BlockScan<int32_t, kHistThreads>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  } tmp;
  __shared__ uint32_t keys[kHistThreads * kHistItems + 1];
  __shared__ int32_t hpos[kHistThreads * kHistItems + 1];
  const int64_t q = blockIdx.x;
  if (q >= count) return;
  const int32_t i = rows[q];
  const int64_t b = offsets[i];
  const int d = (int)(offsets[i + 1] - b);
  uint32_t k[kHistItems];
  const uint32_t pad = (1u << bits) - 1;
#pragma unroll
  for (int u = 0; u < kHistItems; ++u) {
    const int p = threadIdx.x * kHistItems + u;
    k[u] = p < d ? (uint32_t)nd[b + p] : pad;
  }
  Sort(tmp.sort).Sort(k, 0, bits);  // blocked arrangement, ascending
#pragma unroll
  for (int u = 0; u < kHistItems; ++u) keys[threadIdx.x * kHistItems + u] = k[u];
  __syncthreads();
  int32_t nh = 0;
  bool hd[kHistItems];
#pragma unroll
  for (int u = 0; u < kHistItems; ++u) {
    const int p = threadIdx.x * kHistItems + u;
    hd[u] = p < d && (p == 0 || keys[p] != keys[p - 1]);
    nh += hd[u];
  }
  int32_t rank, total;
  Scan(tmp.scan).ExclusiveSum(nh, rank, total);
#pragma unroll
  for (int u = 0; u < kHistItems; ++u) {
    if (hd[u]) {
      hpos[rank] = threadIdx.x * kHistItems + u;
      hkey[b + rank] = (int32_t)k[u];
      ++rank;
    }
  }
  if (threadIdx.x == 0) hpos[total] = d;
  __syncthreads();
  for (int r = threadIdx.x; r < total; r += kHistThreads) hcnt[b + r] = hpos[r + 1] - hpos[r];
  if (threadIdx.x == 0) dcnt[i] = total;
}

// d > 2048: CTA per row, counting instead of sorting.  Degrees are counted
// in shared-memory windows of kHistWin consecutive values (direct-mapped
// counters, native shared atomics); the window's nonzero counters are then
// compacted in ascending order by a block scan.  Windows are visited from
// the smallest degree up, jumping over empty value ranges (next window = the
// smallest degree not yet counted), so a row costs one pass per non-empty
// window (R-MAT22 hubs: 1-8).  Values past the first window are mostly the
// degrees of other hubs -- few -- so the first pass also collects them
// (<= kHistOvf) and counts them by pairwise comparison instead of further
// window passes over the whole row.
#ifndef EFG_HIST_BIG_THREADS
#define EFG_HIST_BIG_THREADS 512
#endif
constexpr int kHistWin = 16384, kHistBigThreads = EFG_HIST_BIG_THREADS, kHistOvf = 2048;
__global__ void __launch_bounds__(kHistBigThreads)
k_hist_count(const int32_t* __restrict__ rows, int64_t count, const int64_t* __restrict__ offsets,
             const int32_t* __restrict__ nd, int32_t* __restrict__ hkey, int32_t* __restrict__ hcnt,
             int32_t* __restrict__ dcnt) {
  extern __shared__ int32_t wcnt[];  // kHistWin
  using Scan = cub::BlockScan<int32_t, kHistBigThreads>;
  using Red = cub::BlockReduce<int32_t, kHistBigThreads>;
  __shared__ union {
    typename Scan::TempStorage scan;
    typename Red::TempStorage red;
  } tmp;
  __shared__ int32_t next_lo, novf;
  __shared__ int32_t ovf[kHistOvf];
  constexpr int kPer = kHistWin / kHistBigThreads;  // counters per thread in the compaction
  const int64_t q = blockIdx.x;
  if (q >= count) return;
  const int32_t i = rows[q];
  const int64_t b = offsets[i];
  const int d = (int)(offsets[i + 1] - b);
  // smallest degree of the row: first window
  int32_t mn = INT32_MAX;
  for (int p = threadIdx.x; p < d; p += kHistBigThreads) mn = min(mn, nd[b + p]);
  mn = Red(tmp.red).Reduce(mn, cub::Min());
  if (threadIdx.x == 0) next_lo = mn;
  __syncthreads();
  int32_t lo = next_lo, base = 0;
  bool first = true;
  while (lo != INT32_MAX) {
    for (int k = threadIdx.x; k < kHistWin; k += kHistBigThreads) wcnt[k] = 0;
    if (threadIdx.x == 0) novf = 0;
    __syncthreads();
    int32_t nxt = INT32_MAX;  // smallest degree beyond this window
    for (int p = threadIdx.x; p < d; p += kHistBigThreads) {
      const int32_t k = nd[b + p];
      if (k >= lo && k - lo < kHistWin) {
        atomicAdd(&wcnt[k - lo], 1);
      } else if (k >= lo) {
        nxt = min(nxt, k);
        if (first) {  // values past the first window: few (hub degrees), kept for one small sort
          const int32_t at = atomicAdd(&novf, 1);
          if (at < kHistOvf) ovf[at] = k;
        }
      }
    }
    nxt = Red(tmp.red).Reduce(nxt, cub::Min());
    if (threadIdx.x == 0) next_lo = nxt;
    __syncthreads();
    // ascending compaction of the nonzero counters: thread t owns [t*kPer, (t+1)*kPer)
    int32_t nz = 0;
#pragma unroll 4
    for (int u = 0; u < kPer; ++u) nz += wcnt[threadIdx.x * kPer + u] != 0;
    int32_t rank, total;
    Scan(tmp.scan).ExclusiveSum(nz, rank, total);
    rank += base;
    for (int u = 0; u < kPer; ++u) {
      const int32_t c = wcnt[threadIdx.x * kPer + u];
      if (c) {
        hkey[b + rank] = lo + threadIdx.x * kPer + u;
        hcnt[b + rank] = c;
        ++rank;
      }
    }
    base += total;
    lo = next_lo;
    __syncthreads();
    if (first) {
      first = false;
      const int32_t no = novf;
      if (no <= kHistOvf) {
        // all values past the first window are in ovf: distinct values and
        // their counts by pairwise comparison (no <= kHistOvf), appended in
        // ascending order after the window's entries.  wcnt is free now.
        for (int e = threadIdx.x; e < no; e += kHistBigThreads) {
          const int32_t x = ovf[e];
          int32_t c = 0;
          bool lead = true;
          for (int f = 0; f < no; ++f) {
            const bool eq = ovf[f] == x;
            c += eq;
            lead &= !(eq && f < e);
          }
          wcnt[e] = lead ? c : 0;
        }
        __syncthreads();
        int32_t mine = 0;
        for (int e = threadIdx.x; e < no; e += kHistBigThreads) {
          if (wcnt[e] == 0) continue;
          const int32_t x = ovf[e];
          int32_t r = 0;
          for (int f = 0; f < no; ++f) r += wcnt[f] != 0 && ovf[f] < x;
          hkey[b + base + r] = x;
          hcnt[b + base + r] = wcnt[e];
          ++mine;
        }
        const int32_t nd_ovf = Red(tmp.red).Sum(mine);
        if (threadIdx.x == 0) next_lo = nd_ovf;
        __syncthreads();
        base += next_lo;
        break;
      }
    }
  }
  if (threadIdx.x == 0) dcnt[i] = base;
}

// Chain table, group of G lanes per row i: for every distinct neighbour
// degree y of i, C_i(y) = sum_a h_a F[y + di - 4 + x_a] - F[2y + di - 4].
template <int G>
__global__ void k_ctab_group(const int32_t* __restrict__ rows, int64_t count, const int64_t* __restrict__ offsets,
                             const int32_t* __restrict__ dcnt, const int32_t* __restrict__ hkey,
                             const int32_t* __restrict__ hcnt, const int32_t* __restrict__ deg,
                             const double* __restrict__ F, double* __restrict__ ctab, int64_t flen,
                             int max_d = 0x7fffffff) {
  const int sub = threadIdx.x & (G - 1);
  int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  if (q >= count) return;
  const int32_t i = rows[q];
  if (dcnt[i] > max_d) return;  // k_ctab_block's
  int64_t b = offsets[i], e = b + dcnt[i];
  int32_t di = deg[i];
  for (int64_t o = b + sub; o < e; o += G) {
    int32_t y = hkey[o];
    int64_t base = (int64_t)y + di - 4;
    double acc = 0.0;
    for (int64_t a = b; a < e; ++a)
      acc += (double)__ldg(hcnt + a) * __ldg(F + EFG_CLAMP(base + __ldg(hkey + a), flen));
    ctab[o] = acc - __ldg(F + EFG_CLAMP(base + y, flen));
  }
}

// Rows with many distinct degrees: one CTA per row, threads over outputs.
// The direct terms' inputs are staged in shared memory (counts as doubles) in
// chunks of kCtabStage entries, and every thread carries up to kCtabOut
// outputs (y = its own + T, + 2T, ...) so one staged (x, h) pair feeds
// kCtabOut F gathers + FMAs.
//
// Far field: inputs are grouped in geometric tiles over x (tile t covers
// x in [base (1.25^t - 1), base (1.25^(t+1) - 1)), base = di - 3).  For a
// tile with centre xc and members x_a = xc + delta_a, Taylor-expanding
// F(s) = s ln s about Z = y + di - 4 + xc,
//   sum_a h_a F(Z + delta_a) = F(Z) (m0 + m1/Z) + m1 + sum_{j=1..K} c_j Z^-j,
//   c_j = (-1)^(j+1) m_{j+1} / (j (j+1)),  m_k = sum_a h_a delta_a^k,
// and Z >= base + x_first bounds |delta|/Z by 0.135 (checked per tile), so
// the truncation at K = 15 is below 1e-16 of the sum.  Tiles of at least
// kExpMin members are expanded (one F gather + K FMAs per output instead of
// one gather per member; R-MAT22: 92 % of the terms); the rest are summed
// term by term.  Fixed per-output summation order (deterministic).
constexpr int kCtabStage = 1024;
#ifndef EFG_CTAB_THREADS
#define EFG_CTAB_THREADS 128
#endif
constexpr int kCtabThreads = EFG_CTAB_THREADS;
constexpr int kCtabOut = 4;
constexpr int kExpK = 15, kExpTiles = 64, kExpGrid = kCtabThreads, kExpMin = 12, kExpMinD = 128;
#ifndef EFG_CTAB_WARP_D
#define EFG_CTAB_WARP_D 128
#endif
constexpr int kCtabWarpD = EFG_CTAB_WARP_D;  // rows with fewer distinct degrees: a warp each, direct
static_assert(kCtabWarpD % 32 == 0 && kCtabWarpD <= 512, "k_ctab_warp: 32 x OUT staged inputs (rows past kExpMinD go direct there)");
constexpr double kExpRatio = 0.135;
#ifndef EFG_EXP_GROWTH
#define EFG_EXP_GROWTH 1.25f
#endif
constexpr float kExpGrowth = EFG_EXP_GROWTH;  // tile t: x in [base (g^t - 1), base (g^(t+1) - 1))

template <int K>
__device__ __forceinline__ void ctab_outputs(const int32_t* __restrict__ sx, const double* __restrict__ sh, int nq,
                                             const int64_t (&base)[kCtabOut], const double* __restrict__ F,
                                             double (&acc)[kCtabOut]) {
  const double* Fb[K];  // per-output table base: one 32-bit index per gather
#pragma unroll
  for (int k = 0; k < K; ++k) Fb[k] = F + base[k];
#pragma unroll 4
  for (int q = 0; q < nq; ++q) {
    const int32_t x = sx[q];
    const double h = sh[q];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = fma(h, __ldg(Fb[k] + x), acc[k]);
  }
}

// Rows of degree > 64 with fewer than kCtabWarpD distinct neighbour degrees
// (half of k_ctab_block's rows at R-MAT22, 4.5 % of its terms): a warp each.
// The inputs (x, h) are staged in the warp's shared slice once, each lane
// carries up to 4 outputs (y = its own + 32, + 64, + 96) and every staged pair
// feeds their F gathers -- the same fma sequence per output as k_ctab_block's
// direct path (inputs in ascending order), so the values are identical.
#ifndef EFG_CTAB_WARPS
#define EFG_CTAB_WARPS 4  // 4 / 8 / 16 warps per CTA: 0.512 / 0.538 / 0.71 ms (r02)
#endif
constexpr int kCtabWarps = EFG_CTAB_WARPS;
template <int OUT>
__global__ void __launch_bounds__(kCtabWarps * 32)
k_ctab_warp(const int32_t* __restrict__ rows, int64_t count, const int64_t* __restrict__ offsets,
            const int32_t* __restrict__ dcnt, const int32_t* __restrict__ hkey, const int32_t* __restrict__ hcnt,
            const int32_t* __restrict__ deg, const double* __restrict__ F, double* __restrict__ ctab, int64_t flen,
            int max_d) {
  __shared__ int32_t sx[kCtabWarps][32 * OUT];
  __shared__ double sh[kCtabWarps][32 * OUT];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (q >= count) return;
  const int32_t i = rows[q];
  const int D = dcnt[i];
  if (D > max_d) return;  // k_ctab_block's
  const int64_t b = offsets[i];
  const int32_t di = deg[i];
  for (int a = lane; a < D; a += 32) {
    sx[w][a] = hkey[b + a];
    sh[w][a] = (double)hcnt[b + a];
  }
  __syncwarp();
  int64_t base[OUT];
  int32_t yk[OUT];
  double acc[OUT];
#pragma unroll
  for (int k = 0; k < OUT; ++k) {
    const int o = lane + 32 * k;
    yk[k] = o < D ? sx[w][o] : sx[w][0];  // past-the-end outputs shadow the first one
    base[k] = (int64_t)yk[k] + di - 4;
    acc[k] = 0.0;
  }
  const int K = (D + 31) >> 5;  // warp-uniform
  for (int a = 0; a < D; ++a) {
    const int32_t x = sx[w][a];
    const double h = sh[w][a];
#pragma unroll
    for (int k = 0; k < OUT; ++k)
      if (k < K) acc[k] = fma(h, __ldg(F + EFG_CLAMP(base[k] + x, flen)), acc[k]);
  }
#pragma unroll
  for (int k = 0; k < OUT; ++k) {
    const int o = lane + 32 * k;
    if (o < D) ctab[b + o] = acc[k] - __ldg(F + EFG_CLAMP(base[k] + yk[k], flen));
  }
}

// tile of input x (fast single precision: a boundary off by one only moves a
// member to a neighbouring tile, and every expanded tile's ratio is checked)
__device__ __forceinline__ int exp_tile(int32_t x, float inv_base, float inv_lg) {
  return (int)fminf(__log2f(fmaf((float)x, inv_base, 1.0f)) * inv_lg, (float)kExpGrid);
}

#ifndef EFG_CTAB_MINB
#define EFG_CTAB_MINB 8  // <= 64 registers: 8 CTAs per SM (measured 2.78 ms vs 3.94 at 1 and 2.84 unbounded)
#endif
__global__ void __launch_bounds__(kCtabThreads, EFG_CTAB_MINB)
k_ctab_block(const int32_t* __restrict__ rows, int64_t nrows, const int64_t* __restrict__ offsets,
             const int32_t* __restrict__ dcnt, const int32_t* __restrict__ hkey, const int32_t* __restrict__ hcnt,
             const int32_t* __restrict__ deg, const double* __restrict__ F, double* __restrict__ ctab,
             int exp_min, int exp_min_d, int64_t flen, int min_d = 0) {
  __shared__ int32_t sx[kCtabStage];
  __shared__ double sh[kCtabStage];
  __shared__ int32_t tbeg[kExpGrid], tend[kExpGrid];
  __shared__ int32_t ebeg[kExpTiles], eend[kExpTiles], exc[kExpTiles];  // expanded tiles: entries, centre
  __shared__ double ecoef[kExpTiles][kExpK + 2];                         // m0, m1, c_1..c_K
  __shared__ int32_t rlo[kExpTiles + 1], rpre[kExpTiles + 2];            // direct ranges: start, prefix
  __shared__ int32_t emp[kExpTiles], wcnt[kCtabThreads / 32], wmem[kCtabThreads / 32];
  __shared__ int32_t sne;
  const int64_t r = blockIdx.x;
  if (r >= nrows) return;
  const int32_t i = rows[r];
  const int64_t b = offsets[i];
  const int D = dcnt[i];
  if (D < min_d) return;  // a warp's row (k_ctab_group<32>)
  const int32_t di = deg[i];
  constexpr int T = kCtabThreads;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int ne = 0, nr = 1;
  if (D >= exp_min_d) {
    const double tb = (double)(di - 3);
    const float inv_base = 1.0f / (float)tb, inv_l125 = 1.0f / log2f(kExpGrowth);
    for (int t = threadIdx.x; t < kExpGrid; t += T) tbeg[t] = -1;
    __syncthreads();
    for (int a = threadIdx.x; a < D; a += T) {
      const int t = exp_tile(hkey[b + a], inv_base, inv_l125);
      if (t < kExpGrid) {
        if (a == 0 || exp_tile(hkey[b + a - 1], inv_base, inv_l125) != t) tbeg[t] = a;
        if (a == D - 1 || exp_tile(hkey[b + a + 1], inv_base, inv_l125) != t) tend[t] = a + 1;
      }
    }
    __syncthreads();
    {  // thread t judges grid tile t; expanded tiles compacted in ascending order by a block scan
      static_assert(kExpGrid == T, "one grid tile per thread");
      const int t = threadIdx.x;
      const int32_t a0 = tbeg[t], a1 = a0 >= 0 ? tend[t] : 0;
      int32_t xc = 0;
      bool ok = a0 >= 0 && a1 - a0 >= exp_min;
      if (ok) {
        const int32_t x0 = hkey[b + a0], x1 = hkey[b + a1 - 1];
        xc = (x0 + x1) >> 1;
        ok = (double)max(xc - x0, x1 - xc) <= kExpRatio * (tb + (double)x0);
      }
      const int own = ok ? a1 - a0 : 0;
      int f = ok, mem = own;  // inclusive warp prefix of (flag, members)
      for (int o = 1; o < 32; o <<= 1) {
        const int fu = __shfl_up_sync(0xffffffffu, f, o), mu = __shfl_up_sync(0xffffffffu, mem, o);
        if (lane >= o) f += fu, mem += mu;
      }
      if (lane == 31) wcnt[w] = f, wmem[w] = mem;
      __syncthreads();
      int fb = 0, mb = 0, ft = 0;
      for (int u = 0; u < T / 32; ++u) {
        if (u < w) fb += wcnt[u], mb += wmem[u];
        ft += wcnt[u];
      }
      const int e = fb + f - ok;  // tiles past kExpTiles stay direct
      if (ok && e < kExpTiles) {
        ebeg[e] = a0;
        eend[e] = a1;
        exc[e] = xc;
        emp[e] = mb + mem - own;  // members of the expanded tiles before e
      }
      const int n_e = min(ft, kExpTiles);
      __syncthreads();
      if (t <= n_e) {  // direct range t = [eend[t-1] or 0, ebeg[t] or D), rpre = direct entries before it
        const int32_t lo = t ? eend[t - 1] : 0;
        const int32_t mp = t < n_e ? emp[t] : (n_e ? emp[n_e - 1] + eend[n_e - 1] - ebeg[n_e - 1] : 0);
        rlo[t] = lo;
        rpre[t] = lo - mp;
        if (t == n_e) rpre[t + 1] = D - mp;
      }
      if (t == 0) sne = n_e;
    }
    __syncthreads();
    ne = sne;
    nr = ne + 1;

    // moments: warp per expanded tile, fixed lane order and butterfly
    for (int e = w; e < ne; e += T / 32) {
      double m[kExpK + 2];
#pragma unroll
      for (int k = 0; k < kExpK + 2; ++k) m[k] = 0.0;
      const int32_t xc = exc[e];
      for (int a = ebeg[e] + lane; a < eend[e]; a += 32) {
        const double dl = (double)(hkey[b + a] - xc);
        double p = (double)hcnt[b + a];
#pragma unroll
        for (int k = 0; k < kExpK + 2; ++k) {
          m[k] += p;
          p *= dl;
        }
      }
#pragma unroll
      for (int k = 0; k < kExpK + 2; ++k)
        for (int o = 16; o; o >>= 1) m[k] += __shfl_xor_sync(0xffffffffu, m[k], o);
      if (lane == 0) {
        ecoef[e][0] = m[0];
        ecoef[e][1] = m[1];
#pragma unroll
        for (int j = 1; j <= kExpK; ++j) ecoef[e][1 + j] = ((j & 1) ? m[j + 1] : -m[j + 1]) / (double)(j * (j + 1));
      }
    }
  } else if (threadIdx.x == 0) {
    rlo[0] = 0;
    rpre[0] = 0;
    rpre[1] = D;
  }
  __syncthreads();
  const int Dd = rpre[nr];  // direct inputs
  for (int o0 = 0; o0 < D; o0 += T * kCtabOut) {
    const int K = min(kCtabOut, (D - o0 + T - 1) / T);  // block-uniform
    int64_t base[kCtabOut];
    int32_t yk[kCtabOut];
    double acc[kCtabOut];
#pragma unroll
    for (int k = 0; k < kCtabOut; ++k) {
      const int o = o0 + threadIdx.x + k * T;
      yk[k] = o < D ? hkey[b + o] : hkey[b];  // past-the-end outputs shadow the first one
      base[k] = (int64_t)yk[k] + di - 4;
      acc[k] = 0.0;
    }
    for (int q0 = 0; q0 < Dd; q0 += kCtabStage) {
      const int nq = min(kCtabStage, Dd - q0);
      __syncthreads();
      for (int q = threadIdx.x; q < nq; q += T) {
        const int qq = q0 + q;
        int lo = 0, hi = nr - 1;  // last range with rpre <= qq
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (rpre[mid] <= qq) lo = mid;
          else hi = mid - 1;
        }
        const int64_t a = b + rlo[lo] + (qq - rpre[lo]);
        sx[q] = hkey[a];
        sh[q] = (double)hcnt[a];
      }
      __syncthreads();
      static_assert(kCtabOut <= 8, "ctab_outputs dispatch covers K <= 8");
      switch (K) {
        case 1: ctab_outputs<1>(sx, sh, nq, base, F, acc); break;
        case 2: ctab_outputs<2>(sx, sh, nq, base, F, acc); break;
        case 3: ctab_outputs<3>(sx, sh, nq, base, F, acc); break;
        case 4: ctab_outputs<4>(sx, sh, nq, base, F, acc); break;
        case 5: ctab_outputs<kCtabOut >= 5 ? 5 : 1>(sx, sh, nq, base, F, acc); break;
        case 6: ctab_outputs<kCtabOut >= 6 ? 6 : 1>(sx, sh, nq, base, F, acc); break;
        case 7: ctab_outputs<kCtabOut >= 7 ? 7 : 1>(sx, sh, nq, base, F, acc); break;
        default: ctab_outputs<kCtabOut>(sx, sh, nq, base, F, acc); break;
      }
    }
    for (int e = 0; e < ne; ++e) {
      const double* co = ecoef[e];
      const int32_t xc = exc[e];
#pragma unroll
      for (int k = 0; k < kCtabOut; ++k) {
        if (k >= K) break;
        const int64_t Z = base[k] + xc;
        const double FZ = __ldg(F + EFG_CLAMP(Z, flen)), t = 1.0 / (double)Z;
        double poly = co[1 + kExpK];
#pragma unroll
        for (int j = kExpK - 1; j >= 1; --j) poly = fma(poly, t, co[1 + j]);
        acc[k] += fma(FZ, fma(co[1], t, co[0]), fma(t, poly, co[1]));
      }
    }
#pragma unroll
    for (int k = 0; k < kCtabOut; ++k) {
      const int o = o0 + threadIdx.x + k * T;
      if (o < D) ctab[b + o] = acc[k] - __ldg(F + EFG_CLAMP(base[k] + yk[k], flen));
    }
  }
}

// ---------------------------------------------------------------- per seed
template <class T>
__device__ __forceinline__ T warp_sum(T x) {
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Block-wide fixed-order sum (deterministic); result valid in thread 0.
template <int THREADS, class T>
__device__ __forceinline__ T block_sum(T x, T* scratch) {
  x = warp_sum(x);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[w] = x;
  __syncthreads();
  T r = 0;
  if (threadIdx.x == 0)
    for (int k = 0; k < THREADS / 32; ++k) r += scratch[k];
  return r;
}

// Chains, pushed.  Seed v's chain term is W_c(v) = sum_{i in A(v)} C_i(dv):
// instead of every seed searching dv in each neighbour's table, each row i
// pushes C_i(d_v) to every neighbour v right after computing its table
// (rows are local: keys and values are contiguous, the lookup stays in
// registers / shared memory).  Pushed values are summed in fixed point per
// node, two words (hi = floor(x), lo = frac(x) 2^32, x = C 2^-e) with a
// per-degree scale 2^e >= dv dmax F(3 dmax) 2^-62 >= W_c(v) 2^-62, so the
// integer sums cannot overflow and keep >= 2^-94 of the bound: exact to far
// below the EF tolerance, and independent of the order of the pushes.  The
// exact integer part of the chain count, sum_i S1(i), is pushed alongside.
struct ChainAcc {
  unsigned long long* wh;  // [n] sum of hi words
  unsigned long long* wl;  // [n] sum of lo words
  unsigned long long* p2;  // [n] sum_{i in A(v)} S1(i)
  double* ws;              // [n] stars: sum_b h_b C_v(x_b)
  double c0;               // dmax F(3 dmax)
};

__host__ __device__ __forceinline__ int chain_exp(int64_t dv, double c0) {
  return ilogb((double)dv * c0) + 1 - 62;
}

__device__ __forceinline__ void chain_push(const ChainAcc& ca, int32_t v, int32_t dv, double val, int64_t s1i) {
  const double x = ldexp(val, -chain_exp(dv, ca.c0));
  const double f = floor(x);
  atomicAdd(ca.wh + v, (unsigned long long)(int64_t)f);
  atomicAdd(ca.wl + v, (unsigned long long)(int64_t)ldexp(x - f, 32));
  atomicAdd(ca.p2 + v, (unsigned long long)s1i);
}

// d <= 32, fused: one warp per row i does the histogram, the chain table and
// the pushes in registers (nothing of H_i or C_i reaches memory).  Lane e
// holds slot e; the sorted degrees' run heads give H_i in lanes 0..D-1; lane
// k computes C_i(key_k) over the D keys (shuffled in), and each slot takes the
// value of its degree's run.  Same table values as k_hist_warp + k_ctab_group
// (same summation order).
#ifndef EFG_SMALL_WARPS
#define EFG_SMALL_WARPS 4
#endif
constexpr int kSmallWarps = EFG_SMALL_WARPS;
__global__ void __launch_bounds__(kSmallWarps * 32)
k_small_rows(const int32_t* __restrict__ rows, int64_t count, const int64_t* __restrict__ offsets,
                             const int32_t* __restrict__ nbr, const int32_t* __restrict__ nd,
                             const int32_t* __restrict__ deg, const double* __restrict__ F,
                             const int64_t* __restrict__ s1, ChainAcc ca, int64_t flen) {
  const int lane = threadIdx.x & 31;
  const int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (q >= count) return;
  const int32_t i = rows[q];
  const int64_t b = offsets[i];
  const int d = (int)(offsets[i + 1] - b);
  const int32_t y = lane < d ? nd[b + lane] : 0x7fffffff;  // this slot's neighbour degree
  (void)deg;
  int32_t x = y;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int32_t o = __shfl_xor_sync(0xffffffffu, x, j);
      const bool up = (lane & k) == 0;
      const bool lower = (lane & j) == 0;
      x = (lower == up) ? min(x, o) : max(x, o);
    }
  }
  const int32_t prev = __shfl_up_sync(0xffffffffu, x, 1);
  const bool head = lane < d && (lane == 0 || x != prev);
  const unsigned heads = __ballot_sync(0xffffffffu, head);
  const int D = __popc(heads);
  // run k (k < D): key and count, gathered into lane k
  __shared__ int2 runs[kSmallWarps][32];
  const int w = threadIdx.x >> 5;
  if (head) {
    const unsigned after = heads & ~((2u << lane) - 1);  // heads after this lane
    const int nxt = after ? __ffs(after) - 1 : d;
    runs[w][__popc(heads & ((1u << lane) - 1))] = make_int2(x, nxt - lane);
  }
  __syncwarp();
  int32_t key = 0x7fffffff, cntk = 0;
  if (lane < D) {
    key = runs[w][lane].x;
    cntk = runs[w][lane].y;
  }
  // chain table: C_i(key_k) = sum_a h_a F[key_k + di - 4 + x_a] - F[2 key_k + di - 4].
  // The only negative argument is an isolated edge (di = 1, key = 1: -1), whose
  // table is exactly 0 (no chain leaves it); clamping to F[0] = 0 keeps it 0
  // without reading before the table.
  const int64_t base = (int64_t)key + d - 4;
  double c = 0.0;
  for (int a = 0; a < D; ++a) {
    const int32_t xa = __shfl_sync(0xffffffffu, key, a);
    const int32_t ha = __shfl_sync(0xffffffffu, cntk, a);
    if (lane < D) c += (double)ha * __ldg(F + EFG_CLAMP(max(base + xa, (int64_t)0), flen));
  }
  if (lane < D) c -= __ldg(F + EFG_CLAMP(max(base + key, (int64_t)0), flen));
  const double hc = warp_sum(lane < D ? (double)cntk * c : 0.0);
  if (lane == 0) ca.ws[i] = hc;
  // pushes: slot e takes C of its degree's run
  int idx = 0;
  for (int k = 0; k < D; ++k)
    if (__shfl_sync(0xffffffffu, key, k) == y) idx = k;
  const double val = __shfl_sync(0xffffffffu, c, idx);
  if (lane < d) chain_push(ca, nbr[b + lane], y, val, s1[i]);
}

// d <= 8 (1.46 M of R-MAT22's 2.18 M rows): the same fused histogram / table /
// pushes with 8 lanes per row, four rows per warp.  The table values and the
// stars term are those of k_small_rows bit for bit (same per-output order;
// the 32-lane reduction tree only adds zeros beyond lane 8).
__global__ void __launch_bounds__(kSmallWarps * 32)
k_small_rows8(const int32_t* __restrict__ rows, int64_t count, const int64_t* __restrict__ offsets,
              const int32_t* __restrict__ nbr, const int32_t* __restrict__ nd, const double* __restrict__ F,
              const int64_t* __restrict__ s1, ChainAcc ca, int64_t flen) {
  const int lane = threadIdx.x & 31, g = lane >> 3, t = lane & 7, w = threadIdx.x >> 5;
  const int64_t q0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 4;
  if (q0 >= count) return;  // warp-uniform
  const int64_t q = q0 + g;
  const bool valid = q < count;
  const int32_t i = valid ? rows[q] : 0;
  const int64_t b = valid ? offsets[i] : 0;
  const int d = valid ? (int)(offsets[i + 1] - b) : 0;
  const int32_t y = t < d ? nd[b + t] : 0x7fffffff;
  int32_t x = y;
#pragma unroll
  for (int k = 2; k <= 8; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int32_t o = __shfl_xor_sync(0xffffffffu, x, j);
      const bool up = (t & k) == 0;
      const bool lower = (t & j) == 0;
      x = (lower == up) ? min(x, o) : max(x, o);
    }
  }
  const int32_t prev = __shfl_up_sync(0xffffffffu, x, 1);
  const bool head = t < d && (t == 0 || x != prev);
  const unsigned heads = (__ballot_sync(0xffffffffu, head) >> (8 * g)) & 0xffu;
  const int D = __popc(heads);
  __shared__ int2 runs[kSmallWarps][32];
  if (head) {
    const unsigned after = heads & ~((2u << t) - 1);
    const int nxt = after ? __ffs(after) - 1 : d;
    runs[w][8 * g + __popc(heads & ((1u << t) - 1))] = make_int2(x, nxt - t);
  }
  __syncwarp();
  int32_t key = 0x7fffffff, cntk = 0;
  if (t < D) {
    key = runs[w][8 * g + t].x;
    cntk = runs[w][8 * g + t].y;
  }
  const int64_t base = (int64_t)key + d - 4;
  double c = 0.0;
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const int32_t xa = __shfl_sync(0xffffffffu, key, 8 * g + a);
    const int32_t ha = __shfl_sync(0xffffffffu, cntk, 8 * g + a);
    if (t < D && a < D) c += (double)ha * __ldg(F + EFG_CLAMP(max(base + xa, (int64_t)0), flen));
  }
  if (t < D) c -= __ldg(F + EFG_CLAMP(max(base + key, (int64_t)0), flen));
  double hc = t < D ? (double)cntk * c : 0.0;
  for (int o = 4; o; o >>= 1) hc += __shfl_xor_sync(0xffffffffu, hc, o);
  if (t == 0 && valid) ca.ws[i] = hc;
  int idx = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (__shfl_sync(0xffffffffu, key, 8 * g + k) == y && k < D) idx = k;
  const double val = __shfl_sync(0xffffffffu, c, 8 * g + idx);
  if (t < d) chain_push(ca, nbr[b + t], y, val, s1[i]);
}

// d > 32: CTA per row.  Keys below kPushDirect (most neighbour degrees) are
// located through a direct-mapped shared table (key -> position; only keys
// present are ever read, so it needs no clearing), larger ones by binary
// search over H_i's keys (shared memory, global beyond kPushKeys).
#ifndef EFG_PUSH_THREADS
#define EFG_PUSH_THREADS 128
#endif
#ifndef EFG_PUSH_SLICES
#define EFG_PUSH_SLICES 8  // k_push_block ms (r02): 4: 1.04, 6: 1.03, 8: 1.07, 12: 1.14, 16: 1.17, 32: 1.43; e2e best at 8
#endif
constexpr int kPushThreads = EFG_PUSH_THREADS, kPushKeys = 4096, kPushDirect = 4096, kPushSlices = EFG_PUSH_SLICES;
#ifndef EFG_PUSH_UNROLL
#define EFG_PUSH_UNROLL 4
#endif
constexpr int kPushUnroll = EFG_PUSH_UNROLL;
__global__ void __launch_bounds__(kPushThreads)
k_push_block(const int32_t* __restrict__ rows, int64_t count, const int64_t* __restrict__ offsets,
             const int32_t* __restrict__ nbr, const int32_t* __restrict__ nd, const int32_t* __restrict__ dcnt,
             const int32_t* __restrict__ hkey, const int32_t* __restrict__ hcnt, const double* __restrict__ ctab,
             const int64_t* __restrict__ s1, ChainAcc ca) {
  __shared__ int32_t sk[kPushKeys];
  __shared__ int16_t pos[kPushDirect];
  __shared__ double red[kPushThreads / 32];
  const int64_t q = blockIdx.x;
  if (q >= count) return;
  const int32_t i = rows[q];
  const int64_t b = offsets[i];
  const int d = (int)(offsets[i + 1] - b);
  const int D = dcnt[i];
  const int32_t* keys = D <= kPushKeys ? sk : hkey + b;
  // the row's slots in gridDim.y slices (long hub rows spread over CTAs);
  // slice 0 also forms the stars term
  const int p0 = (int)((int64_t)d * blockIdx.y / gridDim.y), p1 = (int)((int64_t)d * (blockIdx.y + 1) / gridDim.y);
  double hc = 0.0;
  for (int k = threadIdx.x; k < D; k += kPushThreads) {
    const int32_t kk = hkey[b + k];
    if (D <= kPushKeys) sk[k] = kk;
    if (kk < kPushDirect && k < 32768) pos[kk] = (int16_t)k;
    if (blockIdx.y == 0) hc += (double)hcnt[b + k] * ctab[b + k];
  }
  hc = block_sum<kPushThreads>(hc, red);  // syncs: the tables are complete afterwards
  if (threadIdx.x == 0 && blockIdx.y == 0) ca.ws[i] = hc;
  __syncthreads();
  const int64_t s1i = s1[i];
  // kPushUnroll slots per thread per step: their loads, lookups and table
  // gathers are issued together before the pushes (one slot at a time was a
  // dependent chain: ~23 cycles of long-scoreboard stall per instruction)
  for (int p = p0 + threadIdx.x; p < p1; p += kPushUnroll * kPushThreads) {
    int32_t y[kPushUnroll], vv[kPushUnroll], lo[kPushUnroll];
    double cv[kPushUnroll];
#pragma unroll
    for (int k = 0; k < kPushUnroll; ++k) {
      const int pp = p + k * kPushThreads;
      y[k] = pp < p1 ? nd[b + pp] : -1;
      vv[k] = pp < p1 ? nbr[b + pp] : 0;
    }
#pragma unroll
    for (int k = 0; k < kPushUnroll; ++k) {
      if (y[k] < 0) {
        lo[k] = 0;
      } else if (y[k] < kPushDirect && D <= 32768) {
        lo[k] = pos[y[k]];
      } else {
        int l = 0, h = D - 1;  // y is present: v is a neighbour of i
        while (l < h) {
          const int mid = (l + h) >> 1;
          if (keys[mid] < y[k]) l = mid + 1; else h = mid;
        }
        lo[k] = l;
      }
    }
#pragma unroll
    for (int k = 0; k < kPushUnroll; ++k) cv[k] = y[k] >= 0 ? __ldg(ctab + b + lo[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < kPushUnroll; ++k)
      if (y[k] >= 0) chain_push(ca, vv[k], y[k], cv[k], s1i);
  }
}

// 32 < d <= 256: warp per row, H_i's keys (<= 256) in the warp's shared slice,
// binary search per slot.  (Also taking the 256 < d <= 2048 rows with <= 256
// distinct neighbour degrees measured neutral, r02.)
#ifndef EFG_PUSH_WARPS
#define EFG_PUSH_WARPS 4
#endif
constexpr int kPushWarps = EFG_PUSH_WARPS, kPushWarpKeys = 256;
__global__ void __launch_bounds__(kPushWarps * 32)
k_push_warp256(const int32_t* __restrict__ rows, int64_t count, const int64_t* __restrict__ offsets,
               const int32_t* __restrict__ nbr, const int32_t* __restrict__ nd, const int32_t* __restrict__ dcnt,
               const int32_t* __restrict__ hkey, const int32_t* __restrict__ hcnt, const double* __restrict__ ctab,
               const int64_t* __restrict__ s1, ChainAcc ca) {
  __shared__ int32_t sk[kPushWarps][kPushWarpKeys];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t q = (int64_t)blockIdx.x * kPushWarps + w;
  if (q >= count) return;
  const int32_t i = rows[q];
  const int64_t b = offsets[i];
  const int d = (int)(offsets[i + 1] - b);
  const int D = dcnt[i];
  double hc = 0.0;
  for (int k = lane; k < D; k += 32) {
    sk[w][k] = hkey[b + k];
    hc += (double)hcnt[b + k] * ctab[b + k];
  }
  hc = warp_sum(hc);
  if (lane == 0) ca.ws[i] = hc;
  __syncwarp();
  const int64_t s1i = s1[i];
  for (int p = lane; p < d; p += kPushUnroll * 32) {  // as k_push_block: the slots' loads issued together
    int32_t y[kPushUnroll], vv[kPushUnroll], lo[kPushUnroll];
    double cv[kPushUnroll];
#pragma unroll
    for (int k = 0; k < kPushUnroll; ++k) {
      const int pp = p + 32 * k;
      y[k] = pp < d ? nd[b + pp] : -1;
      vv[k] = pp < d ? nbr[b + pp] : 0;
    }
#pragma unroll
    for (int k = 0; k < kPushUnroll; ++k) {
      int l = 0, h = D - 1;  // y is present: v is a neighbour of i
      while (y[k] >= 0 && l < h) {
        const int mid = (l + h) >> 1;
        if (sk[w][mid] < y[k]) l = mid + 1; else h = mid;
      }
      lo[k] = l;
    }
#pragma unroll
    for (int k = 0; k < kPushUnroll; ++k) cv[k] = y[k] >= 0 ? __ldg(ctab + b + lo[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < kPushUnroll; ++k)
      if (y[k] >= 0) chain_push(ca, vv[k], y[k], cv[k], s1i);
  }
}

// ------------------------------------------------------------- triangles
// W_t(v) = sum over triangles {v,i,j} of F(S-6) - F(S-4), S = dv+di+dj, and
// t(v) = their number.  Every triangle at v is found exactly once through the
// row of its lower-ranked member i: j in Adj+(i) and j in Adj(v) (the edge
// i-j lies in exactly one of Adj+(i), Adj+(j)).  Rows (i in Adj(v)) are long
// -- at R-MAT22 96 % of all probes sit in rows of >= 64 entries -- so a warp
// takes a whole row and its lanes stride it: the Adj+ loads are coalesced and
// kUnroll of them are in flight per lane before the membership probes.
// Membership: shared-memory hash of Adj(v) (load <= 1/4, linear probing) or,
// for hubs, a bitmap over node ids.  Per-lane sums in a fixed assignment,
// reduced in a fixed order (deterministic).

constexpr int kUnroll = 4;

// Bucketised hash map node id -> degree in shared memory: NB buckets of 4
// keys (one 16-byte load per probe, no per-lane probe loop in the common
// case), filled slot 0..3 in order, linear probing over buckets only when a
// bucket is full (rare at load <= 1/4).  With WITH_DEG the matching degree
// comes from a parallel array, otherwise from the global degree array.
template <int NB, bool WITH_DEG>
struct SmemMap {
  int4* keys;           // NB
  int32_t* degs;        // 4 * NB (WITH_DEG)
  const int32_t* gdeg;  // global degrees (!WITH_DEG)
  __device__ __forceinline__ static uint32_t bucket(int32_t key) {
    return ((uint32_t)key * 2654435761u) >> (32 - __builtin_ctz(NB));
  }
  __device__ __forceinline__ void clear(int tid, int nthr) {
    for (int s = tid; s < NB; s += nthr) keys[s] = make_int4(-1, -1, -1, -1);
  }
  __device__ __forceinline__ void insert(int32_t key, int32_t deg) {
    int32_t* flat = reinterpret_cast<int32_t*>(keys);
    for (uint32_t b = bucket(key);; b = (b + 1) & (NB - 1)) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (atomicCAS(&flat[4 * b + k], -1, key) == -1) {
          if (WITH_DEG) degs[4 * b + k] = deg;
          return;
        }
      }
    }
  }
  // phase 1: slot of key or -1 (one 16-byte load; the loop only runs past full buckets)
  __device__ __forceinline__ int32_t probe(int32_t key) const {
    uint32_t b = bucket(key);
    int4 q = keys[b];
    int k = q.x == key ? 0 : q.y == key ? 1 : q.z == key ? 2 : q.w == key ? 3 : -1;
    while (k < 0 && q.w != -1) {  // bucket full: key may sit further on
      b = (b + 1) & (NB - 1);
      q = keys[b];
      k = q.x == key ? 0 : q.y == key ? 1 : q.z == key ? 2 : q.w == key ? 3 : -1;
    }
    return k >= 0 ? (int32_t)(4 * b + k) : -1;
  }
  // phase 2: degree of a key found at `slot`
  __device__ __forceinline__ int32_t finish(int32_t key, int32_t slot) const {
    return WITH_DEG ? degs[slot] : __ldg(gdeg + key);
  }
  static constexpr bool kPhased = false;  // fused lookup schedules better for smem maps
  __device__ __forceinline__ int32_t degree(int32_t key) const {
    uint32_t b = bucket(key);
    int4 q = keys[b];
    while (true) {
      const int k = q.x == key ? 0 : q.y == key ? 1 : q.z == key ? 2 : q.w == key ? 3 : -1;
      if (k >= 0) return WITH_DEG ? degs[4 * b + k] : __ldg(gdeg + key);
      if (q.w == -1) return -1;  // bucket not full: key absent
      b = (b + 1) & (NB - 1);
      q = keys[b];
    }
  }
};



// Exact two-word fixed-point sum of P values (each |P| < 2^45): the value is
// hi 2^32 + lo; both words stay far from overflow for any count < 2^31.
struct Fix2 {
  int64_t hi = 0, lo = 0;
  __device__ __forceinline__ void add(int64_t p) {
    hi += p >> 32;
    lo += p & 0xffffffffll;
  }
};

// One warp over entries [p0, p1) of row `row` (= Adj+(i), s0 = dv + di), in
// phases so that each phase's loads are issued together: kUnroll entry loads,
// kUnroll membership probes, kUnroll degree lookups for the hits, kUnroll
// G-table gathers, then the (fixed-order) accumulation.
template <class Map>
__device__ __forceinline__ void tri_row(const FArgs& a, const int32_t* __restrict__ row, int32_t p0, int32_t p1,
                                        int32_t s0, int lane, const Map& map, int64_t& tri, Fix2& Wt) {
  for (int32_t p = p0 + lane; p < p1; p += 32 * kUnroll) {
    int32_t j[kUnroll], dj[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) j[u] = p + 32 * u < p1 ? __ldg(row + p + 32 * u) : -1;
    if constexpr (Map::kPhased) {
      // the entry's degree streams alongside its label (adjd), so a hit needs
      // only the G gather; labels past the shared bitmap check the global one
      int32_t tag[kUnroll], dd[kUnroll];
      int64_t g[kUnroll];
      const int32_t* rowd = a.adjd + (row - a.adjj);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) dd[u] = j[u] >= 0 ? __ldg(rowd + p + 32 * u) : 0;
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) tag[u] = j[u] >= 0 ? map.probe(j[u]) : -1;
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) dj[u] = tag[u] >= 0 ? map.finish(j[u], tag[u], dd[u]) : -1;
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) g[u] = dj[u] >= 0 ? __ldg(a.PT + EFG_CLAMP(s0 + dj[u], a.flen)) : 0;
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        if (dj[u] >= 0) {
          Wt.add(g[u]);
          ++tri;
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) dj[u] = j[u] >= 0 ? map.degree(j[u]) : -1;
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        if (dj[u] >= 0) {
          Wt.add(__ldg(a.PT + EFG_CLAMP(s0 + dj[u], a.flen)));
          ++tri;
        }
      }
    }
  }
}

// Rows x = first, first+stride, ... < dv of seed v, one warp per row.
// Rows ob+x, x = first, first+stride, ... < nrows (of a seed of degree dv).
template <class Map>
__device__ __forceinline__ void tri_rows(const FArgs& a, int64_t ob, int nrows, int first, int stride, int lane,
                                         const Map& map, int64_t& tri, Fix2& Wt, int dv) {
  for (int x = first; x < nrows; x += stride) {
    const int64_t e = ob + x;
    const int32_t pc = __ldg(a.pc + e);
    if (pc == 0) continue;
    tri_row(a, a.adjj + __ldg(a.offsets + __ldg(a.nbr + e)), 0, pc, dv + __ldg(a.nd + e), lane, map, tri, Wt);
  }
}

// Reverse probing.  A row Adj+(i) much longer than Adj(v) is cheaper to test
// the other way round: each j in Adj(v) is looked up in a global bucketed
// hash of Adj+(i) (built once per pass for |Adj+(i)| >= kRevMin, 4 keys per
// 16-byte bucket, load <= 1/4, located at bucket 2*offsets[i]).  A hit is
// exactly j in Adj+(i), i.e. the same triangle the forward scan would find.
constexpr int kRevMin = 64;
constexpr int kRevKappa = 2;
__device__ __forceinline__ bool use_reverse(int32_t pc, int dv) { return pc >= kRevMin && kRevKappa * dv < pc; }

__device__ __forceinline__ uint32_t rowhash_lg(int32_t pc) { return 32u - __clz(pc - 1); }  // NB = 2^lg >= pc

__device__ __forceinline__ bool rowhash_has(const int4* __restrict__ base, uint32_t lg, int32_t key) {
  const uint32_t mask = (1u << lg) - 1;
  uint32_t b = ((uint32_t)key * 2654435761u) >> (32 - lg);
  while (true) {
    const int4 q = __ldg(base + b);
    if (q.x == key || q.y == key || q.z == key || q.w == key) return true;
    if (q.w == -1) return false;
    b = (b + 1) & mask;
  }
}

// Warp per node with |Adj+(i)| >= kRevMin: clear its buckets, insert its labels.
__global__ void k_rowhash(const int64_t* __restrict__ offsets, const int32_t* __restrict__ dplus,
                          const int32_t* __restrict__ adjj, int64_t n, int4* __restrict__ rowhash) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  const int64_t p0 = offsets[i];
  const int32_t pc = dplus[i];
  if (pc < kRevMin) return;
  const uint32_t lg = rowhash_lg(pc), nb = 1u << lg;
  int4* base = rowhash + 2 * p0;
  for (uint32_t b = lane; b < nb; b += 32) base[b] = make_int4(-1, -1, -1, -1);
  __syncwarp();
  int32_t* flat = reinterpret_cast<int32_t*>(base);
  for (int32_t p = lane; p < pc; p += 32) {
    const int32_t key = adjj[p0 + p];
    for (uint32_t b = (key * 2654435761u) >> (32 - lg);; b = (b + 1) & (nb - 1)) {
      int k = 0;
      for (; k < 4; ++k)
        if (atomicCAS(&flat[4 * b + k], -1, key) == -1) break;
      if (k < 4) break;
    }
  }
}

// dv <= 32: warp per seed (the warp walks the seed's rows one after another;
// long rows are probed in reverse, all 32 lanes at once).
constexpr int kTriWarps = 8;
__global__ void __launch_bounds__(kTriWarps * 32)
k_tri_warp(const int32_t* __restrict__ seeds, int64_t count, FArgs a) {
  __shared__ int4 sK[kTriWarps][32];
  __shared__ int32_t sD[kTriWarps][128];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t qs = (int64_t)blockIdx.x * kTriWarps + w;
  if (qs >= count) return;
  const int32_t v = seeds[qs];
  const int64_t ob = a.offsets[v];
  const int dv = (int)(a.offsets[v + 1] - ob);
  SmemMap<32, true> map{sK[w], sD[w], nullptr};
  map.clear(lane, 32);
  int32_t myl = -1, myd = 0, mypc = 0;
  int64_t myps = 0;
  if (lane < dv) {
    const int32_t i = a.nbr[ob + lane];
    myl = __ldg(a.rank_of + i);
    myd = a.nd[ob + lane];
    mypc = __ldg(a.pc + ob + lane);
    myps = __ldg(a.offsets + i);
  }
  __syncwarp();
  if (lane < dv) map.insert(myl, myd);
  __syncwarp();
  int64_t tri = 0;
  Fix2 Wt;
  const bool rev = lane < dv && use_reverse(mypc, dv);
  unsigned fwd = __ballot_sync(0xffffffffu, lane < dv && mypc > 0 && !rev);
  while (fwd) {
    const int x = __ffs(fwd) - 1;
    fwd &= fwd - 1;
    const int32_t pcx = __shfl_sync(0xffffffffu, mypc, x);
    const int64_t psx = __shfl_sync(0xffffffffu, myps, x);
    const int32_t dx = __shfl_sync(0xffffffffu, myd, x);
    tri_row(a, a.adjj + psx, 0, pcx, dv + dx, lane, map, tri, Wt);
  }
  unsigned rv = __ballot_sync(0xffffffffu, rev);
  while (rv) {
    const int x = __ffs(rv) - 1;
    rv &= rv - 1;
    const int32_t pcx = __shfl_sync(0xffffffffu, mypc, x);
    const int64_t psx = __shfl_sync(0xffffffffu, myps, x);
    const int32_t dx = __shfl_sync(0xffffffffu, myd, x);
    if (lane < dv && lane != x && rowhash_has(a.rowhash + 2 * psx, rowhash_lg(pcx), myl)) {
      Wt.add(__ldg(a.PT + EFG_CLAMP(dv + dx + myd, a.flen)));
      ++tri;
    }
  }
  tri = warp_sum(tri);
  Wt.hi = warp_sum(Wt.hi);
  Wt.lo = warp_sum(Wt.lo);
  if (lane == 0) {
    a.tri[v - a.seed_lo] = tri;
    a.Wth[v - a.seed_lo] = Wt.hi;
    a.Wtl[v - a.seed_lo] = Wt.lo;
  }
}

// 32 < dv <= MAXD: CTA per seed, warps take rows round-robin.
// smem: 16 * NB (+ 16 * NB with degrees) bytes
template <int THREADS, int NB, bool WITH_DEG>
__global__ void __launch_bounds__(THREADS)
k_tri_seed(const int32_t* __restrict__ seeds, int64_t count, FArgs a) {
  extern __shared__ int4 dyn4[];
  __shared__ int64_t red_i[THREADS / 32], red_h[THREADS / 32], red_l[THREADS / 32];
  const int64_t qs = blockIdx.x;
  if (qs >= count) return;
  const int32_t v = seeds[qs];
  const int64_t ob = a.offsets[v];
  const int dv = (int)(a.offsets[v + 1] - ob);
  SmemMap<NB, WITH_DEG> map{dyn4, reinterpret_cast<int32_t*>(dyn4 + NB), a.deg_by_rank};
  map.clear(threadIdx.x, THREADS);
  __syncthreads();
  for (int x = threadIdx.x; x < dv; x += THREADS) map.insert(__ldg(a.rank_of + a.nbr[ob + x]), a.nd[ob + x]);
  __syncthreads();
  int64_t tri = 0;
  Fix2 Wt;
  tri_rows(a, ob, dv, threadIdx.x >> 5, THREADS / 32, threadIdx.x & 31, map, tri, Wt, dv);
  tri = block_sum<THREADS>(tri, red_i);
  const int64_t wh = block_sum<THREADS>(Wt.hi, red_h);
  const int64_t wl = block_sum<THREADS>(Wt.lo, red_l);
  if (threadIdx.x == 0) {
    a.tri[v - a.seed_lo] = tri;
    a.Wth[v - a.seed_lo] = wh;
    a.Wtl[v - a.seed_lo] = wl;
  }
}

// Hubs (dv > kHashMaxDeg), one 1024-thread CTA per hub, hubs in descending
// work order.  Adj(v) membership in two levels: a shared-memory Bloom filter
// of kFilterBits bits (one multiplicative hash; at most dv/kFilterBits false
// positives) answers most probes, and only filter positives read the hub's
// exact bitmap over node ids in global memory (L2-resident while the hub runs).
constexpr int kHubThreads = 1024;
constexpr uint32_t kFilterWords = 48 * 1024;            // 192 KB of shared memory
constexpr uint32_t kFilterBits = kFilterWords * 32;

// Membership over rank labels: probe targets j come from Adj+ lists, so they
// outrank a neighbour of the hub and are mostly high-degree nodes with small
// labels.  Labels < kFilterBits are answered exactly by the shared-memory
// bitmap; larger labels (rare) read the hub's global bitmap.
struct HubMap {
  const uint32_t* sbm;   // shared: bits of labels < kFilterBits
  const uint32_t* bm;    // global exact bitmap over all labels
  const int32_t* deg;    // degree by rank label
  static constexpr bool kPhased = true;  // global loads: issue each phase's loads together
  // phase 1: shared bitmap (exact), or "ask global" for large labels
  __device__ __forceinline__ int32_t probe(int32_t j) const {
    if ((uint32_t)j < kFilterBits) return ((sbm[j >> 5] >> (j & 31)) & 1u) ? 0 : -1;
    return 1;
  }
  // phase 2: large labels check the exact global bit
  __device__ __forceinline__ int32_t finish(int32_t j, int32_t tag, int32_t d) const {
    if (tag == 0) return d;
    return ((__ldg(bm + (j >> 5)) >> (j & 31)) & 1u) ? d : -1;
  }
};

// Hub work is cut into tasks of kHubRows consecutive rows, so the largest
// hubs spread over many SMs; each task rebuilds the filter (dv bits, well
// below its probe count) and writes a partial merged per hub in task order.
#ifndef EFG_HUB_ROWS
#define EFG_HUB_ROWS 8192  // k_mid_big R-MAT22 10.40 / 10.28 / 10.26 ms at 4096 / 8192 / 16384; Chung-Lu 0.90 at 8192, 1.31 at 16384 (r02)
#endif
constexpr int64_t kHubRows = EFG_HUB_ROWS;
#ifndef EFG_MID_SMALL_DEG
#define EFG_MID_SMALL_DEG 256  // listing middles of degree <= this in small CTAs (k_list_counts' split)
#endif

struct HubTasks {
  const int32_t* seed;  // [ntasks]
  const int32_t* x0;    // [ntasks] first row
  const int32_t* x1;    // [ntasks] end row
  int64_t* ptri;
  int64_t* pWh;
  int64_t* pWl;
};

__global__ void __launch_bounds__(kHubThreads, 1)
k_tri_hub(HubTasks tk, int64_t ntasks, const uint32_t* __restrict__ bitmaps, int64_t words,
          const int32_t* __restrict__ hub_slot, FArgs a) {
  extern __shared__ uint32_t filt[];  // kFilterWords
  __shared__ int64_t red_i[kHubThreads / 32], red_h[kHubThreads / 32], red_l[kHubThreads / 32];
  const int64_t t = blockIdx.x;
  if (t >= ntasks) return;
  const int32_t v = tk.seed[t];
  const int64_t ob = a.offsets[v];
  const int dv = (int)(a.offsets[v + 1] - ob);
  for (uint32_t k = threadIdx.x; k < kFilterWords; k += kHubThreads) filt[k] = 0u;
  __syncthreads();
  for (int x = threadIdx.x; x < dv; x += kHubThreads) {
    const int32_t r = __ldg(a.rank_of + a.nbr[ob + x]);
    if ((uint32_t)r < kFilterBits) atomicOr(&filt[r >> 5], 1u << (r & 31));
  }
  __syncthreads();
  HubMap map{filt, bitmaps + (int64_t)hub_slot[v] * words, a.deg_by_rank};
  int64_t tri = 0;
  Fix2 Wt;
  const int x0 = tk.x0[t];
  tri_rows(a, ob + x0, tk.x1[t] - x0, threadIdx.x >> 5, kHubThreads / 32, threadIdx.x & 31, map, tri, Wt, dv);
  tri = block_sum<kHubThreads>(tri, red_i);
  const int64_t wh = block_sum<kHubThreads>(Wt.hi, red_h);
  const int64_t wl = block_sum<kHubThreads>(Wt.lo, red_l);
  if (threadIdx.x == 0) {
    tk.ptri[t] = tri;
    tk.pWh[t] = wh;
    tk.pWl[t] = wl;
  }
}

// Hub task count (degrees only: it is read back with the list counts).
__global__ void k_hub_count(const int32_t* __restrict__ hubs, const int64_t* __restrict__ nhubs_dev,
                            const int64_t* __restrict__ offsets, unsigned long long* __restrict__ ntasks) {
  const int64_t nhubs = *nhubs_dev;
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nhubs; h += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = hubs[h];
    atomicAdd(ntasks, (unsigned long long)ceil_div(offsets[v + 1] - offsets[v], kHubRows));
  }
}

// Class counts of a listing pass from the rank order (labels are in
// descending degree order, so "degree > T" is a label prefix): the triangle
// classes' sizes and the hub task count, straight into the count slots.
__device__ __forceinline__ int64_t ranks_above_deg(const int32_t* __restrict__ deg_by_rank, int64_t n, int32_t t) {
  int64_t lo = 0, hi = n;  // first rank of degree <= t
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (deg_by_rank[mid] > t) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__global__ void k_list_counts(const int32_t* __restrict__ deg_by_rank, int64_t n, int64_t* __restrict__ c,
                              int slot_s, int slot_1, int slot_2, int slot_3, int slot_hub, int slot_tasks) {
  __shared__ int64_t red[8];
  const int64_t g32 = ranks_above_deg(deg_by_rank, n, 32), g256 = ranks_above_deg(deg_by_rank, n, EFG_MID_SMALL_DEG),
                g1024 = ranks_above_deg(deg_by_rank, n, 1024), ghub = ranks_above_deg(deg_by_rank, n, kHashMaxDeg);
  static_assert(EFG_MID_SMALL_DEG < 1024, "the listing's small / big split below the tr3 bound");
  int64_t t = 0;
  for (int64_t r = threadIdx.x; r < ghub; r += blockDim.x) t += ceil_div(deg_by_rank[r], kHubRows);
  t = block_sum<256>(t, red);
  if (threadIdx.x == 0) {
    c[slot_s] = n - g32;
    c[slot_1] = g32 - g256;
    c[slot_2] = g256 - g1024;
    c[slot_3] = g1024 - ghub;
    c[slot_hub] = ghub;
    c[slot_tasks] = t;
  }
}

// Triangle probes of each hub (sort key for the hub order).
__global__ void __launch_bounds__(256) k_hub_work(const int32_t* __restrict__ hubs, int64_t nhubs,
                                                  const int64_t* __restrict__ offsets,
                                                  const int32_t* __restrict__ nbr, const int32_t* __restrict__ dplus,
                                                  int64_t* __restrict__ work) {
  // a CTA per hub: sum of |Adj+(u)| over the hub's row (dplus gathers, L2-resident)
  __shared__ int64_t red[8];
  const int64_t h = blockIdx.x;
  if (h >= nhubs) return;
  const int32_t v = hubs[h];
  int64_t w = 0;
  for (int64_t p = offsets[v] + threadIdx.x; p < offsets[v + 1]; p += 256) w += __ldg(dplus + __ldg(nbr + p));
  w = block_sum<256>(w, red);
  if (threadIdx.x == 0) work[h] = w;
}

__global__ void k_hub_ntasks(const int32_t* __restrict__ hubs, int64_t nhubs, const int64_t* __restrict__ offsets,
                             int64_t* __restrict__ nt) {
  const int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (h < nhubs) nt[h] = ceil_div(offsets[hubs[h] + 1] - offsets[hubs[h]], kHubRows);
  if (h == nhubs) nt[h] = 0;
}

// Task records (thread per hub, tasks of one hub contiguous, hubs in order).
__global__ void k_hub_tasks(const int32_t* __restrict__ hubs, int64_t nhubs, const int64_t* __restrict__ offsets,
                            const int64_t* __restrict__ tstart, int32_t* __restrict__ tseed,
                            int32_t* __restrict__ tx0, int32_t* __restrict__ tx1) {
  const int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (h >= nhubs) return;
  const int32_t v = hubs[h];
  const int64_t dv = offsets[v + 1] - offsets[v];
  for (int64_t t = tstart[h], x = 0; t < tstart[h + 1]; ++t, x += kHubRows) {
    tseed[t] = v;
    tx0[t] = (int32_t)x;
    tx1[t] = (int32_t)(x + kHubRows < dv ? x + kHubRows : dv);
  }
}

__global__ void k_hub_merge(const int32_t* __restrict__ hubs, int64_t nhubs, const int64_t* __restrict__ tstart,
                            const int64_t* __restrict__ ptri, const int64_t* __restrict__ pWh,
                            const int64_t* __restrict__ pWl, FArgs a) {
  const int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (h >= nhubs) return;
  int64_t tri = 0, wh = 0, wl = 0;
  for (int64_t t = tstart[h]; t < tstart[h + 1]; ++t) {
    tri += ptri[t];
    wh += pWh[t];
    wl += pWl[t];
  }
  const int32_t v = hubs[h];
  a.tri[v - a.seed_lo] = tri;
  a.Wth[v - a.seed_lo] = wh;
  a.Wtl[v - a.seed_lo] = wl;
}

__global__ void k_hub_bitmaps(const int32_t* __restrict__ hubs, int64_t nhubs, const int64_t* __restrict__ offsets,
                              const int32_t* __restrict__ nbr, const int32_t* __restrict__ rank_of,
                              uint32_t* __restrict__ bitmaps, int64_t words, int32_t* __restrict__ hub_slot) {
  int64_t h = blockIdx.x;
  if (h >= nhubs) return;
  int32_t v = hubs[h];
  if (threadIdx.x == 0) hub_slot[v] = (int32_t)h;
  uint32_t* bm = bitmaps + h * words;
  for (int64_t p = offsets[v] + threadIdx.x; p < offsets[v + 1]; p += blockDim.x) {
    int32_t i = rank_of[nbr[p]];
    atomicOr(bm + (i >> 5), 1u << (i & 31));
  }
}

// ------------------------------------------------------- triangle listing
// Whole-graph passes list every triangle once instead of once per member.
// Triangle {u, v, w} with rank(u) > rank(v) > rank(w) (u the lowest in the
// degree order, v the middle) is found by v's CTA: for every lower-ranked
// neighbour u of v (a "row"), Adj+(u) is scanned (coalesced, 4 loads in
// flight per lane) against a shared-memory map of Adj+(v), which is short
// (|Adj+| <= sqrt(2m); 813 at R-MAT22) even for hubs.  Probes: sum over u of
// |Adj+(u)|^2 = 7.1e9 at R-MAT22, against 2.2e10 for the per-seed scan.
// All three members receive the same correction G(du+dv+dw): v sums its own
// in registers, u's arrive once per row, w's are summed per entry of Adj+(v)
// and reach global memory once per (v, chunk of rows, entry).  Sums are in
// fixed point (P = rint(G 2^40), |P| < 2^45: error <= 2^-41 per triangle,
// far below the 1e-12 floor of the EF tolerance) with integer additions,
// which commute, so the result does not depend on scheduling.  Global words
// per node: (sum of s >> 32, sum of s & (2^32-1), count), never overflowing
// (a row has < 2^16 hits, a node < 2^31 partial sums).
#ifndef EFG_MID_BIG_THREADS
#define EFG_MID_BIG_THREADS 320
#endif
#ifndef EFG_MID_WARPS
#define EFG_MID_WARPS 4  // k_mid_warp ms (r02): 4: 0.746, 8: 0.795, 16: 0.853
#endif
constexpr int kMidWarps = EFG_MID_WARPS;  // k_mid_warp: warps (middles) per CTA
constexpr int kMidThreads = 256;
constexpr int kMidNB = 512;         // shared map of Adj+(v): <= 1024 keys at load <= 1/2
constexpr int kMidLgNB = 9;
// Big middles: CTAs of 10 warps, 4 per SM (48 registers: 40 warps, as 5 x 8),
// each with Adj+(v) parts of 1024 entries and chunks of 512 rows (48 KB of
// shared memory).  Measured k_mid_big, R-MAT22 (r02): 8 warps x 5 CTAs with
// parts / chunks of 1024 / 256: 11.06 ms; 768 / 512 (same shared memory):
// 10.62; 640 / 512: 11.26; 10 warps x 4 CTAs, 768 / 512: 10.37, 1024 / 512:
// 10.27; 12 warps x 3 CTAs: 10.88.  Fewer, larger chunks halve the barrier
// waits and entry flushes; fewer CTAs per SM build fewer Adj+(v) bitmaps.
#ifndef EFG_MID_MAXP
#define EFG_MID_MAXP 1024
#endif
constexpr int kMidMaxP = EFG_MID_MAXP;  // longer Adj+(v) are processed in parts of this size
#ifndef EFG_MID_CHUNK
#define EFG_MID_CHUNK 512
#endif
// rows between entry flushes: 32-bit entry words cannot overflow (per entry and chunk at most
// kMidChunk hits of Q < 2^45: low pieces < 512 * 2^22 = 2^31, high pieces < 512 * 2^23 = 2^32)
constexpr int kMidChunk = EFG_MID_CHUNK;
static_assert(kMidChunk <= 512, "entry words would overflow");
// probe-loop unroll (entries per lane per step), measured per loop: bitmap scan with
// the 8-byte word+prefix entries 4 for long rows, 2 / 1 for rows whose scan is at most
// 64 / 32 entries (k_mid_big 12.25 -> 11.80 ms; peeking at labels 31 / 63 of longer
// rows to shorten their step measured slower: 12.38), r02; hash 4 in big CTAs, 2 in
// small (1 for scans of at most 32 entries)
#ifndef EFG_MID_UNROLL_BM
#define EFG_MID_UNROLL_BM 4
#endif
#ifndef EFG_MID_BIG_MINB
#define EFG_MID_BIG_MINB 4
#endif
constexpr int kMidUnrollBm = EFG_MID_UNROLL_BM;
#ifndef EFG_MID_ADAPT_U
#define EFG_MID_ADAPT_U 1
#endif
constexpr bool kMidAdaptU = EFG_MID_ADAPT_U;
#ifndef EFG_MID_U1_SPAN
#define EFG_MID_U1_SPAN 32
#endif
#ifndef EFG_MID_U2_SPAN
#define EFG_MID_U2_SPAN 64
#endif
#ifndef EFG_MID_H1_SPAN
#define EFG_MID_H1_SPAN 32
#endif



constexpr int kMidSmallDeg = EFG_MID_SMALL_DEG;  // middle vertices of degree <= this run in small CTAs

// CTA shapes of k_mid_block: big (hub tasks and degree > kMidSmallDeg) and
// small (32 < degree <= kMidSmallDeg, where |Adj+(v)| and the rows are few).
struct MidBig {
  static constexpr int kThreads = EFG_MID_BIG_THREADS, kNB = kMidNB, kLgNB = kMidLgNB, kMaxP = kMidMaxP,
                       kChunk = kMidChunk;
  static constexpr int kBmWords = 2048;  // label bitmap for rank(v) <= 65536 (same shared bytes as the hash)
  static constexpr int kUnrollHash = 4;
};
// small middles (33..256): CTAs of 3 warps (14 per SM, shared-memory bound):
// a middle has ~30 rows, so fewer warps wait less at its barriers; measured
// k_mid_small 2.32 ms with 4 warps x 12, 2.24 with 3 x 14, 2.74 with 6 x 8
#ifndef EFG_MID_SMALL_THREADS
#define EFG_MID_SMALL_THREADS 96
#endif
#ifndef EFG_MID_SMALL_MINB
#define EFG_MID_SMALL_MINB 16
#endif
#ifndef EFG_MID_SMALL_UNROLL
#define EFG_MID_SMALL_UNROLL 2
#endif
#ifndef EFG_MID_SMALL_CHUNK
#define EFG_MID_SMALL_CHUNK 256
#endif
struct MidSmall {
  static constexpr int kThreads = EFG_MID_SMALL_THREADS, kNB = 128, kLgNB = 7, kMaxP = kMidSmallDeg < 256 ? kMidSmallDeg : 256,
                       kChunk = EFG_MID_SMALL_CHUNK;
  static constexpr int kBmWords = 0;
  static constexpr int kUnrollHash = EFG_MID_SMALL_UNROLL;
};
constexpr int kListScale = 40;      // P = rint(G * 2^40)
constexpr int64_t kListMaxDeg = 1000000;  // |G(3 dmax)| < 32

struct MArgs {
  const int64_t* offsets;
  const int32_t* nbr;
  const int32_t* nd;        // degree per slot, or null: gathered from deg (distributed listing: other parts' rows)
  const int32_t* deg;
  const int32_t* dplus;     // |Adj+(v)|: Adj+(v) at adjj[offsets[v], offsets[v] + dplus[v])
  const int32_t* adjj;
  const int32_t* adjd;
  const int32_t* rank_of;
  const int32_t* by_rank;
  const int32_t* deg_by_rank;
  const int64_t* PT;        // fixed-point G
  const uint64_t* PQ;       // Q = -P >= 0 (G < 0 on every reachable S): the block listing's table
  int64_t flen;             // PT length (bounds-checked builds)
  int32_t bm_lim;           // label bitmap for parts with lim <= this (else the hash; EFG_MID_BM_LIMIT, tests)
  unsigned long long* acc;  // [4 n] per node: (hi, lo, count, pad)
  int64_t n, n32;           // labels < n32: degree > 32
  int64_t nhubs, ntasks;    // labels < nhubs come as ntasks row-range tasks
  int32_t part, nparts;     // distributed pass: this part takes work units u with u % nparts == part
  int32_t nunits;           // k_mid_block work units of this launch: ntasks hub tasks, then labels
  int64_t label0;           // first label of the launch's label units
};

__global__ void k_gfix(const double* __restrict__ G, int64_t len, int64_t* __restrict__ PT, uint64_t* __restrict__ PQ) {
  const int64_t S = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (S < len) {
    const int64_t p = (int64_t)rint(ldexp(G[S], kListScale));
    PT[S] = p;
    PQ[S] = (uint64_t)(-p);
  }
}

// one partial sum (|s| < 2^63) and its triangle count into a node's words
__device__ __forceinline__ void red_node(unsigned long long* acc, int32_t node, int64_t s, uint64_t c) {
  unsigned long long* p = acc + 4 * (int64_t)node;
  atomicAdd(p, (unsigned long long)(s >> 32));
  atomicAdd(p + 1, (unsigned long long)(s & 0xffffffffll));
  atomicAdd(p + 2, (unsigned long long)c);
}

// v's own share, kept as two words so that any number of rows fits
struct Acc2 {
  int64_t hi = 0, lo = 0;
  uint32_t c = 0;
  __device__ __forceinline__ void add_row(int64_t s, uint32_t n) {
    hi += s >> 32;
    lo += s & 0xffffffffll;
    c += n;
  }
};

// shared bucketed map label -> position in Adj+(v) (NB buckets of 4, key -1 = empty)
// slot of key past a full first bucket (rare at load <= 1/4), or -1
__device__ __forceinline__ int32_t smap_slot_slow(const int4* __restrict__ keys, uint32_t lg, uint32_t b, int32_t key) {
  const uint32_t mask = (1u << lg) - 1;
  while (true) {
    b = (b + 1) & mask;
    const int4 q = keys[b];
    const int k = q.x == key ? 0 : q.y == key ? 1 : q.z == key ? 2 : q.w == key ? 3 : -1;
    if (k >= 0) return (int32_t)(4 * b + k);
    if (q.w == -1) return -1;
  }
}
template <class V>
__device__ __forceinline__ int32_t smap_find(const int4* __restrict__ keys, const V* __restrict__ vals, uint32_t lg,
                                             int32_t key) {
  const uint32_t b = ((uint32_t)key * 2654435761u) >> (32 - lg);
  const int4 q = keys[b];
  int32_t slot = q.x == key ? (int32_t)(4 * b) : q.y == key ? (int32_t)(4 * b + 1)
               : q.z == key ? (int32_t)(4 * b + 2) : q.w == key ? (int32_t)(4 * b + 3) : -1;
  if (slot < 0 && q.w != -1) slot = smap_slot_slow(keys, lg, b, key);
  return slot >= 0 ? (int32_t)vals[slot] : -1;
}
template <class V>
__device__ __forceinline__ void smap_insert(int4* keys, V* vals, uint32_t lg, int32_t key, int32_t val) {
  int32_t* flat = reinterpret_cast<int32_t*>(keys);
  const uint32_t mask = (1u << lg) - 1;
  for (uint32_t b = ((uint32_t)key * 2654435761u) >> (32 - lg);; b = (b + 1) & mask)
    for (int k = 0; k < 4; ++k)
      if (atomicCAS(&flat[4 * b + k], -1, key) == -1) {
        vals[4 * b + k] = (V)val;
        return;
      }
}

// Warp sums on the native reduction unit (REDUX): a 32-bit count directly,
// a 64-bit row sum (|s| < 2^57 per lane) as three 26/26/12-bit pieces that
// cannot overflow 32 bits over 32 lanes.
__device__ __forceinline__ uint32_t warp_count(uint32_t c) { return __reduce_add_sync(0xffffffffu, c); }
__device__ __forceinline__ int64_t warp_sum64(int64_t x) {
  const uint32_t p0 = (uint32_t)(x & 0x3ffffff), p1 = (uint32_t)((x >> 26) & 0x3ffffff);
  const int32_t p2 = (int32_t)(x >> 52);
  const uint64_t s0 = __reduce_add_sync(0xffffffffu, p0), s1 = __reduce_add_sync(0xffffffffu, p1);
  const int64_t s2 = __reduce_add_sync(0xffffffffu, p2);
  return (int64_t)s0 + ((int64_t)s1 << 26) + (s2 << 52);
}

// Explicit shared-window loads for the listing's probe loop: the map base is
// converted once, so the loop carries a 32-bit address instead of
// re-deriving the shared window of a generic pointer on every probe.
__device__ __forceinline__ int4 lds128(uint32_t addr) {
  int4 v;
  asm("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ int32_t lds32(uint32_t addr) {
  int32_t v;
  asm("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ int32_t lds_s16(uint32_t addr) {
  short v;
  asm("ld.shared.s16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ void reds_add(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// The bitmap form of mid_scan (labels < lim <= 32 kBmWords): a running row
// pointer and the row's Q-table base stay in registers; one 8-byte shared
// load per entry gives membership and, with a popcount, the position in
// Adj+(v).  Branch-free up to the hit: the key is clamped to lim (the bitmap
// holds a zero word at lim >> 5 whose prefix is |part|, and lim is never a
// member), so every lane's position is a valid index and w's degree is read
// unpredicated; only the Q gather and the hit are predicated.  The row is
// label-sorted, so the scan is past lim exactly when some lane's last entry is.
template <int U, class Hit>
__device__ __forceinline__ void mid_scan_bm(const int32_t* __restrict__ row, int32_t pu, int32_t lim,
                                            const uint64_t* __restrict__ PQ, uint32_t s0, uint32_t bmb, uint32_t db,
                                            int lane, Hit hit, int64_t flen = 0) {
  const int32_t* __restrict__ rp = row + lane;
  for (int32_t q = lane; q - lane < pu; q += 32 * U, rp += 32 * U) {
    int32_t j[U], y[U];
    bool h[U];
    uint64_t g[U];
#pragma unroll
    for (int k = 0; k < U; ++k) j[k] = q + 32 * k < pu ? __ldg(rp + 32 * k) : INT32_MAX;
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint32_t key = (uint32_t)min(j[k], lim);
      const uint2 wp = lds64(bmb + 8u * (key >> 5));
      const uint32_t bit = __funnelshift_l(0u, 1u, key);  // 1 << (key & 31): the wrapping shift, no mask
      h[k] = (wp.x & bit) != 0u;
      y[k] = (int32_t)(wp.y + __popc(wp.x & (bit - 1)));
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint32_t S = s0 + (uint32_t)lds32(db + 4u * (uint32_t)y[k]);  // 32-bit index: one wide multiply-add
      g[k] = h[k] ? __ldg(PQ + EFG_CLAMP(S, flen)) : 0ull;
    }
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (h[k]) hit(y[k], j[k], g[k]);
    if (__any_sync(0xffffffffu, j[U - 1] >= lim)) break;
  }
}

// The hash form of the scan (Adj+(v) parts whose labels reach past the
// bitmap): a bucketed map label -> packed entry (position | degree << 10) at
// NB = 2^lg buckets of 4 keys (kb) and 4 values (pvb), load <= 1/4.  One
// 16-byte load answers the common case; a bucket that is full and misses
// continues the linear probe (rare).  Labels >= lim are never members, so no
// clamp; a miss reads the value of slot 0 (unused) and only the Q gather and
// the hit are predicated, as in mid_scan_bm.
constexpr int kPosBits = 10;  // entry positions < kMidMaxP <= 1024
static_assert(kMidMaxP <= (1 << kPosBits) && kMidSmallDeg <= (1 << kPosBits), "packed hash entries hold positions in kPosBits");
static_assert(kListMaxDeg < (int64_t(1) << (32 - kPosBits)), "packed hash entries hold degrees <= kListMaxDeg above the position");
__device__ __forceinline__ int32_t mslot_slow(uint32_t kb, uint32_t lg, uint32_t b, int32_t key) {
  const uint32_t mask = (1u << lg) - 1;
  while (true) {
    b = (b + 1) & mask;
    const int4 q = lds128(kb + 16 * b);
    const int k = q.x == key ? 0 : q.y == key ? 1 : q.z == key ? 2 : q.w == key ? 3 : -1;
    if (k >= 0) return (int32_t)(4 * b + k);
    if (q.w == -1) return -1;
  }
}
template <int U, class Hit>
__device__ __forceinline__ void mid_scan_hash(const int32_t* __restrict__ row, int32_t pu, int32_t lim,
                                              const uint64_t* __restrict__ PQ, uint32_t s0, uint32_t kb, uint32_t pvb,
                                              uint32_t lg, int lane, Hit hit, int64_t flen = 0) {
  const int32_t* __restrict__ rp = row + lane;
  for (int32_t q = lane; q - lane < pu; q += 32 * U, rp += 32 * U) {
    int32_t j[U], fs[U];
    uint64_t g[U];
#pragma unroll
    for (int k = 0; k < U; ++k) j[k] = q + 32 * k < pu ? __ldg(rp + 32 * k) : INT32_MAX;
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int32_t key = j[k];
      const uint32_t b = ((uint32_t)key * 2654435761u) >> (32 - lg);
      const int4 e = lds128(kb + 16 * b);
      // at most one key of the bucket matches: the slot as a sum of selects (no branches)
      const bool m0 = e.x == key, m1 = e.y == key, m2 = e.z == key, m3 = e.w == key;
      const int32_t sl = (int32_t)(4 * b) + (m1 ? 1 : 0) + (m2 ? 2 : 0) + (m3 ? 3 : 0);
      fs[k] = (m0 | m1 | m2 | m3) ? sl : -1;
      if (fs[k] < 0 && e.w != -1) fs[k] = mslot_slow(kb, lg, b, key);
    }
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const uint32_t pv = (uint32_t)lds32(pvb + 4u * (uint32_t)max(fs[k], 0));
      fs[k] = fs[k] >= 0 ? (int32_t)(pv & ((1u << kPosBits) - 1)) : -1;
      const uint32_t S = s0 + (pv >> kPosBits);
      g[k] = fs[k] >= 0 ? __ldg(PQ + EFG_CLAMP(S, flen)) : 0ull;
    }
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (fs[k] >= 0) hit(fs[k], j[k], g[k]);
    if (__any_sync(0xffffffffu, j[U - 1] >= lim)) break;
  }
}

// first position of a label-sorted Adj+ row (length pu) holding a label >= lim
__device__ __forceinline__ int32_t row_lower_bound(const int32_t* __restrict__ row, int32_t pu, int32_t lim) {
  int32_t lo = 0, hi = pu;
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (__ldg(row + mid) < lim) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ bool above(int32_t dj, int32_t j, int32_t dv, int32_t v) {
  return dj > dv || (dj == dv && j > v);
}

// dv <= 32 (labels >= n32): warp per v.  Lane e holds slot e of v's row;
// Adj+(v) is the set of lanes whose neighbour ranks above v (a shared hash
// label -> lane).  The rows (lower-ranked neighbours u) are short here
// (|Adj+(u)| <= du <= dv <= 32), so they are scanned FLAT: the warp lays all
// rows' entries end to end (exclusive scan of |Adj+(u)|, each flat position
// tagged with its row in shared memory) and probes 32 of them per step,
// whatever row they belong to -- a row-at-a-time scan left most lanes idle
// (WS-4M: ~10 rows of ~10 entries per seed against 64-lane steps).  Entries
// at or past v's own label (Adj+(u) is label-sorted) fail the `< rank(v)`
// test.  u's and w's sums go to shared 32-bit pieces of Q = -P (at most 32
// hits per row and per entry: no overflow), v's stay in registers.
constexpr int kMidFlat = 1024;  // 32 rows x 32 entries
#ifndef EFG_MID_WARP_EXACT
#define EFG_MID_WARP_EXACT 1
#endif
constexpr bool kMidWarpExact = EFG_MID_WARP_EXACT;
__global__ void __launch_bounds__(kMidWarps * 32)
k_mid_warp(MArgs a) {
  __shared__ int4 sK[kMidWarps][32];
  __shared__ int8_t sV[kMidWarps][128];
  __shared__ int32_t sE[kMidWarps][32];  // degree of each slot's neighbour (entries of Adj+(v) among them)
  __shared__ uint32_t sQ[kMidWarps][6][32];  // per lane: row pieces lo / hi / count, entry pieces lo / hi / count
  __shared__ int8_t sRow[kMidWarps][kMidFlat];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t r = a.n32 + ((int64_t)blockIdx.x * kMidWarps + w) * a.nparts + a.part;
  if (r >= a.n) return;
  const int32_t v = __ldg(a.by_rank + r);
  const int64_t ob = __ldg(a.offsets + v);
  const int32_t dv = (int32_t)(__ldg(a.offsets + v + 1) - ob);
  int32_t u = -1, du = 0, pu = 0;
  int64_t psu = 0;
  bool up = false;
  if (lane < dv) {
    u = __ldg(a.nbr + ob + lane);
    du = a.nd ? __ldg(a.nd + ob + lane) : __ldg(a.deg + u);
    up = above(du, u, dv, v);
    pu = __ldg(a.dplus + u);
    psu = __ldg(a.offsets + u);  // Adj+(u) starts at u's own row (slot space)
  }
  if (__ballot_sync(0xffffffffu, up) == 0) return;  // Adj+(v) empty: no triangle has v in the middle
  sK[w][lane] = make_int4(-1, -1, -1, -1);
  sE[w][lane] = du;
#pragma unroll
  for (int k = 0; k < 6; ++k) sQ[w][k][lane] = 0;
  // flat layout of the rows' entries: each row up to v's own label (Adj+(u) is
  // label-sorted; a binary search per lane, rows in parallel, halves the flat
  // length against scanning whole rows)
  int32_t len = 0;
  if (lane < dv && !up && pu >= 2) len = kMidWarpExact ? row_lower_bound(a.adjj + psu, pu, (int32_t)r) : pu;
  int32_t incl = len;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int32_t st = incl - len, total = __shfl_sync(0xffffffffu, incl, 31);
  for (int32_t p = 0; p < len; ++p) sRow[w][EFG_CLAMP(st + p, kMidFlat)] = (int8_t)lane;
  __syncwarp();
  if (up) smap_insert(sK[w], sV[w], 5, __ldg(a.rank_of + u), lane);
  __syncwarp();
  const uint32_t qb = (uint32_t)__cvta_generic_to_shared(&sQ[w][0][0]);
  const int32_t lim = (int32_t)r;
  Acc2 av;
  for (int32_t f0 = 0; f0 < total; f0 += 32) {
    const int32_t f = f0 + lane;
    const bool valid = f < total;
    const int32_t rr = valid ? (int32_t)sRow[w][f] : 0;
    const int32_t st_r = __shfl_sync(0xffffffffu, st, rr);
    const int64_t ps_r = __shfl_sync(0xffffffffu, psu, rr);
    const int32_t s0_r = dv + __shfl_sync(0xffffffffu, du, rr);
    const int32_t j = valid ? __ldg(a.adjj + ps_r + (f - st_r)) : INT32_MAX;
    const int32_t y = j < lim ? smap_find(sK[w], sV[w], 5, j) : -1;
    if (y >= 0) {
      const int64_t g = __ldg(a.PT + EFG_CLAMP(s0_r + sE[w][y], a.flen));
      av.add_row(g, 1);
      const uint64_t Q = (uint64_t)(-g);
      const uint32_t lo = (uint32_t)(Q & 0x3fffff), hi = (uint32_t)(Q >> 22);
      reds_add(qb + 4u * (0 * 32 + rr), lo);  // u's share (row rr)
      reds_add(qb + 4u * (1 * 32 + rr), hi);
      reds_add(qb + 4u * (2 * 32 + rr), 1u);
      reds_add(qb + 4u * (3 * 32 + y), lo);   // w's share (entry y)
      reds_add(qb + 4u * (4 * 32 + y), hi);
      reds_add(qb + 4u * (5 * 32 + y), 1u);
    }
  }
  __syncwarp();
  if (lane < dv) {
    if (sQ[w][2][lane]) {  // a row: u's share
      const uint64_t Q = ((uint64_t)sQ[w][1][lane] << 22) + sQ[w][0][lane];
      red_node(a.acc, u, -(int64_t)Q, sQ[w][2][lane]);
    }
    if (sQ[w][5][lane]) {  // an entry of Adj+(v): w's share
      const uint64_t Q = ((uint64_t)sQ[w][4][lane] << 22) + sQ[w][3][lane];
      red_node(a.acc, u, -(int64_t)Q, sQ[w][5][lane]);
    }
  }
  const int64_t vh = warp_sum(av.hi), vl = warp_sum(av.lo);
  const uint32_t vc = warp_count(av.c);
  if (lane == 0 && vc) {
    unsigned long long* q = a.acc + 4 * (int64_t)v;
    atomicAdd(q, (unsigned long long)vh);
    atomicAdd(q + 1, (unsigned long long)vl);
    atomicAdd(q + 2, (unsigned long long)vc);
  }
}

// dv > 32 (labels < n32, hubs first): CTA per v, warps take rows.  Entry
// sums of Adj+(v) in shared memory as 32-bit words (Q = -P split 22 + 23
// bits, count), flushed every kMidChunk rows.
template <class C>
struct MidSmem {
  // Adj+(v) as a map label -> position: a bitmap over labels [0, rank(v)),
  // each 32-bit word stored beside the popcount of the words before it (one
  // 8-byte shared load answers both membership and position: positions are
  // label ranks, Adj+ rows are sorted), when rank(v) is small enough, else a
  // bucketed hash
  union {
    struct {
      int4 lk[C::kNB];
      uint32_t lv[4 * C::kNB];  // packed entry: position | degree << kPosBits
    };
    uint2 bmp[C::kBmWords + 1];  // {bitmap word, popcount of the words before it}; + the zero word at lim >> 5
  };
  int64_t rps[C::kChunk];  // compacted rows of the current chunk: Adj+(u) start,
  int32_t ru[C::kChunk], rdu[C::kChunk], rpu[C::kChunk];  // u, du, |Adj+(u)|
  int32_t node[C::kMaxP], edeg[C::kMaxP + 1];  // edeg[np]: read (unused) by the bitmap scan's misses
  uint32_t elo[C::kMaxP], ehi[C::kMaxP], ec[C::kMaxP];
  int32_t nrows;
  int32_t wtot[C::kThreads / 32];
};

template <bool PART, class C>
__device__ __forceinline__ void mid_block_body(const MArgs& a, const HubTasks& tk) {
  constexpr int kMidThreads = C::kThreads, kMidLgNB = C::kLgNB, kMidMaxP = C::kMaxP,
                kMidChunk = C::kChunk;
  __shared__ MidSmem<C> sm;
  const uint32_t kb = (uint32_t)__cvta_generic_to_shared(sm.lk), vb = (uint32_t)__cvta_generic_to_shared(sm.lv);
  const uint32_t eb_lo = (uint32_t)__cvta_generic_to_shared(sm.elo), eb_hi = (uint32_t)__cvta_generic_to_shared(sm.ehi),
                 eb_c = (uint32_t)__cvta_generic_to_shared(sm.ec), db = (uint32_t)__cvta_generic_to_shared(sm.edeg);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int NW = kMidThreads / 32;
  int32_t v, x0, x1;
  // work unit of this part (PART: grid sized per part, units u % nparts == part)
  const int32_t unit = PART ? (int32_t)blockIdx.x * a.nparts + a.part : (int32_t)blockIdx.x;
  if (PART && unit >= a.nunits) return;
  if (unit < a.ntasks) {  // a row range of a hub
    v = tk.seed[unit];
    x0 = tk.x0[unit];
    x1 = tk.x1[unit];
  } else {
    v = __ldg(a.by_rank + a.label0 + (unit - a.ntasks));
    x0 = 0;
    x1 = (int32_t)(__ldg(a.offsets + v + 1) - __ldg(a.offsets + v));
  }
  const int64_t ob = __ldg(a.offsets + v);
  const int32_t dv = (int32_t)(__ldg(a.offsets + v + 1) - ob);
  const int64_t pb = __ldg(a.offsets + v);
  const int32_t pv = __ldg(a.dplus + v);
  const int32_t labv = __ldg(a.rank_of + v);
  if (pv == 0) return;  // no triangle has v in the middle
  Acc2 av;
  // Adj+(v) in parts of kMidMaxP entries (one part unless |Adj+(v)| > kMidMaxP);
  // a part's rows stop at its last label
  for (int32_t q0 = 0; q0 < pv; q0 += kMidMaxP) {
    const int32_t np = min(pv - q0, kMidMaxP);
    const int32_t lim = q0 + np < pv ? __ldg(a.adjj + pb + q0 + np) : labv;
    const uint32_t lgl = min(32u - __clz(max(np, 2) - 1), (uint32_t)kMidLgNB);  // NB = min(2^lgl >= np, kMidNB)
    (void)EFG_DCHECK(np <= (1 << kPosBits));
    const bool use_bm = C::kBmWords > 0 && lim <= 32 * C::kBmWords && lim <= a.bm_lim;  // block-uniform
    const int nbw = use_bm ? (lim + 31) >> 5 : 0;
    __syncthreads();
    if (use_bm) {
      for (int b = threadIdx.x; b < nbw; b += blockDim.x) sm.bmp[b] = make_uint2(0u, 0u);
      if (threadIdx.x == 0) sm.bmp[nbw] = make_uint2(0u, (uint32_t)np);  // the word of key lim: no member, prefix |part|
    } else {
      for (int b = threadIdx.x; b < (1 << lgl); b += blockDim.x) sm.lk[b] = make_int4(-1, -1, -1, -1);
    }
    __syncthreads();
    if (threadIdx.x == 0) sm.nrows = 0;  // the part's first chunk count (read after the next barrier)
    for (int t = threadIdx.x; t < np; t += blockDim.x) {
      const int32_t l = __ldg(a.adjj + pb + q0 + t);
      if (use_bm) atomicOr(&sm.bmp[l >> 5].x, 1u << (l & 31));
      const int32_t dl = __ldg(a.deg_by_rank + l);
      if (!use_bm) smap_insert(sm.lk, sm.lv, lgl, l, t | (dl << kPosBits));
      sm.node[t] = __ldg(a.by_rank + l);
      sm.edeg[t] = dl;
      sm.elo[t] = 0;
      sm.ehi[t] = 0;
      sm.ec[t] = 0;
    }
    if (use_bm) {
      // exclusive prefix of the words' popcounts: thread t owns words [t*per, (t+1)*per)
      __syncthreads();
      constexpr int per = C::kBmWords > 0 ? (C::kBmWords + kMidThreads - 1) / kMidThreads : 1;
      int tot = 0;
#pragma unroll
      for (int k = 0; k < per; ++k) {
        const int wi = threadIdx.x * per + k;
        tot += wi < nbw ? __popc(sm.bmp[wi].x) : 0;
      }
      int incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) sm.wtot[w] = incl;
      __syncthreads();
      int base = incl - tot;
      for (int k = 0; k < w; ++k) base += sm.wtot[k];
#pragma unroll
      for (int k = 0; k < per; ++k) {
        const int wi = threadIdx.x * per + k;
        if (wi < nbw) {
          sm.bmp[wi].y = (uint32_t)base;
          base += __popc(sm.bmp[wi].x);
        }
      }
    }
    const uint32_t bmb = (uint32_t)__cvta_generic_to_shared(sm.bmp);
    for (int32_t c0 = x0; c0 < x1; c0 += kMidChunk) {
      // compact the chunk's rows (lower-ranked u with |Adj+(u)| >= 2) into shared memory
      // (the count was zeroed before the part's setup barriers / in the previous chunk's flush)
      __syncthreads();
      for (int32_t x = c0 + threadIdx.x; x < min(x1, c0 + kMidChunk); x += blockDim.x) {
        const int64_t e = ob + x;
        const int32_t u = __ldg(a.nbr + e), du = a.nd ? __ldg(a.nd + e) : __ldg(a.deg + u);
        const int32_t pu = above(du, u, dv, v) ? 0 : __ldg(a.dplus + u);
        const bool keep = pu >= 2;
        const unsigned m = __ballot_sync(__activemask(), keep);
        int base = 0;
        const int leader = __ffs(__activemask()) - 1;
        if (lane == leader && m) base = atomicAdd(&sm.nrows, __popc(m));
        base = __shfl_sync(__activemask(), base, leader);
        if (keep) {
          const int k = base + __popc(m & ((1u << lane) - 1));
          sm.ru[k] = u;
          sm.rdu[k] = du;
          sm.rpu[k] = pu;
          sm.rps[k] = __ldg(a.offsets + u);
        }
      }
      __syncthreads();
      const int32_t nr = sm.nrows;
      for (int32_t x = w; x < nr; x += NW) {
        const int32_t u = sm.ru[x], du = sm.rdu[x], pu = sm.rpu[x];
        const int64_t psu = sm.rps[x];
        uint64_t rq = 0;  // the lane's sum of Q = -P over the row's hits
        uint32_t rc = 0;
        const auto hit = [&](int32_t y, int32_t, uint64_t q) {
          rq += q;
          ++rc;
          reds_add(eb_lo + 4 * y, (uint32_t)(q & 0x3fffff));
          reds_add(eb_hi + 4 * y, (uint32_t)(q >> 22));
          reds_add(eb_c + 4 * y, 1u);
        };
        // the map kind is block-uniform: one loop per kind, no branch in the probe
        // the unroll follows the row: the scan covers at most min(|Adj+(u)|, lim) entries
        // (distinct labels below lim), so short scans take one step of 32 / 64 lanes
        // instead of a 128-lane step
        const int32_t span = min(pu, lim);
        if (use_bm && kMidAdaptU && span <= EFG_MID_U1_SPAN)
          mid_scan_bm<1>(a.adjj + psu, pu, lim, a.PQ, (uint32_t)(dv + du), bmb, db, lane, hit, a.flen);
        else if (use_bm && kMidAdaptU && span <= EFG_MID_U2_SPAN)
          mid_scan_bm<2>(a.adjj + psu, pu, lim, a.PQ, (uint32_t)(dv + du), bmb, db, lane, hit, a.flen);
        else if (use_bm)
          mid_scan_bm<kMidUnrollBm>(a.adjj + psu, pu, lim, a.PQ, (uint32_t)(dv + du), bmb, db, lane, hit, a.flen);
        else if (kMidAdaptU && span <= EFG_MID_H1_SPAN)
          mid_scan_hash<1>(a.adjj + psu, pu, lim, a.PQ, (uint32_t)(dv + du), kb, vb, lgl, lane, hit, a.flen);
        else
          mid_scan_hash<C::kUnrollHash>(a.adjj + psu, pu, lim, a.PQ, (uint32_t)(dv + du), kb, vb, lgl, lane, hit,
                                        a.flen);
        rc = warp_count(rc);
        if (rc) {
          const int64_t rs = -warp_sum64((int64_t)rq);  // the row's sum of P (|lane sums| < 2^57)
          if (lane == 0) {
            red_node(a.acc, u, rs, rc);
            av.add_row(rs, rc);
          }
        }
      }
      __syncthreads();
      for (int t = threadIdx.x; t < np; t += blockDim.x) {
        if (t == 0) sm.nrows = 0;  // the next chunk's count (read again after its first barrier)
        if (sm.ec[t]) {
          const uint64_t q = ((uint64_t)sm.ehi[t] << 22) + sm.elo[t];
          red_node(a.acc, sm.node[t], -(int64_t)q, sm.ec[t]);
          sm.elo[t] = 0;
          sm.ehi[t] = 0;
          sm.ec[t] = 0;
        }
      }
    }
  }
  // v's own share: each warp's lane 0 holds its rows' part (integer words, any order): no block reduction
  if (lane == 0 && av.c) {
    unsigned long long* q = a.acc + 4 * (int64_t)v;
    atomicAdd(q, (unsigned long long)av.hi);
    atomicAdd(q + 1, (unsigned long long)av.lo);
    atomicAdd(q + 2, (unsigned long long)av.c);
  }
}

// Launch shapes: 4 CTAs of 320 threads per SM for the big instantiation (<= 51
// registers; round 1 with 256-thread CTAs: 5 per SM 14.6 ms against 15.6 at 63
// registers / 4), 12 for the small.
template <bool PART>
__global__ void __launch_bounds__(MidBig::kThreads, EFG_MID_BIG_MINB) k_mid_big(MArgs a, HubTasks tk) {
  mid_block_body<PART, MidBig>(a, tk);
}
template <bool PART>
__global__ void __launch_bounds__(MidSmall::kThreads, EFG_MID_SMALL_MINB) k_mid_small(MArgs a, HubTasks tk) {
  mid_block_body<PART, MidSmall>(a, tk);
}

// Per-seed results of the listing: t(v) and the two W_t words.
__global__ void k_list_out(const unsigned long long* __restrict__ acc, FArgs a, int64_t count) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= count) return;
  const unsigned long long* p = acc + 4 * (a.seed_lo + q);
  a.tri[q] = (int64_t)p[2];
  a.Wth[q] = (int64_t)p[0];
  a.Wtl[q] = (int64_t)p[1];
}

// Epilogue: closed-form T and mass, W, EF = ln T - W/T, flags.
__global__ void k_epilogue(FArgs a, int64_t count, double* __restrict__ ef, int64_t* __restrict__ total,
                           uint8_t* __restrict__ flags, int64_t* __restrict__ T_out, double* __restrict__ W_out) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= count) return;
  const int64_t v = a.seed_lo + q;
  const int64_t dv = a.offsets[v + 1] - a.offsets[v];
  const int64_t s1v = a.s1[v];
  const int64_t tri = a.tri[q];
  // chains: sum_i [(di-1)(dv+di-4) + S1(i) - dv] = S2 + (dv-5) S1 - 2dv^2 + 4dv + sum_i S1(i)
  const int64_t Tc = a.s2[v] + (dv - 5) * s1v - 2 * dv * dv + 4 * dv + (int64_t)a.cp2[v];
  const int64_t T = dv * (dv - 1) * (dv - 4) + 2 * (dv - 1) * s1v + Tc - 8 * tri;
  const int64_t mass = dv * (dv - 1) + s1v - dv;
  // W_t = X 2^-40 with X = Wth 2^32 + Wtl, converted from the canonical split
  // (0 <= lo < 2^32): a function of the exact integer only, so every triangle
  // path and every sharding gives the same double
  const int64_t xh = a.Wth[q] + (a.Wtl[q] >> 32), xl = a.Wtl[q] & 0xffffffffll;
  const double Wt = ldexp((double)xh, 32 - kListScale) + ldexp((double)xl, -kListScale);
  // W_c from its two words, canonical split likewise
  const int64_t ch = (int64_t)a.cwh[v] + ((int64_t)a.cwl[v] >> 32), cl = (int64_t)a.cwl[v] & 0xffffffffll;
  const int ce = chain_exp(dv, a.c0);
  const double Wc = dv > 0 ? ldexp((double)ch, ce) + ldexp((double)cl, ce - 32) : 0.0;
  const double W = (a.cws[v] + Wc) + 4.0 * Wt;
  double e = 0.0;
  // entropy >= 0: clamp the last-ulp cancellation of ln T - W/T when only one
  // positive-degree cluster class exists (EF mathematically 0)
  if (T > 0) e = fmax(log((double)T) - W / (double)T, 0.0);
  ef[q] = e;
  if (total) total[q] = mass;
  flags[q] = mass == 0 ? 1 : (T == 0 ? 2 : 0);
  if (T_out) T_out[q] = T;
  if (W_out) W_out[q] = W;
}

// Cluster totals |C(v)| = dv(dv-1) + S1(v) - dv (the epilogue's `mass`).
__global__ void k_mass(const int64_t* __restrict__ offsets, const int64_t* __restrict__ s1, int64_t n,
                       int64_t* __restrict__ total) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int64_t dv = offsets[v + 1] - offsets[v];
  total[v] = dv * (dv - 1) + s1[v] - dv;
}

struct DegRange {
  const int64_t* offsets;
  int64_t lo, hi;           // lo < dv <= hi
  __host__ __device__ bool operator()(const int32_t& v) const {
    int64_t d = offsets[v + 1] - offsets[v];
    return d > lo && d <= hi;
  }
};

// Seeds of r satisfying pred -> out (ascending); the count lands in *count_dev
// (device memory, read back with all other counts in one synchronisation).
template <class Pred>
void select_seeds(Context& ctx, SeedRange r, Pred pred, int32_t* out, int64_t* count_dev) {
  cudaStream_t s = ctx.stream;
  size_t tmp = 0;
  cub::CountingInputIterator<int32_t> it((int32_t)r.lo);
  const int64_t cnt = r.hi - r.lo;
  EFG_CUDA_CHECK(cub::DeviceSelect::If(nullptr, tmp, it, out, count_dev, cnt, pred, s));
  EFG_REGION("cub::DeviceSelect::If", s,
             EFG_CUDA_CHECK(cub::DeviceSelect::If(ctx.buf("cub").get(tmp), tmp, it, out, count_dev, cnt, pred, s)));
}

__global__ void k_seed_work(const int64_t* __restrict__ offsets, const int32_t* __restrict__ pcv,
                            const int32_t* __restrict__ dcnt, int64_t n, int64_t* __restrict__ work) {
  const int lane = threadIdx.x & 31;
  int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (v >= n) return;
  int64_t b = offsets[v], e = offsets[v + 1];
  int64_t w = 0;
  for (int64_t p = b + lane; p < e; p += 32) w += pcv[p] + 8;  // triangle probes + chain lookup
  w = warp_sum(w);
  if (lane == 0) {
    int64_t D = dcnt[v];
    work[v] = w + D * (D + 1) / 2 + 64;
  }
}

// The part's S1 / S2 into its words (nodes [lo, hi); zeros elsewhere).
__global__ void k_part_s12(const int64_t* __restrict__ s1, const int64_t* __restrict__ s2, int64_t lo, int64_t hi,
                           unsigned long long* __restrict__ w1, unsigned long long* __restrict__ w2) {
  const int64_t v = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= hi) return;
  w1[v] = (unsigned long long)s1[v];
  w2[v] = (unsigned long long)s2[v];
}

// Row work of the distributed pass per node, in units of a quarter adjacency
// slot: a per-row cost (launch share, histogram, small-row table), the slots
// (neighbour degrees, orientation, sort, pushes) and the chain table (~ |D_i|^2,
// |D_i| <= d, capped where the far-field expansion takes over).  Weights fitted
// to measured per-part times on R-MAT22 (tools/dist_estimate.py, N = 4 and 8:
// per row 0.73 ns, per slot 0.072 ns, per capped d^2 5.1e-5 ns).
__global__ void k_part_weight(const int64_t* __restrict__ offsets, int64_t n, int64_t* __restrict__ w) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int64_t d = offsets[v + 1] - offsets[v], dc = d < 1024 ? d : 1024;
  w[v] = 40 + 4 * d + dc * dc / 350;
}

// bounds[p] = first node whose inclusive work prefix reaches p * total / nparts
__global__ void k_part_search(const int64_t* __restrict__ prefix, int64_t n, int32_t nparts,
                              int64_t* __restrict__ bounds) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > nparts) return;
  if (p == 0 || p == nparts) {
    bounds[p] = p == 0 ? 0 : n;
    return;
  }
  const double target = (double)prefix[n - 1] * p / nparts;
  int64_t lo = 0, hi = n;  // first v with prefix[v] >= target, cut after it
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((double)prefix[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  bounds[p] = lo + 1 < n ? lo + 1 : n;
}

}  // namespace

void part_bounds(Context& ctx, const CSRView& g, int32_t nparts, int64_t* bounds) {
  cudaStream_t s = ctx.stream;
  const int64_t n = g.n;
  const int B = 256;
  int64_t* w = ctx.buf("pb_w").as<int64_t>(2 * n + nparts + 1);
  int64_t* pre = w + n;
  int64_t* db = w + 2 * n;
  EFG_LAUNCH(k_part_weight, ceil_div(n, B), B, 0, s, g.offsets, n, w);
  size_t tmp = 0;
  EFG_CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, tmp, w, pre, n, s));
  EFG_REGION("cub::DeviceScan::InclusiveSum", s,
             EFG_CUDA_CHECK(cub::DeviceScan::InclusiveSum(ctx.buf("cub").get(tmp), tmp, w, pre, n, s)));
  EFG_LAUNCH(k_part_search, 1, 64 * ceil_div(nparts + 1, 64), 0, s, pre, n, nparts, db);
  EFG_CUDA_CHECK(cudaMemcpyAsync(bounds, db, (nparts + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  EFG_CUDA_CHECK(cudaStreamSynchronize(s));
  for (int p = 1; p <= nparts; ++p) bounds[p] = std::max(bounds[p], bounds[p - 1]);
}

// Segment bounds of listed rows (CUB segmented sort over non-contiguous rows).

// Class lists by degree (all known before any histogram is built).
struct Lists {
  int32_t *hw8, *hw, *hs, *hb, *hl;  // histogram rows: d <= 8, <= 32, <= 256, <= 2048, > 2048 (all nodes)
  int32_t *cg, *cb;               // chain tables: d <= 64, > 64 (all nodes)
  int32_t *trs, *tr1, *tr2, *tr3, *hub;  // triangles
};
enum Slot {
  kHW8, kHW, kHS, kHB, kHL, kCG, kCB, kTrS, kTr1, kTr2, kTr3, kHubs, kNTasks, kNSlots
};
// per-chunk counts of the node-class lists (histograms, chain tables): class
// c in [kHW8, kCB], chunk k -> kNSlots + c * kMaxChunks + k
constexpr int kNCounts = kNSlots + (kCB + 1) * kMaxChunks;
__host__ __device__ constexpr int cslot(int c, int k) { return kNSlots + c * kMaxChunks + k; }
constexpr int64_t kHistWarpMax = 32, kHistBlockMax = kHistThreads * kHistItems, kCtabGroupMax = 64;
#ifndef EFG_CLASS_KERNELS
#define EFG_CLASS_KERNELS 1
#endif
constexpr bool kClassKernels = EFG_CLASS_KERNELS;

// Row-class lists in one pass over the degrees (instead of one CUB selection
// per class): tiles of kClsTile rows, per-tile class counts, a scan of the
// tile counts per class, then each tile scatters its rows in id order (the
// same ascending lists as a selection).  Classes: histogram class 0..4 (d <=
// 8, <= 32, <= 256, <= kHistBlockMax, above) and chain-table class 5 / 6
// (32 < d <= 64, d > 64); 12-bit fields of packed per-thread counts.
constexpr int kClsThreads = 256, kClsPer = 8, kClsTile = kClsThreads * kClsPer;
struct ClassArgs {
  const int32_t* deg;
  int64_t r0, r1;
  int32_t ntiles, nclasses;  // 5 (histograms only) or 7
  int32_t* list[7];
  int64_t* tcount;  // [7][ntiles]
  int64_t* tbase;   // [7][ntiles]
};
// per-thread packed counts of its kClsPer rows: hist classes (5 x 12 bits) and chain-table classes (2 x 12 bits)
__device__ __forceinline__ void cls_counts(const ClassArgs& a, int64_t v0, uint64_t& hc, uint32_t& cc) {
  hc = 0;
  cc = 0;
#pragma unroll
  for (int i = 0; i < kClsPer; ++i) {
    const int64_t v = v0 + i;
    if (v >= a.r1) break;
    const int32_t d = __ldg(a.deg + v);
    const int h = d <= 8 ? 0 : d <= 32 ? 1 : d <= 256 ? 2 : d <= (int32_t)(kHistThreads * kHistItems) ? 3 : 4;
    hc += 1ull << (12 * h);
    if (a.nclasses > 5 && d > 32) cc += 1u << (d > 64 ? 12 : 0);
  }
}
__global__ void __launch_bounds__(kClsThreads) k_class_count(ClassArgs a) {
  using BR64 = cub::BlockReduce<uint64_t, kClsThreads>;
  using BR32 = cub::BlockReduce<uint32_t, kClsThreads>;
  __shared__ typename BR64::TempStorage t64;
  __shared__ typename BR32::TempStorage t32;
  const int tile = blockIdx.x;
  uint64_t hc;
  uint32_t cc;
  cls_counts(a, a.r0 + (int64_t)tile * kClsTile + threadIdx.x * kClsPer, hc, cc);
  hc = BR64(t64).Sum(hc);
  cc = BR32(t32).Sum(cc);
  if (threadIdx.x == 0) {
    for (int c = 0; c < 5; ++c) a.tcount[(int64_t)c * a.ntiles + tile] = (int64_t)((hc >> (12 * c)) & 0xfff);
    for (int c = 5; c < a.nclasses; ++c) a.tcount[(int64_t)c * a.ntiles + tile] = (int64_t)((cc >> (12 * (c - 5))) & 0xfff);
  }
}
// block c: exclusive scan of class c's tile counts; its total into cdev[c]
__global__ void __launch_bounds__(1024) k_class_scan(ClassArgs a, int64_t* __restrict__ cdev) {
  using BS = cub::BlockScan<int64_t, 1024>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int64_t carry;
  const int c = blockIdx.x;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int32_t t0 = 0; t0 < a.ntiles; t0 += 1024) {
    const int32_t t = t0 + threadIdx.x;
    const int64_t x = t < a.ntiles ? a.tcount[(int64_t)c * a.ntiles + t] : 0;
    int64_t ex, tot;
    BS(tmp).ExclusiveSum(x, ex, tot);
    const int64_t base = carry;
    if (t < a.ntiles) a.tbase[(int64_t)c * a.ntiles + t] = base + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry = base + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) cdev[c] = carry;
}
__global__ void __launch_bounds__(kClsThreads) k_class_scatter(ClassArgs a) {
  using BS64 = cub::BlockScan<uint64_t, kClsThreads>;
  using BS32 = cub::BlockScan<uint32_t, kClsThreads>;
  __shared__ typename BS64::TempStorage t64;
  __shared__ typename BS32::TempStorage t32;
  const int tile = blockIdx.x;
  const int64_t v0 = a.r0 + (int64_t)tile * kClsTile + threadIdx.x * kClsPer;
  uint64_t hc;
  uint32_t cc;
  cls_counts(a, v0, hc, cc);
  BS64(t64).ExclusiveSum(hc, hc);
  BS32(t32).ExclusiveSum(cc, cc);
  int64_t pos[7];
#pragma unroll
  for (int c = 0; c < 5; ++c) pos[c] = a.tbase[(int64_t)c * a.ntiles + tile] + (int64_t)((hc >> (12 * c)) & 0xfff);
#pragma unroll
  for (int c = 5; c < 7; ++c)
    pos[c] = c < a.nclasses ? a.tbase[(int64_t)c * a.ntiles + tile] + (int64_t)((cc >> (12 * (c - 5))) & 0xfff) : 0;
#pragma unroll
  for (int i = 0; i < kClsPer; ++i) {
    const int64_t v = v0 + i;
    if (v >= a.r1) break;
    const int32_t d = __ldg(a.deg + v);
    const int h = d <= 8 ? 0 : d <= 32 ? 1 : d <= 256 ? 2 : d <= (int32_t)(kHistThreads * kHistItems) ? 3 : 4;
#pragma unroll
    for (int c = 0; c < 5; ++c)
      if (c == h) a.list[c][pos[c]++] = (int32_t)v;
    if (a.nclasses > 5 && d > 32) {
      if (d > 64) a.list[6][pos[6]++] = (int32_t)v;
      else a.list[5][pos[5]++] = (int32_t)v;
    }
  }
}

// per-chunk runs of the row-class lists: chunk k of class c = ids in [row[k], row[k+1])
struct ChunkLists {
  const int32_t* list[kCB + 1];
  int nlists, nchunks;
  int64_t row[kMaxChunks + 1];
};
__device__ __forceinline__ int64_t ids_below(const int32_t* __restrict__ l, int64_t len, int64_t x) {
  int64_t lo = 0, hi = len;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (l[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__global__ void k_chunk_counts(ChunkLists cl, int64_t* __restrict__ cdev) {
  const int c = threadIdx.x / kMaxChunks, k = threadIdx.x % kMaxChunks;
  if (c >= cl.nlists || k >= cl.nchunks) return;
  const int64_t len = cdev[c];  // the class's total (slot c)
  cdev[cslot(c, k)] = ids_below(cl.list[c], len, cl.row[k + 1]) - ids_below(cl.list[c], len, cl.row[k]);
}
// first entry of chunk k's run in class list cls (host, from the read-back counts)
static inline int64_t lstart(const int64_t* c, int cls, int k) {
  int64_t s = 0;
  for (int j = 0; j < k; ++j) s += c[cslot(cls, j)];
  return s;
}

// Node-class lists.  Histogram and chain-table classes are selected once over
// all rows; chunk k's run of list X starts at X + lstart(c, X, k), so their
// kernels can run on a chunk as soon as its neighbours are resident.
// row_lists: the per-chunk histogram / chain-table classes; tri_lists (with
// seeds): the triangle classes and the hub list.
static Lists make_lists(Context& ctx, const Prepared& P, const Staging& stg, SeedRange r, int64_t* cdev, bool seeds,
                        bool row_lists = true, bool tri_lists = true) {
  const int64_t n = P.g.n, cnt = r.hi - r.lo;
  auto list = [&](const char* name, int64_t len) { return ctx.buf(name).as<int32_t>(len > 0 ? len : 1); };
  const int64_t* off = P.g.offsets;
  Lists L{};
  if (row_lists) {
  L.hw8 = list("f_l_hw8", n);
  L.hw = list("f_l_hw", n);
  L.hs = list("f_l_hs", n);
  L.hb = list("f_l_hb", n);
  L.hl = list("f_l_hl", n);
  if (seeds) {
    L.cg = list("f_l_cg", n);
    L.cb = list("f_l_cb", n);
  }
  // one selection per class over all the chunks' rows (ids ascending); chunk
  // k's part is the run of ids in [row[k], row[k+1]) (k_chunk_counts), at
  // lstart(c, cls, k) -- 7 selections instead of 7 per chunk (each a few
  // launches: 28 of them were 2 ms on the staged path before any row work)
  const SeedRange all{stg.row[0], stg.row[stg.nchunks]};
  static_assert(kHistWarpMax == 32 && kCtabGroupMax == 64, "k_class_* hard-code the class bounds");
  if (kClassKernels) {
    ClassArgs ca{};
    ca.deg = P.deg;
    ca.r0 = all.lo;
    ca.r1 = all.hi;
    ca.ntiles = (int32_t)ceil_div(all.hi - all.lo, (int64_t)kClsTile);
    ca.nclasses = seeds ? 7 : 5;
    int32_t* lists7[7] = {L.hw8, L.hw, L.hs, L.hb, L.hl, L.cg, L.cb};
    for (int c = 0; c < 7; ++c) ca.list[c] = lists7[c];
    ca.tcount = ctx.buf("f_cls_tiles").as<int64_t>(2 * 7 * (int64_t)std::max(ca.ntiles, 1));
    ca.tbase = ca.tcount + 7 * (int64_t)std::max(ca.ntiles, 1);
    if (ca.ntiles > 0) {
      EFG_LAUNCH(k_class_count, ca.ntiles, kClsThreads, 0, ctx.stream, ca);
      EFG_LAUNCH(k_class_scan, ca.nclasses, 1024, 0, ctx.stream, ca, cdev);
      EFG_LAUNCH(k_class_scatter, ca.ntiles, kClsThreads, 0, ctx.stream, ca);
    }
  } else {
    select_seeds(ctx, all, DegRange{off, -1, 8}, L.hw8, cdev + kHW8);
    select_seeds(ctx, all, DegRange{off, 8, kHistWarpMax}, L.hw, cdev + kHW);
    select_seeds(ctx, all, DegRange{off, kHistWarpMax, 256}, L.hs, cdev + kHS);
    select_seeds(ctx, all, DegRange{off, 256, kHistBlockMax}, L.hb, cdev + kHB);
    select_seeds(ctx, all, DegRange{off, kHistBlockMax, INT64_MAX}, L.hl, cdev + kHL);
    if (seeds) {
      select_seeds(ctx, all, DegRange{off, kHistWarpMax, kCtabGroupMax}, L.cg, cdev + kCG);
      select_seeds(ctx, all, DegRange{off, kCtabGroupMax, INT64_MAX}, L.cb, cdev + kCB);
    }
  }
  ChunkLists cl{};
  const int32_t* lists[kCB + 1] = {L.hw8, L.hw, L.hs, L.hb, L.hl, L.cg, L.cb};
  for (int c = 0; c <= kCB; ++c) cl.list[c] = lists[c];
  cl.nlists = seeds ? kCB + 1 : kHL + 1;
  cl.nchunks = stg.nchunks;
  for (int k = 0; k <= stg.nchunks; ++k) cl.row[k] = stg.row[k];
  EFG_LAUNCH(k_chunk_counts, 1, 64, 0, ctx.stream, cl, cdev);
  }
  if (!seeds || !tri_lists) return L;
  L.trs = list("f_l_trs", cnt);
  L.tr1 = list("f_l_tr1", cnt);
  L.tr2 = list("f_l_tr2", cnt);
  L.tr3 = list("f_l_tr3", cnt);
  L.hub = list("f_l_hub", cnt);
  select_seeds(ctx, r, DegRange{off, -1, 32}, L.trs, cdev + kTrS);
  select_seeds(ctx, r, DegRange{off, 32, 256}, L.tr1, cdev + kTr1);
  select_seeds(ctx, r, DegRange{off, 256, 1024}, L.tr2, cdev + kTr2);
  select_seeds(ctx, r, DegRange{off, 1024, kHashMaxDeg}, L.tr3, cdev + kTr3);
  select_seeds(ctx, r, DegRange{off, kHashMaxDeg, INT64_MAX}, L.hub, cdev + kHubs);
  return L;
}

// Neighbour-degree histograms H_i for every node (slot space, see H build).
static void build_histograms(Context& ctx, const Prepared& P, const Lists& L, const int64_t* c, const Staging& stg,
                             int k, int32_t* hkey, int32_t* hcnt, int32_t* dcnt, bool small_rows = true) {
  cudaStream_t s = ctx.stream;
  const int B = 256;
  const int64_t* off = P.g.offsets;
  const int64_t nw = c[cslot(kHW, k)], ns = c[cslot(kHS, k)], nb = c[cslot(kHB, k)], nl = c[cslot(kHL, k)];
  if (small_rows) {
    const int64_t nw8 = c[cslot(kHW8, k)];
    EFG_LAUNCH(k_hist_warp, ceil_div(nw8 * 32, B), B, 0, s, L.hw8 + lstart(c, kHW8, k), nw8, off, P.nd, hkey, hcnt,
               dcnt);
    EFG_LAUNCH(k_hist_warp, ceil_div(nw * 32, B), B, 0, s, L.hw + lstart(c, kHW, k), nw, off, P.nd, hkey, hcnt, dcnt);
  }
  int bits = 1;
  while (bits < 31 && (int64_t(1) << bits) <= (int64_t)P.dmax + 1) ++bits;
  EFG_LAUNCH(k_hist_warp8, ceil_div(ns * 32, kHistW8Warps * 32), kHistW8Warps * 32, 0, s, L.hs + lstart(c, kHS, k), ns,
             off, P.nd,
             hkey, hcnt, dcnt);
  EFG_LAUNCH((k_hist_block<kHistThreads, kHistItems>), nb, kHistThreads, 0, s, L.hb + lstart(c, kHB, k), nb, off, P.nd,
             hkey, hcnt,
             dcnt, bits);
  if (nl) {
    const int smw = kHistWin * (int)sizeof(int32_t);
    EFG_CUDA_CHECK(cudaFuncSetAttribute(k_hist_count, cudaFuncAttributeMaxDynamicSharedMemorySize, smw));
    EFG_LAUNCH(k_hist_count, nl, kHistBigThreads, smw, s, L.hl + lstart(c, kHL, k), nl, off, P.nd, hkey, hcnt, dcnt);
  }
}

static int64_t read_counts(Context& ctx, const int64_t* cdev, int64_t* c) {
  EFG_CUDA_CHECK(cudaMemcpyAsync(c, cdev, kNCounts * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx.stream));
  EFG_CUDA_CHECK(cudaStreamSynchronize(ctx.stream));
  return 0;
}

void factorized_work(Context& ctx, Prepared& P, int64_t* d_work) {
  const int64_t n = P.g.n, m2 = P.g.m2 > 0 ? P.g.m2 : 1;
  Staging one;
  one.row[1] = n;
  one.slot[1] = P.g.m2;
  int64_t* cdev = ctx.buf("f_counts").as<int64_t>(kNCounts);
  EFG_CUDA_CHECK(cudaMemsetAsync(cdev, 0, kNCounts * sizeof(int64_t), ctx.stream));
  Lists L = make_lists(ctx, P, one, SeedRange{0, n}, cdev, false);
  int64_t c[kNCounts];
  read_counts(ctx, cdev, c);
  int32_t* hkey = ctx.buf("f_hkey").as<int32_t>(m2);
  int32_t* hcnt = ctx.buf("f_hcnt").as<int32_t>(m2);
  int32_t* dcnt = ctx.buf("f_dcnt").as<int32_t>(n);
  build_histograms(ctx, P, L, c, one, 0, hkey, hcnt, dcnt);
  const int B = 256;
  EFG_LAUNCH(k_seed_work, ceil_div(n * 32, B), B, 0, ctx.stream, P.g.offsets, P.pc, dcnt, n, d_work);
}

// The pass has two host synchronisations: dmax (prepare_head) and one
// batched read of every class count; the rest is launched back to back.  With
// staged host inputs the per-row work (neighbour degrees, histograms, chain
// tables) of each row chunk runs while the next chunk is still copied.
PrepInfo ef_factorized(Context& ctx, const CSRView& g, const Staging& stg, SeedRange r, double* ef, int64_t* total,
                       uint8_t* flags, int64_t* T_out, double* W_out, efg_stats* st, const DistPart* dp) {
  cudaStream_t s = ctx.stream;
  const int64_t n = g.n, m2 = g.m2 > 0 ? g.m2 : 1;
  const int B = 256;
  size_t tmp = 0;
  const int64_t cnt = r.hi - r.lo;
  Prepared P;
  if (st) EFG_CUDA_CHECK(cudaEventRecord(ctx.ev[2], s));
  const int dmode = dp ? dp->mode : -1;
  auto& dh = ctx.dist_head;
  if ((dmode == kDistList || dmode == kDistTables) && dh.valid && dh.P.g.offsets == g.offsets && dh.P.g.nbr == g.nbr && dh.P.g.n == n &&
      dh.P.g.m2 == g.m2) {
    P = dh.P;  // the rows part's degrees, tables and rank labels on this graph are still resident
  } else {
    prepare_head(ctx, g, true, P);
  }
  // distributed parts work on their node range, as one resident chunk
  Staging own;
  if (dp) {
    own.nchunks = 1;
    own.row[0] = dp->node_lo;
    own.row[1] = dp->node_hi;
    if (dmode != kDistRepl) {  // the caller's (exchanged) Adj+ rows and |Adj+|
      P.adjj = dp->adjp;
      P.dplus = dp->dplus;
    }
  }
  const Staging& rows = dp ? own : stg;
  // ---- phase 1: class lists and counts on the device, one read-back
  int64_t* cdev = ctx.buf("f_counts").as<int64_t>(kNCounts);
  EFG_CUDA_CHECK(cudaMemsetAsync(cdev, 0, kNCounts * sizeof(int64_t), s));
  // whole-graph passes list triangles (they gather |Adj+(u)| from dplus); the
  // per-seed triangle path reads it per slot from the slot table
  const bool listing = dp || (r.lo == 0 && r.hi == n && P.dmax <= kListMaxDeg);
  const bool tables = dmode == -1 || dmode == kDistRepl || dmode == kDistTables;  // chain tables and pushes here
  Lists L = make_lists(ctx, P, rows, r, cdev, true, tables, !listing);
  if (dp) {
    EFG_REQUIRE(P.dmax <= kListMaxDeg, "distributed pass: maximum degree above the listing bound");
    if (dmode == kDistRepl || dmode == kDistRows) {  // the tables / listing parts add into these words
      EFG_CUDA_CHECK(cudaMemsetAsync(dp->words, 0, kDistWords * n * sizeof(unsigned long long), s));
      EFG_CUDA_CHECK(cudaMemsetAsync(dp->ws, 0, n * sizeof(double), s));
    }
  }
  if (!listing)
    EFG_LAUNCH(k_hub_count, 2 * ctx.num_sms, 256, 0, s, L.hub, cdev + kHubs, g.offsets,
               reinterpret_cast<unsigned long long*>(cdev + kNTasks));
  else if (dmode != kDistRows && dmode != kDistTables)
    EFG_LAUNCH(k_list_counts, 1, 256, 0, s, P.deg_by_rank, n, cdev, kTrS, kTr1, kTr2, kTr3, kHubs, kNTasks);
  int64_t c[kNCounts];
  read_counts(ctx, cdev, c);
  // ---- phase 2: no further host synchronisation; per row chunk as it arrives
  int32_t* dcnt = ctx.buf("f_dcnt").as<int32_t>(n);
  int32_t* hkey = nullptr;
  int32_t* hcnt = nullptr;
  ChainAcc ca{};
  if (dmode != kDistList) {
    double* ctab = nullptr;
    if (tables) {
      hkey = ctx.buf("f_hkey").as<int32_t>(m2);
      hcnt = ctx.buf("f_hcnt").as<int32_t>(m2);
      ctab = ctx.buf("f_ctab").as<double>(m2);
      unsigned long long* acc = dp ? dp->words : ctx.buf("f_chain_acc").as<unsigned long long>(3 * n);
      if (!dp) EFG_CUDA_CHECK(cudaMemsetAsync(acc, 0, 3 * n * sizeof(unsigned long long), s));
      ca.wh = acc;
      ca.wl = acc + n;
      ca.p2 = acc + 2 * n;
      ca.ws = dp ? dp->ws : ctx.buf("f_chain_ws").as<double>(n);
      const double d3 = 3.0 * (P.dmax > 1 ? P.dmax : 1);
      ca.c0 = (P.dmax > 1 ? P.dmax : 1) * d3 * log(d3);
    }
    if (dmode == kDistRepl) prepare_rows(ctx, P, 0, n, 0, g.m2);  // every row's orientation, no exchange
    for (int k = 0; k < rows.nchunks; ++k) {
      if (!dp && stg.ready[k]) EFG_CUDA_CHECK(cudaStreamWaitEvent(s, stg.ready[k], 0));
      if (dmode == -1 || dmode == kDistRows)
        prepare_rows(ctx, P, rows.row[k], rows.row[k + 1], rows.slot[k], rows.slot[k + 1]);
      if (!tables) continue;
      build_histograms(ctx, P, L, c, rows, k, hkey, hcnt, dcnt, false);
      // rows with d <= 32: histogram, chain table and pushes fused in registers
      // (d <= 8: four rows per warp)
      const int64_t nsm8 = c[cslot(kHW8, k)], nsm = c[cslot(kHW, k)];
      EFG_LAUNCH(k_small_rows8, ceil_div(ceil_div(nsm8, 4), kSmallWarps), kSmallWarps * 32, 0, s,
                 L.hw8 + lstart(c, kHW8, k), nsm8, g.offsets, g.nbr, P.nd, P.ftab, P.s1, ca, P.ftab_len);
      EFG_LAUNCH(k_small_rows, ceil_div(nsm, kSmallWarps), kSmallWarps * 32, 0, s, L.hw + lstart(c, kHW, k), nsm,
                 g.offsets, g.nbr, P.nd, P.deg, P.ftab, P.s1, ca, P.ftab_len);
      // chain tables C_i(y): rows with 32 < d <= 64 by 8-lane groups, the rest by CTAs
      const int64_t ng = c[cslot(kCG, k)], nb = c[cslot(kCB, k)];
      EFG_LAUNCH(k_ctab_group<8>, ceil_div(ng * 8, B), B, 0, s, L.cg + lstart(c, kCG, k), ng, g.offsets, dcnt, hkey, hcnt, P.deg,
                 P.ftab, ctab, P.ftab_len);
      // rows of degree > 64: fewer than kCtabWarpD distinct neighbour degrees (half of them,
      // no far-field expansion) a warp each, the rest a CTA each
      EFG_LAUNCH(k_ctab_block, nb, kCtabThreads, 0, s, L.cb + lstart(c, kCB, k), nb, g.offsets, dcnt, hkey, hcnt, P.deg, P.ftab,
                 ctab, kExpMin, kExpMinD, P.ftab_len, kCtabWarpD);
      if (kCtabWarpD > 0)
        EFG_LAUNCH(k_ctab_warp<kCtabWarpD / 32>, ceil_div(nb, kCtabWarps), kCtabWarps * 32, 0, s, L.cb + lstart(c, kCB, k), nb, g.offsets, dcnt, hkey,
                   hcnt, P.deg, P.ftab, ctab, P.ftab_len, kCtabWarpD - 1);
      // chains pushed from the rows whose tables are now complete
      const int64_t ps1 = c[cslot(kHS, k)], pb = c[cslot(kHB, k)], pl = c[cslot(kHL, k)];
      EFG_LAUNCH(k_push_warp256, ceil_div(ps1, kPushWarps), kPushWarps * 32, 0, s, L.hs + lstart(c, kHS, k), ps1, g.offsets, g.nbr,
                 P.nd, dcnt, hkey, hcnt, ctab, P.s1, ca);
      EFG_LAUNCH(k_push_block, pb, kPushThreads, 0, s, L.hb + lstart(c, kHB, k), pb, g.offsets, g.nbr, P.nd, dcnt, hkey, hcnt, ctab,
                 P.s1, ca);
      // rows of degree > 2048 in kPushSlices slices each (a hub row is one CTA's long serial loop otherwise)
      EFG_LAUNCH(k_push_block, dim3((unsigned)pl, kPushSlices), kPushThreads, 0, s, L.hl + lstart(c, kHL, k), pl, g.offsets, g.nbr,
                 P.nd, dcnt, hkey, hcnt, ctab, P.s1, ca);
    }
    if (dmode == kDistRepl || dmode == kDistRows) {  // the part's S1 / S2 into the words (the finish needs them)
      const int64_t cntp = dp->node_hi - dp->node_lo;
      if (cntp > 0)
        EFG_LAUNCH(k_part_s12, ceil_div(cntp, B), B, 0, s, P.s1, P.s2, dp->node_lo, dp->node_hi,
                   dp->words + 7 * n, dp->words + 8 * n);
    }
    if (stg.total_host && !dp && r.lo == 0 && r.hi == n && n > 0) {
      // S1 is complete: cluster totals now, their read-back overlaps the listing
      EFG_LAUNCH(k_mass, ceil_div(n, B), B, 0, s, g.offsets, P.s1, n, total);
      EFG_CUDA_CHECK(cudaEventRecord(ctx.aux_ev[0], s));
      EFG_CUDA_CHECK(cudaStreamWaitEvent(ctx.copy_stream, ctx.aux_ev[0], 0));
      EFG_CUDA_CHECK(cudaMemcpyAsync(stg.total_host, total, n * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                     ctx.copy_stream));
      EFG_CUDA_CHECK(cudaEventRecord(ctx.aux_ev[1], ctx.copy_stream));
      ctx.total_sent = true;
      total = nullptr;
    }
    if (dmode == kDistRows) {
      // the part's rows sorted; the caller exchanges Adj+ rows and |Adj+| (overlapping the tables part),
      // then runs the listing part
      prepare_tail(ctx, P, true, false, dp->node_lo, dp->node_hi);
      if (st) EFG_CUDA_CHECK(cudaEventRecord(ctx.ev[3], s));
      dh.P = P;
      dh.valid = true;
      return PrepInfo{P.dmax, P.sum_c2};
    }
    if (dmode == kDistTables) {
      if (st) EFG_CUDA_CHECK(cudaEventRecord(ctx.ev[3], s));
      return PrepInfo{P.dmax, P.sum_c2};
    }
    prepare_tail(ctx, P, true, !listing);
  }
  if (st) EFG_CUDA_CHECK(cudaEventRecord(ctx.ev[3], s));
  const PrepInfo info{P.dmax, P.sum_c2};
  if (cnt <= 0 && !dp) return info;
  FArgs a;
  a.offsets = P.g.offsets;
  a.nbr = P.g.nbr;
  a.nd = P.nd;
  a.s1 = P.s1;
  a.F = P.ftab;
  a.flen = P.ftab_len;
  a.G = P.gtab;
  a.pc = P.pc;
  a.adjj = P.adjj;
  a.adjd = P.adjd;
  a.deg = P.deg;
  a.rank_of = P.rank_of;
  a.deg_by_rank = P.deg_by_rank;
  a.dcnt = dcnt;
  a.hkey = hkey;
  a.hcnt = hcnt;
  a.seed_lo = r.lo;
  a.s2 = P.s2;
  a.cwh = ca.wh;
  a.cwl = ca.wl;
  a.cp2 = ca.p2;
  a.cws = ca.ws;
  a.c0 = ca.c0;
  a.tri = ctx.buf("f_tri").as<int64_t>(cnt > 0 ? cnt : 1);
  a.Wth = ctx.buf("f_Wth").as<int64_t>(cnt > 0 ? cnt : 1);
  a.Wtl = ctx.buf("f_Wtl").as<int64_t>(cnt > 0 ? cnt : 1);
  {
    int64_t* PT = ctx.buf("l_pt").as<int64_t>(P.ftab_len);
    uint64_t* PQ = ctx.buf("l_pq").as<uint64_t>(P.ftab_len);
    EFG_LAUNCH(k_gfix, ceil_div(P.ftab_len, B), B, 0, s, P.gtab, P.ftab_len, PT, PQ);
    a.PT = PT;
    a.PQ = PQ;
  }
  // 2. triangles: listed once each for whole-graph passes, else per seed (the long kernels first)
  const int64_t nhubs = c[kHubs], ntasks = c[kNTasks];
  // hub tasks (hubs in descending work order, kHubRows rows each) serve both triangle paths
  HubTasks tk{};
  int64_t* tstart = nullptr;
  int32_t* hs = nullptr;
  if (nhubs) {
    {  // hubs in descending triangle-probe order (the longest hub tasks start first); a listing
       // pass takes the hub list from the rank order (labels [0, nhubs) are the hubs)
      const int32_t* hubs = listing ? P.by_rank : L.hub;
      int64_t* hw = ctx.buf("f_hub_work").as<int64_t>(2 * nhubs + 2);
      EFG_LAUNCH(k_hub_work, nhubs, 256, 0, s, hubs, nhubs, g.offsets, g.nbr, P.dplus, hw);
      int64_t* hw_sorted = hw + nhubs;
      hs = ctx.buf("f_hub_sorted").as<int32_t>(nhubs);
      EFG_CUDA_CHECK(
          cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, hw, hw_sorted, hubs, hs, nhubs, 0, 64, s));
      EFG_REGION("cub::DeviceRadixSort::SortPairsDescending", s,
                 EFG_CUDA_CHECK(cub::DeviceRadixSort::SortPairsDescending(ctx.buf("cub").get(tmp), tmp, hw,
                                                                          hw_sorted, hubs, hs, nhubs, 0, 64, s)));
    }
    int64_t* hnt = ctx.buf("f_hub_nt").as<int64_t>(nhubs + 1);
    tstart = ctx.buf("f_hub_tstart").as<int64_t>(nhubs + 1);
    EFG_LAUNCH(k_hub_ntasks, ceil_div(nhubs + 1, B), B, 0, s, hs, nhubs, P.g.offsets, hnt);
    EFG_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, hnt, tstart, nhubs + 1, s));
    EFG_REGION("cub::DeviceScan::ExclusiveSum", s,
               EFG_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(ctx.buf("cub").get(tmp), tmp, hnt, tstart, nhubs + 1, s)));
    int32_t* tseed = ctx.buf("f_hub_tseed").as<int32_t>(ntasks);
    int32_t* tx0 = ctx.buf("f_hub_tx0").as<int32_t>(ntasks);
    int32_t* tx1 = ctx.buf("f_hub_tx1").as<int32_t>(ntasks);
    EFG_LAUNCH(k_hub_tasks, ceil_div(nhubs, B), B, 0, s, hs, nhubs, P.g.offsets, tstart, tseed, tx0, tx1);
    tk.seed = tseed;
    tk.x0 = tx0;
    tk.x1 = tx1;
    if (st) st->terms = ntasks;
  }
  if (listing) {
    MArgs ma;
    unsigned long long* acc = dp ? dp->words + 3 * n : ctx.buf("l_acc").as<unsigned long long>(4 * n);
    if (!dp) EFG_CUDA_CHECK(cudaMemsetAsync(acc, 0, 4 * n * sizeof(unsigned long long), s));
    ma.offsets = P.g.offsets;
    ma.nbr = P.g.nbr;
    ma.nd = dp && dp->mode == kDistList ? nullptr : P.nd;
    ma.deg = P.deg;
    ma.dplus = P.dplus;
    ma.adjj = P.adjj;
    ma.adjd = P.adjd;
    ma.rank_of = P.rank_of;
    ma.by_rank = P.by_rank;
    ma.deg_by_rank = P.deg_by_rank;
    ma.PT = a.PT;
    ma.PQ = a.PQ;
    ma.flen = P.ftab_len;
    ma.bm_lim = INT32_MAX;
    if (const char* e = getenv("EFG_MID_BM_LIMIT")) ma.bm_lim = atoi(e);  // tests: the hash path on every part
    ma.acc = acc;
    ma.n = n;
    ma.n32 = c[kTr1] + c[kTr2] + c[kTr3] + c[kHubs];  // whole-graph pass: nodes of degree > 32
    ma.nhubs = nhubs;                                  // labels [0, nhubs): degree > kHashMaxDeg
    ma.ntasks = ntasks;
    ma.nparts = dp ? dp->nparts : 1;
    ma.part = dp ? dp->part : 0;
    // big CTAs: hub tasks and labels [nhubs, n256); small CTAs: labels [n256, n32)
    const int64_t n256 = c[kTr2] + c[kTr3] + c[kHubs];
    ma.label0 = nhubs;
    ma.nunits = (int32_t)(ntasks + (n256 - nhubs));
    MArgs ms = ma;
    ms.ntasks = 0;
    ms.label0 = n256;
    ms.nunits = (int32_t)(ma.n32 - n256);
    if (dp) {
      EFG_LAUNCH(k_mid_big<true>, ceil_div(ma.nunits, ma.nparts), MidBig::kThreads, 0, s, ma, tk);
      EFG_LAUNCH(k_mid_small<true>, ceil_div(ms.nunits, ms.nparts), MidSmall::kThreads, 0, s, ms, tk);
    } else {
      EFG_LAUNCH(k_mid_big<false>, ma.nunits, MidBig::kThreads, 0, s, ma, tk);
      EFG_LAUNCH(k_mid_small<false>, ms.nunits, MidSmall::kThreads, 0, s, ms, tk);
    }
    EFG_LAUNCH(k_mid_warp, ceil_div(ceil_div(n - ma.n32, ma.nparts), kMidWarps), kMidWarps * 32, 0, s, ma);
    if (dp) return info;  // the caller reduces the words over all parts, then ef_finish
    EFG_LAUNCH(k_list_out, ceil_div(cnt, B), B, 0, s, acc, a, cnt);
  } else if (nhubs) {
    // exact bitmaps over rank labels, per-task partials merged in task order
    const int64_t words = ceil_div(n, 32);
    uint32_t* bms = ctx.buf("f_bitmaps").as<uint32_t>(nhubs * words);
    int32_t* hub_slot = ctx.buf("f_hub_slot").as<int32_t>(n);
    EFG_CUDA_CHECK(cudaMemsetAsync(bms, 0, nhubs * words * sizeof(uint32_t), s));
    EFG_LAUNCH(k_hub_bitmaps, nhubs, 1024, 0, s, L.hub, nhubs, P.g.offsets, P.g.nbr, P.rank_of, bms, words, hub_slot);
    tk.ptri = ctx.buf("f_hub_ptri").as<int64_t>(ntasks);
    tk.pWh = ctx.buf("f_hub_pWh").as<int64_t>(ntasks);
    tk.pWl = ctx.buf("f_hub_pWl").as<int64_t>(ntasks);
    const int smh = kFilterWords * 4;
    EFG_CUDA_CHECK(cudaFuncSetAttribute(k_tri_hub, cudaFuncAttributeMaxDynamicSharedMemorySize, smh));
    EFG_LAUNCH(k_tri_hub, ntasks, kHubThreads, smh, s, tk, ntasks, bms, words, hub_slot, a);
    EFG_LAUNCH(k_hub_merge, ceil_div(nhubs, B), B, 0, s, hs, nhubs, tstart, tk.ptri, tk.pWh, tk.pWl, a);
  }
  if (!listing) {
    int4* rowhash = ctx.buf("f_rowhash").as<int4>(2 * m2);  // bucket 2*offsets[i] starts Adj+(i)'s hash
    EFG_LAUNCH(k_rowhash, ceil_div(n * 32, B), B, 0, s, P.g.offsets, P.dplus, P.adjj, n, rowhash);
    a.rowhash = rowhash;
    // buckets of 4 keys: dv <= 256 at load <= 1/8 with degrees, dv <= 1024 / 4096 at load <= 1/4
    auto k_tri_seed_256 = k_tri_seed<128, 512, true>;
    auto k_tri_seed_1024 = k_tri_seed<256, 1024, true>;
    auto k_tri_seed_4096 = k_tri_seed<512, kHashMaxDeg, false>;
    const int sm3 = 16 * kHashMaxDeg;
    EFG_CUDA_CHECK(cudaFuncSetAttribute(k_tri_seed_1024, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 1024));
    EFG_CUDA_CHECK(cudaFuncSetAttribute(k_tri_seed_4096, cudaFuncAttributeMaxDynamicSharedMemorySize, sm3));
    EFG_LAUNCH(k_tri_seed_4096, c[kTr3], 512, sm3, s, L.tr3, c[kTr3], a);
    EFG_LAUNCH(k_tri_seed_1024, c[kTr2], 256, 32 * 1024, s, L.tr2, c[kTr2], a);
    EFG_LAUNCH(k_tri_seed_256, c[kTr1], 128, 32 * 512, s, L.tr1, c[kTr1], a);
    EFG_LAUNCH(k_tri_warp, ceil_div(c[kTrS], kTriWarps), kTriWarps * 32, 0, s, L.trs, c[kTrS], a);
  }
  // 3. chains (and stars, from the seed's own chain table): warp per row (dv <= 1024), CTA per row above
  // 5. epilogue
  EFG_LAUNCH(k_epilogue, ceil_div(cnt, B), B, 0, s, a, cnt, ef, total, flags, T_out, W_out);
  return info;
}

// Epilogue of a distributed pass for seeds r, from the words and stars terms
// reduced over all parts (ef_factorized with a DistPart).
void ef_finish(Context& ctx, const CSRView& g, SeedRange r, const unsigned long long* words, const double* ws,
               double* ef, int64_t* total, uint8_t* flags, int64_t* T_out, double* W_out) {
  cudaStream_t s = ctx.stream;
  const int B = 256;
  const int64_t n = g.n, cnt = r.hi - r.lo;
  if (cnt <= 0) return;
  // S1 / S2 arrive in the reduced words (every part wrote its own rows');
  // dmax (the chain words' fixed-point scale) from the degrees
  Prepared P;
  const auto& dh = ctx.dist_head;
  if (dh.valid && dh.P.g.offsets == g.offsets && dh.P.g.nbr == g.nbr && dh.P.g.n == n && dh.P.g.m2 == g.m2)
    P = dh.P;  // the distributed parts' head on this graph
  else
    prepare_head(ctx, g, false, P);
  P.s1 = const_cast<int64_t*>(reinterpret_cast<const int64_t*>(words + 7 * n));
  P.s2 = const_cast<int64_t*>(reinterpret_cast<const int64_t*>(words + 8 * n));
  FArgs a{};
  a.offsets = g.offsets;
  a.s1 = P.s1;
  a.s2 = P.s2;
  a.cwh = words;
  a.cwl = words + n;
  a.cp2 = words + 2 * n;
  a.cws = ws;
  const double d3 = 3.0 * (P.dmax > 1 ? P.dmax : 1);
  a.c0 = (P.dmax > 1 ? P.dmax : 1) * d3 * log(d3);
  a.seed_lo = r.lo;
  a.tri = ctx.buf("f_tri").as<int64_t>(cnt);
  a.Wth = ctx.buf("f_Wth").as<int64_t>(cnt);
  a.Wtl = ctx.buf("f_Wtl").as<int64_t>(cnt);
  EFG_LAUNCH(k_list_out, ceil_div(cnt, B), B, 0, s, words + 3 * n, a, cnt);
  EFG_LAUNCH(k_epilogue, ceil_div(cnt, B), B, 0, s, a, cnt, ef, total, flags, T_out, W_out);
}

EFG_CHECK_ACCESSOR(check_line_factor)

}  // namespace efg
