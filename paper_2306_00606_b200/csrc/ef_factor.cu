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
//   * stars without the triangle term depend on (di, dj) only, so they are a
//     self-convolution of v's neighbour-degree histogram H_v (|D_v|^2 terms
//     instead of C(dv,2));
//   * chains through i without the triangle term depend on v only through
//     dv, so C_i(y) = sum_x H_i(x) F(y+di-4+x) - F(2y+di-4) is tabulated
//     once per (i, distinct neighbour degree y) and looked up by each seed;
//   * a cluster whose three nodes form a triangle has degree D-2 instead of
//     D = dv+di+dj-4; each triangle at v carries star weight 2 and two chains
//     (v->i->j, v->j->i), so the correction is 4 (F(D-2) - F(D)) per triangle,
//     found once per seed through the degree-ordered orientation Adj+.
// T and mass have closed forms given the triangle count t(v):
//   T    = 2C(dv,2)(dv-4) + 2(dv-1)S1(v) + sum_i [(di-1)(dv+di-4) + S1(i) - dv] - 8 t(v)
//   mass = dv(dv-1) + S1(v) - dv          (test_expected_force.py:139-147)
// All sums run in a fixed order per seed (no atomics on values), so results
// are bitwise reproducible and independent of sharding.
#include <cub/cub.cuh>

#include "common.cuh"
#include "efg_internal.cuh"

namespace efg {

namespace {

struct FArgs {
  const int64_t* offsets;
  const int32_t* nbr;
  const int32_t* nd;
  const int32_t* deg;
  const int64_t* s1;
  const double* F;
  const int64_t* offp;
  const int2* adjp;
  const int64_t* hoff;
  const int32_t* hkey;
  const int32_t* hcnt;
  const double* ctab;
  int64_t n;
  int64_t seed_lo;
  double* ef;
  int64_t* total;
  uint8_t* flags;
  int64_t* T_out;
  double* W_out;
};

// ---------------------------------------------------------------- H build
// Warp per row: number of distinct values in the sorted neighbour-degree row.
__global__ void k_rle_count(const int64_t* __restrict__ offsets, const int32_t* __restrict__ snd,
                            int64_t n, int64_t* __restrict__ dcnt) {
  const int lane = threadIdx.x & 31;
  int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (v >= n) return;
  int64_t b = offsets[v], e = offsets[v + 1];
  int c = 0;
  for (int64_t p = b + lane; p < e; p += 32) c += (p == b) || (snd[p] != snd[p - 1]);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) dcnt[v] = c;
}

// Warp per row: (key, count) runs of the sorted row, ascending key.  Heads
// are compacted first (their row-relative positions parked in hcnt), then
// each run length is the distance to the next head.
__global__ void k_rle_fill(const int64_t* __restrict__ offsets, const int32_t* __restrict__ snd, int64_t n,
                           const int64_t* __restrict__ hoff, int32_t* __restrict__ hkey,
                           int32_t* __restrict__ hcnt) {
  const int lane = threadIdx.x & 31;
  int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (v >= n) return;
  const int64_t b = offsets[v], e = offsets[v + 1];
  const int64_t h0 = hoff[v], h1 = hoff[v + 1];
  int64_t out = h0;
  for (int64_t p0 = b; p0 < e; p0 += 32) {
    int64_t p = p0 + lane;
    bool head = p < e && ((p == b) || (snd[p] != snd[p - 1]));
    unsigned mask = __ballot_sync(0xffffffffu, head);
    if (head) {
      int64_t slot = out + __popc(mask & ((1u << lane) - 1));
      hkey[slot] = snd[p];
      hcnt[slot] = (int32_t)(p - b);
    }
    out += __popc(mask);
  }
  __syncwarp();
  for (int64_t s0 = h0; s0 < h1; s0 += 32) {
    int64_t sl = s0 + lane;
    int32_t cur = 0, nxt = 0;
    if (sl < h1) {
      cur = hcnt[sl];
      nxt = sl + 1 < h1 ? hcnt[sl + 1] : (int32_t)(e - b);
    }
    __syncwarp();
    if (sl < h1) hcnt[sl] = nxt - cur;
    __syncwarp();
  }
}

// Chain table, group of G lanes per row i: for every distinct neighbour
// degree y of i, C_i(y) = sum_a h_a F[y + di - 4 + x_a] - F[2y + di - 4].
template <int G>
__global__ void k_ctab_group(const int64_t* __restrict__ hoff, const int32_t* __restrict__ hkey,
                             const int32_t* __restrict__ hcnt, const int32_t* __restrict__ deg,
                             const double* __restrict__ F, int64_t n, int64_t big, double* __restrict__ ctab) {
  const int sub = threadIdx.x & (G - 1);
  int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  if (i >= n) return;
  int64_t b = hoff[i], e = hoff[i + 1];
  if (e - b > big) return;  // k_ctab_block
  int32_t di = deg[i];
  for (int64_t o = b + sub; o < e; o += G) {
    int32_t y = hkey[o];
    int64_t base = (int64_t)y + di - 4;
    double acc = 0.0;
    for (int64_t a = b; a < e; ++a) acc += (double)__ldg(hcnt + a) * __ldg(F + base + __ldg(hkey + a));
    ctab[o] = acc - __ldg(F + base + y);
  }
}

// Rows with many distinct degrees: one CTA per row, threads over outputs.
__global__ void k_ctab_block(const int32_t* __restrict__ rows, int64_t nrows, const int64_t* __restrict__ hoff,
                             const int32_t* __restrict__ hkey, const int32_t* __restrict__ hcnt,
                             const int32_t* __restrict__ deg, const double* __restrict__ F,
                             double* __restrict__ ctab) {
  int64_t r = blockIdx.x;
  if (r >= nrows) return;
  int32_t i = rows[r];
  int64_t b = hoff[i], e = hoff[i + 1];
  int32_t di = deg[i];
  for (int64_t o = b + threadIdx.x; o < e; o += blockDim.x) {
    int32_t y = hkey[o];
    int64_t base = (int64_t)y + di - 4;
    double acc = 0.0;
    for (int64_t q = b; q < e; ++q) acc += (double)__ldg(hcnt + q) * __ldg(F + base + __ldg(hkey + q));
    ctab[o] = acc - __ldg(F + base + y);
  }
}

struct BigRow {
  const int64_t* hoff;
  int64_t big;
  __host__ __device__ bool operator()(const int32_t& i) const { return hoff[i + 1] - hoff[i] > big; }
};

// ---------------------------------------------------------------- per seed
__device__ __forceinline__ double ctab_lookup(const FArgs& a, int32_t i, int32_t y) {
  int64_t lo = a.hoff[i], hi = a.hoff[i + 1] - 1;
  while (lo < hi) {  // y is present: v (degree y) is a neighbour of i
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(a.hkey + mid) < y) lo = mid + 1; else hi = mid;
  }
  return __ldg(a.ctab + lo);
}

__device__ __forceinline__ void finalize(const FArgs& a, int32_t v, int64_t dv, int64_t Tc, int64_t tri,
                                         double Ws, double Wc, double Wt) {
  const int64_t s1v = a.s1[v];
  const int64_t T = dv * (dv - 1) * (dv - 4) + 2 * (dv - 1) * s1v + Tc - 8 * tri;
  const int64_t mass = dv * (dv - 1) + s1v - dv;
  const double W = (Ws + Wc) + 4.0 * Wt;
  double efv = 0.0;
  if (T > 0) efv = log((double)T) - W / (double)T;
  uint8_t fl = mass == 0 ? 1 : (T == 0 ? 2 : 0);
  const int64_t o = v - a.seed_lo;
  a.ef[o] = efv;
  a.total[o] = mass;
  a.flags[o] = fl;
  if (a.T_out) a.T_out[o] = T;
  if (a.W_out) a.W_out[o] = W;
}

template <class T>
__device__ __forceinline__ T warp_sum(T x) {
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Seeds with dv <= 32: one warp per seed.  A is kept sorted in shared memory
// and membership is a 5-step binary search.
constexpr int kWarpSeedWarps = 8;
__global__ void __launch_bounds__(kWarpSeedWarps * 32)
k_seed_warp(const int32_t* __restrict__ seeds, int64_t count, FArgs a) {
  __shared__ int32_t sA[kWarpSeedWarps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t q = (int64_t)blockIdx.x * kWarpSeedWarps + w;
  if (q >= count) return;
  const int32_t v = seeds[q];
  const int64_t ob = a.offsets[v];
  const int32_t dv = (int32_t)(a.offsets[v + 1] - ob);
  int32_t i = -1, di = 0;
  int64_t Tc = 0;
  double Wc = 0.0;
  if (lane < dv) {
    i = a.nbr[ob + lane];
    di = a.nd[ob + lane];
    Tc = (int64_t)(di - 1) * (dv + di - 4) + a.s1[i] - dv;
    Wc = ctab_lookup(a, i, dv);
  }
  sA[w][lane] = lane < dv ? i : 0x7fffffff;
  __syncwarp();
  // stars over H_v (|D_v| <= dv <= 32)
  const int64_t hb = a.hoff[v];
  const int D = (int)(a.hoff[v + 1] - hb);
  int32_t xa = 0, ha = 0;
  if (lane < D) {
    xa = a.hkey[hb + lane];
    ha = a.hcnt[hb + lane];
  }
  const int64_t c = dv - 4;
  double Ws = 0.0;
  for (int bb = 0; bb < D; ++bb) {
    int32_t xb = __shfl_sync(0xffffffffu, xa, bb);
    int32_t hbv = __shfl_sync(0xffffffffu, ha, bb);
    if (lane < bb) Ws += (double)((int64_t)ha * hbv) * a.F[c + xa + xb];
  }
  if (lane < D) Ws += (double)((int64_t)ha * (ha - 1) / 2) * a.F[c + 2 * xa];
  Ws *= 2.0;
  // triangles: 4 groups of 8 lanes, group g walks Adj+(A[x]) for x = g, g+4, ...
  const int g = lane >> 3, sub = lane & 7;
  int64_t tri = 0;
  double Wt = 0.0;
  for (int x = g; x < dv; x += 4) {
    const int32_t ii = sA[w][x];
    const int32_t dix = a.nd[ob + x];
    const int64_t pb = a.offp[ii], pe = a.offp[ii + 1];
    for (int64_t p = pb + sub; p < pe; p += 8) {
      const int2 jd = a.adjp[p];
      // binary search in sorted sA[w][0..dv)
      int lo = 0, hi = dv;
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (sA[w][mid] < jd.x) lo = mid + 1; else hi = mid;
      }
      if (lo < dv && sA[w][lo] == jd.x) {
        const int64_t S = (int64_t)dv + dix + jd.y;
        Wt += a.F[S - 6] - a.F[S - 4];
        ++tri;
      }
    }
  }
  Tc = warp_sum(Tc);
  tri = warp_sum(tri);
  Ws = warp_sum(Ws);
  Wc = warp_sum(Wc);
  Wt = warp_sum(Wt);
  if (lane == 0) finalize(a, v, dv, Tc, tri, Ws, Wc, Wt);
}

__device__ __forceinline__ uint32_t hslot(int32_t key, int shift) {
  return ((uint32_t)key * 2654435761u) >> shift;
}

// Block-wide fixed-order reductions (deterministic).
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
  return r;  // valid in thread 0
}

// Seeds with 32 < dv <= SLOTS/2: one CTA per seed, A in a shared-memory hash
// set (open addressing, load <= 1/2).  Seeds with larger dv (hubs) use a
// per-CTA bitmap over node ids in global memory (BITMAP = true).
template <int THREADS, int SLOTS, bool BITMAP>
__global__ void __launch_bounds__(THREADS)
k_seed_block(const int32_t* __restrict__ seeds, int64_t count, FArgs a, uint32_t* __restrict__ bitmaps,
             int64_t bitmap_words) {
  extern __shared__ int32_t table[];  // SLOTS entries (unused when BITMAP)
  __shared__ double red_d[THREADS / 32];
  __shared__ int64_t red_i[THREADS / 32];
  const int64_t q = blockIdx.x;
  if (q >= count) return;
  const int32_t v = seeds[q];
  const int64_t ob = a.offsets[v];
  const int32_t dv = (int32_t)(a.offsets[v + 1] - ob);
  constexpr int kShift = 32 - __builtin_ctz(SLOTS);
  uint32_t* bm = BITMAP ? bitmaps + (int64_t)blockIdx.x * bitmap_words : nullptr;
  if (!BITMAP) {
    for (int s = threadIdx.x; s < SLOTS; s += THREADS) table[s] = -1;
    __syncthreads();
  }
  // insert A; per-neighbour chain terms
  int64_t Tc = 0;
  double Wc = 0.0;
  for (int x = threadIdx.x; x < dv; x += THREADS) {
    const int32_t i = a.nbr[ob + x];
    const int32_t di = a.nd[ob + x];
    Tc += (int64_t)(di - 1) * (dv + di - 4) + a.s1[i] - dv;
    Wc += ctab_lookup(a, i, dv);
    if (BITMAP) {
      atomicOr(bm + (i >> 5), 1u << (i & 31));
    } else {
      uint32_t s = hslot(i, kShift);
      while (atomicCAS(&table[s], -1, i) != -1) s = (s + 1) & (SLOTS - 1);
    }
  }
  // stars over H_v: thread handles rows a = t, t+THREADS, ...
  const int64_t hb = a.hoff[v];
  const int D = (int)(a.hoff[v + 1] - hb);
  const int64_t c = dv - 4;
  double Ws = 0.0;
  for (int ra = threadIdx.x; ra < D; ra += THREADS) {
    const int32_t xa = a.hkey[hb + ra];
    const int64_t ha = a.hcnt[hb + ra];
    double acc = (double)(ha * (ha - 1) / 2) * a.F[c + 2 * xa];
    const int64_t base = c + xa;
    for (int rb = ra + 1; rb < D; ++rb) acc += (double)(ha * __ldg(a.hcnt + hb + rb)) * __ldg(a.F + base + __ldg(a.hkey + hb + rb));
    Ws += acc;
  }
  Ws *= 2.0;
  __syncthreads();  // membership structure complete
  if (BITMAP) __threadfence_block();
  // triangles: groups of 8 lanes walk Adj+(A[x])
  constexpr int G = 8, NG = THREADS / G;
  const int grp = threadIdx.x / G, sub = threadIdx.x & (G - 1);
  int64_t tri = 0;
  double Wt = 0.0;
  for (int x = grp; x < dv; x += NG) {
    const int32_t ii = a.nbr[ob + x];
    const int32_t dix = a.nd[ob + x];
    const int64_t pb = a.offp[ii], pe = a.offp[ii + 1];
    for (int64_t p = pb + sub; p < pe; p += G) {
      const int2 jd = a.adjp[p];
      bool hit;
      if (BITMAP) {
        hit = (__ldcg(bm + (jd.x >> 5)) >> (jd.x & 31)) & 1u;
      } else {
        uint32_t s = hslot(jd.x, kShift);
        int32_t k;
        while ((k = table[s]) != jd.x && k != -1) s = (s + 1) & (SLOTS - 1);
        hit = k == jd.x;
      }
      if (hit) {
        const int64_t S = (int64_t)dv + dix + jd.y;
        Wt += a.F[S - 6] - a.F[S - 4];
        ++tri;
      }
    }
  }
  Tc = block_sum<THREADS>(Tc, red_i);
  tri = block_sum<THREADS>(tri, red_i);
  Ws = block_sum<THREADS>(Ws, red_d);
  Wc = block_sum<THREADS>(Wc, red_d);
  Wt = block_sum<THREADS>(Wt, red_d);
  if (threadIdx.x == 0) finalize(a, v, dv, Tc, tri, Ws, Wc, Wt);
}

struct DegClass {
  const int32_t* deg;
  int32_t lo, hi;  // lo < deg <= hi
  __host__ __device__ bool operator()(const int32_t& v) const {
    int32_t d = deg[v];
    return d > lo && d <= hi;
  }
};

}  // namespace

// Class boundaries (by dv): warp | block-S | block-M | block-L | hub bitmap.
static constexpr int32_t kClassHi[5] = {32, 256, 2048, 16384, 0x7fffffff};

namespace {
__global__ void k_seed_work(const int64_t* __restrict__ offsets, const int32_t* __restrict__ nbr,
                            const int64_t* __restrict__ offp, const int64_t* __restrict__ hoff, int64_t n,
                            int64_t* __restrict__ work) {
  const int lane = threadIdx.x & 31;
  int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (v >= n) return;
  int64_t b = offsets[v], e = offsets[v + 1];
  int64_t w = 0;
  for (int64_t p = b + lane; p < e; p += 32) {
    int32_t i = nbr[p];
    w += offp[i + 1] - offp[i] + 8;  // triangle probes + chain lookup
  }
  w = warp_sum(w);
  if (lane == 0) {
    int64_t D = hoff[v + 1] - hoff[v];
    work[v] = w + D * (D + 1) / 2 + 64;
  }
}
}  // namespace

// Neighbour-degree histograms H_i for every node (sorted distinct degrees +
// counts).  Returns the number of entries.
static int64_t build_histograms(Context& ctx, Prepared& P, int64_t*& hoff, int32_t*& hkey, int32_t*& hcnt) {
  cudaStream_t s = ctx.stream;
  const int64_t n = P.g.n, m2 = P.g.m2;
  const int B = 256;
  EFG_REQUIRE(m2 < (int64_t(1) << 31), "adjacency too large for the segmented sort (2m >= 2^31)");
  // 1. neighbour-degree histograms H_i (sorted distinct degrees + counts)
  int32_t* snd = ctx.buf("f_snd").as<int32_t>(m2);
  size_t tmp = 0;
  EFG_CUDA_CHECK(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp, P.nd, snd, (int)m2, (int)n, P.g.offsets,
                                                    P.g.offsets + 1, s));
  EFG_REGION("cub::DeviceSegmentedSort::SortKeys", s, EFG_CUDA_CHECK(cub::DeviceSegmentedSort::SortKeys(ctx.buf("cub").get(tmp), tmp, P.nd, snd, (int)m2, (int)n,
                                                    P.g.offsets, P.g.offsets + 1, s)));
  int64_t* dcnt = ctx.buf("f_dcnt").as<int64_t>(n + 1);
  hoff = ctx.buf("f_hoff").as<int64_t>(n + 1);
  EFG_LAUNCH(k_rle_count, ceil_div(n * 32, B), B, 0, s, P.g.offsets, snd, n, dcnt);
  EFG_CUDA_CHECK(cudaMemsetAsync(dcnt + n, 0, sizeof(int64_t), s));
  EFG_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, dcnt, hoff, n + 1, s));
  EFG_REGION("cub::DeviceScan::ExclusiveSum", s, EFG_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(ctx.buf("cub").get(tmp), tmp, dcnt, hoff, n + 1, s)));
  int64_t nh = 0;
  EFG_CUDA_CHECK(cudaMemcpyAsync(&nh, hoff + n, sizeof nh, cudaMemcpyDeviceToHost, s));
  EFG_CUDA_CHECK(cudaStreamSynchronize(s));
  hkey = ctx.buf("f_hkey").as<int32_t>(nh);
  hcnt = ctx.buf("f_hcnt").as<int32_t>(nh);
  EFG_LAUNCH(k_rle_fill, ceil_div(n * 32, B), B, 0, s, P.g.offsets, snd, n, hoff, hkey, hcnt);
  return nh;
}

void factorized_work(Context& ctx, Prepared& P, int64_t* d_work) {
  int64_t* hoff;
  int32_t *hkey, *hcnt;
  build_histograms(ctx, P, hoff, hkey, hcnt);
  const int B = 256;
  EFG_LAUNCH(k_seed_work, ceil_div(P.g.n * 32, B), B, 0, ctx.stream, P.g.offsets, P.g.nbr, P.offp, hoff, P.g.n,
             d_work);
}

void ef_factorized(Context& ctx, Prepared& P, SeedRange r, double* ef, int64_t* total, uint8_t* flags,
                   int64_t* T_out, double* W_out, efg_stats* st) {
  cudaStream_t s = ctx.stream;
  const int64_t n = P.g.n;
  const int B = 256;
  size_t tmp = 0;
  int64_t* hoff;
  int32_t *hkey, *hcnt;
  const int64_t nh = build_histograms(ctx, P, hoff, hkey, hcnt);
  double* ctab = ctx.buf("f_ctab").as<double>(nh);
  // 2. chain tables: rows with <= kBig distinct degrees by 8-lane groups, the rest by CTAs
  {
    const int64_t kBig = 64;
    int32_t* rows = ctx.buf("f_rows").as<int32_t>(n);
    int64_t* nrows_d = ctx.buf("f_nrows").as<int64_t>(1);
    EFG_LAUNCH(k_ctab_group<8>, ceil_div(n * 8, B), B, 0, s, hoff, hkey, hcnt, P.deg, P.ftab, n, kBig, ctab);
    cub::CountingInputIterator<int32_t> rit(0);
    BigRow pred{hoff, kBig};
    EFG_CUDA_CHECK(cub::DeviceSelect::If(nullptr, tmp, rit, rows, nrows_d, n, pred, s));
    EFG_REGION("cub::DeviceSelect::If", s, EFG_CUDA_CHECK(cub::DeviceSelect::If(ctx.buf("cub").get(tmp), tmp, rit, rows, nrows_d, n, pred, s)));
    int64_t nrows = 0;
    EFG_CUDA_CHECK(cudaMemcpyAsync(&nrows, nrows_d, sizeof nrows, cudaMemcpyDeviceToHost, s));
    EFG_CUDA_CHECK(cudaStreamSynchronize(s));
    EFG_LAUNCH(k_ctab_block, nrows, 128, 0, s, rows, nrows, hoff, hkey, hcnt, P.deg, P.ftab, ctab);
  }
  // 3. classify seeds of [lo, hi) by degree
  const int64_t cnt = r.hi - r.lo;
  FArgs a;
  a.offsets = P.g.offsets;
  a.nbr = P.g.nbr;
  a.nd = P.nd;
  a.deg = P.deg;
  a.s1 = P.s1;
  a.F = P.ftab;
  a.offp = P.offp;
  a.adjp = P.adjp;
  a.hoff = hoff;
  a.hkey = hkey;
  a.hcnt = hcnt;
  a.ctab = ctab;
  a.n = n;
  a.seed_lo = r.lo;
  a.ef = ef;
  a.total = total;
  a.flags = flags;
  a.T_out = T_out;
  a.W_out = W_out;
  if (cnt <= 0) return;
  int32_t* lists = ctx.buf("f_lists").as<int32_t>(5 * cnt);
  int64_t* ncls_d = ctx.buf("f_ncls").as<int64_t>(5);
  cub::CountingInputIterator<int32_t> it((int32_t)r.lo);
  for (int k = 0; k < 5; ++k) {
    DegClass pred{P.deg, k ? kClassHi[k - 1] : 0, kClassHi[k]};
    EFG_CUDA_CHECK(cub::DeviceSelect::If(nullptr, tmp, it, lists + k * cnt, ncls_d + k, cnt, pred, s));
    EFG_REGION("cub::DeviceSelect::If", s, EFG_CUDA_CHECK(
        cub::DeviceSelect::If(ctx.buf("cub").get(tmp), tmp, it, lists + k * cnt, ncls_d + k, cnt, pred, s)));
  }
  int64_t ncls[5];
  EFG_CUDA_CHECK(cudaMemcpyAsync(ncls, ncls_d, sizeof ncls, cudaMemcpyDeviceToHost, s));
  EFG_CUDA_CHECK(cudaStreamSynchronize(s));
  // 4. hubs first (long CTAs), then descending classes
  const int64_t words = ceil_div(n, 32);
  if (ncls[4]) {
    uint32_t* bms = ctx.buf("f_bitmaps").as<uint32_t>(ncls[4] * words);
    EFG_CUDA_CHECK(cudaMemsetAsync(bms, 0, ncls[4] * words * sizeof(uint32_t), s));
    EFG_LAUNCH((k_seed_block<1024, 32, true>), ncls[4], 1024, 0, s, lists + 4 * cnt, ncls[4], a, bms, words);
  }
  if (ncls[3]) {
    auto kern = k_seed_block<512, 32768, false>;
    EFG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 * 4));
    EFG_LAUNCH(kern, ncls[3], 512, 32768 * 4, s, lists + 3 * cnt, ncls[3], a, nullptr, 0);
  }
  if (ncls[2]) EFG_LAUNCH((k_seed_block<256, 4096, false>), ncls[2], 256, 4096 * 4, s, lists + 2 * cnt, ncls[2], a, nullptr, 0);
  if (ncls[1]) EFG_LAUNCH((k_seed_block<128, 512, false>), ncls[1], 128, 512 * 4, s, lists + 1 * cnt, ncls[1], a, nullptr, 0);
  if (ncls[0]) EFG_LAUNCH(k_seed_warp, ceil_div(ncls[0], kWarpSeedWarps), kWarpSeedWarps * 32, 0, s, lists, ncls[0], a);
  if (st) st->terms = nh;
}

}  // namespace efg
