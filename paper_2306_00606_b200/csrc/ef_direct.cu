// K3 (direct) -- per-seed enumeration of every star and chain cluster.
//
// The original formulation (expected_force.py:345-418 `ef_vertex_centric`,
// PAPER.md:116,155): for seed v every star pair (i, j), i<j in Adj(v)
// (weight 2, :375-382) and every chain v->i->k, k in Adj(i)\{v} (weight 1,
// :383-390) is visited, its out-degree computed as the degree sum minus the
// internal edges, and T = sum w d, W = sum w d ln d accumulated on the fly
// (no per-cluster data leaves registers).  Internal edges:
//   * chain v->i->k is internal iff k in Adj(v): shared-memory hash of Adj(v)
//     (dv <= 4096) or a global bitmap over node ids (hubs);
//   * star {v,i,j} is internal iff j in Adj(i) -- which is exactly the set of
//     chain hits v->i->j.  Each triangle pair is met twice by the chain walks
//     (from i and from j), so each hit moves half of the star weight:
//     W += F(D-2) - F(D), T -= 2.  Stars are therefore enumerated without a
//     membership test.
// Load balance follows the per-seed work w(v) = C(dv,2) + sum_{i in A} di
// (K2): each seed is cut into fixed-size tasks of kTaskItems items, one CTA
// per task, and a seed's task partials are merged in task order (a fixed
// split independent of the device count -> deterministic results).
#include <cub/cub.cuh>

#include "common.cuh"
#include "efg_internal.cuh"

namespace efg {

namespace {

constexpr int kThreads = 256;
constexpr int64_t kTaskItems = 32768;
constexpr int kHashSlots = 8192;          // smem hash for dv <= 4096
constexpr int kHashMaxDeg = kHashSlots / 2;

struct DArgs {
  const int64_t* offsets;
  const int32_t* nbr;
  const int32_t* nd;
  const int64_t* s1;
  const double* F;
  const int64_t* cp;        // [2m] exclusive prefix of nd within each row
  const int64_t* tstart;    // [cnt+1] first task of seed lo+q
  const int32_t* task_seed; // [ntasks]
  const int32_t* hub_slot;  // [n] bitmap index for dv > kHashMaxDeg, else -1
  const uint32_t* bitmaps;
  int64_t words;
  int64_t seed_lo;
  int64_t* pT;
  double* pW;
  int64_t flen;             // F table length (bounds-checked builds)
};

__device__ __forceinline__ uint32_t hslot(int32_t key) { return ((uint32_t)key * 2654435761u) >> 19; }

template <class T>
__device__ __forceinline__ T warp_sum(T x) {
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Star pair index q in [0, C(dv,2)) -> (x, y), x < y, row-major over x.
__device__ __forceinline__ void unrank_pair(int64_t q, int64_t dv, int64_t& x, int64_t& y) {
  // rows x hold dv-1-x pairs; first index of row x: x*dv - x(x+1)/2
  double fd = (double)dv;
  double disc = (2.0 * fd - 1.0) * (2.0 * fd - 1.0) - 8.0 * (double)q;
  int64_t xx = (int64_t)((2.0 * fd - 1.0 - sqrt(disc > 0 ? disc : 0.0)) * 0.5);
  if (xx < 0) xx = 0;
  auto first = [&](int64_t r) { return r * dv - r * (r + 1) / 2; };
  while (xx > 0 && first(xx) > q) --xx;
  while (first(xx + 1) <= q) ++xx;
  x = xx;
  y = q - first(xx) + xx + 1;
}

__global__ void __launch_bounds__(kThreads)
k_direct_task(DArgs a, int64_t ntasks) {
  __shared__ int32_t table[kHashSlots];
  __shared__ int64_t redT[kThreads / 32];
  __shared__ double redW[kThreads / 32];
  const int64_t task = blockIdx.x;
  if (task >= ntasks) return;
  const int32_t v = a.task_seed[task];
  const int64_t ob = a.offsets[v];
  const int64_t dv = a.offsets[v + 1] - ob;
  const int64_t first_task = a.tstart[v - a.seed_lo];
  const int64_t nstar = dv * (dv - 1) / 2;
  const int64_t wv = nstar + a.s1[v];
  const int64_t q0 = (task - first_task) * kTaskItems;
  const int64_t q1 = q0 + kTaskItems < wv ? q0 + kTaskItems : wv;
  const bool use_bm = dv > kHashMaxDeg;
  const uint32_t* bm = use_bm ? a.bitmaps + (int64_t)a.hub_slot[v] * a.words : nullptr;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = dv - 4;
  int64_t T = 0;
  double W = 0.0;
  // chain items need membership of Adj(v)
  if (!use_bm && q1 > nstar) {
    for (int s = threadIdx.x; s < kHashSlots; s += kThreads) table[s] = -1;
    __syncthreads();
    for (int64_t x = threadIdx.x; x < dv; x += kThreads) {
      int32_t i = a.nbr[ob + x];
      uint32_t s = hslot(i);
      while (atomicCAS(&table[s], -1, i) != -1) s = (s + 1) & (kHashSlots - 1);
    }
    __syncthreads();
  }
  // stars: items [q0, min(q1, nstar))
  for (int64_t q = q0 + threadIdx.x; q < q1 && q < nstar; q += kThreads) {
    int64_t x, y;
    unrank_pair(q, dv, x, y);
    int64_t d = c + a.nd[ob + x] + a.nd[ob + y];
    T += 2 * d;
    W += 2.0 * a.F[EFG_CLAMP(d, a.flen)];
  }
  // chains: items [max(q0, nstar), q1), warp-cooperative over 32 consecutive items
  const int64_t cs = q0 > nstar ? q0 : nstar;
  for (int64_t base = cs + (int64_t)w * 32; base < q1; base += kThreads) {
    const int64_t q = base + lane;
    // lane 0: row x0 of the warp's first item (upper_bound in the row prefix)
    int64_t x0 = 0;
    if (lane == 0) {
      int64_t r = base - nstar, lo = 0, hi = dv;  // last x with cp[x] <= r
      while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (a.cp[ob + mid] <= r) lo = mid; else hi = mid;
      }
      x0 = lo;
    }
    x0 = __shfl_sync(0xffffffffu, x0, 0);
    // boundaries of the next 32 rows; each lane counts how many it passes
    int64_t bnd = x0 + 1 + lane < dv ? a.cp[ob + x0 + 1 + lane] : INT64_MAX;
    const int64_t r = q - nstar;
    int k = 0;
#pragma unroll
    for (int s = 16; s; s >>= 1) {
      int64_t b = __shfl_sync(0xffffffffu, bnd, k + s - 1);
      if (k + s <= 32 && b <= r) k += s;
    }
    {
      int64_t b = __shfl_sync(0xffffffffu, bnd, k < 32 ? k : 31);
      if (k < 32 && b <= r) ++k;
    }
    if (q < q1) {
      const int64_t x = EFG_CLAMP(x0 + k, dv);
      const int32_t i = a.nbr[ob + x];
      const int64_t di = a.nd[ob + x];
      const int64_t t = r - a.cp[ob + x];
      const int64_t oi = a.offsets[i];
      const int32_t kk = a.nbr[oi + t];
      if (kk != v) {
        const int64_t dk = a.nd[oi + t];
        bool tri;
        if (use_bm) {
          tri = (__ldg(bm + (kk >> 5)) >> (kk & 31)) & 1u;
        } else {
          uint32_t s = hslot(kk);
          int32_t key;
          while ((key = table[s]) != kk && key != -1) s = (s + 1) & (kHashSlots - 1);
          tri = key == kk;
        }
        const int64_t D = c + di + dk;
        if (tri) {
          T += (D - 2) - 2;
          W += 2.0 * a.F[EFG_CLAMP(D - 2, a.flen)] - a.F[EFG_CLAMP(D, a.flen)];
        } else {
          T += D;
          W += a.F[EFG_CLAMP(D, a.flen)];
        }
      }
    }
  }
  // fixed-order CTA reduction
  T = warp_sum(T);
  W = warp_sum(W);
  if (lane == 0) {
    redT[w] = T;
    redW[w] = W;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t tt = 0;
    double ww = 0.0;
    for (int k = 0; k < kThreads / 32; ++k) {
      tt += redT[k];
      ww += redW[k];
    }
    a.pT[task] = tt;
    a.pW[task] = ww;
  }
}

// Warp per row: cp[e] = sum of nd over the row before e.
__global__ void k_row_prefix(const int64_t* __restrict__ offsets, const int32_t* __restrict__ nd, int64_t lo,
                             int64_t hi, int64_t* __restrict__ cp) {
  const int lane = threadIdx.x & 31;
  int64_t v = lo + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (v >= hi) return;
  int64_t b = offsets[v], e = offsets[v + 1];
  int64_t carry = 0;
  for (int64_t p0 = b; p0 < e; p0 += 32) {
    int64_t p = p0 + lane;
    int64_t x = p < e ? nd[p] : 0;
    int64_t incl = x;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (p < e) cp[p] = carry + incl - x;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
}

__global__ void k_task_counts(const int64_t* __restrict__ offsets, const int64_t* __restrict__ s1, int64_t lo,
                              int64_t cnt, int64_t* __restrict__ ntask) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q > cnt) return;
  if (q == cnt) {
    ntask[q] = 0;
    return;
  }
  int64_t v = lo + q;
  int64_t dv = offsets[v + 1] - offsets[v];
  int64_t w = dv * (dv - 1) / 2 + s1[v];
  ntask[q] = w > 0 ? ceil_div(w, kTaskItems) : 1;
}

__global__ void k_task_fill(const int64_t* __restrict__ tstart, int64_t lo, int64_t cnt,
                            int32_t* __restrict__ task_seed) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= cnt) return;
  for (int64_t t = tstart[q]; t < tstart[q + 1]; ++t) task_seed[t] = (int32_t)(lo + q);
}

__global__ void k_hub_bitmaps(const int32_t* __restrict__ hubs, int64_t nhubs, const int64_t* __restrict__ offsets,
                              const int32_t* __restrict__ nbr, uint32_t* __restrict__ bitmaps, int64_t words,
                              int32_t* __restrict__ hub_slot) {
  int64_t h = blockIdx.x;
  if (h >= nhubs) return;
  int32_t v = hubs[h];
  if (threadIdx.x == 0) hub_slot[v] = (int32_t)h;
  uint32_t* bm = bitmaps + h * words;
  for (int64_t p = offsets[v] + threadIdx.x; p < offsets[v + 1]; p += blockDim.x) {
    int32_t i = nbr[p];
    atomicOr(bm + (i >> 5), 1u << (i & 31));
  }
}

__global__ void k_direct_epilogue(const int64_t* __restrict__ offsets, const int64_t* __restrict__ s1,
                                  const int64_t* __restrict__ tstart, const int64_t* __restrict__ pT,
                                  const double* __restrict__ pW, int64_t lo, int64_t cnt, double* __restrict__ ef,
                                  int64_t* __restrict__ total, uint8_t* __restrict__ flags, int64_t* T_out,
                                  double* W_out) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= cnt) return;
  int64_t v = lo + q;
  int64_t dv = offsets[v + 1] - offsets[v];
  int64_t T = 0;
  double W = 0.0;
  for (int64_t t = tstart[q]; t < tstart[q + 1]; ++t) {
    T += pT[t];
    W += pW[t];
  }
  int64_t mass = dv * (dv - 1) + s1[v] - dv;
  double e = 0.0;
  // entropy >= 0: clamp the last-ulp cancellation of ln T - W/T when only one
  // positive-degree cluster class exists (EF mathematically 0)
  if (T > 0) e = fmax(log((double)T) - W / (double)T, 0.0);
  ef[q] = e;
  total[q] = mass;
  flags[q] = mass == 0 ? 1 : (T == 0 ? 2 : 0);
  if (T_out) T_out[q] = T;
  if (W_out) W_out[q] = W;
}

__global__ void k_direct_work(const int64_t* __restrict__ offsets, const int64_t* __restrict__ s1, int64_t n,
                              int64_t* __restrict__ work) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  int64_t dv = offsets[v + 1] - offsets[v];
  work[v] = dv * (dv - 1) / 2 + s1[v] + 64;
}

struct HubPred {
  const int32_t* deg;
  __host__ __device__ bool operator()(const int32_t& v) const { return deg[v] > kHashMaxDeg; }
};

}  // namespace

void direct_work(Context& ctx, Prepared& P, int64_t* d_work) {
  EFG_LAUNCH(k_direct_work, ceil_div(P.g.n, 256), 256, 0, ctx.stream, P.g.offsets, P.s1, P.g.n, d_work);
}

void ef_direct(Context& ctx, Prepared& P, SeedRange r, double* ef, int64_t* total, uint8_t* flags,
               int64_t* T_out, double* W_out, efg_stats* st) {
  cudaStream_t s = ctx.stream;
  const int B = 256;
  const int64_t n = P.g.n;
  const int64_t cnt = r.hi - r.lo;
  if (cnt <= 0) return;
  size_t tmp = 0;
  // tasks
  int64_t* ntask = ctx.buf("d_ntask").as<int64_t>(cnt + 1);
  int64_t* tstart = ctx.buf("d_tstart").as<int64_t>(cnt + 1);
  EFG_LAUNCH(k_task_counts, ceil_div(cnt + 1, B), B, 0, s, P.g.offsets, P.s1, r.lo, cnt, ntask);
  EFG_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, ntask, tstart, cnt + 1, s));
  EFG_REGION("cub::DeviceScan::ExclusiveSum", s, EFG_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(ctx.buf("cub").get(tmp), tmp, ntask, tstart, cnt + 1, s)));
  int64_t ntasks = 0;
  EFG_CUDA_CHECK(cudaMemcpyAsync(&ntasks, tstart + cnt, sizeof ntasks, cudaMemcpyDeviceToHost, s));
  // hubs needing a bitmap
  int32_t* hubs = ctx.buf("d_hubs").as<int32_t>(cnt);
  int64_t* nh_d = ctx.buf("d_nhubs").as<int64_t>(1);
  cub::CountingInputIterator<int32_t> it((int32_t)r.lo);
  HubPred pred{P.deg};
  EFG_CUDA_CHECK(cub::DeviceSelect::If(nullptr, tmp, it, hubs, nh_d, cnt, pred, s));
  EFG_REGION("cub::DeviceSelect::If", s, EFG_CUDA_CHECK(cub::DeviceSelect::If(ctx.buf("cub").get(tmp), tmp, it, hubs, nh_d, cnt, pred, s)));
  int64_t nhubs = 0;
  EFG_CUDA_CHECK(cudaMemcpyAsync(&nhubs, nh_d, sizeof nhubs, cudaMemcpyDeviceToHost, s));
  EFG_CUDA_CHECK(cudaStreamSynchronize(s));
  int32_t* task_seed = ctx.buf("d_task_seed").as<int32_t>(ntasks);
  EFG_LAUNCH(k_task_fill, ceil_div(cnt, B), B, 0, s, tstart, r.lo, cnt, task_seed);
  const int64_t words = ceil_div(n, 32);
  uint32_t* bitmaps = ctx.buf("d_bitmaps").as<uint32_t>(nhubs * words + 1);
  int32_t* hub_slot = ctx.buf("d_hub_slot").as<int32_t>(n);
  if (nhubs) {
    EFG_CUDA_CHECK(cudaMemsetAsync(bitmaps, 0, nhubs * words * sizeof(uint32_t), s));
    EFG_LAUNCH(k_hub_bitmaps, nhubs, 1024, 0, s, hubs, nhubs, P.g.offsets, P.g.nbr, bitmaps, words, hub_slot);
  }
  // row prefixes for the seeds' rows
  int64_t* cp = ctx.buf("d_cp").as<int64_t>(P.g.m2);
  EFG_LAUNCH(k_row_prefix, ceil_div(cnt * 32, B), B, 0, s, P.g.offsets, P.nd, r.lo, r.hi, cp);
  int64_t* pT = ctx.buf("d_pT").as<int64_t>(ntasks);
  double* pW = ctx.buf("d_pW").as<double>(ntasks);
  DArgs a{P.g.offsets, P.g.nbr, P.nd, P.s1, P.ftab, cp, tstart, task_seed, hub_slot, bitmaps, words, r.lo, pT, pW,
          P.ftab_len};
  EFG_LAUNCH(k_direct_task, ntasks, kThreads, 0, s, a, ntasks);
  EFG_LAUNCH(k_direct_epilogue, ceil_div(cnt, B), B, 0, s, P.g.offsets, P.s1, tstart, pT, pW, r.lo, cnt, ef, total,
             flags, T_out, W_out);
  if (st) st->terms = ntasks;
}

EFG_CHECK_ACCESSOR(check_line_direct)

}  // namespace efg
