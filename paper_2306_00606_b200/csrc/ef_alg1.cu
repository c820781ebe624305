// K3b -- Algorithm 1 of the paper: the cluster-centric
// middle-triplet scatter, kept as an independent cross-check engine
// (engine "alg1", EFG_ENGINE_ALG1).
//
//   for every middle v, for every pair i < j in Adj(v):
//     d = |Adj v| + |Adj i| + |Adj j| - 4, minus 2 if i ~ j     (lines 7-8)
//     H_i(d) += 1, H_j(d) += 1, H_v(d) += 2                     (lines 9-11)
//   EF(v) = Entropy(H_v)                                        (line 13)
//
// The histograms are never materialised: what the entropy needs of H_x is
// mass = sum of counts, T = sum count*d and W = sum count*F(d), F(d) = d ln d
// (expected_force.py:312-324), so each triplet adds (1, d, F(d)) to i and j
// and (2, 2d, 2F(d)) to v.  v is fixed per work task: its share is summed in
// registers and reduced once per task; i's and j's go out as global atomics
// (mass and T as exact 64-bit integers, W as fp64: its summation order
// follows the atomics, so W -- and EF -- may differ in the last bits from run
// to run, unlike the factorised and direct engines).  The edge test i ~ j is
// a binary search in the shorter of the two sorted rows (the reference's
// `connected`, expected_force.py:363-368).  This decomposition shares nothing
// with the factorised engine (degree classes, triangle listing) nor with the
// direct engine (per-seed walks): a third, independent route to the same
// mass, T and EF.  Cost: C(dv, 2) pairs per middle, three atomics per
// endpoint -- a cross-check for graphs up to a few 1e9 triplets, not a fast
// path.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "common.cuh"
#include "efg_internal.cuh"

namespace efg {

namespace {

constexpr int kAlgThreads = 256;
constexpr int64_t kAlgPairs = 65536;  // pairs per work task (hubs split over many CTAs)

// pair index q in [0, C(d, 2)) -> (x, y), x < y, row-major over x
__device__ __forceinline__ void pair_of(int64_t q, int64_t d, int64_t& x, int64_t& y) {
  // x = largest with x d - x (x + 1) / 2 <= q
  const double b = 2.0 * (double)d - 1.0;
  int64_t xx = (int64_t)((b - sqrt(b * b - 8.0 * (double)q)) * 0.5);
  if (xx < 0) xx = 0;
  while (xx > 0 && xx * d - xx * (xx + 1) / 2 > q) --xx;
  while ((xx + 1) * d - (xx + 1) * (xx + 2) / 2 <= q) ++xx;
  x = xx;
  y = q - (xx * d - xx * (xx + 1) / 2) + xx + 1;
}

// j in Adj(i)?  binary search in the shorter sorted row
__device__ __forceinline__ bool adjacent(const int64_t* __restrict__ offsets, const int32_t* __restrict__ nbr,
                                         int32_t i, int64_t di, int32_t j, int64_t dj) {
  if (di > dj) {
    const int32_t t = i;
    i = j;
    j = t;
    di = dj;
  }
  const int32_t* row = nbr + offsets[i];
  int64_t lo = 0, hi = di;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(row + mid) < j) lo = mid + 1;
    else hi = mid;
  }
  return lo < di && __ldg(row + lo) == j;
}

__global__ void k_alg1_ntask(const int64_t* __restrict__ offsets, int64_t n, int64_t* __restrict__ nt) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v > n) return;
  if (v == n) {
    nt[v] = 0;
    return;
  }
  const int64_t d = offsets[v + 1] - offsets[v];
  nt[v] = ceil_div(d * (d - 1) / 2, kAlgPairs);
}

__global__ void k_alg1_fill(const int64_t* __restrict__ tstart, int64_t n, int32_t* __restrict__ task_v) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  for (int64_t t = tstart[v]; t < tstart[v + 1]; ++t) task_v[t] = (int32_t)v;
}

struct AlgAcc {
  unsigned long long* mass;  // [n]
  unsigned long long* T;     // [n]
  double* W;                 // [n]
};

__global__ void __launch_bounds__(kAlgThreads)
k_alg1_task(const int64_t* __restrict__ offsets, const int32_t* __restrict__ nbr, const int32_t* __restrict__ nd,
            const double* __restrict__ F, int64_t flen, const int64_t* __restrict__ tstart,
            const int32_t* __restrict__ task_v, int64_t ntasks, AlgAcc acc) {
  __shared__ int64_t rT[kAlgThreads / 32];
  __shared__ double rW[kAlgThreads / 32];
  const int64_t t = blockIdx.x;
  if (t >= ntasks) return;
  const int32_t v = task_v[t];
  const int64_t ob = offsets[v], dv = offsets[v + 1] - ob;
  const int64_t npairs = dv * (dv - 1) / 2;
  const int64_t q0 = (t - tstart[v]) * kAlgPairs, q1 = min(q0 + kAlgPairs, npairs);
  int64_t Tv = 0;
  double Wv = 0.0;
  for (int64_t q = q0 + threadIdx.x; q < q1; q += kAlgThreads) {
    int64_t x, y;
    pair_of(q, dv, x, y);
    x = EFG_CLAMP(x, dv);
    y = EFG_CLAMP(y, dv);
    const int32_t i = nbr[ob + x], j = nbr[ob + y];
    const int64_t di = nd[ob + x], dj = nd[ob + y];
    const int64_t d = dv + di + dj - 4 - (adjacent(offsets, nbr, i, di, j, dj) ? 2 : 0);  // lines 7-8
    const double f = F[EFG_CLAMP(d, flen)];
    Tv += 2 * d;  // line 11: H_v(d) += 2
    Wv += 2.0 * f;
    atomicAdd(acc.mass + i, 1ull);  // line 9
    atomicAdd(acc.T + i, (unsigned long long)d);
    atomicAdd(acc.W + i, f);
    atomicAdd(acc.mass + j, 1ull);  // line 10
    atomicAdd(acc.T + j, (unsigned long long)d);
    atomicAdd(acc.W + j, f);
  }
  // v's share of the task, once
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) {
    Tv += __shfl_xor_sync(0xffffffffu, Tv, o);
    Wv += __shfl_xor_sync(0xffffffffu, Wv, o);
  }
  if (lane == 0) {
    rT[w] = Tv;
    rW[w] = Wv;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t tt = 0;
    double ww = 0.0;
    for (int k = 0; k < kAlgThreads / 32; ++k) {
      tt += rT[k];
      ww += rW[k];
    }
    atomicAdd(acc.mass + v, (unsigned long long)(2 * (q1 - q0)));
    atomicAdd(acc.T + v, (unsigned long long)tt);
    atomicAdd(acc.W + v, ww);
  }
}

// line 13: EF = entropy of H_v from (mass, T, W); flags as expected_force.py:325-327
__global__ void k_alg1_epilogue(AlgAcc acc, int64_t lo, int64_t cnt, double* __restrict__ ef,
                                int64_t* __restrict__ total, uint8_t* __restrict__ flags, int64_t* T_out,
                                double* W_out) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= cnt) return;
  const int64_t v = lo + q;
  const int64_t mass = (int64_t)acc.mass[v], T = (int64_t)acc.T[v];
  const double W = acc.W[v];
  ef[q] = T > 0 ? fmax(log((double)T) - W / (double)T, 0.0) : 0.0;
  total[q] = mass;
  flags[q] = mass == 0 ? 1 : (T == 0 ? 2 : 0);
  if (T_out) T_out[q] = T;
  if (W_out) W_out[q] = W;
}

}  // namespace

void ef_alg1(Context& ctx, Prepared& P, SeedRange r, double* ef, int64_t* total, uint8_t* flags, int64_t* T_out,
             double* W_out, efg_stats* st) {
  cudaStream_t s = ctx.stream;
  const int B = 256;
  const int64_t n = P.g.n, cnt = r.hi - r.lo;
  if (cnt <= 0) return;
  // every middle contributes to its neighbours: the whole graph is processed, seeds [lo, hi) are reported
  AlgAcc acc;
  acc.mass = ctx.buf("a1_mass").as<unsigned long long>(n);
  acc.T = ctx.buf("a1_T").as<unsigned long long>(n);
  acc.W = ctx.buf("a1_W").as<double>(n);
  EFG_CUDA_CHECK(cudaMemsetAsync(acc.mass, 0, n * sizeof(unsigned long long), s));
  EFG_CUDA_CHECK(cudaMemsetAsync(acc.T, 0, n * sizeof(unsigned long long), s));
  EFG_CUDA_CHECK(cudaMemsetAsync(acc.W, 0, n * sizeof(double), s));
  int64_t* nt = ctx.buf("a1_nt").as<int64_t>(n + 1);
  int64_t* tstart = ctx.buf("a1_tstart").as<int64_t>(n + 1);
  EFG_LAUNCH(k_alg1_ntask, ceil_div(n + 1, B), B, 0, s, P.g.offsets, n, nt);
  size_t tmp = 0;
  EFG_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, nt, tstart, n + 1, s));
  EFG_REGION("cub::DeviceScan::ExclusiveSum", s,
             EFG_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(ctx.buf("cub").get(tmp), tmp, nt, tstart, n + 1, s)));
  int64_t ntasks = 0;
  EFG_CUDA_CHECK(cudaMemcpyAsync(&ntasks, tstart + n, sizeof ntasks, cudaMemcpyDeviceToHost, s));
  EFG_CUDA_CHECK(cudaStreamSynchronize(s));
  int32_t* task_v = ctx.buf("a1_task_v").as<int32_t>(ntasks > 0 ? ntasks : 1);
  EFG_LAUNCH(k_alg1_fill, ceil_div(n, B), B, 0, s, tstart, n, task_v);
  EFG_LAUNCH(k_alg1_task, ntasks, kAlgThreads, 0, s, P.g.offsets, P.g.nbr, P.nd, P.ftab, P.ftab_len, tstart, task_v,
             ntasks, acc);
  EFG_LAUNCH(k_alg1_epilogue, ceil_div(cnt, B), B, 0, s, acc, r.lo, cnt, ef, total, flags, T_out, W_out);
  if (st) st->terms = ntasks;
}

EFG_CHECK_ACCESSOR(check_line_alg1)

}  // namespace efg
