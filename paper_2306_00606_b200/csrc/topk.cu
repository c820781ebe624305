// K5 -- key-node ranking on the device.
//
// No reference function: the semantics come from the reference's consumers,
// `np.argsort(ef, kind="stable")` (analysis.py:240) read from the top, with
// ties going to the lower id (analysis.py:101), i.e. np.lexsort((ids, -ef))[:k].
// Implementation: stable LSD radix sort of (ef, id) pairs in descending key
// order (CUB; equal keys keep ascending id), first k ids.
#include <cub/cub.cuh>

#include "common.cuh"
#include "efg_internal.cuh"

namespace efg {

namespace {
__global__ void k_topk_init(const double* __restrict__ ef, int64_t n, double* __restrict__ keys,
                            int64_t* __restrict__ ids) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  double x = ef[t];
  keys[t] = x == 0.0 ? 0.0 : x;  // canonical +0.0 so that -0.0 ties with 0.0 like lexsort
  ids[t] = t;
}
}  // namespace

void topk_device(Context& ctx, const double* d_ef, int64_t n, int64_t k, int64_t* d_ids_out) {
  cudaStream_t s = ctx.stream;
  if (n <= 0 || k <= 0) return;
  const int B = 256;
  double* keys = ctx.buf("t_keys").as<double>(n);
  double* keys2 = ctx.buf("t_keys2").as<double>(n);
  int64_t* ids = ctx.buf("t_ids").as<int64_t>(n);
  int64_t* ids2 = ctx.buf("t_ids2").as<int64_t>(n);
  EFG_LAUNCH(k_topk_init, ceil_div(n, B), B, 0, s, d_ef, n, keys, ids);
  size_t tmp = 0;
  EFG_CUDA_CHECK(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, keys, keys2, ids, ids2, n, 0, 64, s));
  EFG_REGION("cub::DeviceRadixSort::SortPairsDescending", s, EFG_CUDA_CHECK(
      cub::DeviceRadixSort::SortPairsDescending(ctx.buf("cub").get(tmp), tmp, keys, keys2, ids, ids2, n, 0, 64, s)));
  EFG_CUDA_CHECK(cudaMemcpyAsync(d_ids_out, ids2, (k < n ? k : n) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
}

// ---------------------------------------------------------------------------
// Ranking consumers, built on the same sort.
//
// rank_ascending_device: np.argsort(ef, kind="stable") -- the EF ranking the
//   immunization windows are cut from (analysis.py:240).  Stable LSD radix sort
//   of (canonical ef, id) ascending: equal keys keep ascending id.
// ef_bins_device: ef_bins (analysis.py:84-103) -- the number of distinct EF
//   values, k targets lo + i*(hi-lo)/(k-1) with exactly the reference's IEEE
//   operation order, and per target argmin |ef - target| with ties to the
//   lowest id (np.argmin).  |ef - t| >= 0, so its bit pattern orders like the
//   value and a 64-bit atomicMin finds the minimum; a second pass takes the
//   lowest id attaining it.  Both passes are integer atomics: deterministic.
namespace {
constexpr int kRankThreads = 256;

__global__ void k_distinct(const double* __restrict__ sorted, int64_t n, unsigned long long* __restrict__ cnt) {
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    local += (i == 0 || sorted[i] != sorted[i - 1]) ? 1ull : 0ull;
  for (int o = 16; o; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(cnt, local);
}

__global__ void k_bin_targets(const double* __restrict__ sorted, int64_t n, int64_t k, double* __restrict__ targets,
                              unsigned long long* __restrict__ best, unsigned long long* __restrict__ rep) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= k) return;
  const double lo = sorted[0], hi = sorted[n - 1];
  // analysis.py:97: lo if k == 1 else lo + i * (hi - lo) / (k - 1), no contraction
  targets[i] = k == 1 ? lo : __dadd_rn(lo, __ddiv_rn(__dmul_rn((double)i, __dsub_rn(hi, lo)), (double)(k - 1)));
  best[i] = ~0ull;
  rep[i] = ~0ull;
}

__global__ void k_nearest_diff(const double* __restrict__ ef, int64_t n, const double* __restrict__ targets, int64_t k,
                               unsigned long long* __restrict__ best) {
  for (int64_t t = 0; t < k; ++t) {
    const double tg = targets[t];
    unsigned long long local = ~0ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      unsigned long long b = (unsigned long long)__double_as_longlong(fabs(__dsub_rn(ef[i], tg)));
      local = b < local ? b : local;
    }
    for (int o = 16; o; o >>= 1) {
      unsigned long long x = __shfl_down_sync(0xffffffffu, local, o);
      local = x < local ? x : local;
    }
    if ((threadIdx.x & 31) == 0 && local != ~0ull) atomicMin(best + t, local);
  }
}

__global__ void k_nearest_id(const double* __restrict__ ef, int64_t n, const double* __restrict__ targets, int64_t k,
                             const unsigned long long* __restrict__ best, unsigned long long* __restrict__ rep) {
  for (int64_t t = 0; t < k; ++t) {
    const double tg = targets[t];
    const unsigned long long want = best[t];
    unsigned long long local = ~0ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      unsigned long long b = (unsigned long long)__double_as_longlong(fabs(__dsub_rn(ef[i], tg)));
      if (b == want && (unsigned long long)i < local) local = (unsigned long long)i;
    }
    for (int o = 16; o; o >>= 1) {
      unsigned long long x = __shfl_down_sync(0xffffffffu, local, o);
      local = x < local ? x : local;
    }
    if ((threadIdx.x & 31) == 0 && local != ~0ull) atomicMin(rep + t, local);
  }
}

// Sorted canonical keys (ascending) and their ids, in ctx buffers.
void sort_ascending(Context& ctx, const double* d_ef, int64_t n, double** keys_out, int64_t** ids_out) {
  cudaStream_t s = ctx.stream;
  double* keys = ctx.buf("t_keys").as<double>(n);
  double* keys2 = ctx.buf("t_keys2").as<double>(n);
  int64_t* ids = ctx.buf("t_ids").as<int64_t>(n);
  int64_t* ids2 = ctx.buf("t_ids2").as<int64_t>(n);
  EFG_LAUNCH(k_topk_init, ceil_div(n, kRankThreads), kRankThreads, 0, s, d_ef, n, keys, ids);
  size_t tmp = 0;
  EFG_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, keys2, ids, ids2, n, 0, 64, s));
  EFG_REGION("cub::DeviceRadixSort::SortPairs", s, EFG_CUDA_CHECK(
      cub::DeviceRadixSort::SortPairs(ctx.buf("cub").get(tmp), tmp, keys, keys2, ids, ids2, n, 0, 64, s)));
  *keys_out = keys2;
  *ids_out = ids2;
}

int grid_for(Context& ctx, int64_t n) {
  int64_t g = ceil_div(n, kRankThreads);
  int64_t cap = (int64_t)ctx.num_sms * 8;
  return (int)(g < cap ? (g > 0 ? g : 1) : cap);
}
}  // namespace

void rank_ascending_device(Context& ctx, const double* d_ef, int64_t n, int64_t* d_order) {
  if (n <= 0) return;
  double* keys;
  int64_t* ids;
  sort_ascending(ctx, d_ef, n, &keys, &ids);
  EFG_CUDA_CHECK(cudaMemcpyAsync(d_order, ids, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx.stream));
}

int64_t ef_bins_device(Context& ctx, const double* d_ef, int64_t n, int64_t k, double* d_targets, int64_t* d_rep) {
  cudaStream_t s = ctx.stream;
  double* keys;
  int64_t* ids;
  sort_ascending(ctx, d_ef, n, &keys, &ids);
  unsigned long long* words = ctx.buf("t_bin_words").as<unsigned long long>(2 * k + 1);
  unsigned long long* best = words;
  unsigned long long* rep = words + k;
  unsigned long long* cnt = words + 2 * k;
  EFG_CUDA_CHECK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
  EFG_LAUNCH(k_distinct, grid_for(ctx, n), kRankThreads, 0, s, keys, n, cnt);
  unsigned long long distinct = 0;
  EFG_CUDA_CHECK(cudaMemcpyAsync(&distinct, cnt, sizeof(distinct), cudaMemcpyDeviceToHost, s));
  EFG_CUDA_CHECK(cudaStreamSynchronize(s));
  if ((int64_t)distinct < k) return (int64_t)distinct;
  EFG_LAUNCH(k_bin_targets, ceil_div(k, kRankThreads), kRankThreads, 0, s, keys, n, k, d_targets, best, rep);
  EFG_LAUNCH(k_nearest_diff, grid_for(ctx, n), kRankThreads, 0, s, d_ef, n, d_targets, k, best);
  EFG_LAUNCH(k_nearest_id, grid_for(ctx, n), kRankThreads, 0, s, d_ef, n, d_targets, k, best, rep);
  EFG_CUDA_CHECK(cudaMemcpyAsync(d_rep, rep, k * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  return (int64_t)distinct;
}

}  // namespace efg
