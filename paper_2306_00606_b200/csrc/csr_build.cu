// K1 -- device CSR builder.  Replaces efgraph/graph.py:147-190 `build_graph`
// and must produce the SAME arrays bit for bit:
//   drop self-loops (:159); orig_ids = sorted distinct endpoints (:163);
//   reject n >= 2^31 (:165-166); dense ids by lower_bound (:167-168);
//   dedupe canonical lo*n+hi codes (:169); symmetrise and sort by (src, dst)
//   (:174-178); offsets from per-source counts (:180-181).
// All outputs are canonical (sorted / unique), so any exact implementation
// matches the reference.  Sorts are CUB LSD radix sorts limited to the bits
// the keys actually use.
#include <cub/cub.cuh>

#include "common.cuh"
#include "efg_internal.cuh"

namespace efg {

namespace {

// Endpoint flags: self-loops contribute no endpoints (graph.py:159).
__global__ void k_mark_loops(const int64_t* __restrict__ edges, int64_t k, uint8_t* __restrict__ flag2) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= k) return;
  bool ok = edges[2 * t] != edges[2 * t + 1];
  flag2[2 * t] = ok;
  flag2[2 * t + 1] = ok;
}

__device__ __forceinline__ int64_t lower_bound64(const int64_t* __restrict__ a, int64_t n, int64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_codes(const int64_t* __restrict__ edges, int64_t k, const int64_t* __restrict__ orig,
                        int64_t n, uint64_t* __restrict__ codes) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= k) return;
  int64_t u = edges[2 * t], v = edges[2 * t + 1];
  if (u == v) {
    codes[t] = ~0ull;  // sorts last, trimmed by the unique count
    return;
  }
  int64_t lo = lower_bound64(orig, n, u < v ? u : v);
  int64_t hi = lower_bound64(orig, n, u < v ? v : u);
  codes[t] = (uint64_t)lo * (uint64_t)n + (uint64_t)hi;
}

__global__ void k_symmetrise(const uint64_t* __restrict__ codes, int64_t m, int64_t n,
                             uint64_t* __restrict__ keys) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= m) return;
  uint64_t c = codes[t];
  uint64_t lo = c / (uint64_t)n, hi = c % (uint64_t)n;
  keys[t] = c;                                   // (lo, hi)
  keys[m + t] = hi * (uint64_t)n + lo;           // (hi, lo)
}

__global__ void k_split_keys(const uint64_t* __restrict__ keys, int64_t m2, int64_t n,
                             int32_t* __restrict__ nbr, int64_t* __restrict__ offsets) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= m2) return;
  uint64_t key = keys[t];
  int64_t src = (int64_t)(key / (uint64_t)n);
  nbr[t] = (int32_t)(key % (uint64_t)n);
  // offsets[v] = first position whose src >= v; every node has degree >= 1
  int64_t prev = t ? (int64_t)(keys[t - 1] / (uint64_t)n) : -1;
  for (int64_t v = prev + 1; v <= src; ++v) offsets[v] = t;
  if (t == m2 - 1) offsets[n] = m2;
}

__global__ void k_shift(int64_t* __restrict__ x, int64_t cnt, int64_t delta) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < cnt) x[t] += delta;
}

int bits_for(uint64_t maxval) {
  int b = 1;
  while (b < 64 && (maxval >> b)) ++b;
  return b;
}

}  // namespace

// Build the CSR of `k` raw (u, v) int64 pairs already resident on the device.
void build_csr_device(Context& ctx, const int64_t* d_edges, int64_t k, DeviceCSR& out) {
  cudaStream_t s = ctx.stream;
  out.n = 0;
  out.m = 0;
  if (k == 0) return;
  const int B = 256;
  // 1. endpoints of non-loop pairs -> sorted distinct = orig_ids
  int64_t* ends = ctx.buf("k1_ends").as<int64_t>(2 * k);  // radix double buffer
  int64_t* ends_sorted = ctx.buf("k1_ends_sorted").as<int64_t>(2 * k);
  uint8_t* flag2 = ctx.buf("k1_flag2").as<uint8_t>(2 * k);
  int64_t* dnum = ctx.buf("k1_num").as<int64_t>(4);
  EFG_LAUNCH(k_mark_loops, ceil_div(k, B), B, 0, s, d_edges, k, flag2);
  // compact away self-loop endpoints
  size_t tmp = 0;
  EFG_CUDA_CHECK(cub::DeviceSelect::Flagged(nullptr, tmp, d_edges, flag2, ends_sorted, dnum, 2 * k, s));
  EFG_REGION("cub::DeviceSelect::Flagged", s, EFG_CUDA_CHECK(cub::DeviceSelect::Flagged(ctx.buf("cub").get(tmp), tmp, d_edges, flag2, ends_sorted, dnum, 2 * k, s)));
  int64_t nend = 0;
  EFG_CUDA_CHECK(cudaMemcpyAsync(&nend, dnum, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  EFG_CUDA_CHECK(cudaStreamSynchronize(s));
  if (nend == 0) return;
  // id range -> number of radix bits (ids may be any int64, like the
  // reference's np.unique; sort them as unsigned offsets from the minimum)
  EFG_CUDA_CHECK(cub::DeviceReduce::Min(nullptr, tmp, ends_sorted, dnum + 1, nend, s));
  EFG_REGION("cub::DeviceReduce::Min", s, EFG_CUDA_CHECK(cub::DeviceReduce::Min(ctx.buf("cub").get(tmp), tmp, ends_sorted, dnum + 1, nend, s)));
  EFG_CUDA_CHECK(cub::DeviceReduce::Max(nullptr, tmp, ends_sorted, dnum + 2, nend, s));
  EFG_REGION("cub::DeviceReduce::Max", s, EFG_CUDA_CHECK(cub::DeviceReduce::Max(ctx.buf("cub").get(tmp), tmp, ends_sorted, dnum + 2, nend, s)));
  int64_t mm[2] = {0, 0};
  EFG_CUDA_CHECK(cudaMemcpyAsync(mm, dnum + 1, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  EFG_CUDA_CHECK(cudaStreamSynchronize(s));
  const int64_t minid = mm[0];
  EFG_LAUNCH(k_shift, ceil_div(nend, B), B, 0, s, ends_sorted, nend, -minid);
  int idbits = bits_for((uint64_t)mm[1] - (uint64_t)minid);
  uint64_t* ukeys = reinterpret_cast<uint64_t*>(ends_sorted);
  uint64_t* ukeys_alt = reinterpret_cast<uint64_t*>(ends);
  EFG_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, ukeys, ukeys_alt, nend, 0, idbits, s));
  EFG_REGION("cub::DeviceRadixSort::SortKeys", s, EFG_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(ctx.buf("cub").get(tmp), tmp, ukeys, ukeys_alt, nend, 0, idbits, s)));
  int64_t* orig = ctx.buf("k1_orig").as<int64_t>(nend);
  EFG_CUDA_CHECK(cub::DeviceSelect::Unique(nullptr, tmp, ukeys_alt, reinterpret_cast<uint64_t*>(orig), dnum, nend, s));
  EFG_REGION("cub::DeviceSelect::Unique", s, EFG_CUDA_CHECK(cub::DeviceSelect::Unique(ctx.buf("cub").get(tmp), tmp, ukeys_alt, reinterpret_cast<uint64_t*>(orig), dnum, nend, s)));
  int64_t n = 0;
  EFG_CUDA_CHECK(cudaMemcpyAsync(&n, dnum, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  EFG_CUDA_CHECK(cudaStreamSynchronize(s));
  EFG_REQUIRE(n < (int64_t(1) << 31), "graph too large: " + std::to_string(n) + " nodes exceeds int32 id space");
  EFG_LAUNCH(k_shift, ceil_div(n, B), B, 0, s, orig, n, minid);
  // 2. canonical dense codes, dedupe
  uint64_t* codes = ctx.buf("k1_codes").as<uint64_t>(k);
  uint64_t* codes_sorted = ctx.buf("k1_codes_sorted").as<uint64_t>(k);
  EFG_LAUNCH(k_codes, ceil_div(k, B), B, 0, s, d_edges, k, orig, n, codes);
  int cbits = bits_for((uint64_t)n * (uint64_t)n);
  // self-loops carry ~0: sort on all 64 bits only if any exist; else on cbits
  int64_t nloops = k - nend / 2;
  int sort_bits = nloops ? 64 : cbits;
  EFG_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, codes, codes_sorted, k, 0, sort_bits, s));
  EFG_REGION("cub::DeviceRadixSort::SortKeys", s, EFG_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(ctx.buf("cub").get(tmp), tmp, codes, codes_sorted, k, 0, sort_bits, s)));
  EFG_CUDA_CHECK(cub::DeviceSelect::Unique(nullptr, tmp, codes_sorted, codes, dnum, k - nloops, s));
  EFG_REGION("cub::DeviceSelect::Unique", s, EFG_CUDA_CHECK(cub::DeviceSelect::Unique(ctx.buf("cub").get(tmp), tmp, codes_sorted, codes, dnum, k - nloops, s)));
  int64_t m = 0;
  EFG_CUDA_CHECK(cudaMemcpyAsync(&m, dnum, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  EFG_CUDA_CHECK(cudaStreamSynchronize(s));
  // 3. symmetrise, sort by (src, dst), split
  uint64_t* keys = ctx.buf("k1_keys").as<uint64_t>(2 * m);
  uint64_t* keys_sorted = ctx.buf("k1_keys_sorted").as<uint64_t>(2 * m);
  EFG_LAUNCH(k_symmetrise, ceil_div(m, B), B, 0, s, codes, m, n, keys);
  EFG_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys, keys_sorted, 2 * m, 0, cbits, s));
  EFG_REGION("cub::DeviceRadixSort::SortKeys", s, EFG_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(ctx.buf("cub").get(tmp), tmp, keys, keys_sorted, 2 * m, 0, cbits, s)));
  out.alloc(n, m);
  EFG_LAUNCH(k_split_keys, ceil_div(2 * m, B), B, 0, s, keys_sorted, 2 * m, n, out.nbr, out.offsets);
  EFG_CUDA_CHECK(cudaMemcpyAsync(out.orig_ids, orig, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  out.n = n;
  out.m = m;
}

}  // namespace efg
