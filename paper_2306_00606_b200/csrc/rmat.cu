// Device R-MAT sampler, bit-identical to efgraph/graph.py:204-246
// `generate_rmat`.
//
// The reference draws numpy PCG64 doubles rng.random((batch, scale)) and
// inserts canonical pair codes lo*side+hi into a Python set until `target`
// distinct codes exist, or until cap = 20*target pairs were drawn
// (graph.py:213-246).  The double stream does not depend on the batch sizes,
// so the edge set is "the first `target` distinct non-loop codes of the pair
// stream" (all distinct codes of the first `cap` pairs when truncated).
// Here every thread jumps the 128-bit PCG64 LCG to its first draw
// (square-and-multiply advance) and emits the codes of its pairs; a stable
// radix sort by code yields each code's first stream index; the cutoff is the
// target-th smallest first index; the surviving codes feed the CSR builder.
#include <cub/cub.cuh>

#include "common.cuh"
#include "efg_internal.cuh"

namespace efg {

namespace {

typedef unsigned __int128 u128;
__device__ __host__ inline u128 mk128(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }
__device__ inline u128 pcg_mult() { return mk128(0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull); }

// state advanced by `delta` LCG steps (pcg_advance_lcg_128)
__device__ inline u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

// numpy PCG64 next_uint64: step, then XSL-RR output of the new state
__device__ inline uint64_t pcg_next(u128& state, u128 inc) {
  state = state * pcg_mult() + inc;
  const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
  const unsigned rot = (unsigned)(state >> 122);
  return (x >> rot) | (x << ((64 - rot) & 63));
}

constexpr int kPairsPerThread = 32;

__global__ void k_rmat_codes(uint64_t s_hi, uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, int scale, double a,
                             double ab, double abc, int64_t npairs, uint64_t loop_code,
                             uint64_t* __restrict__ codes, int32_t* __restrict__ idx) {
  const int64_t t0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * kPairsPerThread;
  if (t0 >= npairs) return;
  const u128 inc = mk128(i_hi, i_lo);
  u128 st = pcg_advance(mk128(s_hi, s_lo), inc, (uint64_t)t0 * scale);
  const uint64_t side = 1ull << scale;
  for (int k = 0; k < kPairsPerThread && t0 + k < npairs; ++k) {
    uint64_t u = 0, v = 0;
    for (int c = 0; c < scale; ++c) {
      const double r = (double)(pcg_next(st, inc) >> 11) * (1.0 / 9007199254740992.0);
      const uint64_t bit = 1ull << (scale - 1 - c);
      if (r >= ab) u |= bit;                                   // graph.py:227
      if ((r >= a && r < ab) || r >= abc) v |= bit;            // graph.py:228
    }
    const int64_t t = t0 + k;
    codes[t] = u == v ? loop_code : (u < v ? u : v) * side + (u < v ? v : u);
    idx[t] = (int32_t)t;
  }
}

// first occurrence of each distinct code in the sorted stream (loops excluded)
__global__ void k_first_flags(const uint64_t* __restrict__ sc, int64_t n, uint64_t loop_code,
                              uint8_t* __restrict__ flag) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  flag[k] = sc[k] != loop_code && (k == 0 || sc[k] != sc[k - 1]);
}

__global__ void k_keep_before(const uint64_t* __restrict__ sc, const int32_t* __restrict__ sidx,
                              const uint8_t* __restrict__ first, int64_t n, const int32_t* __restrict__ cut_dev,
                              uint8_t* __restrict__ keep) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  keep[k] = first[k] && sidx[k] <= *cut_dev;
}

__global__ void k_codes_to_pairs(const uint64_t* __restrict__ codes, int64_t m, int scale,
                                 int64_t* __restrict__ pairs) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const uint64_t c = codes[k];
  pairs[2 * k] = (int64_t)(c >> scale);
  pairs[2 * k + 1] = (int64_t)(c & ((1ull << scale) - 1));
}

int bits_of(uint64_t x) {
  int b = 1;
  while (b < 64 && (x >> b)) ++b;
  return b;
}

}  // namespace

// Returns (edges drawn into the context CSR) and whether the attempt cap truncated.
void rmat_build_device(Context& ctx, int scale, int64_t avg_degree, const double* probs, const uint64_t* state,
                       const uint64_t* inc, bool& truncated, DeviceCSR& out) {
  cudaStream_t s = ctx.stream;
  EFG_REQUIRE(scale >= 1 && scale <= 30, "scale must be in [1, 30]");
  EFG_REQUIRE(avg_degree >= 1, "avg_degree must be >= 1");
  const double a = probs[0], b = probs[1], c = probs[2];
  const double ab = a + b, abc = a + b + c;  // same expression order as graph.py:227-228
  const int64_t side = int64_t(1) << scale;
  const int64_t target = side * avg_degree / 2;
  const int64_t cap = 20 * target;
  EFG_REQUIRE(cap < (int64_t(1) << 31), "attempt cap exceeds the int32 stream index");
  const uint64_t loop_code = (uint64_t)1 << (2 * scale);
  const int kbits = bits_of(loop_code);
  const int B = 256;
  size_t tmp = 0;
  int64_t npairs = std::min<int64_t>(cap, target + target / 4 + 4096);
  int64_t ndist = 0;
  for (;;) {
    uint64_t* codes = ctx.buf("r_codes").as<uint64_t>(2 * npairs);
    int32_t* idx = ctx.buf("r_idx").as<int32_t>(2 * npairs);
    uint8_t* flag = ctx.buf("r_flag").as<uint8_t>(npairs);
    int64_t* cnt = ctx.buf("r_cnt").as<int64_t>(2);
    EFG_LAUNCH(k_rmat_codes, ceil_div(ceil_div(npairs, kPairsPerThread), B), B, 0, s, (uint64_t)state[1],
               (uint64_t)state[0], (uint64_t)inc[1], (uint64_t)inc[0], scale, a, ab, abc, npairs, loop_code, codes,
               idx);
    uint64_t* sc = codes + npairs;
    int32_t* sidx = idx + npairs;
    EFG_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, codes, sc, idx, sidx, npairs, 0, kbits, s));
    EFG_REGION("cub::DeviceRadixSort::SortPairs", s,
               EFG_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(ctx.buf("cub").get(tmp), tmp, codes, sc, idx, sidx,
                                                              npairs, 0, kbits, s)));
    EFG_LAUNCH(k_first_flags, ceil_div(npairs, B), B, 0, s, sc, npairs, loop_code, flag);
    // first stream index of every distinct code
    int32_t* firsts = idx;  // reuse the unsorted index buffer
    EFG_CUDA_CHECK(cub::DeviceSelect::Flagged(nullptr, tmp, sidx, flag, firsts, cnt, npairs, s));
    EFG_REGION("cub::DeviceSelect::Flagged", s,
               EFG_CUDA_CHECK(cub::DeviceSelect::Flagged(ctx.buf("cub").get(tmp), tmp, sidx, flag, firsts, cnt,
                                                         npairs, s)));
    EFG_CUDA_CHECK(cudaMemcpyAsync(&ndist, cnt, sizeof ndist, cudaMemcpyDeviceToHost, s));
    EFG_CUDA_CHECK(cudaStreamSynchronize(s));
    if (ndist >= target || npairs == cap) {
      truncated = ndist < target;
      uint8_t* keep = ctx.buf("r_keep").as<uint8_t>(npairs);
      int32_t* cut = ctx.buf("r_cut").as<int32_t>(1);
      if (!truncated) {
        // cutoff = target-th smallest first index
        int32_t* sf = ctx.buf("r_sorted_firsts").as<int32_t>(ndist);
        EFG_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, firsts, sf, ndist, 0, bits_of(npairs), s));
        EFG_REGION("cub::DeviceRadixSort::SortKeys", s,
                   EFG_CUDA_CHECK(cub::DeviceRadixSort::SortKeys(ctx.buf("cub").get(tmp), tmp, firsts, sf, ndist, 0,
                                                                 bits_of(npairs), s)));
        EFG_CUDA_CHECK(cudaMemcpyAsync(cut, sf + target - 1, sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
      } else {
        const int32_t all = (int32_t)npairs;
        EFG_CUDA_CHECK(cudaMemcpyAsync(cut, &all, sizeof all, cudaMemcpyHostToDevice, s));
      }
      EFG_LAUNCH(k_keep_before, ceil_div(npairs, B), B, 0, s, sc, sidx, flag, npairs, cut, keep);
      uint64_t* kept = codes;  // reuse
      EFG_CUDA_CHECK(cub::DeviceSelect::Flagged(nullptr, tmp, sc, keep, kept, cnt + 1, npairs, s));
      EFG_REGION("cub::DeviceSelect::Flagged", s,
                 EFG_CUDA_CHECK(cub::DeviceSelect::Flagged(ctx.buf("cub").get(tmp), tmp, sc, keep, kept, cnt + 1,
                                                           npairs, s)));
      int64_t m = 0;
      EFG_CUDA_CHECK(cudaMemcpyAsync(&m, cnt + 1, sizeof m, cudaMemcpyDeviceToHost, s));
      EFG_CUDA_CHECK(cudaStreamSynchronize(s));
      int64_t* pairs = ctx.buf("r_pairs").as<int64_t>(2 * (m > 0 ? m : 1));
      EFG_LAUNCH(k_codes_to_pairs, ceil_div(m, B), B, 0, s, kept, m, scale, pairs);
      build_csr_device(ctx, pairs, m, out);
      return;
    }
    npairs = std::min<int64_t>(cap, 2 * npairs);
  }
}

}  // namespace efg
