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

}  // namespace efg
