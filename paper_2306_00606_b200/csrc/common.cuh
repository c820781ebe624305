// Shared helpers for the efg sm_100a kernels (no torch types anywhere).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace efg {

// Status codes of the C ABI (include/efg.h).
enum Status : int {
  EFG_OK = 0,
  EFG_INVALID = 1,   // -> ValueError
  EFG_CUDA = 2,      // -> OSError subclass (device error)
  EFG_NCCL = 3,
  EFG_OOM = 4,
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define EFG_CUDA_CHECK(expr)                                                        \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      throw ::efg::Error(_e == cudaErrorMemoryAllocation ? ::efg::EFG_OOM            \
                                                         : ::efg::EFG_CUDA,          \
                         std::string(#expr) + ": " + cudaGetErrorString(_e) +        \
                             " (" __FILE__ ":" + std::to_string(__LINE__) + ")");    \
    }                                                                               \
  } while (0)

#define EFG_REQUIRE(cond, msg)                                                      \
  do {                                                                              \
    if (!(cond)) throw ::efg::Error(::efg::EFG_INVALID, (msg));                      \
  } while (0)

// Bounds-checked builds (-DEFG_BOUNDS_CHECK, tools/build_variant.sh checked):
// the compute-sanitizer is closed on the B200 pool, so the risky device
// indices (table gathers, shared-map positions, row ranges) are checked in
// the kernels themselves.  A failed check records its source line in a
// per-translation-unit device word (first failure wins) and the index is
// clamped to 0, so the kernel completes without touching memory out of
// bounds; the C ABI turns a recorded line into a status-2 error after the
// call (efg_check_failures).  Release builds compile the checks away.
#ifdef EFG_BOUNDS_CHECK
static __device__ int efg_check_line = 0;
#define EFG_DCHECK(cond) ((cond) ? true : (atomicCAS(&efg_check_line, 0, __LINE__), false))
#define EFG_CLAMP(idx, len) (EFG_DCHECK((int64_t)(idx) >= 0 && (int64_t)(idx) < (int64_t)(len)) ? (idx) : 0)
// host: read and clear this translation unit's failure line
#define EFG_CHECK_ACCESSOR(fn)                                                     \
  int fn() {                                                                       \
    int v = 0, z = 0;                                                              \
    cudaMemcpyFromSymbol(&v, efg_check_line, sizeof v);                            \
    cudaMemcpyToSymbol(efg_check_line, &z, sizeof z);                              \
    return v;                                                                      \
  }
#else
#define EFG_DCHECK(cond) true
#define EFG_CLAMP(idx, len) (idx)
#define EFG_CHECK_ACCESSOR(fn) \
  int fn() { return 0; }
#endif

constexpr int kWarp = 32;
constexpr int kNumSMs = 148;   // B200; queried at runtime as well

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Grow-only device scratch buffer owned by a context.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void* get(size_t need) {
    if (need == 0) need = 16;
    if (need > bytes) {
      if (p) EFG_CUDA_CHECK(cudaFree(p));
      p = nullptr;
      bytes = 0;
      size_t want = need + need / 8;
      EFG_CUDA_CHECK(cudaMalloc(&p, want));
      bytes = want;
    }
    return p;
  }
  template <class T>
  T* as(size_t count) { return static_cast<T*>(get(count * sizeof(T))); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

// Launch bookkeeping.  Every kernel launch in the library goes through
// EFG_LAUNCH (count is exact: stats.launches); library calls that launch
// their own kernels (CUB) go through EFG_REGION.  When the context's profiler
// is on, both record a CUDA event pair on the launching stream so per-kernel
// device times are measured live (efg_profile_report).
struct Profiler;
extern thread_local int64_t g_launches;
extern thread_local int64_t g_lib_calls;
extern thread_local Profiler* g_prof;
void prof_begin(Profiler*, const char* name, cudaStream_t s);
void prof_end(Profiler*, cudaStream_t s);

inline int64_t grid_count(int64_t g) { return g; }
inline int64_t grid_count(dim3 g) { return (int64_t)g.x * g.y * g.z; }
#define EFG_LAUNCH(kernel, grid, block, smem, stream, ...)                         \
  do {                                                                              \
    if (::efg::grid_count(grid) > 0) {                                              \
      if (::efg::g_prof) ::efg::prof_begin(::efg::g_prof, #kernel, (stream));       \
      kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);                   \
      EFG_CUDA_CHECK(cudaGetLastError());                                           \
      if (::efg::g_prof) ::efg::prof_end(::efg::g_prof, (stream));                  \
      ++::efg::g_launches;                                                          \
    }                                                                               \
  } while (0)

#define EFG_REGION(name, stream, ...)                                              \
  do {                                                                              \
    if (::efg::g_prof) ::efg::prof_begin(::efg::g_prof, (name), (stream));          \
    __VA_ARGS__;                                                                    \
    if (::efg::g_prof) ::efg::prof_end(::efg::g_prof, (stream));                    \
    ++::efg::g_lib_calls;                                                           \
  } while (0)

// Warp bitonic sort of 32*I keys, I per lane in blocked order, ascending
// (within-lane stages are register min/max, cross-lane stages shuffles).
template <int I>
__device__ __forceinline__ void warp_bitonic(uint32_t (&x)[I], int lane) {
#pragma unroll
  for (int k = 2; k <= 32 * I; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < I) {
#pragma unroll
        for (int i = 0; i < I; ++i) {
          const int pi = i ^ j;
          if (pi > i) {
            const bool up = ((lane * I + i) & k) == 0;
            const uint32_t lo = min(x[i], x[pi]), hi = max(x[i], x[pi]);
            x[i] = up ? lo : hi;
            x[pi] = up ? hi : lo;
          }
        }
      } else {
        const int lj = j / I;
        const bool lower = (lane & lj) == 0;
#pragma unroll
        for (int i = 0; i < I; ++i) {
          const uint32_t y = __shfl_xor_sync(0xffffffffu, x[i], lj);
          const bool up = ((lane * I + i) & k) == 0;
          x[i] = (lower == up) ? min(x[i], y) : max(x[i], y);
        }
      }
    }
  }
}

}  // namespace efg
