// Shared device helpers and host-side error plumbing for the C-ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <utility>

#include "moempmc.h"

namespace mp {

constexpr int kChunk = 128;       // tokens per rank/histogram chunk (= GEMM M tile)
constexpr int kBlockMRows = 128;  // rows per GEMM M tile (pieces in split_m mode)

__host__ __device__ inline int cdiv(int a, int b) { return (a + b - 1) / b; }

// Programmatic dependent launch: let the next kernel in the stream start launching
// (its CTAs fill SMs as ours retire and run their prologue), and block until the
// previous kernel has completed and its writes are visible. Both are no-ops when the
// launch carries no programmatic dependency.
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }


// Block-wide inclusive sum for up to 1024 threads (blockDim multiple of 32).
__device__ inline int block_sum(int v, int* red /* >= 32 ints smem */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int t = (lane < nw) ? red[lane] : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

__device__ inline int block_max(int v, int* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int t = (lane < nw) ? red[lane] : INT_MIN;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t = max(t, __shfl_xor_sync(0xffffffffu, t, o));
  return t;
}

// In-place exclusive scan of n ints in shared memory by the whole block.
// Returns the total. Each thread owns a contiguous run (keeps order).
__device__ inline int block_exclusive_scan(int* a, int n, int* red /* >= 33 ints */) {
  const int nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int b = threadIdx.x * per, e = min(n, b + per);
  int s = 0;
  for (int i = b; i < e; ++i) s += a[i];
  // exclusive scan of per-thread sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = nt >> 5;
  int incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __syncthreads();
  if (lane == 31) red[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = (lane < nw) ? red[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < nw) red[lane] = wi - w;  // exclusive warp offsets
    if (lane == 31) red[32] = wi;       // total
  }
  __syncthreads();
  int run = red[warp] + incl - s;
  for (int i = b; i < e; ++i) {
    const int x = a[i];
    a[i] = run;
    run += x;
  }
  const int total = red[32];
  __syncthreads();
  return total;
}

// Router workspace (mp_router_workspace_bytes): [xhl: T x 2d bf16][xb: T f32][count + list: T+1 i32][wabs: d f32]
struct RouterWs {
  void* xhl;
  float* xb;
  int32_t* count;
  int32_t* list;
  static size_t al(size_t x) { return (x + 255) & ~size_t(255); }
  RouterWs(void* ws, int T, int d) {
    char* p = (char*)ws;
    xhl = p;
    p += al((size_t)2 * T * 2 * d);
    xb = (float*)p;
    p += al(sizeof(float) * (size_t)T);
    count = (int32_t*)p;
    list = count + 1;
  }
};

// Kernel launch through cudaLaunchKernelEx. Kernels still bracket their dependent reads
// with griddep_wait() so programmatic edges could be enabled per launch; in the whole-step
// CUDA graph programmatic edges measured slower (5.51 vs 5.34 ms/step, round 1), so none
// are requested.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.numAttrs = 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace mp

#define MP_CUDA_TRY(expr)                                                                  \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess) {                                                               \
      mp_set_last_error("%s:%d: %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return MP_ERR_CUDA;                                                                  \
    }                                                                                      \
  } while (0)

#define MP_REQUIRE(cond, code, ...)      \
  do {                                   \
    if (!(cond)) {                       \
      mp_set_last_error(__VA_ARGS__);    \
      return (code);                     \
    }                                    \
  } while (0)

// defined in capi.cu
extern "C" void mp_set_last_error(const char* fmt, ...);
