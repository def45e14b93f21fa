// Per-SM rate of loading an MMA A operand into TENSOR memory through registers (no shared
// memory): every CTA (one per SM) streams k-blocks of a 128-row bf16 tile (rows `ld` elements
// apart, L2-resident) -- each k-block 128 rows x 64 bf16 -- with W loader warps per TMEM lane
// quadrant, D k-blocks of loads in flight per thread, and writes them with tcgen05.st. Answers
// whether an A-from-TMEM grouped GEMM (whose shared memory then carries only the weights)
// could be fed fast enough.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_11537_b200/csrc \
//        tools/tmem_load_probe.cu -o /tmp/tmem_load_probe && /tmp/tmem_load_probe
#include <cuda_runtime.h>
#include <cstdio>

#include "ptx.cuh"

using namespace mp;

__device__ __forceinline__ uint4 ldg_nc(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// W warps per quadrant: warp w -> quadrant w % 4, column part w / 4 (64 / W bf16 of the k-block)
template <int W, int D>
__global__ void __launch_bounds__(128 * W, 1) k_tmem_load(const __nv_bfloat16* __restrict__ a, int ld, int nkb,
                                                          int rows_total, unsigned long long* ns) {
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_slot;
  constexpr int Q = 8 / W;  // uint4 (8 bf16) per thread per k-block
  const int q = warp & 3, part = warp >> 2;
  const int row = (blockIdx.x * 128 + q * 32 + lane) % rows_total;
  const uint4* src = reinterpret_cast<const uint4*>(a + (size_t)row * ld) + part * Q;
  const uint32_t taddr = tbase + (static_cast<uint32_t>(q * 32) << 16) + part * (Q * 4);
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  uint4 buf[D][Q];
#pragma unroll
  for (int s = 0; s < D; ++s)
#pragma unroll
    for (int i = 0; i < Q; ++i) buf[s][i] = ldg_nc(src + (size_t)s * 8 + i);
  for (int kb = 0; kb < nkb; kb += D) {
#pragma unroll
    for (int s = 0; s < D; ++s) {
      uint32_t r[4 * Q];
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        r[4 * i] = buf[s][i].x, r[4 * i + 1] = buf[s][i].y, r[4 * i + 2] = buf[s][i].z, r[4 * i + 3] = buf[s][i].w;
      }
      const int nxt = kb + s + D;
      if (nxt < nkb)
#pragma unroll
        for (int i = 0; i < Q; ++i) buf[s][i] = ldg_nc(src + (size_t)(nxt % 48) * 8 + i);
      const uint32_t col = taddr + ((kb + s) & 3) * 32;
      if constexpr (Q == 8) {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(col),
            "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
            "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
            "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
            "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
            : "memory");
      } else if constexpr (Q == 4) {
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
            ::"r"(col), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
            "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
            : "memory");
      } else {
        tmem_st8(col, r);
      }
    }
  }
  tmem_st_wait();
  __syncthreads();
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) ns[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tbase, 256);
  }
}

template <int W, int D>
static void run(const __nv_bfloat16* a, int ld, int rows_total, unsigned long long* ns, int nsm) {
  const int nkb = 480;  // 10 units of K = 3072
  auto k = k_tmem_load<W, D>;
  for (int rep = 0; rep < 2; ++rep) k<<<nsm, 128 * W>>>(a, ld, nkb, rows_total, ns);
  cudaDeviceSynchronize();
  unsigned long long h[1024];
  cudaMemcpy(h, ns, sizeof(unsigned long long) * nsm, cudaMemcpyDeviceToHost);
  double mx = 0, mean = 0;
  for (int i = 0; i < nsm; ++i) {
    mx = h[i] > mx ? h[i] : mx;
    mean += h[i];
  }
  mean /= nsm;
  const double bytes = 128.0 * 128 * nkb;  // per CTA
  printf("W=%d warps/quadrant D=%d in flight: %.1f GB/s per SM (mean), %.1f TB/s chip (slowest CTA) [%s]\n", W, D,
         bytes / mean, bytes * nsm / mx / 1e3, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int ld = 3072, rows_total = 16384;  // H of GEMM2: 16384 rows x 3072 bf16 (100 MB)
  __nv_bfloat16* a;
  cudaMalloc(&a, sizeof(__nv_bfloat16) * (size_t)rows_total * ld);
  cudaMemset(a, 0, sizeof(__nv_bfloat16) * (size_t)rows_total * ld);
  unsigned long long* ns;
  cudaMalloc(&ns, sizeof(unsigned long long) * 1024);
  run<1, 1>(a, ld, rows_total, ns, nsm);
  run<1, 2>(a, ld, rows_total, ns, nsm);
  run<1, 3>(a, ld, rows_total, ns, nsm);
  run<2, 2>(a, ld, rows_total, ns, nsm);
  run<2, 4>(a, ld, rows_total, ns, nsm);
  run<4, 4>(a, ld, rows_total, ns, nsm);
  run<4, 6>(a, ld, rows_total, ns, nsm);
  return 0;
}
