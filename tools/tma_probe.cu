// Per-SM TMA ingest probe: every CTA (one per SM) streams 2-D tiles of an L2-resident
// bf16 buffer into a STAGES-deep shared-memory ring (mbarrier tx completion), the
// consumer releases each stage immediately. Reports bytes/s per SM and chip-wide for
// box sizes and ring depths, to separate the GEMM core's per-SM operand ingest limit
// from MMA / epilogue effects.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_11537_b200/csrc \
//        tools/tma_probe.cu -o /tmp/tma_probe -lcuda && /tmp/tma_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace mp;

template <int STAGES>
__global__ void __launch_bounds__(64, 1) k_probe(const __grid_constant__ CUtensorMap tm, int box_rows, int iters,
                                                 int rows_total, unsigned long long* cycles, int priv = 0) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stage_bytes = box_rows * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * stage_bytes);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const long long t0 = clock64();
  if (threadIdx.x == 0) {  // producer
    uint32_t stage = 0, phase = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&empty[stage], phase ^ 1);
      mbar_arrive_expect_tx(&full[stage], stage_bytes);
      // priv > 0: every CTA cycles over its own priv boxes (no two SMs read the same line)
      const int row = priv ? (int)(((long long)blockIdx.x * priv + (i % priv)) * box_rows)
                           : ((blockIdx.x * 7 + i) * box_rows) % rows_total;
      tma_load_2d(smem + stage * stage_bytes, &tm, &full[stage], 0, row);
      if (++stage == STAGES) stage = 0, phase ^= 1;
    }
  } else if (threadIdx.x == 32) {  // consumer
    uint32_t stage = 0, phase = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&full[stage], phase);
      mbar_arrive(&empty[stage]);
      if (++stage == STAGES) stage = 0, phase ^= 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
}

template <int STAGES>
__global__ void __launch_bounds__(64, 1) k_probe3(const __grid_constant__ CUtensorMap tm, int box_bytes, int iters,
                                                  int blocks_total, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * box_bytes);
  uint64_t* empty = full + STAGES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    uint32_t stage = 0, phase = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&empty[stage], phase ^ 1);
      mbar_arrive_expect_tx(&full[stage], box_bytes);
      const int z = ((blockIdx.x * 7 + i) * 2) % blocks_total;
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
              smem_u32(smem + stage * box_bytes)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(&full[stage])), "r"(0), "r"(0), "r"(z)
          : "memory");
      if (++stage == STAGES) stage = 0, phase ^= 1;
    }
  } else if (threadIdx.x == 32) {
    uint32_t stage = 0, phase = 0;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(&full[stage], phase);
      mbar_arrive(&empty[stage]);
      if (++stage == STAGES) stage = 0, phase ^= 1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

// Chip-wide TMA throughput with DISJOINT per-SM regions: an L2-resident working set (each CTA
// cycles over its own boxes) and an HBM stream (each CTA reads its own slice once).
static void private_regions(int nsm) {
  auto enc = get_encode();
  const int box_rows = 256, sbytes = box_rows * 128;
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * nsm);
  for (size_t total_mb : {size_t(48), size_t(4096)}) {
    const size_t bytes_total = total_mb << 20;
    const int per = (int)(bytes_total / sbytes / nsm);  // boxes per CTA
    const long long rows_total = (long long)per * nsm * box_rows;
    void* buf;
    cudaMalloc(&buf, (size_t)rows_total * 128);
    cudaMemset(buf, 1, (size_t)rows_total * 128);
    CUtensorMap tm;
    cuuint64_t dims[2] = {64, (cuuint64_t)rows_total};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int stages = 6, smem = stages * sbytes + 2 * stages * 8 + 2048;
    cudaFuncSetAttribute((void*)k_probe<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = total_mb > 1024 ? per : (64 << 20) / sbytes;  // HBM: each box once
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      k_probe<6><<<nsm, 64, smem>>>(tm, box_rows, iters, (int)0, cyc, per);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    const double bytes = (double)nsm * iters * sbytes;
    printf("private regions, %s (%zu MB): 32 KB boxes, 6 stages: %7.1f GB/s per SM, %6.2f TB/s chip (%s)\n",
           total_mb > 1024 ? "HBM stream" : "L2-resident", total_mb, bytes / nsm / (ms * 1e-3) / 1e9,
           bytes / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    cudaFree(buf);
  }
  cudaFree(cyc);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  private_regions(nsm);
  const int rows_total = 1 << 16;  // 64K rows x 128 B = 8 MB: L2-resident
  void* buf;
  cudaMalloc(&buf, (size_t)rows_total * 128);
  cudaMemset(buf, 1, (size_t)rows_total * 128);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * nsm);
  auto enc = get_encode();
  for (int box_rows : {64, 128, 256}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {64, (cuuint64_t)rows_total};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int stages : {2, 4, 6}) {
      const int sbytes = box_rows * 128;
      const int smem = stages * sbytes + 2 * stages * 8 + 2048;
      if (smem > 227 * 1024) continue;
      const int iters = (64 << 20) / sbytes;  // 64 MB per CTA
      void* kern = stages == 2 ? (void*)k_probe<2> : stages == 4 ? (void*)k_probe<4> : (void*)k_probe<6>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (stages == 2) k_probe<2><<<nsm, 64, smem>>>(tm, box_rows, iters, rows_total, cyc);
        if (stages == 4) k_probe<4><<<nsm, 64, smem>>>(tm, box_rows, iters, rows_total, cyc);
        if (stages == 6) k_probe<6><<<nsm, 64, smem>>>(tm, box_rows, iters, rows_total, cyc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)nsm * iters * sbytes;
      std::vector<unsigned long long> h(nsm);
      cudaMemcpy(h.data(), cyc, sizeof(unsigned long long) * nsm, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (auto v : h) mx = v > mx ? v : mx;
      printf("box %3d rows (%5d B)  stages %d: %7.1f GB/s per SM, %6.2f TB/s chip, %.1f B/clk per SM (%s)\n", box_rows,
             sbytes, stages, bytes / nsm / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e12,
             (double)iters * sbytes / (double)mx, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // 3-D boxes {64 cols, 256 rows, 2 tiles} = 64 KB per operation (two 32 KB SW128 tiles)
  {
    const int tiles = rows_total / 256;
    CUtensorMap tm;
    cuuint64_t dims[3] = {64, 256, (cuuint64_t)tiles};
    cuuint64_t strides[2] = {128, 256 * 128};
    cuuint32_t box[3] = {64, 256, 2};
    cuuint32_t es[3] = {1, 1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int bb = 65536;
    for (int stages : {2, 3}) {
      const int smem = stages * bb + 2 * stages * 8 + 2048;
      const int iters = (64 << 20) / bb;
      void* kern = stages == 2 ? (void*)k_probe3<2> : (void*)k_probe3<3>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (stages == 2) k_probe3<2><<<nsm, 64, smem>>>(tm, bb, iters, tiles, cyc);
        if (stages == 3) k_probe3<3><<<nsm, 64, smem>>>(tm, bb, iters, tiles, cyc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)nsm * iters * bb;
      printf("3-D box 64 KB (2 x 256 rows)  stages %d: %7.1f GB/s per SM, %6.2f TB/s chip (%s)\n", stages,
             bytes / nsm / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
