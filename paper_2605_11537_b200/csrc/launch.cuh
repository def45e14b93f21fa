// Host-side helpers: TMA tensor-map encoding (driver entry point fetched at
// run time, no -lcuda link) and the persistent GEMM launcher.
#pragma once
#include <cudaTypedefs.h>

#include "common.cuh"
#include "gemm2_sm100.cuh"
#include "gemm_sm100.cuh"

namespace mp {

int num_sms();

int gemm_bf16(const void* A, const void* B, void* C, int M, int N, int K, int c_dtype, int ldc, const float* bias,
              int act, int sig_from, int store_hint, void* stream, int grid_cap = 0);
int ffn_grid();   // persistent grid of the grouped expert GEMMs (mp_set_sm_partition)
int pred_grid();  // persistent grid of the predictor GEMMs

// 2-D bf16 row-major [rows x cols] tensor map, box = [box_rows x 64 cols], SWIZZLE_128B.
int make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t row_stride_elems,
                   uint32_t box_rows);

int make_tmap_bf16_store(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t row_stride_elems);

int make_tmap_f32(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t row_stride_elems,
                  uint32_t box_rows);

template <int BN, int STAGES, class Sched, class Epi, class Kind = KindBF16, int ASTAGES = 0>
int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const Sched& sched, const Epi& epi, int grid,
                cudaStream_t st, const CUtensorMap* tc = nullptr) {
  auto kern = k_umma_gemm<BN, STAGES, Sched, Epi, Kind, ASTAGES>;
  const int smem = GemmSmem<BN, STAGES, ASTAGES>::kBytes;
  static_assert(GemmSmem<BN, STAGES, ASTAGES>::kBytes <= 232448, "GEMM shared memory over the sm_100 limit");
  static bool configured = false;  // one attribute call per instantiation
  if (!configured) {
    MP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  if (grid < 1) grid = 1;
  CUtensorMap none{};
  MP_CUDA_TRY(launch_pdl(kern, dim3(grid), dim3(kGemmThreads), smem, st, ta, tb, sched, epi, tc ? *tc : none));
  return MP_OK;
}

template <int BN, int STAGES, class Sched, class Epi>
int launch_gemm2(const CUtensorMap& ta, const CUtensorMap& tb, const Sched& sched, const Epi& epi, int grid,
                 cudaStream_t st, const CUtensorMap* tc = nullptr) {
  auto kern = k_umma_gemm2<BN, STAGES, Sched, Epi>;
  const int smem = Gemm2Smem<BN, STAGES>::kBytes;
  static bool configured = false;
  if (!configured) {
    MP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  if (grid < 2) grid = 2;
  grid &= ~1;  // whole clusters
  CUtensorMap none{};
  kern<<<grid, kGemmThreads, smem, st>>>(ta, tb, sched, epi, tc ? *tc : none);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

}  // namespace mp
