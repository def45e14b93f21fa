// Float64 GEMM for the predictor trainer (reference src/predictor.py:238-334: the SRU
// projections, the head logits and every weight / input gradient are numpy float64 matmuls).
//
//   C[M x N] = op(A)[M x K] . op(B)[K x N] + beta * C      (row-major, ld = row stride)
//   op(A) = A (ta = 0, A[m][k] at A[m*lda + k]) or A^T (ta = 1, A[k][m] at A[k*lda + m])
//   op(B) = B (tb = 0, B[k][n] at B[k*ldb + n]) or B^T (tb = 1, B[n][k] at B[n*ldb + k])
//
// 64 x 64 output tile per block of 256 threads (4 x 4 outputs each, DFMA), K staged through
// shared memory 16 at a time with the next slab prefetched into registers while the current
// one is multiplied. Off the inference path (training only); float64 like the reference.
#include "common.cuh"

namespace mp {

constexpr int kDT = 64;  // tile edge
constexpr int kDK = 16;  // K slab

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_dgemm(int M, int N, int K, const double* __restrict__ A, int lda,
                                               const double* __restrict__ B, int ldb, double beta,
                                               double* __restrict__ C, int ldc) {
  __shared__ double As[kDK][kDT + 1], Bs[kDK][kDT + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * kDT, n0 = blockIdx.x * kDT;
  double acc[4][4] = {};
  // loader mapping: 1024 elements per slab and operand, 4 per thread
  auto load = [&](int k0, double (&ra)[4], double (&rb)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = threadIdx.x + 256 * i;
      // A slab element (m, k): contiguous along k when !TA, along m when TA
      int m, k;
      if (TA) { k = idx >> 6; m = idx & 63; } else { m = idx >> 4; k = idx & 15; }
      const int gm = m0 + m, gk = k0 + k;
      ra[i] = (gm < M && gk < K) ? (TA ? A[(size_t)gk * lda + gm] : A[(size_t)gm * lda + gk]) : 0.0;
      int n, kb;
      if (TB) { n = idx >> 4; kb = idx & 15; } else { kb = idx >> 6; n = idx & 63; }
      const int gn = n0 + n, gkb = k0 + kb;
      rb[i] = (gn < N && gkb < K) ? (TB ? B[(size_t)gn * ldb + gkb] : B[(size_t)gkb * ldb + gn]) : 0.0;
    }
  };
  auto store = [&](const double (&ra)[4], const double (&rb)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = threadIdx.x + 256 * i;
      if (TA) As[idx >> 6][idx & 63] = ra[i]; else As[idx & 15][idx >> 4] = ra[i];
      if (TB) Bs[idx & 15][idx >> 4] = rb[i]; else Bs[idx >> 6][idx & 63] = rb[i];
    }
  };
  double ra[4], rb[4];
  load(0, ra, rb);
  for (int k0 = 0; k0 < K; k0 += kDK) {
    __syncthreads();
    store(ra, rb);
    __syncthreads();
    if (k0 + kDK < K) load(k0 + kDK, ra, rb);
#pragma unroll
    for (int k = 0; k < kDK; ++k) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[k][ty + 16 * i];
        b[i] = Bs[k][tx + 16 * i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= N) continue;
      double* c = C + (size_t)m * ldc + n;
      *c = beta == 0.0 ? acc[i][j] : acc[i][j] + beta * *c;
    }
  }
}

}  // namespace mp

using namespace mp;

extern "C" int mp_dgemm(int ta, int tb, int M, int N, int K, const double* A, int lda, const double* B, int ldb,
                        double beta, double* C, int ldc, void* stream) {
  MP_REQUIRE(M >= 0 && N >= 0 && K >= 0 && lda >= 0 && ldb >= 0 && ldc >= 0, MP_ERR_CONFIG,
             "mp_dgemm: bad sizes M=%d N=%d K=%d", M, N, K);
  MP_REQUIRE(ldc >= N && lda >= (ta ? M : K) && ldb >= (tb ? K : N), MP_ERR_CONFIG, "mp_dgemm: leading dimensions");
  if (M == 0 || N == 0) return MP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 grid(cdiv(N, kDT), cdiv(M, kDT)), block(256);
  if (!ta && !tb) k_dgemm<false, false><<<grid, block, 0, st>>>(M, N, K, A, lda, B, ldb, beta, C, ldc);
  else if (!ta && tb) k_dgemm<false, true><<<grid, block, 0, st>>>(M, N, K, A, lda, B, ldb, beta, C, ldc);
  else if (ta && !tb) k_dgemm<true, false><<<grid, block, 0, st>>>(M, N, K, A, lda, B, ldb, beta, C, ldc);
  else k_dgemm<true, true><<<grid, block, 0, st>>>(M, N, K, A, lda, B, ldb, beta, C, ldc);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}
