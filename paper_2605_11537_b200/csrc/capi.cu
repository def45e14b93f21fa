// C-ABI plumbing: error strings, device info, TMA map encoding, the generic
// dense tcgen05 GEMM entry point and the replica copy.
#include <stdarg.h>
#include <string.h>

#include <algorithm>
#include <mutex>

#include "epilogues.cuh"
#include "launch.cuh"

static thread_local char g_err[1024] = "";

extern "C" void mp_set_last_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char* mp_last_error(void) { return g_err; }
extern "C" int mp_abi_version(void) { return MP_ABI_VERSION; }

extern "C" int mp_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  int dev = 0;
  MP_CUDA_TRY(cudaGetDevice(&dev));
  cudaDeviceProp p;
  MP_CUDA_TRY(cudaGetDeviceProperties(&p, dev));
  if (sm_count) *sm_count = p.multiProcessorCount;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  return MP_OK;
}

namespace mp {

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t row_stride_elems,
                   uint32_t box_rows) {
  auto enc = get_encode();
  MP_REQUIRE(enc != nullptr, MP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  MP_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0 && (row_stride_elems * 2) % 16 == 0, MP_ERR_CONFIG,
             "tensor map: base and row stride must be 16-byte aligned");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_elems * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MP_REQUIRE(r == CUDA_SUCCESS, MP_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) rows=%llu cols=%llu", (int)r,
             (unsigned long long)rows, (unsigned long long)cols);
  return MP_OK;
}

}  // namespace mp

using namespace mp;

extern "C" int mp_gemm_bf16(const void* A, const void* B, void* C, int M, int N, int K, int c_dtype, int ldc,
                            const float* bias, int act, int sig_from, void* stream) {
  MP_REQUIRE(M >= 1 && N >= 64 && K >= 64 && K % 64 == 0 && N % 64 == 0, MP_ERR_CONFIG,
             "mp_gemm_bf16: need K%%64==0, N%%64==0 (M=%d N=%d K=%d)", M, N, K);
  MP_REQUIRE(ldc >= N || ldc == 0, MP_ERR_CONFIG, "mp_gemm_bf16: ldc < N");
  cudaStream_t st = (cudaStream_t)stream;
  const int bn = (N % 256 == 0) ? 256 : (N % 128 == 0 ? 128 : 64);
  CUtensorMap ta, tb;
  int rc = make_tmap_bf16(&ta, A, M, K, K, kBlockM);
  if (rc) return rc;
  rc = make_tmap_bf16(&tb, B, N, K, K, bn);
  if (rc) return rc;
  DenseSched s{M, N / bn, K / 64, bn};
  const int units = cdiv(M, kBlockM) * (N / bn);
  const int grid = units < num_sms() ? units : num_sms();
  if (c_dtype == 0) {
    EpiStoreBf16 e{(__nv_bfloat16*)C, ldc, bias, act, sig_from};
    if (bn == 256) return launch_gemm<256, 4>(ta, tb, s, e, grid, st);
    if (bn == 128) return launch_gemm<128, 6>(ta, tb, s, e, grid, st);
    return launch_gemm<64, 8>(ta, tb, s, e, grid, st);
  } else {
    EpiStoreF32 e{(float*)C, ldc, bias, act, sig_from};
    if (bn == 256) return launch_gemm<256, 4>(ta, tb, s, e, grid, st);
    if (bn == 128) return launch_gemm<128, 6>(ta, tb, s, e, grid, st);
    return launch_gemm<64, 8>(ta, tb, s, e, grid, st);
  }
}

namespace mp {
__global__ void k_f32_to_bf16(const float4* __restrict__ x, uint2* __restrict__ y, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = x[i];
    y[i] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
  }
}
}  // namespace mp

extern "C" int mp_f32_to_bf16(const float* x, void* y, size_t n, void* stream) {
  MP_REQUIRE(n % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0, MP_ERR_CONFIG,
             "mp_f32_to_bf16: n %% 4 != 0 or misaligned");
  const size_t n4 = n / 4;
  const int grid = (int)std::min<size_t>((n4 + 255) / 256, (size_t)num_sms() * 8);
  if (n4) k_f32_to_bf16<<<grid, 256, 0, (cudaStream_t)stream>>>((const float4*)x, (uint2*)y, n4);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_replica_copy(void* dst, const void* src, size_t bytes, void* stream) {
  MP_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return MP_OK;
}
