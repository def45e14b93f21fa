// C-ABI plumbing: error strings, device info, TMA map encoding, the generic
// dense tcgen05 GEMM entry point.
#include <cstring>
#include <vector>
#include <stdarg.h>
#include <string.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "epilogues.cuh"
#include "launch.cuh"
#ifdef MP_DIAG
#include "gemm2_sm100.cuh"
#endif

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

// SM partition for the two-stream (predictor || MoE layers) schedule: persistent grids of
// the grouped expert GEMMs and of the predictor GEMMs; 0 = every SM.
static int g_ffn_sms = 0, g_pred_sms = 0;
int ffn_grid() { return g_ffn_sms > 0 ? std::min(g_ffn_sms, num_sms()) : num_sms(); }
int pred_grid() { return g_pred_sms > 0 ? std::min(g_pred_sms, num_sms()) : num_sms(); }

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

// 2-D bf16 row-major store map for EpiStoreBf16Tma: box = [32 rows x 32 cols] (64 B rows), SWIZZLE_64B.
int make_tmap_bf16_store(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t row_stride_elems) {
  auto enc = get_encode();
  MP_REQUIRE(enc != nullptr, MP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  MP_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0 && (row_stride_elems * 2) % 16 == 0, MP_ERR_CONFIG,
             "tensor map: base and row stride must be 16-byte aligned");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_elems * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MP_REQUIRE(r == CUDA_SUCCESS, MP_ERR_CUDA, "cuTensorMapEncodeTiled(store) failed (%d)", (int)r);
  return MP_OK;
}

// 2-D fp32 row-major tensor map, box = [box_rows x 32 cols] (128 B), SWIZZLE_128B (TF32 operands).
int make_tmap_f32(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t row_stride_elems,
                  uint32_t box_rows) {
  auto enc = get_encode();
  MP_REQUIRE(enc != nullptr, MP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  MP_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0 && (row_stride_elems * 4) % 16 == 0, MP_ERR_CONFIG,
             "tensor map: base and row stride must be 16-byte aligned");
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_elems * 4};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  MP_REQUIRE(r == CUDA_SUCCESS, MP_ERR_CUDA, "cuTensorMapEncodeTiled(f32) failed (%d)", (int)r);
  return MP_OK;
}

}  // namespace mp

using namespace mp;

namespace mp {
// store_hint (TMA-store epilogue only): 0 none, 1 L2 evict_last (the output is consumed right
// away, e.g. the SRU u/f/r read by the scan: layer 102 -> 98 us), 2 evict_first
int gemm_bf16(const void* A, const void* B, void* C, int M, int N, int K, int c_dtype, int ldc, const float* bias,
              int act, int sig_from, int store_hint, void* stream, int grid_cap) {
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
  const int cap = grid_cap > 0 ? std::min(grid_cap, num_sms()) : num_sms();
  const int grid = units < cap ? units : cap;
#ifdef MP_DIAG
  const bool diag_lsu = getenv("MP_DIAG_LSU") != nullptr;  // diagnostic: st.global epilogue
  if (getenv("MP_DIAG_HINT")) store_hint = atoi(getenv("MP_DIAG_HINT"));
#else
  constexpr bool diag_lsu = false;
#endif
  if (c_dtype == 0 && bn == 256 && ldc > 0 && !diag_lsu) {  // bf16 tile through TMA bulk stores
    CUtensorMap tc;
    rc = make_tmap_bf16_store(&tc, C, M, N, ldc);
    if (rc) return rc;
    EpiStoreBf16Tma et{(__nv_bfloat16*)C, ldc, bias, act, sig_from, store_hint};
#ifdef MP_DIAG
    if (getenv("MP_DIAG_PAIR")) {
      CUtensorMap tb2;
      rc = make_tmap_bf16(&tb2, B, N, K, K, 128);
      if (rc) return rc;
      Dense2Sched s2{M, N / 256, K / 64, 256};
      const int units2 = cdiv(M, 2 * kBlockM) * (N / 256);
      return launch_gemm2<256, 6>(ta, tb2, s2, et, std::min(2 * units2, grid & ~1), st, &tc);
    }
#endif
    return launch_gemm<256, 4>(ta, tb, s, et, grid, st, &tc);
  }
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
}  // namespace mp

extern "C" int mp_gemm_bf16(const void* A, const void* B, void* C, int M, int N, int K, int c_dtype, int ldc,
                            const float* bias, int act, int sig_from, void* stream) {
  return gemm_bf16(A, B, C, M, N, K, c_dtype, ldc, bias, act, sig_from, 0, stream, 0);
}

extern "C" int mp_set_sm_partition(int ffn_sms, int predictor_sms) {
  MP_REQUIRE(ffn_sms >= 0 && predictor_sms >= 0, MP_ERR_CONFIG, "mp_set_sm_partition: negative SM count");
  g_ffn_sms = ffn_sms;
  g_pred_sms = predictor_sms;
  return MP_OK;
}

namespace mp {
__global__ void k_f32_to_bf16(const float4* __restrict__ x, uint2* __restrict__ y, size_t n4) {
  griddep_launch_dependents();
  griddep_wait();
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
  if (n4) MP_CUDA_TRY(launch_pdl(k_f32_to_bf16, dim3(grid), dim3(256), 0, (cudaStream_t)stream, (const float4*)x, (uint2*)y, n4));
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

// ---------------------------------------------------------------- graphs and events
// Stream capture / replay of a whole pipeline step, and timing events that stay
// valid inside captured graphs (recorded as external event nodes).
extern "C" int mp_graph_begin(void* stream) {
  MP_CUDA_TRY(cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeThreadLocal));
  return MP_OK;
}

extern "C" int mp_graph_end(void* stream, void** graph_exec) {
  cudaGraph_t g = nullptr;
  MP_CUDA_TRY(cudaStreamEndCapture((cudaStream_t)stream, &g));
  cudaGraphExec_t ex = nullptr;
  const cudaError_t e = cudaGraphInstantiateWithFlags(&ex, g, 0);
  cudaGraphDestroy(g);
  MP_CUDA_TRY(e);
  *graph_exec = (void*)ex;
  return MP_OK;
}

// mp_graph_end that also reports how many kernel nodes the captured graph holds (the
// launches one replay issues; memset / memcpy / event nodes are not counted).
extern "C" int mp_graph_end_counted(void* stream, void** graph_exec, int32_t* kernel_nodes) {
  cudaGraph_t g = nullptr;
  MP_CUDA_TRY(cudaStreamEndCapture((cudaStream_t)stream, &g));
  size_t n = 0;
  cudaError_t e = cudaGraphGetNodes(g, nullptr, &n);
  std::vector<cudaGraphNode_t> nodes(n);
  if (e == cudaSuccess && n) e = cudaGraphGetNodes(g, nodes.data(), &n);
  // kernel nodes of THIS library (namespace mp): collectives (NCCL) and torch copies captured
  // into the same graph are not counted
  int32_t k = 0;
  for (size_t i = 0; e == cudaSuccess && i < n; ++i) {
    cudaGraphNodeType t;
    e = cudaGraphNodeGetType(nodes[i], &t);
    if (e != cudaSuccess || t != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams kp = {};
    const char* name = nullptr;
    if (cudaGraphKernelNodeGetParams(nodes[i], &kp) == cudaSuccess && kp.func != nullptr &&
        cudaFuncGetName(&name, kp.func) == cudaSuccess && name != nullptr)
      k += std::strncmp(name, "_ZN2mp", 6) == 0 || std::strncmp(name, "mp::", 4) == 0 ||
           std::strncmp(name, "void mp::", 9) == 0;  // mangled or demangled
    else
      k += 1;  // name unavailable: count it
    (void)cudaGetLastError();
  }
  cudaGraphExec_t ex = nullptr;
  if (e == cudaSuccess) e = cudaGraphInstantiateWithFlags(&ex, g, 0);
  cudaGraphDestroy(g);
  MP_CUDA_TRY(e);
  *graph_exec = (void*)ex;
  if (kernel_nodes) *kernel_nodes = k;
  return MP_OK;
}

extern "C" int mp_graph_launch(void* graph_exec, void* stream) {
  MP_CUDA_TRY(cudaGraphLaunch((cudaGraphExec_t)graph_exec, (cudaStream_t)stream));
  return MP_OK;
}

extern "C" int mp_graph_destroy(void* graph_exec) {
  MP_CUDA_TRY(cudaGraphExecDestroy((cudaGraphExec_t)graph_exec));
  return MP_OK;
}

extern "C" int mp_event_create(void** ev) {
  cudaEvent_t e;
  MP_CUDA_TRY(cudaEventCreate(&e));
  *ev = (void*)e;
  return MP_OK;
}

extern "C" int mp_event_record(void* ev, void* stream) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  MP_CUDA_TRY(cudaStreamIsCapturing((cudaStream_t)stream, &cs));
  if (cs == cudaStreamCaptureStatusActive)
    MP_CUDA_TRY(cudaEventRecordWithFlags((cudaEvent_t)ev, (cudaStream_t)stream, cudaEventRecordExternal));
  else
    MP_CUDA_TRY(cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)stream));
  return MP_OK;
}

extern "C" int mp_event_elapsed_ms(void* a, void* b, float* ms) {
  MP_CUDA_TRY(cudaEventElapsedTime(ms, (cudaEvent_t)a, (cudaEvent_t)b));
  return MP_OK;
}

extern "C" int mp_event_destroy(void* ev) {
  MP_CUDA_TRY(cudaEventDestroy((cudaEvent_t)ev));
  return MP_OK;
}

// Keep [ptr, ptr + bytes) resident in L2 for kernels launched on `stream` (persisting
// access-policy window; bytes = 0 clears it). Used for the residual stream, which is
// re-read by every layer's router, gather and combine while 1.2 GB of weights stream by.
extern "C" int mp_l2_persist(void* ptr, size_t bytes, float hit_ratio, void* stream) {
  int dev = 0;
  MP_CUDA_TRY(cudaGetDevice(&dev));
  int max_win = 0, max_persist = 0;
  MP_CUDA_TRY(cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev));
  MP_CUDA_TRY(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
  const size_t win = std::min(bytes, (size_t)max_win);
  MP_CUDA_TRY(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min(win, (size_t)max_persist)));
  cudaStreamAttrValue attr = {};
  attr.accessPolicyWindow.base_ptr = ptr;
  attr.accessPolicyWindow.num_bytes = win;
  attr.accessPolicyWindow.hitRatio = win ? hit_ratio : 0.f;
  attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  MP_CUDA_TRY(cudaStreamSetAttribute((cudaStream_t)stream, cudaStreamAttributeAccessPolicyWindow, &attr));
  return MP_OK;
}


extern "C" int mp_enable_peer_access(int peer_device) {
  int dev = 0, can = 0;
  MP_CUDA_TRY(cudaGetDevice(&dev));
  if (peer_device == dev) return MP_OK;
  MP_CUDA_TRY(cudaDeviceCanAccessPeer(&can, dev, peer_device));
  MP_REQUIRE(can, MP_ERR_CONFIG, "mp_enable_peer_access: device %d cannot access device %d", dev, peer_device);
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    (void)cudaGetLastError();  // clear the sticky-free status
    return MP_OK;
  }
  MP_CUDA_TRY(e);
  return MP_OK;
}

#ifdef MP_DIAG
extern "C" __attribute__((visibility("default"))) int mp_debug_set_mma(int flags) {
  MP_CUDA_TRY(cudaMemcpyToSymbol(mp::g_diag_mma, &flags, sizeof(int)));
  return MP_OK;
}
extern "C" __attribute__((visibility("default"))) int mp_debug_set_epi(int flags) {
  MP_CUDA_TRY(cudaMemcpyToSymbol(mp::g_diag_epi, &flags, sizeof(int)));
  return MP_OK;
}

// Diagnostic build only: the dense CTA-pair (cta_group::2) GEMM on the same operands as
// mp_gemm_bf16 (bf16 out through TMA stores; ldc == 0: no stores), for single-vs-pair probes.
extern "C" __attribute__((visibility("default"))) int mp_debug_gemm_pair(const void* A, const void* B, void* C, int M,
                                                                         int N, int K, int ldc, void* stream) {
  MP_REQUIRE(M >= 1 && K % 64 == 0 && N % 256 == 0, MP_ERR_CONFIG, "mp_debug_gemm_pair: K%%64, N%%256");
  cudaStream_t st = (cudaStream_t)stream;
  CUtensorMap ta, tb, tc;
  int rc = make_tmap_bf16(&ta, A, M, K, K, kBlockM);
  if (!rc) rc = make_tmap_bf16(&tb, B, N, K, K, 128);
  if (rc) return rc;
  Dense2Sched s{M, N / 256, K / 64, 256};
  const int units = cdiv(M, 2 * kBlockM) * (N / 256);
  const int grid = std::min(2 * units, num_sms() & ~1);
  if (ldc > 0) {
    rc = make_tmap_bf16_store(&tc, C, M, N, ldc);
    if (rc) return rc;
    EpiStoreBf16Tma et{(__nv_bfloat16*)C, ldc, nullptr, 0, 0, 0};
    return launch_gemm2<256, 6>(ta, tb, s, et, grid, st, &tc);
  }
  EpiStoreBf16 e{(__nv_bfloat16*)C, 0, nullptr, 0, 0};
  return launch_gemm2<256, 6>(ta, tb, s, e, grid, st);
}
#endif
