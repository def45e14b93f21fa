// K6 gather + K7 grouped expert FFN (tcgen05) + K8 residual combine fused into
// the GEMM2 epilogue.
//
// Reference: expert_forward  v @ relu(u @ x)   (src/router_oracle.py:101-111)
//            _run_layers     stream[t] = stream[t] + delta (src/router_oracle.py:127-134)
// Weights keep the reference layouts, which are already K-major for the B
// operand: expert_u (E, F, d) -> rows e*F + f, K = d; expert_v (E, d, F) ->
// rows e*d + j, K = F (zero padded to dp % 64 == 0, Fp % 256 == 0).
// Rows are the slot-grouped permutation from mp_exec_map, so every replica
// segment is a contiguous run of A rows; replicas of one expert alias the same
// weight rows (no copies on one GPU).
#include "epilogues.cuh"
#include "gemm2_sm100.cuh"
#include "launch.cuh"

#include <algorithm>

extern "C" int mp_ffn_down_bn(int dp);

namespace mp {

// xperm[row] = bf16(x[tok_of_row[row]]); one warp per row, 8-byte lanes. All of a
// row's loads are issued before the first store (row length known at compile time
// for the common widths).
template <int KQ>  // dp / 4 float4 per row; 0 = runtime
__global__ void k_gather_rows(const float* __restrict__ x, int T, int dp, const int32_t* __restrict__ tok_of_row,
                              __nv_bfloat16* __restrict__ xperm) {
  griddep_launch_dependents();
  griddep_wait();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const int t = __ldg(&tok_of_row[row]);
  const float4* src = reinterpret_cast<const float4*>(x + (size_t)t * dp);
  uint2* dst = reinterpret_cast<uint2*>(xperm + (size_t)row * dp);
  if constexpr (KQ > 0) {
    constexpr int N = (KQ + 31) / 32;
    float4 v[N];
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (lane + 32 * i < KQ) v[i] = __ldg(&src[lane + 32 * i]);
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (lane + 32 * i < KQ) dst[lane + 32 * i] = make_uint2(pack_bf16x2(v[i].x, v[i].y), pack_bf16x2(v[i].z, v[i].w));
  } else {
    for (int k = lane; k < dp / 4; k += 32) {
      const float4 v = __ldg(&src[k]);
      dst[k] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
    }
  }
}

static cudaError_t gather_rows(const float* x, int T, int dp, const int32_t* tok_of_row, __nv_bfloat16* xperm,
                               cudaStream_t st) {
  const dim3 grid(cdiv(T * 32, 256)), block(256);
  if (dp == 768) return launch_pdl(k_gather_rows<192>, grid, block, 0, st, x, T, dp, tok_of_row, xperm);
  if (dp == 1024) return launch_pdl(k_gather_rows<256>, grid, block, 0, st, x, T, dp, tok_of_row, xperm);
  return launch_pdl(k_gather_rows<0>, grid, block, 0, st, x, T, dp, tok_of_row, xperm);
}

static inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

// dst[g][nt][kb][r][c] = src[g*N + nt*BN + r][kb*64 + c], 16-byte granules.
__global__ void k_tile_kmajor(const uint4* __restrict__ src, uint4* __restrict__ dst, int G, int N, int K, int BN) {
  griddep_launch_dependents();
  griddep_wait();
  const size_t total = (size_t)G * N * K / 8;
  const int kq = K / 8;  // 16-byte granules per source row
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t row = i / kq;
    const int gk = (int)(i - row * kq);  // granule within the row
    const int g = (int)(row / N), n = (int)(row - (size_t)g * N);
    const int nt = n / BN, r = n - nt * BN, kb = gk / 8, c = gk - kb * 8;
    const size_t o = ((((size_t)g * (N / BN) + nt) * (K / 64) + kb) * BN + r) * 8 + c;
    dst[o] = src[i];
  }
}

}  // namespace mp

using namespace mp;

extern "C" int mp_ffn_up_bn(int Fp) {
  (void)Fp;
  return 256;  // GEMM1 column tile (a 192-column variant measured slower)
}

// GEMM2 column tile of the single-CTA kernel: 192 when it divides dp (d = 768: 4 slices of
// 192 with a 5-deep operand ring instead of 3 slices of 256 with a 4-deep ring -- GEMM2
// 142 -> 137.5 us per layer). The CTA-pair kernels read V tiled at 256 (flags bit 6).
extern "C" int mp_ffn_down_bn(int dp) {
  if (dp % 192 == 0) return 192;
  return (dp % 256 == 0) ? 256 : (dp % 128 == 0 ? 128 : 64);
}

extern "C" int mp_tile_kmajor(const void* src, void* dst, int G, int N, int K, int BN, void* stream) {
  MP_REQUIRE(G >= 1 && N % BN == 0 && K % 64 == 0 && (BN == 64 || BN == 128 || BN == 192 || BN == 256), MP_ERR_CONFIG,
             "mp_tile_kmajor: need N %% BN == 0, K %% 64 == 0 (N=%d K=%d BN=%d)", N, K, BN);
  const size_t total = (size_t)G * N * K / 8;
  const int grid = (int)std::min<size_t>((total + 255) / 256, (size_t)num_sms() * 16);
  k_tile_kmajor<<<grid, 256, 0, (cudaStream_t)stream>>>((const uint4*)src, (uint4*)dst, G, N, K, BN);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" size_t mp_ffn_workspace_bytes(int T, int dp, int Fp) {
  return al(sizeof(__nv_bfloat16) * (size_t)T * dp) + al(sizeof(__nv_bfloat16) * (size_t)T * Fp) +
         al(sizeof(int32_t) * (size_t)T);
}

static int tmap_b(CUtensorMap* tb, const void* w, int E, int N, int K, int bn, int tiled, int box_rows) {
  if (tiled) return make_tmap_bf16(tb, w, (uint64_t)E * N * (K / 64), 64, 64, box_rows);
  return make_tmap_bf16(tb, w, (uint64_t)E * N, K, K, box_rows);
}

// flags: bit 0 = pre-tiled weights (mp_tile_kmajor), bit 1 = CTA-pair (cta_group::2) kernels over
//        paired pieces (split_m = 3 piece layout), bit 5 = GEMM2 stores its rows (y[row] = ...)
//        instead of the residual add, bit 6 = V tiled with 256-column slices (the pair layout)
static int ffn_up(int T, int dp, int Fp, int E, const void* u, const int32_t* piece_row, const int32_t* piece_rows,
                  const int32_t* exp_begin, const __nv_bfloat16* xperm, __nv_bfloat16* hid, int flags,
                  cudaStream_t st, const int32_t* piece_wbase = nullptr, int W = 0) {
  // GEMM1: hid = relu(xperm . U_e^T)   [rows x Fp], BN = 256, H written by TMA bulk stores
  // with an L2 evict_last hint (GEMM2 re-reads it right away: GEMM1 151 -> 142 us)
  const int tiled = flags & 1, pair = (flags >> 1) & 1;
  CUtensorMap ta, tb, tc;
  int rc = make_tmap_bf16(&ta, xperm, T, dp, dp, kBlockM);
  if (!rc) rc = tmap_b(&tb, u, piece_wbase ? W : E, Fp, dp, 256, tiled, pair ? 128 : 256);
  if (!rc) rc = make_tmap_bf16_store(&tc, hid, T, Fp, Fp);
  if (rc) return rc;
  EpiStoreBf16Tma et{hid, Fp, nullptr, 1, 0, 1};
  if (pair) {
    Seg2Sched s{piece_row, piece_rows, exp_begin, E, Fp / 256, 256, Fp, dp / 64, tiled};
    return launch_gemm2<256, 6>(ta, tb, s, et, num_sms() & ~1, st, &tc);
  }
  SegSched s{piece_row, piece_rows, exp_begin, E, Fp / 256, 256, Fp, dp / 64, tiled, 0};
  s.piece_wbase = piece_wbase;
  return launch_gemm<256, 4>(ta, tb, s, et, ffn_grid(), st, &tc);
}

static int ffn_down(float* y, int T, int dp, int Fp, int E, const void* v, const int32_t* tok_of_row,
                    const int32_t* piece_row, const int32_t* piece_rows, const int32_t* exp_begin,
                    const __nv_bfloat16* hid, int flags, cudaStream_t st, const int32_t* piece_wbase = nullptr,
                    int W = 0, float* const* peer_x = nullptr, int peer_T = 1) {
  // GEMM2: y[tok] += hid . V_e^T   [rows x dp], scatter + residual epilogue
  const int tiled = flags & 1, pair = (flags >> 1) & 1;
  const int bn = (pair || (flags & 64)) ? 256 : mp_ffn_down_bn(dp);
  MP_REQUIRE(dp % bn == 0, MP_ERR_CONFIG, "ffn_down: dp=%d not a multiple of the V tile %d", dp, bn);
  CUtensorMap ta, tb;
  int rc = make_tmap_bf16(&ta, hid, T, Fp, Fp, kBlockM);
  if (!rc) rc = tmap_b(&tb, v, piece_wbase ? W : E, dp, Fp, bn, tiled, pair ? bn / 2 : bn);
  if (rc) return rc;
  EpiScatterAdd e{y, dp, tok_of_row, (flags >> 5) & 1, peer_x, peer_T};
  if (pair) {
    Seg2Sched s{piece_row, piece_rows, exp_begin, E, dp / bn, bn, dp, Fp / 64, tiled};
    return launch_gemm2<256, 6>(ta, tb, s, e, num_sms() & ~1, st);
  }
  // units walked backwards: the H rows GEMM1 wrote last are still in L2
  SegSched s{piece_row, piece_rows, exp_begin, E, dp / bn, bn, dp, Fp / 64, tiled, 1};
  s.piece_wbase = piece_wbase;
  if (bn == 256) return launch_gemm<256, 4>(ta, tb, s, e, ffn_grid(), st);
  if (bn == 192) return launch_gemm<192, 5>(ta, tb, s, e, ffn_grid(), st);
  if (bn == 128) return launch_gemm<128, 6>(ta, tb, s, e, ffn_grid(), st);
  MP_REQUIRE(bn == 64, MP_ERR_CONFIG, "ffn_down: no kernel for BN %d", bn);
  return launch_gemm<64, 8>(ta, tb, s, e, ffn_grid(), st);
}

#define FFN_CHECKS()                                                                                            \
  MP_REQUIRE(T >= 1 && E >= 1, MP_ERR_CONFIG, "ffn: bad T/E");                                                  \
  MP_REQUIRE(dp % 64 == 0 && Fp % 256 == 0, MP_ERR_CONFIG, "ffn: need dp%%64==0 and Fp%%256==0 (dp=%d Fp=%d)", dp, \
             Fp);                                                                                               \
  MP_REQUIRE(ws_bytes >= mp_ffn_workspace_bytes(T, dp, Fp), MP_ERR_CONFIG, "ffn: workspace too small");          \
  __nv_bfloat16* xperm = (__nv_bfloat16*)ws;                                                                    \
  __nv_bfloat16* hid = (__nv_bfloat16*)((char*)ws + al(sizeof(__nv_bfloat16) * (size_t)T * dp));                \
  (void)xperm;                                                                                                  \
  (void)hid;

extern "C" int mp_ffn_gather(const float* x, int T, int dp, int Fp, int E, const int32_t* tok_of_row, void* ws,
                             size_t ws_bytes, void* stream) {
  FFN_CHECKS();
  MP_CUDA_TRY(gather_rows(x, T, dp, tok_of_row, xperm, (cudaStream_t)stream));
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_ffn_up(int T, int dp, int Fp, int E, const void* u, int flags, const int32_t* piece_row,
                         const int32_t* piece_rows, const int32_t* exp_begin, void* ws, size_t ws_bytes,
                         void* stream) {
  FFN_CHECKS();
  return ffn_up(T, dp, Fp, E, u, piece_row, piece_rows, exp_begin, xperm, hid, flags, (cudaStream_t)stream);
}

extern "C" int mp_ffn_down(float* y, int T, int dp, int Fp, int E, const void* v, int flags,
                           const int32_t* tok_of_row, const int32_t* piece_row, const int32_t* piece_rows,
                           const int32_t* exp_begin, void* ws, size_t ws_bytes, void* stream) {
  FFN_CHECKS();
  return ffn_down(y, T, dp, Fp, E, v, tok_of_row, piece_row, piece_rows, exp_begin, hid, flags,
                  (cudaStream_t)stream);
}

// Expert parallelism over peer memory: row r's result is ADDED into rank (dst_of_row[r] / T_home)'s
// residual stream, token dst_of_row[r] % T_home, through the peer pointers peer_x (device array of
// G float*, NVLink P2P addresses) -- the combine fused into GEMM2's epilogue, no return all-to-all.
extern "C" int mp_ffn_down_peer(float* const* peer_x, int T_home, int T, int dp, int Fp, int E, const void* v,
                                int flags, const int32_t* dst_of_row, const int32_t* piece_row,
                                const int32_t* piece_rows, const int32_t* exp_begin, void* ws, size_t ws_bytes,
                                void* stream) {
  FFN_CHECKS();
  MP_REQUIRE(peer_x != nullptr && T_home >= 1 && !(flags & 2) && !(flags & 32), MP_ERR_CONFIG,
             "mp_ffn_down_peer: needs the peer table, T_home >= 1, single-CTA kernels and residual adds");
  return ffn_down(nullptr, T, dp, Fp, E, v, dst_of_row, piece_row, piece_rows, exp_begin, hid, flags,
                  (cudaStream_t)stream, nullptr, 0, peer_x, T_home);
}

// Physical replicas: B operand rows of piece p come from weight slot piece_wbase[p] of a pool of W
// expert-sized slots (same pre-tiled layout), single-CTA kernels only.
extern "C" int mp_ffn_up_pool(int T, int dp, int Fp, int E, int W, const void* pool_u, int flags,
                              const int32_t* piece_row, const int32_t* piece_rows, const int32_t* exp_begin,
                              const int32_t* piece_wbase, void* ws, size_t ws_bytes, void* stream) {
  FFN_CHECKS();
  MP_REQUIRE((flags & 1) && !(flags & 2) && piece_wbase != nullptr && W >= 1, MP_ERR_CONFIG,
             "mp_ffn_up_pool: needs pre-tiled single-CTA weights and a piece -> slot table");
  return ffn_up(T, dp, Fp, E, pool_u, piece_row, piece_rows, exp_begin, xperm, hid, flags, (cudaStream_t)stream,
                piece_wbase, W);
}

extern "C" int mp_ffn_down_pool(float* y, int T, int dp, int Fp, int E, int W, const void* pool_v, int flags,
                                const int32_t* tok_of_row, const int32_t* piece_row, const int32_t* piece_rows,
                                const int32_t* exp_begin, const int32_t* piece_wbase, void* ws, size_t ws_bytes,
                                void* stream) {
  FFN_CHECKS();
  MP_REQUIRE((flags & 1) && !(flags & 2) && piece_wbase != nullptr && W >= 1, MP_ERR_CONFIG,
             "mp_ffn_down_pool: needs pre-tiled single-CTA weights and a piece -> slot table");
  return ffn_down(y, T, dp, Fp, E, pool_v, tok_of_row, piece_row, piece_rows, exp_begin, hid, flags,
                  (cudaStream_t)stream, piece_wbase, W);
}

extern "C" int mp_moe_ffn(const float* x, float* y, int T, int dp, int Fp, int E, const void* u, const void* v,
                          const int32_t* tok_of_row, const int32_t* piece_row, const int32_t* piece_rows,
                          const int32_t* exp_begin, void* ws, size_t ws_bytes, void* stream) {
  FFN_CHECKS();
  cudaStream_t st = (cudaStream_t)stream;
  MP_CUDA_TRY(gather_rows(x, T, dp, tok_of_row, xperm, st));
  MP_CUDA_TRY(cudaGetLastError());
  int rc = ffn_up(T, dp, Fp, E, u, piece_row, piece_rows, exp_begin, xperm, hid, 0, st);
  if (rc) return rc;
  return ffn_down(y, T, dp, Fp, E, v, tok_of_row, piece_row, piece_rows, exp_begin, hid, 0, st);
}

// Diagnostics: per-CTA start/end %globaltimer (ns) of the last grouped-GEMM launch (n <= 1024).
extern "C" int mp_debug_cta_times(unsigned long long* t0, unsigned long long* t1, int n) {
  MP_REQUIRE(n >= 1 && n <= 1024, MP_ERR_CONFIG, "mp_debug_cta_times: n in [1, 1024]");
  MP_CUDA_TRY(cudaMemcpyFromSymbol(t0, mp::g_cta_t0, sizeof(unsigned long long) * n));
  MP_CUDA_TRY(cudaMemcpyFromSymbol(t1, mp::g_cta_t1, sizeof(unsigned long long) * n));
  return MP_OK;
}

#ifdef MP_DIAG
extern "C" __attribute__((visibility("default"))) int mp_debug_unit_trace(unsigned long long* out, int n) {
  MP_REQUIRE(n >= 1 && n <= mp::kTraceUnits, MP_ERR_CONFIG, "mp_debug_unit_trace: n in [1, %d]", mp::kTraceUnits);
  for (int k = 0; k < 4; ++k)
    MP_CUDA_TRY(cudaMemcpyFromSymbol(out + (size_t)k * n, mp::g_unit_t, sizeof(unsigned long long) * n,
                                     sizeof(unsigned long long) * mp::kTraceUnits * k));
  return MP_OK;
}
#endif
