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
#include "gemm_mc_sm100.cuh"
#include "gemm_mt_sm100.cuh"
#include "launch.cuh"

#include <algorithm>
#include <cstdlib>

extern "C" int mp_ffn_down_bn(int dp);

namespace mp {

// xperm[row] = bf16(x[tok_of_row[row]]); one warp per row, 8-byte lanes. All of a
// row's loads are issued before the first store (row length known at compile time
// for the common widths).
template <int KQ>  // dp / 4 float4 per row; 0 = runtime
__global__ void k_gather_rows(const float* __restrict__ x, int T, int dp, const int32_t* __restrict__ tok_of_row,
                              __nv_bfloat16* __restrict__ xperm, int32_t* __restrict__ done) {
  griddep_launch_dependents();
  griddep_wait();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= T) return;
  const int t = __ldg(&tok_of_row[row]);
  if (done && lane == 0) done[row] = 0;  // GEMM2's per-piece consumption counters
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
                               cudaStream_t st, int32_t* done = nullptr) {
  const dim3 grid(cdiv(T * 32, 256)), block(256);
  if (dp == 768) return launch_pdl(k_gather_rows<192>, grid, block, 0, st, x, T, dp, tok_of_row, xperm, done);
  if (dp == 1024) return launch_pdl(k_gather_rows<256>, grid, block, 0, st, x, T, dp, tok_of_row, xperm, done);
  return launch_pdl(k_gather_rows<0>, grid, block, 0, st, x, T, dp, tok_of_row, xperm, done);
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
  static const bool bn192 = getenv("MP_GEMM1_BN192") != nullptr;  // A/B switch: 192-column GEMM1 units
  return (bn192 && Fp % 192 == 0) ? 192 : 256;
}

// GEMM2 column tile: 192 when it divides dp (d = 768: 4 slices of 192 with a 5-deep operand
// ring instead of 3 slices of 256 with a 4-deep ring -- GEMM2 142 -> 137.5 us per layer);
// MP_GEMM2_BN256=1 restores 256. The CTA-pair and multi-tile kernels always use 256.
extern "C" int mp_ffn_down_bn(int dp) {
  static const bool bn256 = getenv("MP_GEMM2_BN256") != nullptr;  // A/B switch
  if (!bn256 && dp % 192 == 0) return 192;
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

template <int BN, int STAGES, int CL, class Epi>
static int launch_gemm_mc(const CUtensorMap& ta, const CUtensorMap& tb, const SegMcSched<CL>& s, const Epi& e,
                          cudaStream_t st) {
  auto kern = k_umma_gemm_mc<BN, STAGES, CL, SegMcSched<CL>, Epi>;
  const int smem = GemmSmem<BN, STAGES>::kBytes;
  static bool configured = false;
  if (!configured) {
    MP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((num_sms() / CL) * CL);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  MP_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta, tb, s, e));
  return MP_OK;
}

// A-multicast cluster size for n_tiles slices (0: not applicable); MP_MC_CL overrides.
static int mc_cluster(int n_tiles) {
  static const int env = getenv("MP_MC_CL") ? atoi(getenv("MP_MC_CL")) : 0;
  if (env) return (n_tiles % env == 0) ? env : 0;
  for (int c : {4, 3, 2})
    if (n_tiles % c == 0) return c;
  return 0;
}

template <int BN, int STAGES, class Epi>
static int launch_seg_mc(int cl, const CUtensorMap& ta, const CUtensorMap& tb, const int32_t* piece_row,
                         const int32_t* piece_rows, const int32_t* exp_begin, int E, int n_tiles, int n_per_expert,
                         int kb, int tiled, const Epi& e, cudaStream_t st) {
  switch (cl) {
    case 2: return launch_gemm_mc<BN, STAGES, 2>(ta, tb, SegMcSched<2>{piece_row, piece_rows, exp_begin, E, n_tiles, BN, n_per_expert, kb, tiled}, e, st);
    case 3: return launch_gemm_mc<BN, STAGES, 3>(ta, tb, SegMcSched<3>{piece_row, piece_rows, exp_begin, E, n_tiles, BN, n_per_expert, kb, tiled}, e, st);
    case 4: return launch_gemm_mc<BN, STAGES, 4>(ta, tb, SegMcSched<4>{piece_row, piece_rows, exp_begin, E, n_tiles, BN, n_per_expert, kb, tiled}, e, st);
  }
  MP_REQUIRE(false, MP_ERR_CONFIG, "ffn: no multicast cluster size divides %d slices", n_tiles);
  return MP_ERR_CONFIG;
}

static int mt_single() {  // profiling switch: one tile per unit through the multi-tile kernel
  static const int v = getenv("MP_MT_SINGLE") != nullptr;
  return v;
}

template <class Epi>
static int launch_ffn_mt(const CUtensorMap& ta, const CUtensorMap& tb, const FfnMtSched& s, const Epi& e,
                         cudaStream_t st) {
  auto kern = k_ffn_mt<Epi>;
  const int smem = MtSmem::kBytes;
  static bool configured = false;
  if (!configured) {
    MP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  kern<<<num_sms(), kGemmThreads, smem, st>>>(ta, tb, s, e);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

// flags: bit 0 = pre-tiled weights, bit 1 = CTA-pair (cta_group::2) kernel over paired pieces,
//        bit 2 = multi-tile units (k_ffn_mt: two accumulator tiles per unit sharing A or B)
static int ffn_up(int T, int dp, int Fp, int E, const void* u, const int32_t* piece_row, const int32_t* piece_rows,
                  const int32_t* exp_begin, const __nv_bfloat16* xperm, __nv_bfloat16* hid, int flags,
                  cudaStream_t st) {
  // GEMM1: hid = relu(xperm . U_e^T)   [rows x Fp], BN = 256
  const int tiled = flags & 1, pair = (flags >> 1) & 1, mt = (flags >> 2) & 1;
  static const bool diag_nostore = getenv("MP_DIAG_NOSTORE") != nullptr;  // profiling switch only
  static const bool tma_store = getenv("MP_STG_EPILOGUE") == nullptr;     // A/B switch: st.global epilogue
  EpiStoreBf16 e{hid, diag_nostore ? 0 : Fp, nullptr, 1, 0};
  CUtensorMap ta, tb;
  int rc = make_tmap_bf16(&ta, xperm, T, dp, dp, kBlockM);
  if (rc) return rc;
  if (mt) {
    MP_REQUIRE(E <= kMtMaxE, MP_ERR_CONFIG, "ffn multi-tile mode: E <= %d", kMtMaxE);
    rc = tmap_b(&tb, u, E, Fp, dp, 256, tiled, 128);
    if (rc) return rc;
    FfnMtSched s{piece_row, piece_rows, exp_begin, E, Fp / 256, dp / 64, Fp, tiled, mt_single()};
    return launch_ffn_mt(ta, tb, s, e, st);
  }
  rc = tmap_b(&tb, u, E, Fp, dp, 256, tiled, pair ? 128 : 256);
  if (rc) return rc;
  if (pair) {
    Seg2Sched s{piece_row, piece_rows, exp_begin, E, Fp / 256, 256, Fp, dp / 64, tiled};
    if (tma_store && !diag_nostore) {  // H through TMA bulk stores, as in the 1-CTA kernel
      CUtensorMap tc;
      rc = make_tmap_bf16_store(&tc, hid, T, Fp, Fp);
      if (rc) return rc;
      EpiStoreBf16Tma et{hid, Fp, nullptr, 1, 0, getenv("MP_H_NO_EVICT_LAST") == nullptr};
      return launch_gemm2<256, 6>(ta, tb, s, et, num_sms() & ~1, st, &tc);
    }
    return launch_gemm2<256, 6>(ta, tb, s, e, num_sms() & ~1, st);
  }
  if (flags & 8) {  // A tile multicast across a cluster of CTAs computing consecutive slices
    const int cl = mc_cluster(Fp / 256);
    if (cl) return launch_seg_mc<256, 4>(cl, ta, tb, piece_row, piece_rows, exp_begin, E, Fp / 256, Fp, dp / 64, tiled, e, st);
  }
  if (tiled && mp_ffn_up_bn(Fp) == 192 && tma_store && !diag_nostore) {  // 5-deep ring, 16 slices per expert
    rc = tmap_b(&tb, u, E, Fp, dp, 192, tiled, 192);
    if (rc) return rc;
    SegSched s{piece_row, piece_rows, exp_begin, E, Fp / 192, 192, Fp, dp / 64, tiled, 0};
    CUtensorMap tc;
    rc = make_tmap_bf16_store(&tc, hid, T, Fp, Fp);
    if (rc) return rc;
    EpiStoreBf16Tma et{hid, Fp, nullptr, 1, 0, getenv("MP_H_NO_EVICT_LAST") == nullptr};
    return launch_gemm<192, 5>(ta, tb, s, et, ffn_grid(), st, &tc);
  }
  SegSched s{piece_row, piece_rows, exp_begin, E, Fp / 256, 256, Fp, dp / 64, tiled, 0};
  if (tma_store && !diag_nostore) {
    CUtensorMap tc;
    rc = make_tmap_bf16_store(&tc, hid, T, Fp, Fp);
    if (rc) return rc;
    // H is re-read by GEMM2 right after: keep it in L2 (GEMM1 151 -> 142 us, GEMM2 +3.5 us)
    static const int keep = getenv("MP_H_NO_EVICT_LAST") == nullptr;  // A/B switch
    EpiStoreBf16Tma et{hid, Fp, nullptr, 1, 0, keep};
    return launch_gemm<256, 4>(ta, tb, s, et, ffn_grid(), st, &tc);
  }
  return launch_gemm<256, 4>(ta, tb, s, e, ffn_grid(), st);
}

static int ffn_down(float* y, int T, int dp, int Fp, int E, const void* v, const int32_t* tok_of_row,
                    const int32_t* piece_row, const int32_t* piece_rows, const int32_t* exp_begin,
                    const __nv_bfloat16* hid, int flags, cudaStream_t st, int32_t* hdone = nullptr) {
  // GEMM2: y[tok] += hid . V_e^T   [rows x dp], scatter + residual epilogue
  const int tiled = flags & 1, pair = (flags >> 1) & 1, mt = (flags >> 2) & 1;
  const int bn = (pair || mt || (flags & 8)) ? 256 : mp_ffn_down_bn(dp);
  CUtensorMap ta, tb;
  int rc = make_tmap_bf16(&ta, hid, T, Fp, Fp, kBlockM);
  if (rc) return rc;
  if (mt) {
    MP_REQUIRE(bn == 256 && E <= kMtMaxE, MP_ERR_CONFIG, "ffn multi-tile mode: dp %% 256 == 0, E <= %d", kMtMaxE);
    rc = tmap_b(&tb, v, E, dp, Fp, bn, tiled, 128);
    if (rc) return rc;
    EpiScatterAdd ea{y, dp, tok_of_row, nullptr, nullptr, 0, 0, (flags >> 5) & 1};
    FfnMtSched s{piece_row, piece_rows, exp_begin, E, dp / 256, Fp / 64, dp, tiled, mt_single()};
    return launch_ffn_mt(ta, tb, s, ea, st);
  }
  rc = tmap_b(&tb, v, E, dp, Fp, bn, tiled, pair ? bn / 2 : bn);
  if (rc) return rc;
  EpiScatterAdd e{y, dp, tok_of_row, nullptr, nullptr, 0, 0, (flags >> 5) & 1};
  if (pair) {
    MP_REQUIRE(bn == 256, MP_ERR_CONFIG, "ffn pair mode needs dp %% 256 == 0");
    Seg2Sched s{piece_row, piece_rows, exp_begin, E, dp / bn, bn, dp, Fp / 64, tiled};
    return launch_gemm2<256, 6>(ta, tb, s, e, num_sms() & ~1, st);
  }
  if ((flags & 8) && bn == 256) {
    const int cl = mc_cluster(dp / 256);
    if (cl) return launch_seg_mc<256, 4>(cl, ta, tb, piece_row, piece_rows, exp_begin, E, dp / 256, dp, Fp / 64, tiled, e, st);
  }
  static const int rev = getenv("MP_GEMM2_FORWARD") ? 0 : 1;  // A/B switch: GEMM2 in GEMM1's unit order
  SegSched s{piece_row, piece_rows, exp_begin, E, dp / bn, bn, dp, Fp / 64, tiled, rev};
  if ((flags & 16) && hdone) {  // drop each piece's H from L2 after its last slice unit
    EpiScatterAdd ed{y, dp, tok_of_row, hdone, hid, Fp, dp / bn};
    if (bn == 256) return launch_gemm<256, 4>(ta, tb, s, ed, ffn_grid(), st);
    if (bn == 192) return launch_gemm<192, 5>(ta, tb, s, ed, ffn_grid(), st);
    if (bn == 128) return launch_gemm<128, 6>(ta, tb, s, ed, ffn_grid(), st);
    MP_REQUIRE(bn == 64, MP_ERR_CONFIG, "ffn_down: no kernel for BN %d", bn);
    return launch_gemm<64, 8>(ta, tb, s, ed, ffn_grid(), st);
  }
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
  int32_t* hdone = (int32_t*)((char*)hid + al(sizeof(__nv_bfloat16) * (size_t)T * Fp));                       \
  (void)xperm;                                                                                                  \
  (void)hid;                                                                                                    \
  (void)hdone;

extern "C" int mp_ffn_gather(const float* x, int T, int dp, int Fp, int E, const int32_t* tok_of_row, void* ws,
                             size_t ws_bytes, void* stream) {
  FFN_CHECKS();
  MP_CUDA_TRY(gather_rows(x, T, dp, tok_of_row, xperm, (cudaStream_t)stream, hdone));
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
                  (cudaStream_t)stream, hdone);
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

// ============================================================================
// Fused expert FFN: GEMM1 (relu) and GEMM2 (scatter + residual) of every piece in
// ONE persistent launch, the hidden activations H kept in an L2-resident ring of
// 128-row slots instead of a T x F HBM buffer (activation traffic costs ~54 us per
// layer at T = 16k when H goes through HBM: tools/ffn_ab.py, FFN_T=4096 vs 16384).
//
// Work list (static round-robin over CTAs, every role walks the same list): the
// pieces (expert order) are cut into chunks of f.chunk consecutive pieces, and
//   G1(0) G1(1) G2(0) G1(2) G2(1) ... G1(C-1) G2(C-2) G2(C-1)
// where inside a segment the units are expert-major, then BN slice, then piece --
// the order of the two-launch path, so CTAs running at the same time still share
// one weight tile through L2. Piece p's H rows live in ring slot p % (3 f.chunk)
// (3 chunks: the slot's previous occupant is two segments older).
// Dependencies point to EARLIER list positions only, so the persistent schedule
// cannot deadlock:
//   GEMM2(p) waits done1[p] == n_tiles1                (H of piece p complete)
//   GEMM1(p) waits done2[p - 3 f.chunk] == n_tiles2     (ring slot drained)
// Writers publish with __threadfence + atomicAdd after a named barrier of the
// epilogue warps; readers acquire, then fence.proxy.async before TMA reads.
// ============================================================================
namespace mp {

constexpr int kFfnChunkMax = 32;          // pieces per chunk (runtime f.chunk <= this)
constexpr int kFfnSlots = 3 * kFfnChunkMax;  // ring capacity (the schedule uses 3 * f.chunk slots)
constexpr int kFfnMaxE = 1024;

struct FfnFused {
  const int32_t* piece_row;
  const int32_t* piece_rows;
  const int32_t* exp_begin;
  const int32_t* tok_of_row;
  int E, nt1, nt2, kb1, kb2;  // F/256, d/256, d/64, F/64
  int F;
  __nv_bfloat16* ring;        // kSlots x 128 x F
  float* x;                   // residual stream (T x ldx)
  int ldx;
  int32_t* done1;
  int32_t* done2;
  int chunk;  // pieces per chunk; slots = 3 * chunk
  // shared-memory tables (set in the kernel prologue)
  const int* eb;    // exp_begin copy (E + 1)
  const int* seg;   // unit prefix over segments (nseg + 1)
  int P, nseg;
};

struct FUnit {
  int kind;  // 0 = GEMM1, 1 = GEMM2, -1 = empty
  int p, e, nt, rows, a_row, b_row;
};

// prologue (all threads): tables in smem; returns the number of units
__device__ int ffn_prepare(FfnFused& f, int* s_eb, int* s_seg) {
  for (int e = threadIdx.x; e <= f.E; e += blockDim.x) s_eb[e] = f.exp_begin[e];
  __syncthreads();
  const int P = s_eb[f.E];
  const int C = (P + f.chunk - 1) / f.chunk;
  const int nseg = 2 * C;
  if (threadIdx.x == 0) {
    int acc = 0, k = 0;
    auto push = [&](int c, int per) {
      s_seg[k++] = acc;
      acc += (min(P, (c + 1) * f.chunk) - c * f.chunk) * per;
    };
    for (int c = 0; c < C; ++c) {
      push(c, f.nt1);  // segment 2c: G1(c)
      if (c >= 1) push(c - 1, f.nt2);  // segment 2c + 1: G2(c - 1)
    }
    if (C >= 1) push(C - 1, f.nt2);
    s_seg[k] = acc;
  }
  __syncthreads();
  f.eb = s_eb;
  f.seg = s_seg;
  f.P = P;
  f.nseg = nseg;
  return nseg > 0 ? s_seg[nseg] : 0;
}

__device__ __forceinline__ FUnit ffn_unit(const FfnFused& f, int u) {
  int lo = 0, hi = f.nseg;  // segment: seg[lo] <= u < seg[lo + 1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (f.seg[mid] <= u) lo = mid; else hi = mid;
  }
  // segment 0 = G1(0); odd k = G1((k + 1) / 2) except the last; even k >= 2 = G2(k / 2 - 1)
  const bool last = lo == f.nseg - 1;
  const int kind = (lo == 0 || ((lo & 1) && !last)) ? 0 : 1;
  const int c = kind == 0 ? (lo + 1) / 2 : (last ? (f.nseg / 2 - 1) : lo / 2 - 1);
  const int nt_all = kind == 0 ? f.nt1 : f.nt2;
  const int a = c * f.chunk, b = min(f.P, a + f.chunk);
  const int local = u - f.seg[lo];
  // expert of the unit: largest e with (clamp(eb[e]) - a) * nt_all <= local
  int el = 0, eh = f.E;
  while (eh - el > 1) {
    const int mid = (el + eh) >> 1;
    const int q = (min(max(f.eb[mid], a), b) - a) * nt_all;
    if (q <= local) el = mid; else eh = mid;
  }
  const int pe0 = min(max(f.eb[el], a), b), pe1 = min(max(f.eb[el + 1], a), b);
  const int cnt = pe1 - pe0;
  const int rem = local - (pe0 - a) * nt_all;
  const int nt = rem / cnt;
  FUnit U;
  U.kind = kind;
  U.p = pe0 + (rem - nt * cnt);
  U.e = el;
  U.nt = nt;
  U.rows = __ldg(&f.piece_rows[U.p]);
  if (U.rows <= 0) {
    U.kind = -1;
    return U;
  }
  if (kind == 0) {
    U.a_row = __ldg(&f.piece_row[U.p]);
    U.b_row = (el * f.nt1 + nt) * f.kb1 * 256;
  } else {
    U.a_row = (U.p % (3 * f.chunk)) * kBlockM;
    U.b_row = (el * f.nt2 + nt) * f.kb2 * 256;
  }
  return U;
}

__device__ __forceinline__ int ld_acquire_gpu(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__global__ void __launch_bounds__(kGemmThreads, 1)
    k_ffn_fused(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmU,
                const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmV, FfnFused f_in) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  constexpr int BN = 256, STAGES = 4;
  using L = GemmSmem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint32_t* scratch_all = reinterpret_cast<uint32_t*>(smem + L::kScratchOffset);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmU);
    tma_prefetch(&tmH);
    tma_prefetch(&tmV);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 2 * BN);
  griddep_launch_dependents();
  griddep_wait();
  FfnFused f = f_in;
  const int nunits = ffn_prepare(f, reinterpret_cast<int*>(smem + L::kPrepOffset),
                                 reinterpret_cast<int*>(smem + L::kPrepOffset) + kFfnMaxE + 1);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      const uint64_t pol_w = policy_evict_first();
      uint32_t stage = 0, phase = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const FUnit U = ffn_unit(f, u);
        if (U.kind < 0) continue;
        const CUtensorMap* ta = U.kind == 0 ? &tmX : &tmH;
        const CUtensorMap* tb = U.kind == 0 ? &tmU : &tmV;
        const int nkb = U.kind == 0 ? f.kb1 : f.kb2;
        if (U.kind == 0) {
          const int prev = U.p - 3 * f.chunk;  // ring slot must be drained by the previous occupant
          if (prev >= 0 && f.piece_rows[prev] > 0)
            while (ld_acquire_gpu(&f.done2[prev]) < f.nt2) __nanosleep(64);
        } else {
          while (ld_acquire_gpu(&f.done1[U.p]) < f.nt1) __nanosleep(64);
          fence_proxy_async_global();  // H was written through the generic proxy
        }
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          mbar_arrive_expect_tx(&full[stage], L::kStageBytes);
          tma_load_2d(sa, ta, &full[stage], kb * kBlockK, U.a_row);
          tma_load_2d_hint(sb, tb, &full[stage], 0, U.b_row + kb * BN, pol_w);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(kBlockM, BN);
      uint32_t stage = 0, phase = 0, tile = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const FUnit U = ffn_unit(f, u);
        if (U.kind < 0) continue;
        const int nkb = U.kind == 0 ? f.kb1 : f.kb2;
        const uint32_t as = tile & 1, aph = (tile >> 1) & 1;
        mbar_wait(&tempty[as], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + as * BN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint8_t* sa = smem + stage * L::kStageBytes;
          const uint64_t adesc = sw128_kmajor_desc(smem_u32(sa));
          const uint64_t bdesc = sw128_kmajor_desc(smem_u32(sa + L::kABytes));
#pragma unroll
          for (int k = 0; k < 4; ++k) umma_bf16(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          umma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[as]);
        ++tile;
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue (2 warpgroups)
    const int q = warp & 3, half = (warp - 4) >> 2;
    const int r = q * 32 + lane;
    const int c0 = half * (BN / 2);
    uint32_t* scratch = scratch_all + (warp - 4) * L::kScratchWordsPerWarp;
    uint32_t tile = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      const FUnit U = ffn_unit(f, u);
      if (U.kind < 0) continue;
      const uint32_t as = tile & 1, aph = (tile >> 1) & 1;
      mbar_wait(&tfull[as], aph);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + as * BN + c0;
      if (U.kind == 0) {
        const Unit V{(U.p % (3 * f.chunk)) * kBlockM, U.rows, U.b_row, U.nt * BN};  // H rows -> ring slot
        EpiStoreBf16 e{f.ring, f.F, nullptr, 1, 0};
        e.template run<BN / 2>(V, 0, r, taddr, c0, nullptr, scratch);
      } else {
        // rows of this piece map to tokens through the piece's permuted rows
        const Unit V{U.a_row, U.rows, U.b_row, U.nt * BN};
        EpiScatterAdd e{f.x, f.ldx, f.tok_of_row + (f.piece_row[U.p] - U.a_row)};
        e.template run<BN / 2>(V, 0, r, taddr, c0, nullptr, scratch);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[as]);
      named_bar_sync(2, 32 * kEpiWarps);  // every epilogue warp finished its stores for this unit
      if (threadIdx.x == 128) {
        __threadfence();
        if (U.kind == 0) {
          fence_proxy_async_global();
          atomicAdd(&f.done1[U.p], 1);
        } else {
          atomicAdd(&f.done2[U.p], 1);
        }
      }
      ++tile;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * BN);
  }
#endif
}

}  // namespace mp

extern "C" size_t mp_ffn_fused_workspace_bytes(int T, int dp, int Fp, int max_pieces) {
  return al(sizeof(__nv_bfloat16) * (size_t)T * dp) + al(sizeof(__nv_bfloat16) * (size_t)kFfnSlots * kBlockM * Fp) +
         al(sizeof(int32_t) * 2 * (size_t)max_pieces);
}

extern "C" int mp_ffn_fused(float* x, int T, int dp, int Fp, int E, const void* u_tiled, const void* v_tiled,
                            const int32_t* tok_of_row, const int32_t* piece_row, const int32_t* piece_rows,
                            const int32_t* exp_begin, int max_pieces, void* ws, size_t ws_bytes, void* stream) {
  MP_REQUIRE(T >= 1 && E >= 1 && E <= kFfnMaxE && dp % 256 == 0 && Fp % 256 == 0, MP_ERR_CONFIG,
             "mp_ffn_fused: need E <= %d, dp %% 256 == 0 and Fp %% 256 == 0", kFfnMaxE);
  constexpr int kTable = GemmSmem<256, 4>::kPrepInts;
  static const int chunk = getenv("MP_FFN_CHUNK") ? std::max(1, std::min(kFfnChunkMax, atoi(getenv("MP_FFN_CHUNK"))))
                                                  : 32;  // A/B switch (8: 6.22, 16: 5.40, 32: 5.23 ms/step)
  MP_REQUIRE(2 * ((max_pieces + chunk - 1) / chunk) + 1 + kFfnMaxE + 1 <= kTable, MP_ERR_CONFIG,
             "mp_ffn_fused: piece capacity %d too large for the schedule table", max_pieces);
  MP_REQUIRE(ws_bytes >= mp_ffn_fused_workspace_bytes(T, dp, Fp, max_pieces), MP_ERR_CONFIG,
             "mp_ffn_fused: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* p = (char*)ws;
  __nv_bfloat16* xperm = (__nv_bfloat16*)p;
  p += al(sizeof(__nv_bfloat16) * (size_t)T * dp);
  __nv_bfloat16* ring = (__nv_bfloat16*)p;
  p += al(sizeof(__nv_bfloat16) * (size_t)kFfnSlots * kBlockM * Fp);
  int32_t* done = (int32_t*)p;
  MP_CUDA_TRY(cudaMemsetAsync(done, 0, sizeof(int32_t) * 2 * (size_t)max_pieces, st));
  MP_CUDA_TRY(gather_rows(x, T, dp, tok_of_row, xperm, st));
  MP_CUDA_TRY(cudaGetLastError());
  CUtensorMap tx, tu, th, tv;
  int rc = make_tmap_bf16(&tx, xperm, T, dp, dp, kBlockM);
  if (!rc) rc = make_tmap_bf16(&tu, u_tiled, (uint64_t)E * Fp * (dp / 64), 64, 64, 256);
  if (!rc) rc = make_tmap_bf16(&th, ring, (uint64_t)kFfnSlots * kBlockM, Fp, Fp, kBlockM);
  if (!rc) rc = make_tmap_bf16(&tv, v_tiled, (uint64_t)E * dp * (Fp / 64), 64, 64, 256);
  if (rc) return rc;
  FfnFused f{piece_row, piece_rows, exp_begin, tok_of_row, E, Fp / 256, dp / 256, dp / 64, Fp / 64, Fp, ring,
             x, dp, done, done + max_pieces, chunk, nullptr, nullptr, 0, 0};
  const int smem = GemmSmem<256, 4>::kBytes;
  static bool configured = false;
  if (!configured) {
    MP_CUDA_TRY(cudaFuncSetAttribute(k_ffn_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  k_ffn_fused<<<num_sms(), kGemmThreads, smem, st>>>(tx, tu, th, tv, f);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

// Diagnostics: per-CTA start/end %globaltimer (ns) of the last grouped-GEMM launch (n <= 1024).
extern "C" int mp_debug_cta_times(unsigned long long* t0, unsigned long long* t1, int n) {
  MP_REQUIRE(n >= 1 && n <= 1024, MP_ERR_CONFIG, "mp_debug_cta_times: n in [1, 1024]");
  MP_CUDA_TRY(cudaMemcpyFromSymbol(t0, mp::g_cta_t0, sizeof(unsigned long long) * n));
  MP_CUDA_TRY(cudaMemcpyFromSymbol(t1, mp::g_cta_t1, sizeof(unsigned long long) * n));
  return MP_OK;
}
