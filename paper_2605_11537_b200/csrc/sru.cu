// K1 (SRU projection GEMM on tcgen05 with fused bias+sigmoid epilogue),
// K2 (SRU recurrence as a chunked associative scan) and K3 (per-layer head
// argmax = predicted expert).
//
// Reference: sru_cell / sru_forward (src/predictor.py:157-195), vectorised form
// _forward_stack (src/predictor.py:238-254); predict_batch (src/predictor.py:212-223).
// The recurrence c_t = f_t c_{t-1} + (1 - f_t) u_t is first-order linear, so a
// chunk of tokens composes into one affine map c_out = A c_in + B
// (A = prod f, B = chunk scan from 0). Pass A computes (A, B) per
// (chunk, channel), pass B scans the chunk carries per channel, pass C replays
// the chunk from its carry and applies the highway output
// h_t = r_t tanh(c_t) + (1 - r_t) x_t. All channel loads are bf16x2 / float2
// vectors, consecutive lanes = consecutive channels (coalesced rows).
#include "epilogues.cuh"
#include "launch.cuh"

namespace mp {

constexpr int kScanChunk = 64;   // tokens per scan chunk
constexpr int kScanThreads = 128;  // channel pairs per block

__device__ __forceinline__ float2 ld_bf16x2(const __nv_bfloat16* p) {
  const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(p);
  return __bfloat1622float2(v);
}

// pass A: grid (cdiv(d/2, 128), nch). ufr row = [u | f | r], 3d bf16.
__global__ void k_scan_aggregate(const __nv_bfloat16* __restrict__ ufr, int T, int d, float* __restrict__ aggA,
                                 float* __restrict__ aggB) {
  const int cp = blockIdx.x * kScanThreads + threadIdx.x;  // channel pair
  if (2 * cp >= d) return;
  const int ch = blockIdx.y;
  const int t0 = ch * kScanChunk, t1 = min(T, t0 + kScanChunk);
  float a0 = 1.f, a1 = 1.f, b0 = 0.f, b1 = 0.f;
  const __nv_bfloat16* p = ufr + (size_t)t0 * 3 * d + 2 * cp;
#pragma unroll 8
  for (int t = t0; t < t1; ++t, p += 3 * d) {
    const float2 u = ld_bf16x2(p), f = ld_bf16x2(p + d);
    b0 = f.x * b0 + (1.f - f.x) * u.x;
    b1 = f.y * b1 + (1.f - f.y) * u.y;
    a0 *= f.x;
    a1 *= f.y;
  }
  const size_t o = (size_t)ch * d + 2 * cp;
  *reinterpret_cast<float2*>(aggA + o) = make_float2(a0, a1);
  *reinterpret_cast<float2*>(aggB + o) = make_float2(b0, b1);
}

// pass B: carry_in[ch] per channel (c_0 = 0 at the start of every batch, or the
// carry of a preceding shard). Loads are hoisted 16 chunks at a time so the
// serial chain only pays FMA latency, not memory latency.
__global__ void k_scan_carry(const float* __restrict__ aggA, const float* __restrict__ aggB, int nch, int d,
                             const float* __restrict__ c0, float* __restrict__ carry) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  float run = c0 ? c0[c] : 0.f;
  int ch = 0;
  for (; ch + 16 <= nch; ch += 16) {
    float a[16], b[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      a[i] = __ldg(&aggA[(size_t)(ch + i) * d + c]);
      b[i] = __ldg(&aggB[(size_t)(ch + i) * d + c]);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      carry[(size_t)(ch + i) * d + c] = run;
      run = fmaf(a[i], run, b[i]);
    }
  }
  for (; ch < nch; ++ch) {
    const size_t o = (size_t)ch * d + c;
    carry[o] = run;
    run = fmaf(aggA[o], run, aggB[o]);
  }
}

// tanh via one exp + one reciprocal (|abs err| ~1e-7; the reference uses np.tanh in f64)
__device__ __forceinline__ float fast_tanh(float x) {
  const float e = __expf(2.f * x);
  return 1.f - 2.f * __frcp_rn(1.f + e);
}

// pass C: replay each chunk from its carry; h = r tanh(c) + (1 - r) x.
__global__ void k_scan_output(const __nv_bfloat16* __restrict__ ufr, const float* __restrict__ x, int T, int d,
                              const float* __restrict__ carry, float* __restrict__ h32,
                              __nv_bfloat16* __restrict__ h16, float* __restrict__ c_last,
                              int32_t* __restrict__ nonfinite) {
  const int cp = blockIdx.x * kScanThreads + threadIdx.x;
  if (2 * cp >= d) return;
  const int ch = blockIdx.y;
  const int t0 = ch * kScanChunk, t1 = min(T, t0 + kScanChunk);
  const float2 cin = *reinterpret_cast<const float2*>(carry + (size_t)ch * d + 2 * cp);
  float c0 = cin.x, c1 = cin.y;
  bool bad = false;
  const __nv_bfloat16* p = ufr + (size_t)t0 * 3 * d + 2 * cp;
#pragma unroll 8
  for (int t = t0; t < t1; ++t, p += 3 * d) {
    const float2 u = ld_bf16x2(p), f = ld_bf16x2(p + d), r = ld_bf16x2(p + 2 * d);
    const float2 xv = *reinterpret_cast<const float2*>(x + (size_t)t * d + 2 * cp);
    c0 = f.x * c0 + (1.f - f.x) * u.x;
    c1 = f.y * c1 + (1.f - f.y) * u.y;
    const float h0 = r.x * fast_tanh(c0) + (1.f - r.x) * xv.x;
    const float h1 = r.y * fast_tanh(c1) + (1.f - r.y) * xv.y;
    bad |= !(isfinite(h0) && isfinite(h1) && isfinite(c0) && isfinite(c1));
    *reinterpret_cast<float2*>(h32 + (size_t)t * d + 2 * cp) = make_float2(h0, h1);
    *reinterpret_cast<__nv_bfloat162*>(h16 + (size_t)t * d + 2 * cp) = __floats2bfloat162_rn(h0, h1);
  }
  if (c_last && t1 == T) *reinterpret_cast<float2*>(c_last + 2 * cp) = make_float2(c0, c1);
  if (bad) atomicOr(nonfinite, 1);  // reference raises NumericError (src/predictor.py:170-171)
}

static inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

// sparsemax rows (src/predictor.py:198-209) in float64, one thread per row:
// insertion-sort descending into local memory, sorted-threshold tau.
__global__ void k_sparsemax(const double* __restrict__ z, int n, int E, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double srt[256];
  const double* zi = z + (size_t)i * E;
  for (int j = 0; j < E; ++j) {
    const double v = zi[j];
    int k = j;
    while (k > 0 && srt[k - 1] < v) {
      srt[k] = srt[k - 1];
      --k;
    }
    srt[k] = v;
  }
  double cum = 0.0, tau_cum = 0.0;
  int ks = 1;
  for (int k = 1; k <= E; ++k) {
    cum += srt[k - 1];
    if (1.0 + k * srt[k - 1] > cum) {
      ks = k;
      tau_cum = cum;
    }
  }
  const double tau = (tau_cum - 1.0) / ks;
  for (int j = 0; j < E; ++j) out[(size_t)i * E + j] = fmax(zi[j] - tau, 0.0);
}

}  // namespace mp

extern "C" int mp_sparsemax_rows(const double* z, int n, int E, double* out, void* stream) {
  MP_REQUIRE(n >= 0 && E >= 1 && E <= 256, MP_ERR_CONFIG, "sparsemax expects a nonempty 1-D vector (E <= 256)");
  if (n == 0) return MP_OK;
  mp::k_sparsemax<<<mp::cdiv(n, 128), 128, 0, (cudaStream_t)stream>>>(z, n, E, out);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

using namespace mp;

extern "C" size_t mp_sru_workspace_bytes(int T, int d) {
  const int nch = cdiv(T, kScanChunk);
  return al(sizeof(__nv_bfloat16) * (size_t)T * 3 * d) + 3 * al(sizeof(float) * (size_t)nch * d);
}

extern "C" int mp_sru_layer(const void* x_bf16, const float* x_f32, const void* w_cat, const float* b_cat, int T,
                            int d, const float* c0, float* h_f32, void* h_bf16, float* c_last, int32_t* nonfinite,
                            void* ws, size_t ws_bytes, void* stream) {
  MP_REQUIRE(T >= 1, MP_ERR_CONFIG, "batch must contain at least one token");
  MP_REQUIRE(d >= 64 && d % 64 == 0, MP_ERR_CONFIG, "mp_sru_layer: d=%d must be a multiple of 64 (pad)", d);
  MP_REQUIRE(ws_bytes >= mp_sru_workspace_bytes(T, d), MP_ERR_CONFIG, "mp_sru_layer: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int nch = cdiv(T, kScanChunk);
  char* p = (char*)ws;
  __nv_bfloat16* ufr = (__nv_bfloat16*)p;
  p += al(sizeof(__nv_bfloat16) * (size_t)T * 3 * d);
  float* aggA = (float*)p;
  p += al(sizeof(float) * (size_t)nch * d);
  float* aggB = (float*)p;
  p += al(sizeof(float) * (size_t)nch * d);
  float* carry = (float*)p;
  // K1: [u | f | r] = x W_cat^T + b ; sigmoid on the f and r blocks
  int rc = mp_gemm_bf16(x_bf16, w_cat, ufr, T, 3 * d, d, 0, 3 * d, b_cat, 2, d, stream);
  if (rc) return rc;
  // K2
  const dim3 g(cdiv(d / 2, kScanThreads), nch);
  k_scan_aggregate<<<g, kScanThreads, 0, st>>>(ufr, T, d, aggA, aggB);
  k_scan_carry<<<cdiv(d, 128), 128, 0, st>>>(aggA, aggB, nch, d, c0, carry);
  k_scan_output<<<g, kScanThreads, 0, st>>>(ufr, x_f32, T, d, carry, h_f32, (__nv_bfloat16*)h_bf16, c_last,
                                            nonfinite);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_heads_argmax(const void* h_bf16, const void* heads, int T, int d, int L, int E, int Eg,
                               int32_t* assign, void* stream) {
  MP_REQUIRE(T >= 1 && L >= 1 && E >= 1 && E <= Eg && Eg >= 32 && Eg <= 256 && (Eg & (Eg - 1)) == 0, MP_ERR_CONFIG,
             "mp_heads_argmax: bad E=%d Eg=%d", E, Eg);
  MP_REQUIRE(d % 64 == 0, MP_ERR_CONFIG, "mp_heads_argmax: d %% 64 != 0");
  cudaStream_t st = (cudaStream_t)stream;
  const int N = ((L * Eg + 63) / 64) * 64;  // heads rows are zero-padded to a multiple of 64
  const int bn = (N % 256 == 0) ? 256 : (N % 128 == 0 ? 128 : 64);
  CUtensorMap ta, tb;
  int rc = make_tmap_bf16(&ta, h_bf16, T, d, d, kBlockM);
  if (rc) return rc;
  rc = make_tmap_bf16(&tb, heads, N, d, d, bn);
  if (rc) return rc;
  DenseSched s{T, N / bn, d / 64, bn};
  EpiGroupArgmax e{assign, T, Eg, E, L};
  const int units = cdiv(T, kBlockM) * (N / bn);
  const int grid = units < num_sms() ? units : num_sms();
  if (bn == 256) return launch_gemm<256, 4>(ta, tb, s, e, grid, st);
  if (bn == 128) return launch_gemm<128, 6>(ta, tb, s, e, grid, st);
  return launch_gemm<64, 8>(ta, tb, s, e, grid, st);
}
