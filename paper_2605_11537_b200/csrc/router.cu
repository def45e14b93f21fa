// K5: true top-1 routing, route_top1 (src/router_oracle.py:90-98):
//   expert(t) = argmax_e  (W_r[e] . x_t)  computed by the reference in float64
//   from float32 inputs, lowest index on ties.
// GPU form: a tensor-core pass over split-bf16 operands (x = x_hi + x_lo,
// w = w_hi + w_lo; acc = x_hi.w_hi + x_hi.w_lo + x_lo.w_hi in fp32) decides
// every token whose top-2 gap exceeds the pass's error bound; the remaining
// near-ties are re-decided exactly like the reference (fp64 dot products of
// the fp32 inputs) by a warp-per-token kernel. The bound per logit is
//   |err| <= 2^-12 * sum_k |x_k| * max_e |w_ek|
// (split residuals ~3*2^-17 plus worst-case fp32 accumulation of 3d terms).
#include "epilogues.cuh"
#include "launch.cuh"

namespace mp {

constexpr float kRouterEps = 1.f / 4096.f;

// xhl[t] = [bf16(x) | bf16(x - bf16(x))], xb[t] = sum_k |x_k| * wabs[k]. one warp per token.
__global__ void k_router_prep(const float* __restrict__ x, int ldx, int T, int d, const float* __restrict__ wabs,
                              __nv_bfloat16* __restrict__ xhl, float* __restrict__ xb, int32_t* __restrict__ count) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = 0;
  if (warp >= T) return;
  const float* xr = x + (size_t)warp * ldx;
  __nv_bfloat16* o = xhl + (size_t)warp * 2 * d;
  float acc = 0.f;
  for (int k = 2 * lane; k < d; k += 64) {
    const float2 v = *reinterpret_cast<const float2*>(xr + k);
    const __nv_bfloat162 hi = __floats2bfloat162_rn(v.x, v.y);
    const float2 hf = __bfloat1622float2(hi);
    const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x - hf.x, v.y - hf.y);
    *reinterpret_cast<__nv_bfloat162*>(o + k) = hi;
    *reinterpret_cast<__nv_bfloat162*>(o + d + k) = lo;
    acc += fabsf(v.x) * wabs[k] + fabsf(v.y) * wabs[k + 1];
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (lane == 0) xb[warp] = acc * 1.0001f + 1e-30f;
}

// exact re-decision of queued tokens: fp64 logits of fp32 inputs, first max wins.
__global__ void k_router_recheck(const float* __restrict__ x, int ldx, int d, const float* __restrict__ w, int E,
                                 const int32_t* __restrict__ count, const int32_t* __restrict__ list,
                                 int32_t* __restrict__ route) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  const int n = *count;
  for (int k = gw; k < n; k += nw) {
    const int t = list[k];
    const float* xr = x + (size_t)t * ldx;
    double best = 0.0;
    int bi = 0;
    for (int e = 0; e < E; ++e) {
      const float* wr = w + (size_t)e * d;
      double s = 0.0;
      for (int j = lane; j < d; j += 32) s += (double)wr[j] * (double)xr[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (e == 0 || s > best) {
        best = s;
        bi = e;
      }
    }
    if (lane == 0) route[t] = bi;
  }
}

static inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace mp

using namespace mp;

extern "C" size_t mp_router_workspace_bytes(int T, int d) {
  return al(sizeof(__nv_bfloat16) * (size_t)T * 2 * d) + al(sizeof(float) * (size_t)T) +
         al(sizeof(int32_t) * ((size_t)T + 1)) + al(sizeof(float) * (size_t)d);
}

// w_abs (d floats, max_e |w_ek|) lives at the end of the workspace and must be filled by
// mp_router_set_weights before the first call for a weight set.
extern "C" int mp_router_weight_absmax(const float* w_f32, int E, int d, float* wabs_out, void* stream);

namespace mp {
__global__ void k_wabs(const float* __restrict__ w, int E, int d, float* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= d) return;
  float m = 0.f;
  for (int e = 0; e < E; ++e) m = fmaxf(m, fabsf(w[(size_t)e * d + k]));
  out[k] = m;
}
}  // namespace mp

extern "C" int mp_router_weight_absmax(const float* w_f32, int E, int d, float* wabs_out, void* stream) {
  k_wabs<<<cdiv(d, 256), 256, 0, (cudaStream_t)stream>>>(w_f32, E, d, wabs_out);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

static int route_gemm(const float* x, int ldx, int T, int d, const void* w_hl, const float* w_f32, int E, int Eg,
                      int32_t* route, const RouterWs& rw, float eps, cudaStream_t st) {
  CUtensorMap ta, tb;
  int rc = make_tmap_bf16(&ta, rw.xhl, T, 2 * d, 2 * d, kBlockM);
  if (rc) return rc;
  rc = make_tmap_bf16(&tb, w_hl, Eg, 2 * d, 2 * d, Eg);
  if (rc) return rc;
  Split3Sched s{T, 1, d / 64, Eg, d};
  EpiRouterTop1 e{route, rw.xb, eps, E, rw.count, rw.list};
  const int units = cdiv(T, kBlockM);
  const int grid = units < num_sms() ? units : num_sms();
  if (Eg == 256) rc = launch_gemm<256, 4>(ta, tb, s, e, grid, st);
  else if (Eg == 128) rc = launch_gemm<128, 6>(ta, tb, s, e, grid, st);
  else rc = launch_gemm<64, 8>(ta, tb, s, e, grid, st);
  if (rc) return rc;
  k_router_recheck<<<num_sms(), 256, 0, st>>>(x, ldx, d, w_f32, E, rw.count, rw.list, route);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

#define ROUTER_CHECKS()                                                                                          \
  MP_REQUIRE(T >= 1 && d % 64 == 0 && ldx >= d && ldx % 2 == 0, MP_ERR_CONFIG, "mp_route_top1: bad T/d/ldx");     \
  MP_REQUIRE(E >= 1 && E <= Eg && (Eg == 64 || Eg == 128 || Eg == 256), MP_ERR_CONFIG,                          \
             "mp_route_top1: E=%d needs Eg in {64,128,256} >= E", E);                                          \
  MP_REQUIRE(ws_bytes >= mp_router_workspace_bytes(T, d), MP_ERR_CONFIG, "mp_route_top1: workspace too small");

extern "C" int mp_route_top1_ex(const float* x, int ldx, int T, int d, const void* w_hl, const float* w_f32,
                                const float* w_abs, int E, int Eg, int32_t* route, void* ws, size_t ws_bytes,
                                void* stream) {
  ROUTER_CHECKS();
  cudaStream_t st = (cudaStream_t)stream;
  const RouterWs rw(ws, T, d);
  k_router_prep<<<cdiv(T * 32, 256), 256, 0, st>>>(x, ldx, T, d, w_abs, (__nv_bfloat16*)rw.xhl, rw.xb, rw.count);
  return route_gemm(x, ldx, T, d, w_hl, w_f32, E, Eg, route, rw, kRouterEps, st);
}

extern "C" int mp_route_top1_prepared(const float* x, int ldx, int T, int d, const void* w_hl, const float* w_f32,
                                      int E, int Eg, int32_t* route, void* ws, size_t ws_bytes, void* stream) {
  ROUTER_CHECKS();
  // xhl / xb were produced by the previous layer's mp_ffn_down_router epilogue (xb summed
  // by atomics in arbitrary order: 1e-4 relative slack on the bound); count was reset
  // by mp_ffn_gather_split.
  return route_gemm(x, ldx, T, d, w_hl, w_f32, E, Eg, route, RouterWs(ws, T, d), kRouterEps * 1.0001f,
                    (cudaStream_t)stream);
}

extern "C" int mp_route_top1(const float* x, int ldx, int T, int d, const void* w_hl, const float* w_f32, int E,
                             int Eg, float w_norm_max, int32_t* route, void* ws, size_t ws_bytes, void* stream) {
  // Convenience form: derives max_e |w_ek| into the workspace tail on every call.
  (void)w_norm_max;
  MP_REQUIRE(ws_bytes >= mp_router_workspace_bytes(T, d), MP_ERR_CONFIG, "mp_route_top1: workspace too small");
  float* wabs = (float*)((char*)ws + mp_router_workspace_bytes(T, d) - al(sizeof(float) * (size_t)d));
  int rc = mp_router_weight_absmax(w_f32, E, d, wabs, stream);
  if (rc) return rc;
  return mp_route_top1_ex(x, ldx, T, d, w_hl, w_f32, wabs, E, Eg, route, ws, ws_bytes, stream);
}
