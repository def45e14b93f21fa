// Epilogues for the tcgen05 GEMM core: each thread owns one accumulator row of
// the 128-row tile and streams its BN fp32 columns out of TMEM 32 at a time.
#pragma once
#include "gemm_sm100.cuh"

namespace mp {

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// sigmoid(x) = 0.5 + 0.5 tanh(x / 2): one MUFU op. The reference clips the argument
// to [-60, 60] (src/predictor.py:24-25), where tanh is already saturated; the result
// is stored as bf16 (2^-9 relative), far coarser than tanh.approx (~2^-11).
__device__ __forceinline__ float sigmoid_clip(float x) { return fmaf(0.5f, tanh_approx(0.5f * x), 0.5f); }

// 32 consecutive fp32 of a broadcast vector (bias) via 8 x 16-byte loads.
__device__ __forceinline__ void add_bias32(float* v, const float* __restrict__ bias) {
  const float4* b4 = reinterpret_cast<const float4*>(bias);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 b = __ldg(&b4[q]);
    v[4 * q + 0] += b.x;
    v[4 * q + 1] += b.y;
    v[4 * q + 2] += b.z;
    v[4 * q + 3] += b.w;
  }
}

// Software-pipelined walk over NC accumulator columns: the TMEM load of chunk
// c+32 is in flight while chunk c is processed. f(c, v[32]) consumes a chunk.
template <int NC, class F>
__device__ __forceinline__ void tmem_chunks(uint32_t taddr, F&& f) {
  uint32_t ra[32], rb[32];
  tmem_ld32_issue(taddr, ra);
  tmem_ld_wait32(ra);
#pragma unroll
  for (int c = 0; c < NC; c += 64) {
    if (c + 32 < NC) tmem_ld32_issue(taddr + c + 32, rb);
    f(c, reinterpret_cast<float*>(ra));
    if (c + 32 < NC) {
      tmem_ld_wait32(rb);
      if (c + 64 < NC) tmem_ld32_issue(taddr + c + 64, ra);
      f(c + 32, reinterpret_cast<float*>(rb));
      if (c + 64 < NC) tmem_ld_wait32(ra);
    }
  }
}

__device__ __forceinline__ void apply_act(float* v, const float* svec, int act, bool sig) {
  if (svec) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] += svec[i];
  }
  if (act == 1) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
  } else if (act == 2 && sig) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = sigmoid_clip(v[i]);
  }
}

// out[row, n0 + c] = act(acc + bias) -> bf16 (act: 0 none, 1 relu, 2 sigmoid for cols >= sig_from)
struct EpiStoreBf16 {
  static constexpr bool kSplitCols = true;
  __nv_bfloat16* out;
  int ldo;
  const float* bias;  // may be null
  int act;
  int sig_from;
  __device__ __forceinline__ const float* colvec() const { return bias; }
  template <int NC>
  __device__ __forceinline__ void run(const Unit& U, int mt, int r, uint32_t taddr, int c0, const float* svec) const {
    const int rr = mt * kBlockM + r;
    const bool ok = rr < U.rows;
    __nv_bfloat16* dst = out + (size_t)(U.a_row + rr) * ldo + U.n0 + c0;
    tmem_chunks<NC>(taddr, [&](int c, float* v) {
      apply_act(v, bias ? svec + c : nullptr, act, U.n0 + c0 + c >= sig_from);
      if (ok && ldo) {  // ldo == 0: diagnostic mode, no stores
        uint4* d4 = reinterpret_cast<uint4*>(dst + c);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 w;
          w.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
          w.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
          w.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
          w.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
          d4[q] = w;
        }
      }
    });
  }
};

// out[row, n0 + c] = act(acc + bias) in fp32
struct EpiStoreF32 {
  static constexpr bool kSplitCols = true;
  float* out;
  int ldo;
  const float* bias;
  int act;
  int sig_from;
  __device__ __forceinline__ const float* colvec() const { return bias; }
  template <int NC>
  __device__ __forceinline__ void run(const Unit& U, int mt, int r, uint32_t taddr, int c0, const float* svec) const {
    const int rr = mt * kBlockM + r;
    const bool ok = rr < U.rows;
    float* dst = out + (size_t)(U.a_row + rr) * ldo + U.n0 + c0;
    tmem_chunks<NC>(taddr, [&](int c, float* v) {
      apply_act(v, bias ? svec + c : nullptr, act, U.n0 + c0 + c >= sig_from);
      if (ok) {
        float4* d4 = reinterpret_cast<float4*>(dst + c);
#pragma unroll
        for (int q = 0; q < 8; ++q) d4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
    });
  }
};

// Grouped-GEMM2 epilogue: ungated residual combine scattered back to token order
// (src/router_oracle.py:127-134: stream[t] = stream[t] + expert_forward(stream[t])).
// Top-1 routing => each token row is owned by exactly one tile row: no atomics.
struct EpiScatterAdd {
  static constexpr bool kSplitCols = true;
  float* x;  // T x ldx fp32 residual stream (updated in place)
  int ldx;
  const int32_t* tok_of_row;
  __device__ __forceinline__ const float* colvec() const { return nullptr; }
  template <int NC>
  __device__ __forceinline__ void run(const Unit& U, int mt, int r, uint32_t taddr, int c0, const float*) const {
    const int rr = mt * kBlockM + r;
    const bool ok = rr < U.rows;
    const int tok = ok ? __ldg(&tok_of_row[U.a_row + rr]) : 0;
    float4* dst = reinterpret_cast<float4*>(x + (size_t)tok * ldx + U.n0 + c0);
    tmem_chunks<NC>(taddr, [&](int c, float* v) {
      if (ok) {
        float4 o[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] = dst[c / 4 + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          o[q].x += v[4 * q + 0];
          o[q].y += v[4 * q + 1];
          o[q].z += v[4 * q + 2];
          o[q].w += v[4 * q + 3];
          dst[c / 4 + q] = o[q];
        }
      }
    });
  }
};

// Per-row argmax over column groups of width `group` (first index wins ties,
// like numpy.argmax). Columns >= valid inside a group are padding.
// out[g * M + row] for group g = global column / group.
struct EpiGroupArgmax {
  static constexpr bool kSplitCols = false;
  int32_t* out;
  int M;
  int group;
  int valid;
  int ngroups;
  __device__ __forceinline__ const float* colvec() const { return nullptr; }
  template <int BN>
  __device__ __forceinline__ void run(const Unit& U, int mt, int r, uint32_t taddr, int, const float*) const {
    const int rr = mt * kBlockM + r;
    const bool ok = rr < U.rows;
    float best = -INFINITY;
    int bi = 0;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      float v[32];
      tmem_ld32(taddr + c, v);
      const int gc = U.n0 + c;
      const int g = gc / group;
      const int base = gc - g * group;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (base + i < valid && v[i] > best) {
          best = v[i];
          bi = base + i;
        }
      }
      if (((gc + 32) % group) == 0) {
        if (ok && g < ngroups) out[(size_t)g * M + U.a_row + rr] = bi;
        best = -INFINITY;
        bi = 0;
      }
    }
  }
};

// Router epilogue: top-1 plus a certification test. The split-bf16 product is
// within err_scale * |x|_2 of the exact fp32-input logit; when the top-2 gap is
// not larger than twice that bound the token is queued for an fp64 re-decision.
struct EpiRouterTop1 {
  static constexpr bool kSplitCols = false;
  int32_t* route;
  const float* xnorm;  // |x_t|_2
  float err_scale;     // bound factor (includes max_e |w_e|_2)
  int valid;           // E
  int32_t* recheck_count;
  int32_t* recheck_list;
  __device__ __forceinline__ const float* colvec() const { return nullptr; }
  template <int BN>
  __device__ __forceinline__ void run(const Unit& U, int mt, int r, uint32_t taddr, int, const float*) const {
    const int rr = mt * kBlockM + r;
    const bool ok = rr < U.rows;
    float b1 = -INFINITY, b2 = -INFINITY;
    int bi = 0;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      float v[32];
      tmem_ld32(taddr + c, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int e = c + i;
        if (e < valid) {
          if (v[i] > b1) {
            b2 = b1;
            b1 = v[i];
            bi = e;
          } else if (v[i] > b2) {
            b2 = v[i];
          }
        }
      }
    }
    if (ok) {
      const int t = U.a_row + rr;
      route[t] = bi;
      if (valid > 1 && !(b1 - b2 > 2.f * err_scale * __ldg(&xnorm[t]))) {
        const int k = atomicAdd(recheck_count, 1);
        recheck_list[k] = t;
      }
    }
  }
};

}  // namespace mp
