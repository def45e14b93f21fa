// Epilogues for the tcgen05 GEMM core: each thread owns one accumulator row of
// the 128-row tile and streams its BN fp32 columns out of TMEM 32 at a time.
#pragma once
#include "gemm_sm100.cuh"

namespace mp {

#ifdef MP_DIAG
// Diagnostic build only: bit 0 = the TMA-store epilogue packs its boxes but issues no store.
static __device__ int g_diag_epi;
#endif

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

// *p += v as one L2 vector reduction (no value returned; sm_90+ .v4.f32)
__device__ __forceinline__ void red_add_v4(float4* p, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
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

// Coalesced bf16 store of one 32-column chunk of the warp's 32 rows: lane = row
// writes its 64 B to warp-private smem (row stride 80 B: conflict-free 16 B
// stores), then each store instruction writes 8 rows x 64 B contiguous
// segments. row_ptr(i) gives the destination of tile row i of this warp (or
// null for rows outside the unit).
template <class RowPtr>
__device__ __forceinline__ void store_chunk_bf16(const float* v, uint32_t* scratch, RowPtr&& row_ptr) {
  const int lane = threadIdx.x & 31;
  uint4* srow = reinterpret_cast<uint4*>(scratch + lane * 20);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 w;
    w.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
    w.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
    w.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
    w.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
    srow[q] = w;
  }
  __syncwarp();
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int row = it * 8 + (lane >> 2), part = lane & 3;
    const uint4 w = *reinterpret_cast<const uint4*>(scratch + row * 20 + part * 4);
    __nv_bfloat16* dst = row_ptr(row);
    if (dst) reinterpret_cast<uint4*>(dst)[part] = w;
  }
  __syncwarp();
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
  __device__ __forceinline__ void run(const Unit& U, int mt, int r, uint32_t taddr, int c0, const float* svec,
                                      uint32_t* scratch) const {
    const int row0 = mt * kBlockM + (r & ~31);  // first unit row of this warp
    __nv_bfloat16* base = out + (size_t)(U.a_row + row0) * ldo + U.n0 + c0;
    const int nvalid = U.rows - row0;
    tmem_chunks<NC>(taddr, [&](int c, float* v) {
      apply_act(v, bias ? svec + c : nullptr, act, U.n0 + c0 + c >= sig_from);
      if (ldo)  // ldo == 0: diagnostic mode, no stores
        store_chunk_bf16(v, scratch, [&](int i) -> __nv_bfloat16* {
          return i < nvalid ? base + (size_t)i * ldo + c : nullptr;
        });
    });
  }
};

// EpiStoreBf16 with the tile written by TMA bulk stores: each warp packs its 32 rows x
// 32 columns (64 B rows) into its scratch as a SWIZZLE_64B box and one lane issues
// cp.async.bulk.tensor (global writes leave the LSU/L1 path; the box lands as whole
// 64 B row segments). Warps whose 32 rows are not all inside the unit (the tail of a
// piece -- the next rows belong to another piece) fall back to st.global.
// tm (the GEMM kernel's tmC parameter): bf16 [rows x ldo] map, box 32 x 32, SWIZZLE_64B
// (make_tmap_bf16_store).
struct EpiStoreBf16Tma {
  static constexpr bool kSplitCols = true;
  static constexpr bool kTmaStore = true;  // the kernel passes its tmC parameter to run()
  __nv_bfloat16* out;
  int ldo;
  const float* bias;
  int act;
  int sig_from;
  int keep_l2;  // 1: stores carry an L2 evict_last hint (the output is re-read right away), 2: evict_first
  __device__ __forceinline__ const float* colvec() const { return bias; }
  template <int NC>
  __device__ __forceinline__ void run(const Unit& U, int mt, int r, uint32_t taddr, int c0, const float* svec,
                                      uint32_t* scratch, const CUtensorMap* tm) const {
    const int lane = threadIdx.x & 31;
    const int row0 = mt * kBlockM + (r & ~31);
    const int nvalid = U.rows - row0;
    __nv_bfloat16* base = out + (size_t)(U.a_row + row0) * ldo + U.n0 + c0;
    uint8_t* box = reinterpret_cast<uint8_t*>(scratch);
    const int sw = (lane >> 1) & 3;  // SWIZZLE_64B: 16-byte chunk q of row `lane` lives at q ^ ((lane / 2) % 4)
    tmem_chunks<NC>(taddr, [&](int c, float* v) {
      apply_act(v, bias ? svec + c : nullptr, act, U.n0 + c0 + c >= sig_from);
      if (nvalid >= 32) {
        if (lane == 0) bulk_wait_read0();  // previous box of this warp has been read
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 w;
          w.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
          w.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
          w.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
          w.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
          *reinterpret_cast<uint4*>(box + lane * 64 + ((q ^ sw) << 4)) = w;
        }
        fence_proxy_async();
        __syncwarp();
#ifdef MP_DIAG
        if (g_diag_epi & 1) {
          __syncwarp();
          return;
        }
#endif
        if (lane == 0) {
          if (keep_l2 == 1)
            tma_store_2d_hint(tm, box, U.n0 + c0 + c, U.a_row + row0, policy_evict_last());
          else if (keep_l2 == 2)  // streaming output: do not evict the GEMM's L2-resident operands
            tma_store_2d_hint(tm, box, U.n0 + c0 + c, U.a_row + row0, policy_evict_first());
          else
            tma_store_2d(tm, box, U.n0 + c0 + c, U.a_row + row0);
          bulk_commit();
        }
      } else if (nvalid > 0) {
        if (lane == 0) bulk_wait_read0();
        __syncwarp();
        store_chunk_bf16(v, scratch, [&](int i) -> __nv_bfloat16* {
          return i < nvalid ? base + (size_t)i * ldo + c : nullptr;
        });
      }
    });
    // no wait here: the next box waits for this warp's previous box to be READ (its smem is
    // reused); the kernel waits for the writes themselves once, before the CTA exits
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
  __device__ __forceinline__ void run(const Unit& U, int mt, int r, uint32_t taddr, int c0, const float* svec,
                                      uint32_t*) const {
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
  int store = 0;              // 1: plain stores (x[tok] = y) -- every target row has exactly one
                              //    writer (the expert-parallel receive buffer needs no zeroing)
  float* const* peer_x = nullptr;  // expert parallelism over peer memory: tok_of_row holds home * peer_T + t
  int peer_T = 1;                  //    and the row is added into rank home's stream (an NVLink peer address)
  __device__ __forceinline__ const float* colvec() const { return nullptr; }
  template <int NC>
  __device__ __forceinline__ void run(const Unit& U, int mt, int r, uint32_t taddr, int c0, const float*,
                                      uint32_t* scratch) const {
    const int lane = threadIdx.x & 31;
    const int rr = mt * kBlockM + r;
    const bool ok = rr < U.rows;
    const int tok = ok ? __ldg(&tok_of_row[U.a_row + rr]) : -1;
    float* rowp = nullptr;  // this thread's destination row (+ the tile's first column)
    if (tok >= 0)
      rowp = (peer_x ? reinterpret_cast<float*>(__ldg(reinterpret_cast<const unsigned long long*>(peer_x) +
                                                      tok / peer_T)) +
                           (size_t)(tok % peer_T) * ldx
                     : x + (size_t)tok * ldx) +
             U.n0 + c0;
    float4* srow = reinterpret_cast<float4*>(scratch + lane * 20);
    const int pq = lane & 3;
    float* tp[4];  // destination row of the row this lane updates in store step `it`
#pragma unroll
    for (int it = 0; it < 4; ++it)
      tp[it] = reinterpret_cast<float*>(
          __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(rowp), it * 8 + (lane >> 2)));
    tmem_chunks<NC>(taddr, [&](int c, float* v) {
      // two 16-column halves: lane = row -> smem, then 8 rows x 64 B per instruction.
      // The residual update is a vector reduction performed in L2 (red.global.add.v4.f32):
      // top-1 routing gives every element exactly one addend, so x + y is rounded once,
      // exactly like a load-add-store, and the order cannot vary.
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          srow[q] = make_float4(v[16 * h + 4 * q], v[16 * h + 4 * q + 1], v[16 * h + 4 * q + 2], v[16 * h + 4 * q + 3]);
        __syncwarp();
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int row = it * 8 + (lane >> 2);
          const float4 a = *reinterpret_cast<const float4*>(scratch + row * 20 + pq * 4);
          if (tp[it] != nullptr) {
            float4* dst = reinterpret_cast<float4*>(tp[it] + c + 16 * h) + pq;
            if (store)
              *dst = a;
            else
              red_add_v4(dst, a);
          }
        }
        __syncwarp();
      }
    });
  }
};

// Per-row argmax over column groups of width `group` (first index wins ties,
// like numpy.argmax). Columns >= valid inside a group are padding.
// out[g * M + row] for group g = global column / group.
// kSplit: the two epilogue warpgroups take one column half each (valid when a group
// never straddles the halves, i.e. group <= BN / 2 and BN / 2 % group == 0).
template <bool kSplit>
struct EpiGroupArgmaxT {
  static constexpr bool kSplitCols = kSplit;
  int32_t* out;
  int M;
  int group;
  int valid;
  int ngroups;
  __device__ __forceinline__ const float* colvec() const { return nullptr; }
  template <int NC>
  __device__ __forceinline__ void run(const Unit& U, int mt, int r, uint32_t taddr, int c0, const float*,
                                      uint32_t*) const {
    const int rr = mt * kBlockM + r;
    const bool ok = rr < U.rows;
    float best = -INFINITY;
    int bi = 0;
#pragma unroll 1
    for (int c = 0; c < NC; c += 32) {
      float v[32];
      tmem_ld32(taddr + c, v);
      const int gc = U.n0 + c0 + c;
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

using EpiGroupArgmax = EpiGroupArgmaxT<false>;

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
  __device__ __forceinline__ void run(const Unit& U, int mt, int r, uint32_t taddr, int, const float*,
                                      uint32_t*) const {
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
