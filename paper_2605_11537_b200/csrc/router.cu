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
  griddep_launch_dependents();
  griddep_wait();
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
  griddep_launch_dependents();
  griddep_wait();
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


// 16-byte shared-memory load (explicit ld.shared: the address never goes through a generic pointer)
__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr)
               : "memory");
  return v;
}

constexpr int kRfConvThreads = 512;  // convert + epilogue threads (warps 4..19): the split-bf16
                                      // conversion is latency bound, 16 warps keep it under the MMA
constexpr int kRouterThreads = 128 + kRfConvThreads;

// Fused router (Eg <= 128): the split of x into bf16 hi/lo and the bound scale
// sum_k |x_k| * wabs_k are computed INSIDE the GEMM. A producer warp (warp 3) streams x
// fp32 k-blocks (two 128 x 32 SWIZZLE_128B boxes) into a 3-deep shared-memory ring; the 16
// convert warps read them into registers and write the bf16 hi / lo operand rows straight
// into TENSOR memory (tcgen05.st), where the MMA reads its A operand: the split operand
// never passes through shared memory, whose bandwidth (TMA writes, converter reads, MMA
// operand reads) bounded the previous form at ~0.85 us per k-block. No T x 2d split buffer
// goes through HBM, no pre-pass launch. Per k-block (64 columns):
//   acc[:, 0:Eg)   += x_hi . w_hi^T + x_lo . w_hi^T     (N = Eg MMA on the lo rows)
//   acc[:, Eg:2Eg) += x_hi . w_lo^T                     (part of one N = 2Eg MMA)
// with B = [w_hi ; w_lo] stacked as 2Eg rows of one tile; logit = acc[e] + acc[Eg + e].
// Roles: warp 0 TMA (B), warp 3 TMA (x), warp 1 MMA, warp 2 TMEM, warps 4..19 convert +
// epilogue (warp w writes TMEM lanes 32 (w % 4) .. +31, k-columns 16 ((w - 4) / 4) .. +15).
// TMEM: the accumulator (2 Eg columns) then kRxAStages operand stages of 64 columns
// ([hi: 32 | lo: 32], two bf16 per column).
constexpr int kRxStages = 3;   // B (router weight) ring
constexpr int kRxXStages = 3;  // x ring (fp32 k-blocks, freed once the converters hold them in registers)
constexpr int kRxAStages = 4;  // TMEM operand stages
constexpr uint32_t kRxTmemCols = 512;
#ifdef MP_DIAG
// Diagnostic build only: per-CTA %globaltimer stamps of the last fused-router launch.
// [0] start, [1] setup done; per k-block kb < 12: [2 + kb] x issued (producer), [14 + kb]
// landed, [26 + kb] read into registers, [38 + kb] TMEM stage free, [50 + kb] TMEM stores
// done (converter warp 4), [62 + kb] operand ready (MMA); [74] accumulator full, [75] end.
static __device__ unsigned long long g_rt[160][80];
#define RT_STAMP(i)                                                                   \
  do {                                                                                \
    unsigned long long t_;                                                            \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                           \
    if (blockIdx.x < 160) g_rt[blockIdx.x][i] = t_;                                   \
  } while (0)
#else
#define RT_STAMP(i) \
  do {              \
  } while (0)
#endif

template <int EG>
struct RxSmem {
  static_assert(2 * EG + kRxAStages * 64 <= (int)kRxTmemCols, "router TMEM columns");
  static constexpr int kB = 2 * EG * 128;
  static constexpr int kXs = 128 * 64 * 4;  // one x k-block: 128 rows x 64 fp32 as two 16 KB boxes
  static constexpr int kXOffset = kRxStages * kB;
  static constexpr int kBarOffset = kXOffset + kRxXStages * kXs;
  // bfull[S], bempty[S], xfull[X], xfree[X], conv[A], aempty[A], tfull, tempty
  static constexpr int kXbOffset = kBarOffset + (2 * kRxStages + 2 * kRxXStages + 2 * kRxAStages + 2) * 8 + 8;
  static constexpr int kPartOffset = kXbOffset + 128 * 4;   // 4 x 128 partial bound sums
  static constexpr int kHistOffset = kPartOffset + 4 * 128 * 4;  // EG ints: the tile's expert histogram
  static constexpr int kTopOffset = kHistOffset + EG * 4;  // per column group: best, second (float), best index
  static constexpr int kBytes = kTopOffset + 3 * (EG / 32) * 128 * 4 + 1024;
};

template <int EG>
__global__ void __launch_bounds__(kRouterThreads, 1)
    k_router_fused_tx(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmX, int T, int d,
                      const float* __restrict__ wabs, int E, int32_t* __restrict__ route, float eps,
                      int32_t* __restrict__ count, int32_t* __restrict__ list,
                      const float* __restrict__ xg, int ldx, const float* __restrict__ w32,
                      int32_t* __restrict__ hist_cc) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  using L = RxSmem<EG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);  // B stage landed
  uint64_t* empty = full + kRxStages;                                     // B stage consumed by the MMA
  uint64_t* xfull = empty + kRxStages;                                    // x stage landed
  uint64_t* xfree = xfull + kRxXStages;                                   // x stage read by every converter
  uint64_t* conv = xfree + kRxXStages;                                    // TMEM operand stage written
  uint64_t* aempty = conv + kRxAStages;                                   // TMEM operand stage consumed
  uint64_t* tfull = aempty + kRxAStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  float* s_xb = reinterpret_cast<float*>(smem + L::kXbOffset);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = d / 64;
  const int units = (T + kBlockM - 1) / kBlockM;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmB);
    tma_prefetch(&tmX);
    for (int s = 0; s < kRxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kRxXStages; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xfree[s], kRfConvThreads / 32);
    }
    for (int s = 0; s < kRxAStages; ++s) {
      mbar_init(&conv[s], kRfConvThreads / 32);
      mbar_init(&aempty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4 * (EG / 32));  // every TMEM-reading epilogue warp
    fence_barrier_init();
  }
  if (threadIdx.x == 0) RT_STAMP(0);
  if (warp == 2) tmem_alloc(tmem_slot, kRxTmemCols);
  griddep_wait();  // x is the previous layer's output
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) RT_STAMP(1);

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ B producer
      uint32_t stage = 0, phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sb = smem + stage * L::kB;
          mbar_arrive_expect_tx(&full[stage], L::kB);
          tma_load_2d(sb, &tmB, &full[stage], kb * 64, 0);
          tma_load_2d(sb + EG * 128, &tmB, &full[stage], d + kb * 64, 0);
          if (++stage == kRxStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {  // ------------------------------------------------ x producer
      uint32_t stage = 0, phase = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&xfree[stage], phase ^ 1);
          uint8_t* sx = smem + L::kXOffset + stage * L::kXs;
          mbar_arrive_expect_tx(&xfull[stage], L::kXs);
          tma_load_2d(sx, &tmX, &xfull[stage], kb * 64, u * kBlockM);  // rows >= T: zero fill
          tma_load_2d(sx + L::kXs / 2, &tmX, &xfull[stage], kb * 64 + 32, u * kBlockM);
          if (kb < 12) RT_STAMP(2 + kb);
          if (++stage == kRxXStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      constexpr uint32_t id_all = idesc_bf16_f32(kBlockM, 2 * EG);
      constexpr uint32_t id_hi = idesc_bf16_f32(kBlockM, EG);
      uint32_t stage = 0, phase = 0, astage = 0, aphase = 0, tile = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++tile) {
        mbar_wait(tempty, (tile & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          mbar_wait(&conv[astage], aphase);
          tc_fence_after();
          if (kb < 12) RT_STAMP(62 + kb);
          const uint64_t bdesc = sw128_kmajor_desc(smem_u32(smem + stage * L::kB));
          const uint32_t ahi = tmem_base + 2 * EG + astage * 64, alo = ahi + 32;
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // K = 16 per MMA = 8 TMEM columns of packed bf16
            umma_bf16_tmem_a(tmem_base, ahi + 8 * k, bdesc + 2 * k, id_all, (kb | k) != 0);
            umma_bf16_tmem_a(tmem_base, alo + 8 * k, bdesc + 2 * k, id_hi, 1);
          }
          umma_commit(&empty[stage]);
          umma_commit(&aempty[astage]);
          if (++stage == kRxStages) {
            stage = 0;
            phase ^= 1;
          }
          if (++astage == kRxAStages) {
            astage = 0;
            aphase ^= 1;
          }
        }
        umma_commit(tfull);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ convert + epilogue
    const int ct = threadIdx.x - 128;  // 0..kRfConvThreads-1
    const int rq = (warp & 3) * 32 + lane;  // tile row = TMEM lane this thread writes
    const int jq = (warp - 4) >> 2;         // 16-column quarter of the k-block
    const int box = jq >> 1, c0 = (jq & 1) * 4;  // x box (32 columns) and first 16-byte chunk inside a 128 B row
    const uint32_t tq = tmem_base + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 2 * EG + 8 * jq;
    float* s_part = reinterpret_cast<float*>(smem + L::kPartOffset);
    int* s_hist = reinterpret_cast<int*>(smem + L::kHistOffset);
    float* s_top = reinterpret_cast<float*>(smem + L::kTopOffset);
    int* s_topi = reinterpret_cast<int*>(s_top + 2 * (EG / 32) * 128);
    if (hist_cc != nullptr) {
      for (int e = ct; e < EG; e += kRfConvThreads) s_hist[e] = 0;
      named_bar_sync(1, kRfConvThreads);
    }
    uint32_t xstage = 0, xphase = 0, astage = 0, aphase = 0, tile = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++tile) {
      const int row_base = u * kBlockM;
      float part = 0.f;
      // bound-scale weights of the next k-block are loaded one iteration ahead (L2 latency off
      // the conversion's critical path)
      const float4* wq = reinterpret_cast<const float4*>(wabs + 16 * jq);
      float4 wn[4] = {__ldg(wq), __ldg(wq + 1), __ldg(wq + 2), __ldg(wq + 3)};
      for (int kb = 0; kb < nkb; ++kb) {
        const float4 w[4] = {wn[0], wn[1], wn[2], wn[3]};
        if (kb + 1 < nkb) {
          const float4* wk = wq + (kb + 1) * 16;
#pragma unroll
          for (int i = 0; i < 4; ++i) wn[i] = __ldg(wk + i);
        }
        mbar_wait(&xfull[xstage], xphase);
        if (warp == 4 && lane == 0 && kb < 12) RT_STAMP(14 + kb);
        const uint32_t sx = smem_u32(smem + L::kXOffset + xstage * L::kXs + box * (L::kXs / 2)) + rq * 128;
        float4 v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = lds_f4(sx + (((c0 + i) ^ (rq & 7)) << 4));
        __syncwarp();
        if (lane == 0) mbar_arrive(&xfree[xstage]);  // this warp is done with the x stage
        if (warp == 4 && lane == 0 && kb < 12) RT_STAMP(26 + kb);
        if (++xstage == kRxXStages) {
          xstage = 0;
          xphase ^= 1;
        }
        const float f[16] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y, v[1].z, v[1].w,
                             v[2].x, v[2].y, v[2].z, v[2].w, v[3].x, v[3].y, v[3].z, v[3].w};
        uint32_t hw[8], lw[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * q], f[2 * q + 1]);
          const float2 hf = __bfloat1622float2(h);
          const __nv_bfloat162 lo = __floats2bfloat162_rn(f[2 * q] - hf.x, f[2 * q + 1] - hf.y);
          hw[q] = *reinterpret_cast<const uint32_t*>(&h);
          lw[q] = *reinterpret_cast<const uint32_t*>(&lo);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
          part += fabsf(f[4 * i]) * w[i].x + fabsf(f[4 * i + 1]) * w[i].y + fabsf(f[4 * i + 2]) * w[i].z +
                  fabsf(f[4 * i + 3]) * w[i].w;
        mbar_wait(&aempty[astage], aphase ^ 1);  // the MMA has read this operand stage
        tc_fence_after();
        if (warp == 4 && lane == 0 && kb < 12) RT_STAMP(38 + kb);
        tmem_st8(tq + astage * 64, hw);
        tmem_st8(tq + astage * 64 + 32, lw);
        tmem_st_wait();
        if (warp == 4 && lane == 0 && kb < 12) RT_STAMP(50 + kb);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[astage]);
        if (++astage == kRxAStages) {
          astage = 0;
          aphase ^= 1;
        }
      }
      s_part[jq * 128 + rq] = part;
      named_bar_sync(1, kRfConvThreads);
      if (jq == 0)
        s_xb[rq] = (s_part[rq] + s_part[128 + rq] + s_part[256 + rq] + s_part[384 + rq]) * 1.0001f + 1e-30f;
      named_bar_sync(1, kRfConvThreads);
      // top-2 logits per row: the (EG / 32) column groups of the accumulator are read by
      // (EG / 32) x 4 warps (warp & 3 = TMEM lane quadrant), then merged in expert order
      constexpr int kParts = EG / 32;
      const int part_id = (warp - 4) >> 2;
      if (part_id < kParts) {
        mbar_wait(tfull, tile & 1);
        tc_fence_after();
        if (warp == 4 && lane == 0) RT_STAMP(74);
        const int r = (warp & 3) * 32 + lane;
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 32 * part_id;
        float a[32], b[32];
        tmem_ld32(taddr, a);
        tmem_ld32(taddr + EG, b);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
        float b1 = -INFINITY, b2 = -INFINITY;
        int bi = 32 * part_id;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int e = 32 * part_id + i;
          const float v = a[i] + b[i];
          if (e < E) {
            if (v > b1) {
              b2 = b1;
              b1 = v;
              bi = e;
            } else if (v > b2) {
              b2 = v;
            }
          }
        }
        s_top[(0 * kParts + part_id) * 128 + r] = b1;
        s_top[(1 * kParts + part_id) * 128 + r] = b2;
        s_topi[part_id * 128 + r] = bi;
      }
      named_bar_sync(1, kRfConvThreads);
      if (warp < 8) {
        const int r = (warp & 3) * 32 + lane;
        float b1 = s_top[r], b2 = s_top[kParts * 128 + r];
        int bi = s_topi[r];
#pragma unroll
        for (int q = 1; q < kParts; ++q) {  // ascending experts: a later group wins only on '>'
          const float c1 = s_top[q * 128 + r], c2 = s_top[(kParts + q) * 128 + r];
          if (c1 > b1) {
            b2 = fmaxf(b1, c2);
            b1 = c1;
            bi = s_topi[q * 128 + r];
          } else {
            b2 = fmaxf(b2, c1);
          }
        }
        const int t = row_base + r;
        if (hist_cc != nullptr) {
          // near ties re-decided here in float64 by the warp (the arithmetic of
          // k_router_recheck), then the tile's histogram for the execution map
          unsigned m = __ballot_sync(0xffffffffu, t < T && E > 1 && !(b1 - b2 > 2.f * eps * s_xb[r]));
          while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            const float* xr = xg + (size_t)(t - lane + j) * ldx;
            double best = 0.0;
            int bj = 0;
            for (int e = 0; e < E; ++e) {
              const float* wr = w32 + (size_t)e * d;
              double sum = 0.0;
              for (int k = lane; k < d; k += 32) sum += (double)wr[k] * (double)xr[k];
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
              if (e == 0 || sum > best) {
                best = sum;
                bj = e;
              }
            }
            if (lane == j) bi = bj;
          }
          if (t < T) {
            route[t] = bi;
            atomicAdd(&s_hist[bi], 1);
          }
        } else if (t < T) {
          route[t] = bi;
          if (E > 1 && !(b1 - b2 > 2.f * eps * s_xb[r])) {  // queued for k_router_recheck
            const int k = atomicAdd(count, 1);
            list[k] = t;
          }
        }
      }
      named_bar_sync(1, kRfConvThreads);
      if (hist_cc != nullptr) {  // the tile is one 128-token chunk of the execution map
        for (int e = ct; e < E; e += kRfConvThreads) {
          hist_cc[(size_t)u * E + e] = s_hist[e];
          s_hist[e] = 0;
        }
        named_bar_sync(1, kRfConvThreads);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) RT_STAMP(75);
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kRxTmemCols);
  }
#endif
}

template <int EG>
static int launch_router_fused_tx(const float* x, int ldx, int T, int d, const void* w_hl, const float* w_abs, int E,
                                  int32_t* route, int32_t* count, int32_t* list, float eps, cudaStream_t st,
                                  const float* w32 = nullptr, int32_t* hist_cc = nullptr) {
  CUtensorMap tb, tx;
  int rc = make_tmap_bf16(&tb, w_hl, EG, 2 * d, 2 * d, EG);
  if (rc) return rc;
  rc = make_tmap_f32(&tx, x, T, d, ldx, kBlockM);
  if (rc) return rc;
  auto kern = k_router_fused_tx<EG>;
  const int smem = RxSmem<EG>::kBytes;
  static_assert(RxSmem<128>::kBytes <= 232448, "router smem");
  static bool configured = false;
  if (!configured) {
    MP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  if (hist_cc == nullptr) MP_CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int32_t), st));
  const int units = cdiv(T, kBlockM);
  MP_CUDA_TRY(launch_pdl(kern, dim3(units < num_sms() ? units : num_sms()), dim3(kRouterThreads), smem, st, tb, tx, T,
                         d, w_abs, E, route, eps, count, list, x, ldx, w32, hist_cc));
  return MP_OK;
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
  griddep_launch_dependents();
  griddep_wait();
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
  MP_CUDA_TRY(launch_pdl(k_router_recheck, dim3(num_sms()), dim3(256), 0, st, x, ldx, d, w_f32, E, rw.count, rw.list, route));
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
  if ((Eg == 64 || Eg == 128) && ldx % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    const int rc = Eg == 128
                       ? launch_router_fused_tx<128>(x, ldx, T, d, w_hl, w_abs, E, route, rw.count, rw.list, kRouterEps, st)
                       : launch_router_fused_tx<64>(x, ldx, T, d, w_hl, w_abs, E, route, rw.count, rw.list, kRouterEps, st);
    if (rc) return rc;
    MP_CUDA_TRY(launch_pdl(k_router_recheck, dim3(num_sms()), dim3(256), 0, st, x, ldx, d, w_f32, E, rw.count, rw.list, route));
    MP_CUDA_TRY(cudaGetLastError());
    return MP_OK;
  }
  // any other layout (Eg = 256, unaligned rows): split pre-pass + split-bf16 GEMM + recheck
  k_router_prep<<<cdiv(T * 32, 256), 256, 0, st>>>(x, ldx, T, d, w_abs, (__nv_bfloat16*)rw.xhl, rw.xb, rw.count);
  return route_gemm(x, ldx, T, d, w_hl, w_f32, E, Eg, route, rw, kRouterEps, st);
}

// Exact routing with the fp64 re-decision of near ties done inside the router's epilogue
// (warp-cooperative, the arithmetic of k_router_recheck), plus each 128-token tile's expert
// histogram written to chunk_hist[tile][e] -- the first stage of mp_exec_map, so
// mp_exec_map_hist can start from the chunk prefixes. One launch for routing + histogram.
extern "C" int mp_route_top1_hist(const float* x, int ldx, int T, int d, const void* w_hl, const float* w_f32,
                                  const float* w_abs, int E, int Eg, int32_t* route, int32_t* chunk_hist, void* ws,
                                  size_t ws_bytes, void* stream) {
  ROUTER_CHECKS();
  MP_REQUIRE((Eg == 64 || Eg == 128) && ldx % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                 chunk_hist != nullptr,
             MP_ERR_CONFIG, "mp_route_top1_hist: needs Eg in {64, 128}, ldx %% 4 == 0, 16-byte aligned x");
  cudaStream_t st = (cudaStream_t)stream;
  const RouterWs rw(ws, T, d);
  return Eg == 128 ? launch_router_fused_tx<128>(x, ldx, T, d, w_hl, w_abs, E, route, rw.count, rw.list, kRouterEps,
                                                 st, w_f32, chunk_hist)
                   : launch_router_fused_tx<64>(x, ldx, T, d, w_hl, w_abs, E, route, rw.count, rw.list, kRouterEps, st,
                                                w_f32, chunk_hist);
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

#ifdef MP_DIAG
extern "C" __attribute__((visibility("default"))) int mp_debug_router_trace(unsigned long long* out) {
  MP_CUDA_TRY(cudaMemcpyFromSymbol(out, mp::g_rt, sizeof(mp::g_rt)));
  return MP_OK;
}
#endif
