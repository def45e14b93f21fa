// K7 + K8 fused: the whole expert FFN  y = V_e relu(U_e x)  of one replica slot in ONE
// persistent tcgen05 kernel, with the hidden activation kept on chip.
//
// Reference: expert_forward  v @ relu(u @ x)      (src/router_oracle.py:101-111)
//            _run_layers     stream[t] += delta   (src/router_oracle.py:127-134)
//
// At Switch-base shapes with 128 experts a layer is bound by streaming 1.2 GB of expert
// weights from HBM (~128 tokens per expert). The kernel is therefore written "weights as
// the M operand" (swap-AB) so a cold expert's few tokens are a narrow N (16..64), not a
// padded 128-row tile, and the hidden activation never leaves the SM:
//
//   work item  = one replica slot (reference: a slot is one server draining its queue,
//                src/simulator.py:66-81) = a contiguous run of permuted rows of expert e,
//                processed as NT-token tiles by one CTA; items are handed out by an atomic
//                ticket in slot order (expert-major, so the CTAs working on the replicas of a
//                hot expert stream the same weight chunks through L2 at the same time).
//   per tile   = X (NT tokens x d, bf16) staged once in smem (GEMM1 B operand, K-major);
//                for each 128-row chunk c of d_ff:
//                  GEMM1  D1[c&1] (128 x N, TMEM) = U_e[c] (128 x d)  . X^T
//                  epilogue: relu -> bf16 -> H[c&1] in smem (GEMM2 B operand, MN-major)
//                  GEMM2  D2[b]   (128 x N, TMEM) += V_e[b, c] (128 x 128) . H[c&1]   b < d/128
//                then D2 -> registers -> quad-lane transpose -> red.global.add.v4.f32 into the
//                fp32 residual stream (top-1: every element gets exactly one addend, so the
//                update is rounded once and cannot vary between runs).
//   MMA order  = G1(0), G1(1), G2(0), G1(2), G2(1), ...: the relu/convert of chunk c overlaps
//                GEMM1 of chunk c+1.
//
// Roles (384 threads, one CTA per SM): warp 0 = TMA producer (X tile + one ring of 16 KB weight
// boxes: U chunk c, then V chunk c-1, ...), warp 1 = MMA issuer, warp 2 = TMEM allocator,
// warp 3 = item scheduler (ticket + slot decode), warps 4..11 = epilogue.
// TMEM: D2 = (d/128) x NT columns, D1 = 2 x NT columns (<= 512).
// Weights are pre-tiled at 128 rows (mp_tile_kmajor BN = 128): U as [E][F/128][d/64][128][64],
// V as [E][d/128][F/64][128][64], so every weight box is one contiguous 16 KB burst.
#include "epilogues.cuh"
#include "launch.cuh"

#include <stdlib.h>

extern "C" size_t mp_ffn_workspace_bytes(int T, int dp, int Fp);

namespace mp {

constexpr int kFusedThreads = 384;
constexpr int kBoxBytes = 128 * 64 * 2;  // one 128-row x 64-col bf16 weight box
constexpr int kItemSlots = 4;

struct FusedArgs {
  const int32_t* piece_row;
  const int32_t* piece_rows;
  const int32_t* exp_begin;  // E + 1
  const int32_t* tok_of_row;
  float* x;                  // residual stream (T x ldx fp32), updated in place
  int* ticket;               // self-resetting work counter (zero before the first launch)
  int E, d, F, ldx, stages, store;
  int prefetch;  // weight boxes prefetched into L2 ahead of the shared-memory ring (0: none)
  int dbg;       // 1: accumulate per-role wait cycles into g_fused_dbg (diagnostics)
  int diag;      // profiling only (wrong results): bit 0 K-major hidden descriptor, bit 1 no GEMM2
                 // MMAs, bit 2 no GEMM1 MMAs
};

// per-CTA wait-cycle counters of the last debug launch: [cta][16]
static __device__ unsigned long long g_fused_dbg[1024 * 16];

// MN-major SWIZZLE_128B operand: rows of 64 bf16 (128 B) along MN, 8 K-rows per 1024 B atom
// (SBO), atoms along MN lbo bytes apart.
__device__ __forceinline__ uint64_t sw128_mnmajor_desc(uint32_t saddr, uint32_t lbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

__device__ __forceinline__ float sel4(float a0, float a1, float a2, float a3, int s) {
  return s == 0 ? a0 : (s == 1 ? a1 : (s == 2 ? a2 : a3));
}

template <int NT>
__global__ void __launch_bounds__(kFusedThreads, 1)
    k_ffn_fused(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmU,
                const __grid_constant__ CUtensorMap tmV, FusedArgs a) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int KB = a.d / 64;   // GEMM1 k-blocks (X tile boxes)
  const int NB = a.d / 128;  // GEMM2 output blocks (D2 accumulators)
  const int NC = a.F / 128;  // d_ff chunks
  const int S = a.stages;
  constexpr int kXBox = NT * 128;        // one X k-block: NT rows x 128 B
  constexpr int kHBuf = 128 * NT * 2;    // one H buffer: 128 K-rows x NT tokens (bf16)
  constexpr int kHAtom = 128 * 128;      // 64 tokens x 128 K-rows
  uint8_t* sx = smem;
  uint8_t* sh = sx + KB * kXBox;
  uint8_t* ring = sh + 2 * kHBuf;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + S * kBoxBytes);
  uint64_t* full = bars;
  uint64_t* empty = full + S;
  uint64_t* xfull = empty + S;
  uint64_t* xempty = xfull + 1;
  uint64_t* t1full = xempty + 1;   // [2]
  uint64_t* t1empty = t1full + 2;  // [2]
  uint64_t* hfull = t1empty + 2;   // [2]
  uint64_t* hempty = hfull + 2;    // [2]
  uint64_t* d2full = hempty + 2;
  uint64_t* d2empty = d2full + 1;
  uint64_t* ifull = d2empty + 1;      // [kItemSlots]
  uint64_t* iempty = ifull + kItemSlots;
  uint64_t* want = iempty + kItemSlots;  // producer -> scheduler: draw the next slot now
  int4* items = reinterpret_cast<int4*>(want + 2);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(items + kItemSlots);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned long long dbgc[12] = {0};
  const long long dbg_t0 = clock64();
#define DBG_WAIT(k, stmt)                          \
  do {                                             \
    const long long _t = a.dbg ? clock64() : 0;    \
    stmt;                                          \
    if (a.dbg) dbgc[k] += clock64() - _t;          \
  } while (0)
  if (threadIdx.x == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmU);
    tma_prefetch(&tmV);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(xfull, 1);
    mbar_init(xempty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&t1full[i], 1);
      mbar_init(&t1empty[i], kEpiWarps);
      mbar_init(&hfull[i], kEpiWarps);
      mbar_init(&hempty[i], 1);
    }
    mbar_init(d2full, 1);
    mbar_init(d2empty, kEpiWarps);
    for (int i = 0; i < kItemSlots; ++i) {
      mbar_init(&ifull[i], 1);
      mbar_init(&iempty[i], 2 + kEpiWarps);  // producer, MMA, epilogue warps
    }
    mbar_init(want, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t d1_col = NB * NT;

  if (warp == 3) {
    if (lane == 0) {
      // ------------------------------------------------------------ item scheduler
      const int npieces = __ldg(&a.exp_begin[a.E]);
      int slot = 0;
      uint32_t ph = 0;
      int e = 0;
      uint32_t wph = 0;
      bool first = true;
      for (;;) {
        // greedy list scheduling: a CTA holds one slot at a time and draws the next one when its
        // producer starts the last d_ff chunk of the current slot (a scheduler that ran ahead would
        // let the first CTAs take all the work)
        if (!first) {
          DBG_WAIT(10, mbar_wait(want, wph));
          wph ^= 1;
        }
        const int t = atomicAdd(a.ticket, 1);
        int4 it = make_int4(-1, 0, 0, 0);
        if (t < npieces) {
          const int rows = __ldg(&a.piece_rows[t]);
          if (rows <= 0) {
            first = true;  // nothing pushed: draw again without waiting
            continue;
          }
          // expert of piece t: exp_begin is non-decreasing; this CTA's tickets increase
          int lo = e, hi = a.E;  // exp_begin[lo] <= t < exp_begin[hi]
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(&a.exp_begin[mid]) <= t) lo = mid; else hi = mid;
          }
          e = lo;
          it = make_int4(t, e, __ldg(&a.piece_row[t]), rows);
        } else if (t == npieces + (int)gridDim.x - 1) {
          atomicExch(a.ticket, 0);  // last draw of the launch: ready for the next one
        }
        first = false;
        mbar_wait(&iempty[slot], ph ^ 1);
        items[slot] = it;
        mbar_arrive(&ifull[slot]);
        if (++slot == kItemSlots) {
          slot = 0;
          ph ^= 1;
        }
        if (it.x < 0) break;
      }
    }
  } else if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      const uint64_t pol_stream = policy_evict_first();
      uint32_t stage = 0, phase = 0, xt = 0;
      int slot = 0;
      uint32_t ph = 0;
      // box sequence of a tile: U(0), U(1), V(0), U(2), V(1), ..., V(NC-1); box i of it in L2 ahead
      const int per_u = KB, per_v = 2 * NB, nbox = NC * (per_u + per_v);
      auto box_of = [&](int e, int i, const CUtensorMap** m) -> int {
        // position i in the sequence -> (map, row)
        if (i < per_u) {
          *m = &tmU;
          return ((e * NC) * KB + i) * 128;
        }
        const int j = i - per_u, c = j / (per_u + per_v) + 1, w = j % (per_u + per_v);
        if (w < per_u && c < NC) {
          *m = &tmU;
          return ((e * NC + c) * KB + w) * 128;
        }
        const int v = c < NC ? w - per_u : w;  // after U(NC-1): only V(NC-1) remains
        *m = &tmV;
        return ((e * NB + v / 2) * (2 * NC) + 2 * (c - 1) + (v & 1)) * 128;
      };
      auto load_box = [&](const CUtensorMap* m, int row) {
        DBG_WAIT(0, mbar_wait(&empty[stage], phase ^ 1));
        mbar_arrive_expect_tx(&full[stage], kBoxBytes);
        tma_load_2d_hint(ring + stage * kBoxBytes, m, &full[stage], 0, row, pol_stream);
        if (++stage == (uint32_t)S) {
          stage = 0;
          phase ^= 1;
        }
      };
      for (;;) {
        mbar_wait(&ifull[slot], ph);
        const int4 it = items[slot];
        mbar_arrive(&iempty[slot]);
        if (++slot == kItemSlots) {
          slot = 0;
          ph ^= 1;
        }
        if (it.x < 0) break;
        const int e = it.y;
        for (int r0 = 0; r0 < it.w; r0 += NT) {
          DBG_WAIT(1, mbar_wait(xempty, (xt & 1) ^ 1));
          ++xt;
          mbar_arrive_expect_tx(xfull, KB * kXBox);
          for (int kb = 0; kb < KB; ++kb) tma_load_2d(sx + kb * kXBox, &tmX, xfull, kb * 64, it.z + r0);
          const int P = r0 == 0 ? a.prefetch : 0;  // later tiles of the slot re-read the same boxes
          for (int i = 0; i < P && i < nbox; ++i) {
            const CUtensorMap* m;
            const int row = box_of(e, i, &m);
            tma_prefetch_2d(m, 0, row);
          }
          const bool last_tile = r0 + NT >= it.w;
          const int signal_at = nbox - (KB + 2 * NB);  // first box of the last d_ff chunk
          for (int i = 0; i < nbox; ++i) {
            if (last_tile && i == signal_at) mbar_arrive(want);
            const CUtensorMap* m;
            if (P && i + P < nbox) {
              const int row = box_of(e, i + P, &m);
              tma_prefetch_2d(m, 0, row);
            }
            const int row = box_of(e, i, &m);
            load_box(m, row);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      uint32_t stage = 0, phase = 0, xt = 0, c1 = 0, hc = 0, tt = 0;
      int slot = 0;
      uint32_t ph = 0;
      for (;;) {
        mbar_wait(&ifull[slot], ph);
        const int4 it = items[slot];
        mbar_arrive(&iempty[slot]);
        if (++slot == kItemSlots) {
          slot = 0;
          ph ^= 1;
        }
        if (it.x < 0) break;
        for (int r0 = 0; r0 < it.w; r0 += NT) {
          const int n = min(NT, it.w - r0);
          const int N = (n + 15) & ~15;
          const uint32_t id1 = idesc_bf16_f32(128, N);
          const uint32_t id2 = id1 | (1u << 16);  // B (hidden chunk) MN-major
          DBG_WAIT(6, mbar_wait(xfull, xt & 1));
          ++xt;
          tc_fence_after();
          for (int c = 0; c <= NC; ++c) {
            if (c < NC) {
              const uint32_t buf = c1 & 1;
              DBG_WAIT(5, mbar_wait(&t1empty[buf], ((c1 >> 1) & 1) ^ 1));
              tc_fence_after();
              const uint32_t dt = tmem_base + d1_col + buf * NT;
              for (int kb = 0; kb < KB; ++kb) {
                DBG_WAIT(2, mbar_wait(&full[stage], phase));
                tc_fence_after();
                const uint64_t ad = sw128_kmajor_desc(smem_u32(ring + stage * kBoxBytes));
                const uint64_t bd = sw128_kmajor_desc(smem_u32(sx + kb * kXBox));
                if (!(a.diag & 4)) {
#pragma unroll
                  for (int k = 0; k < 4; ++k) umma_bf16(dt, ad + 2 * k, bd + 2 * k, id1, (kb | k) != 0);
                }
                umma_commit(&empty[stage]);
                if (++stage == (uint32_t)S) {
                  stage = 0;
                  phase ^= 1;
                }
              }
              umma_commit(&t1full[buf]);
              ++c1;
              if (c == NC - 1) umma_commit(xempty);  // X tile no longer read
            }
            if (c >= 1) {
              const uint32_t hb = hc & 1;
              DBG_WAIT(4, mbar_wait(&hfull[hb], (hc >> 1) & 1));
              if (c == 1) mbar_wait(d2empty, (tt & 1) ^ 1);
              tc_fence_after();
              const uint32_t hbase = smem_u32(sh + hb * kHBuf);
              for (int b = 0; b < NB; ++b) {
                const uint32_t dt = tmem_base + b * NT;
                for (int k2 = 0; k2 < 2; ++k2) {
                  DBG_WAIT(3, mbar_wait(&full[stage], phase));
                  tc_fence_after();
                  const uint64_t ad = sw128_kmajor_desc(smem_u32(ring + stage * kBoxBytes));
                  if (!(a.diag & 2)) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                      if (a.diag & 1) {
                        const uint64_t bd = sw128_kmajor_desc(hbase + k2 * NT * 128) + 2 * k;
                        umma_bf16(dt, ad + 2 * k, bd, id1, (c > 1 || k2 > 0 || k > 0) ? 1u : 0u);
                      } else {
                        const uint64_t bd = sw128_mnmajor_desc(hbase + (k2 * 64 + k * 16) * 128, kHAtom);
                        umma_bf16(dt, ad + 2 * k, bd, id2, (c > 1 || k2 > 0 || k > 0) ? 1u : 0u);
                      }
                    }
                  }
                  umma_commit(&empty[stage]);
                  if (++stage == (uint32_t)S) {
                    stage = 0;
                    phase ^= 1;
                  }
                }
              }
              umma_commit(&hempty[hb]);
              ++hc;
            }
          }
          umma_commit(d2full);
          ++tt;
        }
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int q = warp & 3;            // TMEM lane quadrant
    const int half = (warp - 4) >> 2;  // warpgroup: token half of D1, D2 block parity
    const int r = q * 32 + lane;       // row of the 128-row accumulator owned by this thread
    constexpr int kHalfCols = NT / 2;
    uint32_t c1 = 0, tt = 0;
    int slot = 0;
    uint32_t ph = 0;
    const int i4 = lane & 3;
    for (;;) {
      mbar_wait(&ifull[slot], ph);
      const int4 it = items[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&iempty[slot]);
      if (++slot == kItemSlots) {
        slot = 0;
        ph ^= 1;
      }
      if (it.x < 0) break;
      for (int r0 = 0; r0 < it.w; r0 += NT) {
        const int n = min(NT, it.w - r0);
        for (int c = 0; c < NC; ++c, ++c1) {
          const uint32_t buf = c1 & 1;
          DBG_WAIT(7, mbar_wait(&t1full[buf], (c1 >> 1) & 1));
          tc_fence_after();
          uint32_t v[kHalfCols];
          const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + d1_col + buf * NT + half * kHalfCols;
#pragma unroll
          for (int j = 0; j < kHalfCols; j += 32) tmem_ld32_issue(taddr + j, v + j);
#pragma unroll
          for (int j = 0; j < kHalfCols; j += 32) tmem_ld_wait32(v + j);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&t1empty[buf]);
          // relu -> bf16 -> row r of the MN-major SW128 hidden buffer (tokens along the row)
          DBG_WAIT(8, mbar_wait(&hempty[buf], ((c1 >> 1) & 1) ^ 1));
          uint8_t* hrow = sh + buf * kHBuf + r * 128;
#pragma unroll
          for (int g = 0; g < kHalfCols / 8; ++g) {
            const int tok = half * kHalfCols + g * 8;  // first token of this 16-byte group
            uint4 w;
            w.x = pack_bf16x2(fmaxf(__uint_as_float(v[8 * g + 0]), 0.f), fmaxf(__uint_as_float(v[8 * g + 1]), 0.f));
            w.y = pack_bf16x2(fmaxf(__uint_as_float(v[8 * g + 2]), 0.f), fmaxf(__uint_as_float(v[8 * g + 3]), 0.f));
            w.z = pack_bf16x2(fmaxf(__uint_as_float(v[8 * g + 4]), 0.f), fmaxf(__uint_as_float(v[8 * g + 5]), 0.f));
            w.w = pack_bf16x2(fmaxf(__uint_as_float(v[8 * g + 6]), 0.f), fmaxf(__uint_as_float(v[8 * g + 7]), 0.f));
            const int atom = tok >> 6, ch = (tok & 63) >> 3;
            *reinterpret_cast<uint4*>(hrow + atom * kHAtom + ((ch ^ (r & 7)) << 4)) = w;
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(&hfull[buf]);
        }
        // ---- D2 -> residual stream: lane = output row of block b, columns = tokens
        DBG_WAIT(9, mbar_wait(d2full, tt & 1));
        ++tt;
        tc_fence_after();
        for (int cb = 0; cb < NT; cb += 32) {
          if (cb >= n) break;
          const int jt = cb + lane;
          const int tokv = jt < n ? __ldg(&a.tok_of_row[it.z + r0 + jt]) : -1;
          int tk[8];
#pragma unroll
          for (int m = 0; m < 8; ++m) tk[m] = __shfl_sync(0xffffffffu, tokv, 4 * m + i4);
          for (int b = half; b < NB; b += 2) {
            uint32_t u[32];
            tmem_ld32_issue(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + b * NT + cb, u);
            tmem_ld_wait32(u);
            float* colbase = a.x + b * 128 + q * 32 + (lane & ~3);
#pragma unroll
            for (int m = 0; m < 8; ++m) {
              const float a0 = __uint_as_float(u[4 * m]), a1 = __uint_as_float(u[4 * m + 1]);
              const float a2 = __uint_as_float(u[4 * m + 2]), a3 = __uint_as_float(u[4 * m + 3]);
              // 4 x 4 transpose inside each quad of lanes: lane i4 ends with rows (lane & ~3) + 0..3
              // of token 4m + i4
              const float r1 = __shfl_xor_sync(0xffffffffu, sel4(a0, a1, a2, a3, i4 ^ 1), 1);
              const float r2 = __shfl_xor_sync(0xffffffffu, sel4(a0, a1, a2, a3, i4 ^ 2), 2);
              const float r3 = __shfl_xor_sync(0xffffffffu, sel4(a0, a1, a2, a3, i4 ^ 3), 3);
              const float own = sel4(a0, a1, a2, a3, i4);
              // value from quad lane s is: own (s == i4) or r_(s ^ i4)
              float4 o;
              o.x = sel4(own, r1, r2, r3, 0 ^ i4);
              o.y = sel4(own, r1, r2, r3, 1 ^ i4);
              o.z = sel4(own, r1, r2, r3, 2 ^ i4);
              o.w = sel4(own, r1, r2, r3, 3 ^ i4);
              if (tk[m] >= 0) {
                float4* dst = reinterpret_cast<float4*>(colbase + (size_t)tk[m] * a.ldx);
                if (a.store)
                  *dst = o;
                else
                  red_add_v4(dst, o);
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(d2empty);
      }
    }
  }
  if (a.dbg && lane == 0 && blockIdx.x < 1024) {  // one recorder per role: warps 0, 1, 3, 4
    const int base = blockIdx.x * 16;
    if (warp == 0) for (int k : {0, 1}) g_fused_dbg[base + k] = dbgc[k];
    if (warp == 1) for (int k : {2, 3, 4, 5, 6}) g_fused_dbg[base + k] = dbgc[k];
    if (warp == 4) for (int k : {7, 8, 9}) g_fused_dbg[base + k] = dbgc[k];
    if (warp == 3) g_fused_dbg[base + 10] = dbgc[10];
    if (warp == 4) g_fused_dbg[base + 11] = clock64() - dbg_t0;
  }
#undef DBG_WAIT
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
#endif
}

}  // namespace mp

using namespace mp;

// Token tile of the fused kernel for a model width: D2 (d/128 x NT) + D1 (2 x NT) TMEM columns.
extern "C" int mp_ffn_fused_tile(int dp) {
  if (dp % 128 != 0 || dp <= 0) return 0;
  const int nb = dp / 128;
  if (nb <= 2) return 128;
  if (nb <= 6) return 64;
  return 0;
}

template <int NT>
static int launch_fused(const CUtensorMap& tx, const CUtensorMap& tu, const CUtensorMap& tv, const FusedArgs& a0,
                        cudaStream_t st) {
  FusedArgs a = a0;
  const int fixed = (a.d / 64) * NT * 128 + 2 * 128 * NT * 2;
  const int bars = (2 * a.stages + 14 + 2 * kItemSlots) * 8 + kItemSlots * 16 + 16;
  const int limit = 232448 - 1024;
  int stages = (limit - fixed - bars - 256) / kBoxBytes;
  if (stages > 8) stages = 8;
  MP_REQUIRE(stages >= 3, MP_ERR_CONFIG, "ffn_fused: d=%d leaves %d weight stages", a.d, stages);
  a.stages = stages;
  const int smem = fixed + stages * kBoxBytes + (2 * stages + 14 + 2 * kItemSlots) * 8 + kItemSlots * 16 + 16 + 1024;
  auto kern = k_ffn_fused<NT>;
  static int configured = 0;
  if (configured < smem) {
    MP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = smem;
  }
  MP_CUDA_TRY(launch_pdl(kern, dim3(ffn_grid()), dim3(kFusedThreads), smem, st, tx, tu, tv, a));
  return MP_OK;
}

// y[tok_of_row[row]] (+)= V_e relu(U_e xperm[row]) for every row of every replica slot; U / V
// pre-tiled at 128 rows (mp_tile_kmajor BN = 128); xperm = the bf16 permuted rows in the FFN
// workspace (written by mp_ffn_gather or the execution map's rank kernel). flags bit 5: store
// the rows (y[tok] = ...) instead of adding them.
extern "C" int mp_ffn_fused(float* y, int T, int dp, int Fp, int E, const void* u, const void* v, int flags,
                            const int32_t* tok_of_row, const int32_t* piece_row, const int32_t* piece_rows,
                            const int32_t* exp_begin, void* ws, size_t ws_bytes, void* stream) {
  MP_REQUIRE(T >= 1 && E >= 1, MP_ERR_CONFIG, "ffn_fused: bad T/E");
  const int NT = mp_ffn_fused_tile(dp);
  MP_REQUIRE(NT > 0 && Fp % 128 == 0, MP_ERR_CONFIG, "ffn_fused: need d %% 128 == 0, d <= 768, F %% 128 == 0 (d=%d F=%d)",
             dp, Fp);
  MP_REQUIRE(ws_bytes >= mp_ffn_workspace_bytes(T, dp, Fp), MP_ERR_CONFIG, "ffn_fused: workspace too small");
  const __nv_bfloat16* xperm = (const __nv_bfloat16*)ws;
  CUtensorMap tx, tu, tv;
  int rc = make_tmap_bf16(&tx, xperm, T, dp, dp, NT);
  if (!rc) rc = make_tmap_bf16(&tu, u, (uint64_t)E * Fp * (dp / 64), 64, 64, 128);
  if (!rc) rc = make_tmap_bf16(&tv, v, (uint64_t)E * dp * (Fp / 64), 64, 64, 128);
  if (rc) return rc;
  static const int prefetch = [] {
    const char* s = getenv("MP_FUSED_PREFETCH");  // experiment knob (boxes of 16 KB)
    return s ? atoi(s) : 0;
  }();
  static const int dbg = getenv("MP_FUSED_DEBUG") != nullptr;
  static const int diag = [] {
    const char* s = getenv("MP_FUSED_DIAG");
    return s ? atoi(s) : 0;
  }();
  FusedArgs a{piece_row, piece_rows, exp_begin, tok_of_row, y, ffn_ticket(ws, T, dp, Fp), E, dp, Fp, dp, 0,
              (flags >> 5) & 1, prefetch, dbg, diag};
  cudaStream_t st = (cudaStream_t)stream;
  if (NT == 128) return launch_fused<128>(tx, tu, tv, a, st);
  return launch_fused<64>(tx, tu, tv, a, st);
}

// Diagnostics: per-CTA wait cycles of the last mp_ffn_fused launch run with MP_FUSED_DEBUG set:
// out[cta * 16 + k], k = 0 producer ring-empty, 1 producer X-empty, 2 MMA ring-full (GEMM1),
// 3 MMA ring-full (GEMM2), 4 MMA hidden-full, 5 MMA D1-empty, 6 MMA X-full, 7 epilogue D1-full,
// 8 epilogue hidden-empty, 9 epilogue D2-full, 10 scheduler, 11 epilogue warp lifetime.
extern "C" int mp_debug_fused_waits(unsigned long long* out, int n) {
  MP_REQUIRE(n >= 1 && n <= 1024 * 16, MP_ERR_CONFIG, "mp_debug_fused_waits: n in [1, 16384]");
  MP_CUDA_TRY(cudaMemcpyFromSymbol(out, mp::g_fused_dbg, sizeof(unsigned long long) * n));
  return MP_OK;
}
