// Multi-tile grouped GEMM for the expert FFN (tcgen05, sm_100a).
//
// Why: at T = 16k the grouped FFN GEMMs are bound by the bytes the SMs pull
// through L2 into shared memory (ncu: ~13-14 TB/s of LTS sectors for both
// GEMMs, DRAM at 57-62 %, tensor pipe at 41-48 %), not by DRAM. A 128 x 256
// tile per unit re-reads the 256-row weight slice once per 128-row piece and
// the piece's rows once per weight slice. A unit here computes TWO 128 x 256
// accumulator tiles (all 512 TMEM columns) from one stream of k-blocks:
//   "MM" unit: two pieces of the same expert x one weight slice  (B read once)
//   "NN" unit: one piece x two weight slices                    (A read once)
// which cuts the operand bytes per MMA flop by 25 % on the Switch-base-128
// workload (hot experts have many pieces, cold experts one).
//
// Shared memory is a ring of 16 KB granules (one 128 x 64 bf16 A tile, or one
// 128-row half of a 256-row B slice); a k-block of a unit takes 3 (1x1),
// 4 (MM) or 5 (NN) granules, so the ring depth adapts to the unit kind. Every
// granule has its own full/empty mbarrier; producer and MMA issuer walk the
// same granule sequence, so the parity of granule g is (g / kRing) & 1.
// The two 128-row halves of a B slice always sit in an aligned granule pair
// (the producer skips one granule when needed), so every MMA is M=128, N=256,
// K=16 exactly as in the single-tile kernel: bitwise identical results.
//
// Roles are those of k_umma_gemm (gemm_sm100.cuh): warp 0 TMA, warp 1 MMA,
// warp 2 TMEM, warps 4..11 two epilogue warpgroups; the TMEM accumulator slots
// are a 2-entry ring, a 2-tile unit waits for both.
#pragma once
#include "common.cuh"
#include "gemm_sm100.cuh"

namespace mp {

constexpr int kMtGranule = 16384;
constexpr int kMtRing = 12;
constexpr int kMtMaxE = 1024;
constexpr int kMtBN = 256;

struct MtSmem {
  static constexpr int kRingBytes = kMtRing * kMtGranule;
  static constexpr int kBarOffset = kRingBytes;  // full[R], empty[R], tfull[2], tempty[2]
  static constexpr int kSlotOffset = kBarOffset + (2 * kMtRing + 4) * 8;
  static constexpr int kPrefixOffset = kSlotOffset + 16;                          // int[kMtMaxE + 1]
  static constexpr int kRedOffset = kPrefixOffset + ((kMtMaxE + 1) * 4 + 15) / 16 * 16;  // int[33]
  static constexpr int kScratchOffset = kRedOffset + 144;
  static constexpr int kBytes = kScratchOffset + kEpiWarps * 640 * 4 + 1024;
};

struct MtUnit {
  int na, nb;  // A tiles (pieces) x B slices, na * nb <= 2
  int a_row[2], rows[2];
  int b_row[2], n0[2];
};

// Units per expert e with p pieces and nt BN-slices:
//   MM units (pieces 2q, 2q+1; slice s), s-major then q   -> (p / 2) * nt
//   NN units for an odd last piece (slices 2s, 2s+1)      -> ceil(nt / 2)
// Expert-major order: concurrent CTAs share one weight slice through L2.
struct FfnMtSched {
  const int32_t* piece_row;
  const int32_t* piece_rows;
  const int32_t* exp_begin;  // E + 1 entries (pieces of expert e: [exp_begin[e], exp_begin[e+1]))
  int E, n_tiles, kb, n_per_expert;
  int b_tiled;  // B pre-tiled as [E][n_tiles][kb][256 rows][64 cols]
  int single;   // 1: one tile per unit (pieces x slices), for A/B comparisons

  __device__ int units_of(int e) const {
    const int p = exp_begin[e + 1] - exp_begin[e];
    if (single) return p * n_tiles;
    return (p >> 1) * n_tiles + (p & 1) * ((n_tiles + 1) >> 1);
  }
  __device__ int slice_row(int e, int nt) const {
    return b_tiled ? (e * n_tiles + nt) * kb * kMtBN : e * n_per_expert + nt * kMtBN;
  }
  // pre: exclusive prefix of units_of over experts (E + 1 entries, smem)
  __device__ MtUnit unit(int u, const int* pre) const {
    int lo = 0, hi = E;  // pre[lo] <= u < pre[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pre[mid] <= u) lo = mid; else hi = mid;
    }
    const int e = lo, b = exp_begin[e], p = exp_begin[e + 1] - b;
    int local = u - pre[e];
    MtUnit U;
    if (single) {
      const int s = local / p, q = local - s * p;
      U.na = U.nb = 1;
      U.a_row[0] = U.a_row[1] = piece_row[b + q];
      U.rows[0] = U.rows[1] = piece_rows[b + q];
      U.b_row[0] = U.b_row[1] = slice_row(e, s);
      U.n0[0] = U.n0[1] = s * kMtBN;
      return U;
    }
    const int mm = (p >> 1) * n_tiles;
    if (local < mm) {
      const int half_p = p >> 1;
      const int s = local / half_p, q = local - s * half_p;
      U.na = 2;
      U.nb = 1;
      U.a_row[0] = __ldg(&piece_row[b + 2 * q]);
      U.rows[0] = __ldg(&piece_rows[b + 2 * q]);
      U.a_row[1] = __ldg(&piece_row[b + 2 * q + 1]);
      U.rows[1] = __ldg(&piece_rows[b + 2 * q + 1]);
      U.b_row[0] = U.b_row[1] = slice_row(e, s);
      U.n0[0] = U.n0[1] = s * kMtBN;
    } else {
      local -= mm;
      const int s0 = 2 * local;
      U.na = 1;
      U.nb = (s0 + 1 < n_tiles) ? 2 : 1;
      U.a_row[0] = U.a_row[1] = piece_row[b + p - 1];
      U.rows[0] = U.rows[1] = piece_rows[b + p - 1];
      U.b_row[0] = slice_row(e, s0);
      U.n0[0] = s0 * kMtBN;
      U.b_row[1] = slice_row(e, s0 + 1);
      U.n0[1] = (s0 + 1) * kMtBN;
    }
    return U;
  }
  // coordinates of the 128-row half h of the B slice starting at row brow, k-block k
  __device__ int b_col(int k) const { return b_tiled ? 0 : k * kBlockK; }
  __device__ int b_row(int brow, int k, int h) const { return brow + (b_tiled ? k * kMtBN : 0) + h * 128; }
};

template <class Epi>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_ffn_mt(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, FfnMtSched sched,
             Epi epi) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  using L = MtSmem;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + kMtRing;
  uint64_t* tfull = empty + kMtRing;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::kSlotOffset);
  int* pre = reinterpret_cast<int*>(smem + L::kPrefixOffset);
  int* red = reinterpret_cast<int*>(smem + L::kRedOffset);
  uint32_t* scratch_all = reinterpret_cast<uint32_t*>(smem + L::kScratchOffset);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < kMtRing; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 2 * kMtBN);
  griddep_launch_dependents();
  griddep_wait();
  const int E = sched.E;
  for (int e = threadIdx.x; e < E; e += blockDim.x) pre[e] = sched.units_of(e);
  __syncthreads();
  const int nunits = block_exclusive_scan(pre, E, red);
  if (threadIdx.x == 0) pre[E] = nunits;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int nkb = sched.kb;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      const uint64_t pol_w = policy_evict_first();  // weights stream once per step
      uint32_t slot = 0, phase = 0;
      auto take = [&]() -> uint32_t {
        const uint32_t s = slot;
        mbar_wait(&empty[s], phase ^ 1);
        mbar_arrive_expect_tx(&full[s], kMtGranule);
        if (++slot == kMtRing) {
          slot = 0;
          phase ^= 1;
        }
        return s;
      };
      MtUnit Un = blockIdx.x < nunits ? sched.unit(blockIdx.x, pre) : MtUnit{};
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const MtUnit U = Un;
        if (u + (int)gridDim.x < nunits) Un = sched.unit(u + gridDim.x, pre);  // consumed next iteration
        for (int kb = 0; kb < nkb; ++kb) {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            if (i < U.na) {
              const uint32_t s = take();
              tma_load_2d(smem + s * kMtGranule, &tmA, &full[s], kb * kBlockK, i ? U.a_row[1] : U.a_row[0]);
            }
          }
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (j < U.nb) {
              const int brow = j ? U.b_row[1] : U.b_row[0];
              if (slot & 1) {  // keep the two halves of a B slice in adjacent granules: skip one
                const uint32_t s = slot;
                mbar_wait(&empty[s], phase ^ 1);
                mbar_arrive(&full[s]);
                if (++slot == kMtRing) {
                  slot = 0;
                  phase ^= 1;
                }
              }
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const uint32_t s = take();
                tma_load_2d_hint(smem + s * kMtGranule, &tmB, &full[s], sched.b_col(kb), sched.b_row(brow, kb, h),
                                 pol_w);
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(kBlockM, kMtBN);
      uint32_t slot = 0, phase = 0, tile = 0;
      auto next = [&]() -> uint32_t {
        const uint32_t s = slot;
        mbar_wait(&full[s], phase);
        if (++slot == kMtRing) {
          slot = 0;
          phase ^= 1;
        }
        return s;
      };
      MtUnit Un = blockIdx.x < nunits ? sched.unit(blockIdx.x, pre) : MtUnit{};
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const MtUnit U = Un;
        if (u + (int)gridDim.x < nunits) Un = sched.unit(u + gridDim.x, pre);  // consumed next iteration
        const int ntile = U.na * U.nb;
        for (int t = 0; t < ntile; ++t) mbar_wait(&tempty[(tile + t) & 1], (((tile + t) >> 1) & 1) ^ 1);
        tc_fence_after();
        const bool two = ntile == 2;
        const uint32_t d0 = tmem_base + (tile & 1) * kMtBN, d1 = tmem_base + ((tile + 1) & 1) * kMtBN;
        for (int kb = 0; kb < nkb; ++kb) {
          // granules in producer order: A0 [A1] [skip] B0 (2 adjacent) [[skip] B1 (2 adjacent)]
          const uint32_t a0 = next();
          const uint32_t a1 = U.na == 2 ? next() : a0;
          if (slot & 1) umma_commit(&empty[next()]);
          const uint32_t b0 = next();
          next();
          uint32_t b1 = b0;
          if (U.nb == 2) {
            if (slot & 1) umma_commit(&empty[next()]);
            b1 = next();
            next();
          }
          tc_fence_after();
          const uint64_t da0 = sw128_kmajor_desc(smem_u32(smem + a0 * kMtGranule));
          const uint64_t da1 = sw128_kmajor_desc(smem_u32(smem + a1 * kMtGranule));
          const uint64_t db0 = sw128_kmajor_desc(smem_u32(smem + b0 * kMtGranule));
          const uint64_t db1 = sw128_kmajor_desc(smem_u32(smem + b1 * kMtGranule));
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t acc = (kb | k) != 0;
            umma_bf16(d0, da0 + 2 * k, db0 + 2 * k, idesc, acc);
            if (two) umma_bf16(d1, da1 + 2 * k, db1 + 2 * k, idesc, acc);  // MM: (A1, B0); NN: (A0, B1)
          }
          umma_commit(&empty[a0]);
          if (U.na == 2) umma_commit(&empty[a1]);
          umma_commit(&empty[b0]);
          umma_commit(&empty[b0 + 1]);
          if (U.nb == 2) {
            umma_commit(&empty[b1]);
            umma_commit(&empty[b1 + 1]);
          }
        }
        for (int t = 0; t < ntile; ++t) umma_commit(&tfull[(tile + t) & 1]);
        tile += ntile;
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int r = q * 32 + lane;
    const int c0 = half * (kMtBN / 2);
    uint32_t* scratch = scratch_all + (warp - 4) * 640;
    uint32_t tile = 0;
    MtUnit Un = blockIdx.x < nunits ? sched.unit(blockIdx.x, pre) : MtUnit{};
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      const MtUnit U = Un;
      if (u + (int)gridDim.x < nunits) Un = sched.unit(u + gridDim.x, pre);
      const int ntile = U.na * U.nb;
      for (int t = 0; t < ntile; ++t, ++tile) {
        const uint32_t as = tile & 1, aph = (tile >> 1) & 1;
        mbar_wait(&tfull[as], aph);
        tc_fence_after();
        // second tile: MM -> (A1, B0), NN -> (A0, B1); unit() fills the unused entries with copies
        const Unit V = (t == 0) ? Unit{U.a_row[0], U.rows[0], U.b_row[0], U.n0[0]}
                                : (U.na == 2 ? Unit{U.a_row[1], U.rows[1], U.b_row[0], U.n0[0]}
                                             : Unit{U.a_row[0], U.rows[0], U.b_row[1], U.n0[1]});
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + as * kMtBN + c0;
        epi.template run<kMtBN / 2>(V, 0, r, taddr, c0, nullptr, scratch);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[as]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * kMtBN);
  }
#endif
}

}  // namespace mp
