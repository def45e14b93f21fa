// Cluster variant of the grouped tcgen05 GEMM with the A tile MULTICAST across the
// cluster (sm_100a).
//
// Why: in the grouped expert GEMMs every 128-row piece is multiplied by all N slices
// of its expert's weights, and the single-CTA kernel re-reads the piece's A rows from
// L2 once per slice (GEMM2: the 128 x 3072 hidden rows, 3 times; GEMM1: the 128 x 768
// token rows, 12 times). Removing the A loads altogether takes 27 us off GEMM2 and
// 9 us off GEMM1 at T = 16k (measured), so the operand traffic through L2, not the
// tensor core, is what those microseconds are. Here a cluster of CL CTAs computes CL
// consecutive slices of the SAME piece: CTA 0 loads each A k-block once with
// .multicast::cluster into every CTA's shared memory; each CTA loads its own B slice.
//
// Protocol per smem stage s (CUTLASS-style multicast pipeline):
//   * full[s] (every CTA, count 1): the CTA's producer arms it with A + B bytes; the
//     multicast A copy and the CTA's own B copy complete_tx on it;
//   * empty[s]: each CTA's MMA commits with multicast to its own empty[s] and to CTA 0's;
//     CTA 0's empty[s] therefore counts CL arrivals (all CTAs are done reading stage s)
//     before CTA 0 overwrites A in every CTA; other CTAs count 1 (their own B);
//   * cluster-wide barrier after mbarrier init and before exit (peers arrive / write
//     into this CTA's shared memory).
// MMA (cta_group::1, 128 x BN) and epilogue are those of k_umma_gemm; results are
// bitwise identical.
#pragma once
#include "gemm_sm100.cuh"

namespace mp {

__device__ __forceinline__ uint32_t mc_cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void mc_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load multicast to every CTA in `mask` (same smem offset, complete_tx on each CTA's
// barrier at the same offset).
__device__ __forceinline__ void tma_load_2d_mc(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
// Arrive (when this thread's prior tcgen05 ops complete) on the barrier at the same
// offset in every CTA of `mask`.
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::
                   "r"(smem_u32(bar)),
               "h"(mask)
               : "memory");
}

// Scheduler concept (cluster form): num_units() counts CLUSTER units;
// unit(u, rank) is CTA `rank`'s Unit (same A rows for every rank, own B slice);
// prepare(int*) as in k_umma_gemm.
template <int BN, int STAGES, int CL, class Sched, class Epi>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_umma_gemm_mc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, Sched sched_in,
                   Epi epi) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  using L = GemmSmem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* svec = reinterpret_cast<float*>(smem + L::kVecOffset);
  uint32_t* scratch_all = reinterpret_cast<uint32_t*>(smem + L::kScratchOffset);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = mc_cluster_ctarank();
  constexpr uint16_t kAll = (1u << CL) - 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], rank == 0 ? CL : 1);
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
  Sched sched = sched_in;
  sched.prepare(reinterpret_cast<int*>(smem + L::kPrepOffset));
  tc_fence_before();
  mc_cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  const int nunits = sched.num_units();
  const int nkb = sched.num_kb();

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      const uint64_t pol_stream = policy_evict_first();
      uint32_t stage = 0, phase = 0;
      Unit Un = cid < nunits ? sched.unit(cid, rank) : Unit{};
      for (int u = cid; u < nunits; u += ncl) {
        const Unit U = Un;
        if (u + ncl < nunits) Un = sched.unit(u + ncl, rank);
        const int mtiles = (U.rows + kBlockM - 1) / kBlockM;
        for (int mt = 0; mt < mtiles; ++mt) {
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);  // rank 0: every CTA released the stage
            uint8_t* sa = smem + stage * L::kStageBytes;
            uint8_t* sb = sa + L::kABytes;
            mbar_arrive_expect_tx(&full[stage], L::kStageBytes);
            if (rank == 0)
              tma_load_2d_mc(sa, &tmA, &full[stage], sched.a_kcol(kb), U.a_row + mt * kBlockM, kAll);
            if constexpr (Sched::kStreamB)
              tma_load_2d_hint(sb, &tmB, &full[stage], sched.b_kcol(kb), U.b_row + sched.b_krow(kb), pol_stream);
            else
              tma_load_2d(sb, &tmB, &full[stage], sched.b_kcol(kb), U.b_row + sched.b_krow(kb));
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = KindBF16::idesc(kBlockM, BN);
      const uint16_t rel = static_cast<uint16_t>((1u << rank) | 1u);  // own stage + CTA 0's A gate
      uint32_t stage = 0, phase = 0, tile = 0;
      Unit Un = cid < nunits ? sched.unit(cid, rank) : Unit{};
      for (int u = cid; u < nunits; u += ncl) {
        const Unit U = Un;
        if (u + ncl < nunits) Un = sched.unit(u + ncl, rank);
        const int mtiles = (U.rows + kBlockM - 1) / kBlockM;
        for (int mt = 0; mt < mtiles; ++mt, ++tile) {
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
            umma_commit_mc(&empty[stage], rel);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit(&tfull[as]);
        }
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int r = q * 32 + lane;
    constexpr bool split = Epi::kSplitCols;
    constexpr int NC = split ? BN / 2 : BN;
    const bool active = split || half == 0;
    const int c0 = split ? half * (BN / 2) : 0;
    uint32_t tile = 0;
    Unit Un = cid < nunits ? sched.unit(cid, rank) : Unit{};
    for (int u = cid; u < nunits; u += ncl) {
      const Unit U = Un;
      if (u + ncl < nunits) Un = sched.unit(u + ncl, rank);
      const int mtiles = (U.rows + kBlockM - 1) / kBlockM;
      for (int mt = 0; mt < mtiles; ++mt, ++tile) {
        const uint32_t as = tile & 1, aph = (tile >> 1) & 1;
        mbar_wait(&tfull[as], aph);
        tc_fence_after();
        if (active) {
          const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + as * BN + c0;
          epi.template run<NC>(U, mt, r, taddr, c0, svec + (tile & 1) * BN + c0,
                               scratch_all + (warp - 4) * L::kScratchWordsPerWarp);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[as]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  mc_cluster_sync();  // no CTA leaves while a peer may still multicast into / arrive on it
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * BN);
  }
#endif
}

// Grouped GEMM over replica-segment pieces, cluster form: a cluster unit is
// (expert, group of CL consecutive BN slices, piece), ordered expert-major, then slice
// group, then piece; CTA `rank` computes slice group * CL + rank of the piece.
template <int CL>
struct SegMcSched {
  static constexpr bool kStreamB = true;
  const int32_t* piece_row;
  const int32_t* piece_rows;
  const int32_t* exp_begin;  // E + 1 (staged in shared memory by prepare)
  int E, n_tiles, bn, n_per_expert, kb;
  int b_tiled;
  __device__ void prepare(int* tab) {
    if (E + 1 > 1025) return;
    for (int e = threadIdx.x; e <= E; e += blockDim.x) tab[e] = exp_begin[e];
    __syncthreads();
    exp_begin = tab;
  }
  __device__ int groups() const { return n_tiles / CL; }
  __device__ int num_units() const { return exp_begin[E] * groups(); }
  __device__ Unit unit(int u, int rank) const {
    const int G = groups();
    int lo = 0, hi = E;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (exp_begin[mid] * G <= u) lo = mid; else hi = mid;
    }
    const int b = exp_begin[lo], cnt = exp_begin[lo + 1] - b;
    const int local = u - b * G;
    const int g = local / cnt;
    const int p = b + (local - g * cnt);
    const int nt = g * CL + rank;
    const int brow = b_tiled ? (lo * n_tiles + nt) * kb * bn : lo * n_per_expert + nt * bn;
    return Unit{__ldg(&piece_row[p]), __ldg(&piece_rows[p]), brow, nt * bn};
  }
  __device__ int num_kb() const { return kb; }
  __device__ int a_kcol(int k) const { return k * kBlockK; }
  __device__ int b_kcol(int k) const { return b_tiled ? 0 : k * kBlockK; }
  __device__ int b_krow(int k) const { return b_tiled ? k * bn : 0; }
};

}  // namespace mp
