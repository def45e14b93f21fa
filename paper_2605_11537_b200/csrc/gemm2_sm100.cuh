// CTA-pair (cta_group::2) variant of the tcgen05 GEMM core.
//
// A cluster of two CTAs on one TPC computes a 256 x BN tile with one
// tcgen05.mma.cta_group::2 (M = 256) issued by the leader CTA: each CTA stages
// its own 128 A rows and HALF of the BN B rows, so B traffic into shared memory
// halves compared with two independent 128-row CTAs, and each CTA's TMEM holds
// its 128 accumulator rows. Protocol (as in the CUTLASS sm100 2-SM pipeline):
//   * both CTAs' TMA loads complete on the LEADER's full barrier (peer bit of
//     the barrier address cleared); only the leader arms it, with both CTAs'
//     bytes;
//   * the leader's single MMA thread commits with multicast to the empty
//     barriers (smem ring) and tfull barriers (accumulator) of both CTAs;
//   * both CTAs' epilogue warps release an accumulator stage by arriving on
//     the leader's tempty barrier (remote arrive for the peer).
// For the grouped expert GEMM a cluster work unit is (expert, BN slice, pair of
// pieces): CTA r computes piece 2p + r (pieces are padded to an even count per
// expert, empty pieces have 0 rows and store nothing).
#pragma once
#include "gemm_sm100.cuh"

namespace mp {

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// 2-SM TMA load: data to this CTA's smem, transaction bytes to the leader's barrier.
__device__ __forceinline__ void tma_load_2d_2sm(void* smem_dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                uint64_t policy) {
  const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tmem_alloc_2sm(uint32_t* smem_slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_2sm(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void umma_bf16_2sm(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive (once all prior tcgen05 ops of this thread complete) on the barrier at the
// same smem offset in both CTAs of the pair.
__device__ __forceinline__ void umma_commit_2sm_mc(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

template <int BN, int STAGES>
struct Gemm2Smem {
  static constexpr int kABytes = kBlockM * kBlockK * 2;
  static constexpr int kBBytes = (BN / 2) * kBlockK * 2;  // this CTA's half of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBarOffset = STAGES * kStageBytes;
  static constexpr int kVecOffset = kBarOffset + (2 * STAGES + 4) * 8 + 16;
  static constexpr int kScratchOffset = (kVecOffset + 2 * BN * 4 + 1023) / 1024 * 1024;  // TMA-store boxes
  static constexpr int kScratchWordsPerWarp = 32 * 20;
  static constexpr int kPrepOffset = kScratchOffset + 8 * kScratchWordsPerWarp * 4;
  static constexpr int kBytes = kPrepOffset + 1025 * 4 + 1024;
};

// What every role needs to know about a cluster work unit.
struct PairUnit {
  Unit U;       // this CTA's rows (b_row = tile base, both CTAs)
  int mtiles;   // M tiles of the unit (same for both CTAs)
  int peer_mt;  // M tiles that carry rows in the peer CTA
};

// Scheduler concept (pair form):
//   int num_units() const;                         // cluster work units
//   PairUnit info(int u, int rank) const;          // decoded once per unit per role (prefetched)
//   void prepare(int* table);                      // all threads, before the roles start
//   int num_kb(), a_kcol(kb), b_kcol(kb), b_krow(kb)
template <int BN, int STAGES, class Sched, class Epi>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    k_umma_gemm2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, Sched sched_in,
                 Epi epi, const __grid_constant__ CUtensorMap tmC) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  using L = Gemm2Smem<BN, STAGES>;
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
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * kEpiWarps);  // epilogue warps of both CTAs
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, 2 * BN);
  griddep_launch_dependents();
  griddep_wait();
  Sched sched = sched_in;
  sched.prepare(reinterpret_cast<int*>(smem + L::kPrepOffset));
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int nunits = sched.num_units();
  const int nkb = sched.num_kb();

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer (both CTAs)
      const uint64_t pol_b = Sched::kStreamB ? policy_evict_first() : policy_evict_normal();
      const uint64_t pol_a = policy_evict_normal();
      uint32_t stage = 0, phase = 0;
      PairUnit In = cid < nunits ? sched.info(cid, rank) : PairUnit{};
      for (int u = cid; u < nunits; u += ncl) {
        const PairUnit I = In;
        if (u + ncl < nunits) In = sched.info(u + ncl, rank);  // consumed next iteration
        const Unit U = I.U;
        const int mtiles = I.mtiles;
        // M tiles that carry rows in each CTA: padding pieces / shorter pieces skip their A loads
        const int my_mt = (U.rows + kBlockM - 1) / kBlockM;
        const int peer_mt = I.peer_mt;
        for (int mt = 0; mt < mtiles; ++mt) {
          const bool load_a = mt < my_mt;
          const uint32_t tx = 2 * L::kBBytes + L::kABytes * ((load_a ? 1 : 0) + (mt < peer_mt ? 1 : 0));
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * L::kStageBytes;
            uint8_t* sb = sa + L::kABytes;
            if (leader) mbar_arrive_expect_tx(&full[stage], tx);
            if (load_a) tma_load_2d_2sm(sa, &tmA, &full[stage], sched.a_kcol(kb), U.a_row + mt * kBlockM, pol_a);
            tma_load_2d_2sm(sb, &tmB, &full[stage], sched.b_kcol(kb),
                            U.b_row + sched.b_krow(kb) + (int)rank * (BN / 2), pol_b);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ------------------------------------------------------------ MMA issuer (leader CTA)
      constexpr uint32_t idesc = idesc_bf16_f32(2 * kBlockM, BN);
      uint32_t stage = 0, phase = 0, tile = 0;
      int mt_next = cid < nunits ? sched.info(cid, rank).mtiles : 0;
      for (int u = cid; u < nunits; u += ncl) {
        const int mtiles = mt_next;
        if (u + ncl < nunits) mt_next = sched.info(u + ncl, rank).mtiles;
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
            for (int k = 0; k < kBlockK / 16; ++k)
              umma_bf16_2sm(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
            umma_commit_2sm_mc(&empty[stage]);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit_2sm_mc(&tfull[as]);
        }
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue (both CTAs)
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int r = q * 32 + lane;
    constexpr bool split = Epi::kSplitCols;
    constexpr int NC = split ? BN / 2 : BN;
    const bool active = split || half == 0;
    const int c0 = split ? half * (BN / 2) : 0;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
    uint32_t tile = 0;
    PairUnit In = cid < nunits ? sched.info(cid, rank) : PairUnit{};
    for (int u = cid; u < nunits; u += ncl) {
      const PairUnit I = In;
      if (u + ncl < nunits) In = sched.info(u + ncl, rank);
      const Unit U = I.U;
      const int mtiles = I.mtiles;
      for (int mt = 0; mt < mtiles; ++mt, ++tile) {
        const uint32_t as = tile & 1, aph = (tile >> 1) & 1;
        const float* vec = epi.colvec();
        if (vec != nullptr) {
          const int et = threadIdx.x - 128;
          for (int i = et; i < BN; i += 32 * kEpiWarps) svec[(tile & 1) * BN + i] = __ldg(&vec[U.n0 + i]);
          named_bar_sync(1, 32 * kEpiWarps);
        }
        mbar_wait(&tfull[as], aph);
        tc_fence_after();
        if (active) {
          const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + as * BN + c0;
          if constexpr (TmaStoreOf<Epi>::value)
            epi.template run<NC>(U, mt, r, taddr, c0, svec + (tile & 1) * BN + c0,
                                 scratch_all + (warp - 4) * L::kScratchWordsPerWarp, &tmC);
          else
            epi.template run<NC>(U, mt, r, taddr, c0, svec + (tile & 1) * BN + c0,
                                 scratch_all + (warp - 4) * L::kScratchWordsPerWarp);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader0 + as * 8);
      }
    }
    if constexpr (TmaStoreOf<Epi>::value) {
      if (lane == 0) bulk_wait0();  // this warp's TMA stores complete before the CTA exits
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, 2 * BN);
  }
#endif
}

// Dense pair scheduler: cluster unit = (pair of 128-row M blocks, BN slice).
struct Dense2Sched {
  static constexpr bool kStreamB = false;
  int M, n_tiles, kb, bn;
  __device__ int num_units() const { return ((M + 2 * kBlockM - 1) / (2 * kBlockM)) * n_tiles; }
  __device__ Unit unit(int u, int rank) const {
    const int mbp = u / n_tiles, nb = u - mbp * n_tiles;
    Unit U;
    U.a_row = (2 * mbp + rank) * kBlockM;
    U.rows = min(kBlockM, M - U.a_row);  // <= 0: nothing to store
    U.b_row = nb * bn;
    U.n0 = nb * bn;
    return U;
  }
  __device__ void prepare(int*) {}
  __device__ PairUnit info(int u, int rank) const {
    return PairUnit{unit(u, rank), 1, unit(u, rank ^ 1).rows > 0 ? 1 : 0};
  }
  __device__ int num_kb() const { return kb; }
  __device__ int a_kcol(int k) const { return k * kBlockK; }
  __device__ int b_kcol(int k) const { return k * kBlockK; }
  __device__ int b_krow(int) const { return 0; }
};

// Grouped pair scheduler over piece pairs (pieces padded to an even count per expert).
struct Seg2Sched {
  static constexpr bool kStreamB = true;
  const int32_t* piece_row;
  const int32_t* piece_rows;
  const int32_t* exp_begin;  // E + 1, all even
  int E, n_tiles, bn, n_per_expert, kb;
  int b_tiled;
  __device__ void prepare(int* tab) {
    if (E + 1 > 1025) return;
    for (int e = threadIdx.x; e <= E; e += blockDim.x) tab[e] = exp_begin[e];
    __syncthreads();
    exp_begin = tab;
  }
  __device__ int num_units() const { return (exp_begin[E] >> 1) * n_tiles; }
  __device__ PairUnit info(int u, int rank) const {
    int lo = 0, hi = E;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if ((exp_begin[mid] >> 1) * n_tiles <= u) lo = mid; else hi = mid;
    }
    const int b = exp_begin[lo] >> 1, cnt = (exp_begin[lo + 1] >> 1) - b;
    const int local = u - b * n_tiles;
    const int nt = local / cnt;
    const int pp = b + (local - nt * cnt);
    const int p = 2 * pp + rank;
    const int brow = b_tiled ? (lo * n_tiles + nt) * kb * bn : lo * n_per_expert + nt * bn;
    const int rows = __ldg(&piece_rows[p]), prow = __ldg(&piece_rows[p ^ 1]);
    PairUnit I;
    I.U = Unit{__ldg(&piece_row[p]), rows, brow, nt * bn};
    const int my = (rows + kBlockM - 1) / kBlockM, peer = (prow + kBlockM - 1) / kBlockM;
    I.mtiles = max(max(my, peer), 1);
    I.peer_mt = peer;
    return I;
  }
  __device__ int num_kb() const { return kb; }
  __device__ int a_kcol(int k) const { return k * kBlockK; }
  __device__ int b_kcol(int k) const { return b_tiled ? 0 : k * kBlockK; }
  __device__ int b_krow(int k) const { return b_tiled ? k * bn : 0; }
};

}  // namespace mp
