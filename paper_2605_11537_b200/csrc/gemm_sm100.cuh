// Persistent warp-specialised tcgen05 GEMM core for sm_100a.
//
//   D[128 x BN] = A[128 x K] * B[BN x K]^T      (bf16 in, fp32 accumulate in TMEM)
//
// Roles (384 threads, one CTA per SM):
//   warp 0 lane 0 : TMA producer  (A and B k-blocks of 64 bf16 = one 128 B swizzle atom)
//   warp 1 lane 0 : MMA issuer    (4 x tcgen05.mma 128xBNx16 per k-block)
//   warp 2        : TMEM allocator (2 accumulator stages x BN columns)
//   warps 4..11   : epilogue, two warpgroups (tcgen05.ld -> registers -> caller's
//                   Epilogue); warpgroup h owns accumulator columns [h*BN/2, (h+1)*BN/2)
//                   when the epilogue is column-separable, else warpgroup 0 does all.
// Pipelines: smem ring full/empty (TMA <-> MMA), TMEM full/empty (MMA <-> epilogue).
//
// Work is expressed as "units": a unit is a run of rows [a_row, a_row+rows) of A
// multiplied by one BN-wide slice of B starting at row b_row. A unit with more
// than 128 rows is processed as consecutive 128-row M-tiles by the SAME CTA --
// this is how a replica slot (reference: src/simulator.py:66-81, one server
// draining its queue) maps onto the GPU; splitting an expert into replicas
// splits its rows into independent units. Units are assigned to CTAs
// round-robin (static persistent schedule), so every role walks the same list.
#pragma once
#include "common.cuh"
#include "ptx.cuh"

namespace mp {

constexpr int kBlockM = 128;
constexpr int kBlockK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B atom row
constexpr int kEpiWarps = 8;
constexpr int kGemmThreads = 128 + 32 * kEpiWarps;

struct Unit {
  int a_row;  // first row of A (and of the row-indexed output)
  int rows;   // rows in this unit (>0); ceil(rows/128) M-tiles
  int b_row;  // first row of B (e.g. expert * N + n0)
  int n0;     // output column offset of this BN slice
};

// Epilogues that write through a TMA store map (kernel parameter tmC) declare kTmaStore.
template <class E, class = void>
struct TmaStoreOf {
  static constexpr bool value = false;
};
template <class E>
struct TmaStoreOf<E, decltype(void(E::kTmaStore))> {
  static constexpr bool value = E::kTmaStore;
};

// Per-CTA start / end timestamps (%globaltimer, ns) of the last k_umma_gemm launch of
// this translation unit, for load-balance diagnostics (mp_debug_cta_times reads the
// copy of ffn.cu, i.e. the grouped expert GEMMs).
static __device__ unsigned long long g_cta_t0[1024];
static __device__ unsigned long long g_cta_t1[1024];
#ifdef MP_DIAG
// Diagnostic build only (MP_NVCC_EXTRA=-DMP_DIAG): per-unit %globaltimer stamps of the
// last launch -- [0] producer issues the unit's first load, [1] MMA sees its first k-block,
// [2] MMA has issued its last k-block, [3] CTA.
constexpr int kTraceUnits = 8192;
static __device__ unsigned long long g_unit_t[4][kTraceUnits];
#define MP_TRACE(k, u, v) \
  do {                    \
    if ((u) < kTraceUnits) g_unit_t[k][u] = (v); \
  } while (0)
// bit 0: issue every N = BN MMA as two N = BN/2 MMAs (the A tile is read twice; same result)
static __device__ int g_diag_mma;
#else
#define MP_TRACE(k, u, v) \
  do {                    \
  } while (0)
#endif

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// TMEM columns of the two accumulator stages (allocation is a power of two >= 32)
constexpr uint32_t tmem_cols(int bn) {
  return 2 * bn <= 32 ? 32 : (2 * bn <= 64 ? 64 : (2 * bn <= 128 ? 128 : (2 * bn <= 256 ? 256 : 512)));
}

template <int BN, int STAGES, int ASTAGES = 0>
struct GemmSmem {
  // ASTAGES == 0: one ring of STAGES x (A | B) stages. ASTAGES > 0: separate rings, STAGES
  // B stages then ASTAGES A stages, each with its own full/empty barriers (the weight
  // stream runs further ahead than the L2-resident activations).
  static constexpr int kABytes = kBlockM * kBlockK * 2;
  static constexpr int kBBytes = BN * kBlockK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kARingOffset = STAGES * kBBytes;
  static constexpr int kRingBytes = ASTAGES ? STAGES * kBBytes + ASTAGES * kABytes : STAGES * kStageBytes;
  static constexpr int kBarOffset = kRingBytes;
  static constexpr int kVecOffset = kBarOffset + (2 * STAGES + 2 * ASTAGES + 4) * 8 + 16;
  static constexpr int kScratchOffset = (kVecOffset + 2 * BN * 4 + 1023) / 1024 * 1024;  // TMA-store boxes
  static constexpr int kScratchWordsPerWarp = 32 * 20;  // 32 rows x (16 + 4 pad) words: store transpose
  static constexpr int kPrepOffset = kScratchOffset + 8 * kScratchWordsPerWarp * 4;  // scheduler table (smem)
  static constexpr int kPrepInts = (ASTAGES || BN % 64 != 0 || STAGES * (kBlockM + BN) * kBlockK * 2 > 196608) ? 768 : 2048;
  static constexpr int kBytes = kPrepOffset + kPrepInts * 4 + 1024;  // + alignment slack
};

// Scheduler concept:
//   int num_units() const; Unit unit(int u) const; int num_kb() const;
//   int a_kcol(int kb) const; int b_kcol(int kb) const;
//   void prepare(int* table) -- run by ALL threads before the roles start; may stage
//   read-only scheduling data in shared memory (GemmSmem::kPrepInts ints).
// Every role decodes the NEXT unit while working on the current one, so the
// (global-memory) piece lookups of a grouped GEMM never stall the pipeline.
// Epilogue concept:
//   static constexpr bool kSplitCols;   // columns independent -> two warpgroups split them
//   const float* colvec() const;        // per-column vector (bias) or null; staged in smem per tile
//   template<int NC> void run(const Unit&, int mt, int r, uint32_t taddr, int c0, const float* svec,
//                             uint32_t* scratch) const   (scratch: warp-private smem, 640 words)
//   (r = row inside the 128-row tile owned by this thread; taddr = TMEM address of
//    (lane quadrant, accumulator stage, column c0); the thread handles tile columns
//    [c0, c0 + NC)).

template <int BN, int STAGES, class Sched, class Epi, class Kind = KindBF16, int ASTAGES = 0>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_umma_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, Sched sched_in,
                Epi epi, const __grid_constant__ CUtensorMap tmC) {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 1000)
  using L = GemmSmem<BN, STAGES, ASTAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + STAGES;
  uint64_t* afull = empty + STAGES;  // split rings only
  uint64_t* aempty = afull + ASTAGES;
  uint64_t* tfull = aempty + ASTAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* svec = reinterpret_cast<float*>(smem + L::kVecOffset);  // [2][BN]
  uint32_t* scratch_all = reinterpret_cast<uint32_t*>(smem + L::kScratchOffset);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    if (blockIdx.x < 1024) g_cta_t0[blockIdx.x] = global_ns();
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < ASTAGES; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps);  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, tmem_cols(BN));
  griddep_wait();  // the prologue above overlapped the previous kernel's tail
  Sched sched = sched_in;
  sched.prepare(reinterpret_cast<int*>(smem + L::kPrepOffset));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int nunits = sched.num_units();
  const int nkb = sched.num_kb();

  if (warp == 0 || (ASTAGES > 0 && warp == 3)) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer(s)
      // unified ring: warp 0 loads A and B; split rings: warp 0 loads B, warp 3 loads A
      const bool do_b = warp == 0, do_a = ASTAGES == 0 || warp == 3;
      const uint64_t pol_stream = policy_evict_first();
      uint32_t stage = 0, phase = 0;
      Unit Un = blockIdx.x < nunits ? sched.unit(blockIdx.x) : Unit{};
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const Unit U = Un;
        if (u + (int)gridDim.x < nunits) Un = sched.unit(u + gridDim.x);  // consumed next iteration
        const int mtiles = (U.rows + kBlockM - 1) / kBlockM;
        for (int mt = 0; mt < mtiles; ++mt) {
          for (int kb = 0; kb < nkb; ++kb) {
            if constexpr (ASTAGES == 0) {
              mbar_wait(&empty[stage], phase ^ 1);
              if (mt == 0 && kb == 0) {
                MP_TRACE(0, u, global_ns());
                MP_TRACE(3, u, (unsigned long long)blockIdx.x);
              }
              uint8_t* sa = smem + stage * L::kStageBytes;
              uint8_t* sb = sa + L::kABytes;
              mbar_arrive_expect_tx(&full[stage], L::kStageBytes);
              tma_load_2d(sa, &tmA, &full[stage], sched.a_kcol(kb), U.a_row + mt * kBlockM);
              if constexpr (Sched::kStreamB)  // weights are read once per step: do not let them evict reused tiles
                tma_load_2d_hint(sb, &tmB, &full[stage], sched.b_kcol(kb), U.b_row + sched.b_krow(kb), pol_stream);
              else
                tma_load_2d(sb, &tmB, &full[stage], sched.b_kcol(kb), U.b_row + sched.b_krow(kb));
              if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
              }
            } else if (do_b) {
              mbar_wait(&empty[stage], phase ^ 1);
              uint8_t* sb = smem + stage * L::kBBytes;
              mbar_arrive_expect_tx(&full[stage], L::kBBytes);
              if constexpr (Sched::kStreamB)
                tma_load_2d_hint(sb, &tmB, &full[stage], sched.b_kcol(kb), U.b_row + sched.b_krow(kb), pol_stream);
              else
                tma_load_2d(sb, &tmB, &full[stage], sched.b_kcol(kb), U.b_row + sched.b_krow(kb));
              if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
              }
            } else if (do_a) {
              mbar_wait(&aempty[stage], phase ^ 1);
              uint8_t* sa = smem + L::kARingOffset + stage * L::kABytes;
              mbar_arrive_expect_tx(&afull[stage], L::kABytes);
              tma_load_2d(sa, &tmA, &afull[stage], sched.a_kcol(kb), U.a_row + mt * kBlockM);
              if (++stage == (ASTAGES ? ASTAGES : 1)) {
                stage = 0;
                phase ^= 1;
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = Kind::idesc(kBlockM, BN);
      uint32_t stage = 0, phase = 0, tile = 0;
      uint32_t astage = 0, aphase = 0;
      Unit Un = blockIdx.x < nunits ? sched.unit(blockIdx.x) : Unit{};
      for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const Unit U = Un;
        if (u + (int)gridDim.x < nunits) Un = sched.unit(u + gridDim.x);
        const int mtiles = (U.rows + kBlockM - 1) / kBlockM;
        for (int mt = 0; mt < mtiles; ++mt, ++tile) {
          const uint32_t as = tile & 1, aph = (tile >> 1) & 1;
          mbar_wait(&tempty[as], aph ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + as * BN;
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&full[stage], phase);
            if (mt == 0 && kb == 0) MP_TRACE(1, u, global_ns());
            uint64_t adesc, bdesc;
            if constexpr (ASTAGES == 0) {
              const uint8_t* sa = smem + stage * L::kStageBytes;
              adesc = sw128_kmajor_desc(smem_u32(sa));
              bdesc = sw128_kmajor_desc(smem_u32(sa + L::kABytes));
            } else {
              mbar_wait(&afull[astage], aphase);
              adesc = sw128_kmajor_desc(smem_u32(smem + L::kARingOffset + astage * L::kABytes));
              bdesc = sw128_kmajor_desc(smem_u32(smem + stage * L::kBBytes));
            }
            tc_fence_after();
#ifdef MP_DIAG
            if (BN % 32 == 0 && (g_diag_mma & 1)) {
              constexpr uint32_t idesc_h = Kind::idesc(kBlockM, BN / 2);
              constexpr uint32_t boff = (BN / 2) * 128 / 16;  // B rows BN/2.. : + (BN/2) x 128 B
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                Kind::mma(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc_h, (kb | k) != 0);
                Kind::mma(d_tmem + BN / 2, adesc + 2 * k, bdesc + boff + 2 * k, idesc_h, (kb | k) != 0);
              }
            } else
#endif
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              // advance 32 B of K inside the swizzle atom: +2 in the >>4 address field
              Kind::mma(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
            }
            umma_commit(&empty[stage]);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
            if constexpr (ASTAGES > 0) {
              umma_commit(&aempty[astage]);
              if (++astage == ASTAGES) {
                astage = 0;
                aphase ^= 1;
              }
            }
          }
          umma_commit(&tfull[as]);
          if (mt == mtiles - 1) MP_TRACE(2, u, global_ns());
        }
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int q = warp & 3;            // TMEM lane quadrant this warp may access
    const int half = (warp - 4) >> 2;  // warpgroup index
    const int r = q * 32 + lane;       // row of the tile owned by this thread
    constexpr bool split = Epi::kSplitCols;
    constexpr int NC = split ? BN / 2 : BN;
    const bool active = split || half == 0;
    const int c0 = split ? half * (BN / 2) : 0;
    uint32_t tile = 0;
    Unit Un = blockIdx.x < nunits ? sched.unit(blockIdx.x) : Unit{};
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      const Unit U = Un;
      if (u + (int)gridDim.x < nunits) Un = sched.unit(u + gridDim.x);
      const int mtiles = (U.rows + kBlockM - 1) / kBlockM;
      for (int mt = 0; mt < mtiles; ++mt, ++tile) {
        const uint32_t as = tile & 1, aph = (tile >> 1) & 1;
        const float* vec = epi.colvec();
        if (vec != nullptr) {  // stage this tile's column vector once (all epilogue threads, named barrier 1)
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
        if (lane == 0) mbar_arrive(&tempty[as]);
      }
    }
    if constexpr (TmaStoreOf<Epi>::value) {
      if (lane == 0) bulk_wait0();  // this warp's TMA stores complete before the CTA exits
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_cta_t1[blockIdx.x] = global_ns();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, tmem_cols(BN));
  }
#endif
}

// ------------------------------------------------------------------ schedulers

// Dense C[M x N] = A[M x K] B[N x K]^T, units = (m block, n block), n fastest.
struct DenseSched {
  __device__ void prepare(int*) {}
  static constexpr bool kStreamB = false;
  int M, n_tiles, kb, bn;
  __device__ int num_units() const { return ((M + kBlockM - 1) / kBlockM) * n_tiles; }
  __device__ Unit unit(int u) const {
    const int mb = u / n_tiles, nb = u - mb * n_tiles;
    Unit U;
    U.a_row = mb * kBlockM;
    U.rows = min(kBlockM, M - U.a_row);
    U.b_row = nb * bn;
    U.n0 = nb * bn;
    return U;
  }
  __device__ int num_kb() const { return kb; }
  __device__ int a_kcol(int k) const { return k * kBlockK; }
  __device__ int b_kcol(int k) const { return k * kBlockK; }
  __device__ int b_krow(int) const { return 0; }
};

// Device-built unit list (grouped GEMM over replica segments).
struct ListSched {
  __device__ void prepare(int*) {}
  static constexpr bool kStreamB = false;
  const int4* units;      // {a_row, rows, b_row, n0}
  const int* num_units_p;  // device scalar, written by the planner
  int kb;
  __device__ int num_units() const { return *reinterpret_cast<const volatile int*>(num_units_p); }
  __device__ Unit unit(int u) const {
    const int4 v = __ldg(&units[u]);
    return Unit{v.x, v.y, v.z, v.w};
  }
  __device__ int num_kb() const { return kb; }
  __device__ int a_kcol(int k) const { return k * kBlockK; }
  __device__ int b_kcol(int k) const { return k * kBlockK; }
  __device__ int b_krow(int) const { return 0; }
};

// Grouped GEMM over replica-segment pieces (built on device by mp_exec_map):
// pieces of expert e are [exp_begin[e], exp_begin[e+1]); units are ordered
// expert-major, then BN slice, then piece, so consecutive units (running on
// neighbouring SMs at the same time) share one weight tile through L2.
struct SegSched {
  static constexpr bool kStreamB = true;
  const int32_t* piece_row;
  const int32_t* piece_rows;
  const int32_t* exp_begin;  // E + 1 entries (staged into shared memory by prepare when E < kPrepInts)
  int E, n_tiles, bn, n_per_expert, kb;
  int b_tiled;  // B pre-tiled as [E][n_tiles][kb][bn rows][64 cols]: every TMA box is one contiguous burst
  int reverse;  // 1: walk the unit list backwards (GEMM2 consumes the hidden rows GEMM1 wrote LAST first,
                //    while they are still in L2)
  int prep_cap = 768;  // <= GemmSmem<BN, STAGES>::kPrepInts of the launch
  const int32_t* piece_wbase = nullptr;  // physical replicas: weight slot of each piece (else its expert)
  __device__ void prepare(int* tab) {
    if (E + 1 > prep_cap) return;  // table of GemmSmem::kPrepInts ints; else exp_begin stays global
    for (int e = threadIdx.x; e <= E; e += blockDim.x) tab[e] = exp_begin[e];
    __syncthreads();
    exp_begin = tab;
  }
  __device__ int num_units() const { return exp_begin[E] * n_tiles; }
  __device__ Unit unit(int u) const {
    if (reverse) u = exp_begin[E] * n_tiles - 1 - u;
    int lo = 0, hi = E;  // exp_begin[lo]*n_tiles <= u < exp_begin[hi]*n_tiles
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (exp_begin[mid] * n_tiles <= u) lo = mid; else hi = mid;
    }
    const int b = exp_begin[lo], cnt = exp_begin[lo + 1] - b;
    const int local = u - b * n_tiles;
    const int nt = local / cnt;
    const int p = b + (local - nt * cnt);
    const int wb = piece_wbase ? __ldg(&piece_wbase[p]) : lo;
    const int brow = b_tiled ? (wb * n_tiles + nt) * kb * bn : wb * n_per_expert + nt * bn;
    return Unit{__ldg(&piece_row[p]), __ldg(&piece_rows[p]), brow, nt * bn};
  }
  __device__ int num_kb() const { return kb; }
  __device__ int a_kcol(int k) const { return k * kBlockK; }
  __device__ int b_kcol(int k) const { return b_tiled ? 0 : k * kBlockK; }
  __device__ int b_krow(int k) const { return b_tiled ? k * bn : 0; }
};

// Dense fp32/TF32 GEMM: k-blocks of 32 fp32 (128 B).
struct DenseTf32Sched {
  __device__ void prepare(int*) {}
  static constexpr bool kStreamB = false;
  int M, n_tiles, kb, bn;
  __device__ int num_units() const { return ((M + kBlockM - 1) / kBlockM) * n_tiles; }
  __device__ Unit unit(int u) const {
    const int mb = u / n_tiles, nb = u - mb * n_tiles;
    return Unit{mb * kBlockM, min(kBlockM, M - mb * kBlockM), nb * bn, nb * bn};
  }
  __device__ int num_kb() const { return kb; }
  __device__ int a_kcol(int k) const { return k * 32; }
  __device__ int b_kcol(int k) const { return k * 32; }
  __device__ int b_krow(int) const { return 0; }
};

// Split-bf16 "3-pass" product for fp32-faithful dot products on the tensor
// core: A = [x_hi | x_lo], B = [w_hi | w_lo] (each 2*Kd wide) and
//   acc = x_hi.w_hi + x_hi.w_lo + x_lo.w_hi
// expressed as 3*nk k-blocks with remapped k coordinates.
struct Split3Sched {
  __device__ void prepare(int*) {}
  static constexpr bool kStreamB = false;
  int M, n_tiles, nk, bn, kd;  // kd = padded real K (multiple of 64)
  __device__ int num_units() const { return ((M + kBlockM - 1) / kBlockM) * n_tiles; }
  __device__ Unit unit(int u) const {
    const int mb = u / n_tiles, nb = u - mb * n_tiles;
    Unit U;
    U.a_row = mb * kBlockM;
    U.rows = min(kBlockM, M - U.a_row);
    U.b_row = nb * bn;
    U.n0 = nb * bn;
    return U;
  }
  __device__ int num_kb() const { return 3 * nk; }
  __device__ int a_kcol(int k) const {
    return k < 2 * nk ? (k % nk) * kBlockK : kd + (k - 2 * nk) * kBlockK;
  }
  __device__ int b_kcol(int k) const {
    return k < nk ? k * kBlockK : (k < 2 * nk ? kd + (k - nk) * kBlockK : (k - 2 * nk) * kBlockK);
  }
  __device__ int b_krow(int) const { return 0; }
};

}  // namespace mp
