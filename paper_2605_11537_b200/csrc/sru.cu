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

constexpr int kScanChunk = 32;   // tokens per scan chunk
constexpr int kScanThreads = 128;  // channel pairs per block

__device__ __forceinline__ float2 ld_bf16x2(const __nv_bfloat16* p) {
  const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(p);
  return __bfloat1622float2(v);
}

// pass A: chunk aggregates (A = prod f, B = chunk scan from c = 0) per channel,
// 4 channels per thread, u/f loads software-pipelined 8 tokens deep.
struct bf16x4 {
  __nv_bfloat162 a, b;
};
constexpr int kAggDepth = 16;  // tokens of u/f loads in flight per thread
__global__ void __launch_bounds__(64) k_scan_aggregate(const __nv_bfloat16* __restrict__ ufr, int T, int d,
                                                       float* __restrict__ aggA, float* __restrict__ aggB) {
  griddep_launch_dependents();
  griddep_wait();
  const int cq = blockIdx.x * blockDim.x + threadIdx.x;
  if (4 * cq >= d) return;
  const int ch = blockIdx.y;
  const int t0 = ch * kScanChunk, t1 = min(T, t0 + kScanChunk);
  float a[4] = {1.f, 1.f, 1.f, 1.f}, b[4] = {0.f, 0.f, 0.f, 0.f};
  const size_t ld3 = (size_t)3 * d;
#pragma unroll 1
  for (int tb = t0; tb < t1; tb += kAggDepth) {
    bf16x4 u[kAggDepth], f[kAggDepth];
#pragma unroll
    for (int i = 0; i < kAggDepth; ++i) {
      const int t = min(tb + i, t1 - 1);
      const __nv_bfloat16* p = ufr + (size_t)t * ld3 + 4 * cq;
      u[i] = *reinterpret_cast<const bf16x4*>(p);
      f[i] = *reinterpret_cast<const bf16x4*>(p + d);
    }
#pragma unroll
    for (int i = 0; i < kAggDepth; ++i) {
      if (tb + i < t1) {
        const float2 ua = __bfloat1622float2(u[i].a), ub = __bfloat1622float2(u[i].b);
        const float2 fa = __bfloat1622float2(f[i].a), fb = __bfloat1622float2(f[i].b);
        const float uu[4] = {ua.x, ua.y, ub.x, ub.y}, ff[4] = {fa.x, fa.y, fb.x, fb.y};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          b[j] = fmaf(ff[j], b[j] - uu[j], uu[j]);
          a[j] *= ff[j];
        }
      }
    }
  }
  const size_t o = (size_t)ch * d + 4 * cq;
  *reinterpret_cast<float4*>(aggA + o) = make_float4(a[0], a[1], a[2], a[3]);
  *reinterpret_cast<float4*>(aggB + o) = make_float4(b[0], b[1], b[2], b[3]);
}

// pass B: carry_in[ch] per channel (c_0 = 0 at the start of every batch, or the
// carry of a preceding shard). Hierarchical so the serial depth is
// 3 * sqrt(nch) instead of nch: block = 32 channels x G chunk groups; each
// (group, channel) composes its chunks' affine maps, one thread per channel
// scans the G group maps, then every group replays its chunks from its carry.
// The chunk maps of a group are loaded into registers 16 at a time (independent
// loads in flight) before the serial composition, and reused by the replay.
constexpr int kCarryGroups = 16;
constexpr int kCarryBatch = 16;
__global__ void __launch_bounds__(32 * kCarryGroups) k_scan_carry(const float* __restrict__ aggA, const float* __restrict__ aggB, int nch, int d,
                             const float* __restrict__ c0, float* __restrict__ carry, float* __restrict__ tot) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ float sA[kCarryGroups][32], sB[kCarryGroups][32], sC[kCarryGroups][32];
  const int cl = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cl;
  const int per = cdiv(nch, kCarryGroups);
  const int ch0 = g * per, ch1 = min(nch, ch0 + per);
  const bool act = c < d;
  float A = 1.f, B = 0.f;
  float ra[kCarryBatch], rb[kCarryBatch];
  const bool one_batch = per <= kCarryBatch;  // typical: nch = 512 -> 32 per group -> two batches
  for (int cb = ch0; cb < ch1; cb += kCarryBatch) {
#pragma unroll
    for (int i = 0; i < kCarryBatch; ++i) {
      const int ch = cb + i;
      if (act && ch < ch1) {
        const size_t o = (size_t)ch * d + c;
        ra[i] = __ldg(&aggA[o]);
        rb[i] = __ldg(&aggB[o]);
      }
    }
#pragma unroll
    for (int i = 0; i < kCarryBatch; ++i) {
      if (act && cb + i < ch1) {
        B = fmaf(ra[i], B, rb[i]);  // compose: apply (A,B) first, then (a,b)
        A *= ra[i];
      }
    }
  }
  sA[g][cl] = A;
  sB[g][cl] = B;
  __syncthreads();
  if (g == 0) {
    float run = (act && c0) ? c0[c] : 0.f;
    float all = 1.f;
    for (int h = 0; h < kCarryGroups; ++h) {
      sC[h][cl] = run;
      run = fmaf(sA[h][cl], run, sB[h][cl]);
      all *= sA[h][cl];
    }
    if (tot && act) {  // the whole range as one affine map c_end = all * c_start + (c_end from c_start = 0)
      tot[c] = all;
      tot[d + c] = run;
    }
  }
  __syncthreads();
  if (act) {
    float run = sC[g][cl];
    for (int cb = ch0; cb < ch1; cb += kCarryBatch) {
      if (!one_batch) {
#pragma unroll
        for (int i = 0; i < kCarryBatch; ++i) {
          const int ch = cb + i;
          if (ch < ch1) {
            const size_t o = (size_t)ch * d + c;
            ra[i] = __ldg(&aggA[o]);
            rb[i] = __ldg(&aggB[o]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < kCarryBatch; ++i) {
        const int ch = cb + i;
        if (ch < ch1) {
          carry[(size_t)ch * d + c] = run;
          run = fmaf(ra[i], run, rb[i]);
        }
      }
    }
  }
}

// tanh via one exp + one reciprocal (|abs err| ~1e-7; the reference uses np.tanh in f64)
__device__ __forceinline__ float fast_tanh(float x) {
  const float e = __expf(2.f * x);
  return 1.f - 2.f * __frcp_rn(1.f + e);
}

// pass C: replay each chunk from its carry; h = r tanh(c) + (1 - r) x.
// 4 channels per thread: 8-byte bf16x4 loads of u/f/r, 16-byte x loads/h stores.
__device__ __forceinline__ float4 ld_bf16x4(const __nv_bfloat16* p) {
  const bf16x4 v = *reinterpret_cast<const bf16x4*>(p);
  const float2 lo = __bfloat1622float2(v.a), hi = __bfloat1622float2(v.b);
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}

__device__ __forceinline__ float sru_step(float& c, float u, float f, float r, float x) {
  c = fmaf(f, c - u, u);  // f c + (1 - f) u
  return fmaf(r, fast_tanh(c) - x, x);  // r tanh(c) + (1 - r) x
}

// Loads are software-pipelined kPF tokens deep (raw bf16x4 / float4 kept in
// registers) so each thread keeps ~kPF * 40 B in flight across the serial chain.
constexpr int kPF = 4;
__global__ void __launch_bounds__(64) k_scan_output(const __nv_bfloat16* __restrict__ ufr,
                                                    const float* __restrict__ x, int T, int d,
                                                    const float* __restrict__ carry, float* __restrict__ h32,
                                                    __nv_bfloat16* __restrict__ h16, float* __restrict__ c_last,
                                                    int32_t* __restrict__ nonfinite) {
  griddep_launch_dependents();
  griddep_wait();
  const int cq = blockIdx.x * blockDim.x + threadIdx.x;  // channel quad
  if (4 * cq >= d) return;
  const int ch = blockIdx.y;
  const int t0 = ch * kScanChunk, t1 = min(T, t0 + kScanChunk);
  const float4 cin = *reinterpret_cast<const float4*>(carry + (size_t)ch * d + 4 * cq);
  float c0 = cin.x, c1 = cin.y, c2 = cin.z, c3 = cin.w;
  bool bad = false;
  const size_t ld3 = (size_t)3 * d;
  bf16x4 bu[2][kPF], bfv[2][kPF], br[2][kPF];
  float4 bx[2][kPF];
  auto fetch = [&](int buf, int tb) {
#pragma unroll
    for (int i = 0; i < kPF; ++i) {
      const int t = min(tb + i, t1 - 1);
      const __nv_bfloat16* p = ufr + (size_t)t * ld3 + 4 * cq;
      bu[buf][i] = *reinterpret_cast<const bf16x4*>(p);
      bfv[buf][i] = *reinterpret_cast<const bf16x4*>(p + d);
      br[buf][i] = *reinterpret_cast<const bf16x4*>(p + 2 * d);
      bx[buf][i] = *reinterpret_cast<const float4*>(x + (size_t)t * d + 4 * cq);
    }
  };
  fetch(0, t0);
#pragma unroll 1
  for (int tb = t0; tb < t1; tb += 2 * kPF) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int tc = tb + half * kPF;
      if (tc >= t1) break;
      if (tc + kPF < t1) fetch(half ^ 1, tc + kPF);
#pragma unroll
      for (int i = 0; i < kPF; ++i) {
        const int t = tc + i;
        if (t < t1) {
          const float2 ua = __bfloat1622float2(bu[half][i].a), ub = __bfloat1622float2(bu[half][i].b);
          const float2 fa = __bfloat1622float2(bfv[half][i].a), fb = __bfloat1622float2(bfv[half][i].b);
          const float2 ra = __bfloat1622float2(br[half][i].a), rb = __bfloat1622float2(br[half][i].b);
          const float4 xv = bx[half][i];
          float4 h;
          h.x = sru_step(c0, ua.x, fa.x, ra.x, xv.x);
          h.y = sru_step(c1, ua.y, fa.y, ra.y, xv.y);
          h.z = sru_step(c2, ub.x, fb.x, rb.x, xv.z);
          h.w = sru_step(c3, ub.y, fb.y, rb.y, xv.w);
          bad |= !(isfinite(h.x) && isfinite(h.y) && isfinite(h.z) && isfinite(h.w) && isfinite(c0 + c1 + c2 + c3));
          *reinterpret_cast<float4*>(h32 + (size_t)t * d + 4 * cq) = h;
          bf16x4 hb;
          hb.a = __floats2bfloat162_rn(h.x, h.y);
          hb.b = __floats2bfloat162_rn(h.z, h.w);
          *reinterpret_cast<bf16x4*>(h16 + (size_t)t * d + 4 * cq) = hb;
        }
      }
    }
  }
  if (c_last && t1 == T) *reinterpret_cast<float4*>(c_last + 4 * cq) = make_float4(c0, c1, c2, c3);
  if (bad) atomicOr(nonfinite, 1);  // reference raises NumericError (src/predictor.py:170-171)
}

static inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

// Single-pass form of K2 (default): one launch reads u/f/r/x once and writes h once.
// Block = kSpWarps consecutive 32-token chunks x one strip of 128 channels (lane = 4
// channels). Blocks take tickets in launch order; a block
//   1. computes its chunks' affine maps (c_out = A c_in + B) and the block map,
//   2. publishes the block map (flag 1), looks back over its predecessors in the strip in
//      windows of 32 (flags read by one warp, maps composed backwards per channel) until a
//      predecessor with a published inclusive carry (flag 2; block 0 always has one),
//   3. publishes its own inclusive carry (flag 2), then replays its chunks (u/f re-read hits
//      L2) and applies the highway output.
// A block only waits on blocks with smaller tickets, which are already running.
// Reference: sru_forward (src/predictor.py:177-195); the recurrence is the one of
// k_scan_aggregate / k_scan_carry / k_scan_output above (same per-step arithmetic).
constexpr int kSpWarps = 8;
constexpr int kSpTokens = kSpWarps * kScanChunk;
constexpr int kSpPF = 2;  // replay: tokens per prefetch group (double buffered)
constexpr int kSpAgg = 8;  // u/f tokens in flight per thread in step 1
// 3 blocks per SM (<= 80 registers): all T / 256 x d / 128 blocks of the bench shape resident
// in one wave (two blocks per SM: 74 us, three: 53 us, four with spills: 65 us).

#ifdef MP_DIAG
// Diagnostic build only: per-block (ticket order) %globaltimer stamps of the last k_scan_fused
// launch: [0] ticket taken, [1] chunk maps done, [2] carry-in known, [3] replay done.
static __device__ unsigned long long g_scan_t[1024][4];
#define SCAN_STAMP(b, i)                                             \
  do {                                                               \
    unsigned long long t_;                                           \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));          \
    if ((b) < 1024) g_scan_t[b][i] = t_;                             \
  } while (0)
#else
#define SCAN_STAMP(b, i) \
  do {                   \
  } while (0)
#endif

__device__ __forceinline__ int sp_ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void sp_st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(32 * kSpWarps, 3) k_scan_fused(const __nv_bfloat16* __restrict__ ufr,
                                                              const float* __restrict__ x, int T, int d,
                                                              const float* __restrict__ c0, float* __restrict__ h32,
                                                              __nv_bfloat16* __restrict__ h16,
                                                              float* __restrict__ c_last, int32_t* __restrict__ nonfinite,
                                                              int* flags, float* agg, float* incl, int nblk) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ float sA[kSpWarps][128], sB[kSpWarps][128];
  __shared__ float sCin[128];
  __shared__ float sLA[128], sLB[128];  // look-back: the low half-window's composed map
  __shared__ int s_ticket, s_lo, s_found;
  const int nstr = d / 128 + (d % 128 != 0);
  if (threadIdx.x == 0) s_ticket = atomicAdd(&flags[nstr * nblk], 1);
  __syncthreads();
  const int str = s_ticket % nstr, blk = s_ticket / nstr;
  if (threadIdx.x == 0) SCAN_STAMP(s_ticket, 0);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cq = str * 32 + lane;
  const bool act = 4 * cq < d;
  const int t0 = (blk * kSpWarps + w) * kScanChunk, t1 = min(T, t0 + kScanChunk);
  const size_t ld3 = (size_t)3 * d;
  // ---- 1. chunk maps
  {
    float a[4] = {1.f, 1.f, 1.f, 1.f}, b[4] = {0.f, 0.f, 0.f, 0.f};
    if (act) {
#pragma unroll 1
      for (int tb = t0; tb < t1; tb += kSpAgg) {
        bf16x4 u[kSpAgg], f[kSpAgg];
#pragma unroll
        for (int i = 0; i < kSpAgg; ++i) {
          const int t = min(tb + i, t1 - 1);
          const __nv_bfloat16* p = ufr + (size_t)t * ld3 + 4 * cq;
          u[i] = *reinterpret_cast<const bf16x4*>(p);
          f[i] = *reinterpret_cast<const bf16x4*>(p + d);
        }
#pragma unroll
        for (int i = 0; i < kSpAgg; ++i) {
          if (tb + i < t1) {
            const float2 ua = __bfloat1622float2(u[i].a), ub = __bfloat1622float2(u[i].b);
            const float2 fa = __bfloat1622float2(f[i].a), fb = __bfloat1622float2(f[i].b);
            const float uu[4] = {ua.x, ua.y, ub.x, ub.y}, ff[4] = {fa.x, fa.y, fb.x, fb.y};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              b[j] = fmaf(ff[j], b[j] - uu[j], uu[j]);
              a[j] *= ff[j];
            }
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      sA[w][4 * lane + j] = a[j];
      sB[w][4 * lane + j] = b[j];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) SCAN_STAMP(s_ticket, 1);
  // ---- 2. block map; sA/sB become the exclusive prefix maps of the chunks inside the block
  const int me = str * nblk + blk;
  const int c = threadIdx.x;  // channel of the strip (threads < 128)
  float BA = 1.f, BB = 0.f;
  if (c < 128) {
#pragma unroll
    for (int k = 0; k < kSpWarps; ++k) {
      const float ak = sA[k][c], bk = sB[k][c];
      sA[k][c] = BA;
      sB[k][c] = BB;
      BB = fmaf(ak, BB, bk);
      BA *= ak;
    }
  }
  float cin = 0.f;
  if (blk == 0) {
    if (c < 128) {
      const int ch = str * 128 + c;
      cin = (c0 != nullptr && ch < d) ? c0[ch] : 0.f;
    }
  } else {
    if (c < 128) {
      agg[(size_t)me * 256 + c] = BA;
      agg[(size_t)me * 256 + 128 + c] = BB;
    }
    __syncthreads();  // the release below is cumulative over the block's writes ordered by the barrier
    if (threadIdx.x == 0) sp_st_release(&flags[me], 1);
    // Look back in windows of 32 predecessors: warp 0 waits for their flags; then two threads
    // per channel load their 16 maps of the window at once (one L2 round trip per window)
    // and compose them; the high half (closer to this block) is applied first.
    float MA = 1.f, MB = 0.f;  // composition of the maps of the blocks walked so far
    const int ch = threadIdx.x & 127, hh = threadIdx.x >> 7;
    int base = blk - 1;
    for (;;) {
      if (w == 0) {
        const int idx = base - lane;
        int f = 0;
        if (idx >= 0)
          while ((f = sp_ld_acquire(&flags[str * nblk + idx])) < 1) __nanosleep(32);
        const unsigned m = __ballot_sync(0xffffffffu, f == 2);
        if (lane == 0) {
          s_found = m != 0;
          s_lo = m ? base - (__ffs(m) - 1) : base - 31;
        }
      }
      __syncthreads();
      const int lo = s_lo, found = s_found;
      const int stop = found ? lo + 1 : lo;
      const int jhi = base - 16 * hh;  // this thread's entries: jhi, jhi - 1, ..., jhi - 15 (>= stop)
      float ra[16], rb[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (jhi - i >= stop) {
          const size_t o = (size_t)(str * nblk + jhi - i) * 256 + ch;
          ra[i] = __ldcg(&agg[o]);
          rb[i] = __ldcg(&agg[o + 128]);
        }
      }
      const float ci = (found && hh == 0) ? __ldcg(&incl[(size_t)(str * nblk + lo) * 128 + ch]) : 0.f;
      float HA = 1.f, HB = 0.f;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (jhi - i >= stop) {  // H <- H o map(jhi - i)
          HB = fmaf(HA, rb[i], HB);
          HA *= ra[i];
        }
      }
      if (hh == 1) {
        sLA[ch] = HA;
        sLB[ch] = HB;
      }
      __syncthreads();
      if (hh == 0) {
        MB = fmaf(MA, HB, MB);  // M <- M o high half
        MA *= HA;
        const float LA = sLA[ch], LB = sLB[ch];
        MB = fmaf(MA, LB, MB);  // M <- M o low half
        MA *= LA;
        if (found) cin = fmaf(MA, ci, MB);
      }
      if (found) break;
      base = lo - 1;
      __syncthreads();  // s_lo / s_found reused
    }
  }
  // ---- 3. publish the inclusive carry, then replay
  if (c < 128) {
    incl[(size_t)me * 128 + c] = fmaf(BA, cin, BB);
    sCin[c] = cin;
  }
  __syncthreads();
  if (threadIdx.x == 0) sp_st_release(&flags[me], 2);
  if (threadIdx.x == 0) SCAN_STAMP(s_ticket, 2);
  if (!act || t0 >= T) return;
  float cc[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) cc[j] = fmaf(sA[w][4 * lane + j], sCin[4 * lane + j], sB[w][4 * lane + j]);
  float c0r = cc[0], c1r = cc[1], c2r = cc[2], c3r = cc[3];
  bool bad = false;
  bf16x4 bu[2][kSpPF], bfv[2][kSpPF], br[2][kSpPF];
  float4 bx[2][kSpPF];
  auto fetch = [&](int buf, int tb) {
#pragma unroll
    for (int i = 0; i < kSpPF; ++i) {
      const int t = min(tb + i, t1 - 1);
      const __nv_bfloat16* p = ufr + (size_t)t * ld3 + 4 * cq;
      bu[buf][i] = *reinterpret_cast<const bf16x4*>(p);
      bfv[buf][i] = *reinterpret_cast<const bf16x4*>(p + d);
      br[buf][i] = *reinterpret_cast<const bf16x4*>(p + 2 * d);
      bx[buf][i] = *reinterpret_cast<const float4*>(x + (size_t)t * d + 4 * cq);
    }
  };
  fetch(0, t0);
#pragma unroll 1
  for (int tb = t0; tb < t1; tb += 2 * kSpPF) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int tc = tb + half * kSpPF;
      if (tc >= t1) break;
      if (tc + kSpPF < t1) fetch(half ^ 1, tc + kSpPF);
#pragma unroll
      for (int i = 0; i < kSpPF; ++i) {
        const int t = tc + i;
        if (t < t1) {
          const float2 ua = __bfloat1622float2(bu[half][i].a), ub = __bfloat1622float2(bu[half][i].b);
          const float2 fa = __bfloat1622float2(bfv[half][i].a), fb = __bfloat1622float2(bfv[half][i].b);
          const float2 ra = __bfloat1622float2(br[half][i].a), rb = __bfloat1622float2(br[half][i].b);
          const float4 xv = bx[half][i];
          float4 h;
          h.x = sru_step(c0r, ua.x, fa.x, ra.x, xv.x);
          h.y = sru_step(c1r, ua.y, fa.y, ra.y, xv.y);
          h.z = sru_step(c2r, ub.x, fb.x, rb.x, xv.z);
          h.w = sru_step(c3r, ub.y, fb.y, rb.y, xv.w);
          bad |= !(isfinite(h.x) && isfinite(h.y) && isfinite(h.z) && isfinite(h.w) &&
                   isfinite(c0r + c1r + c2r + c3r));
          *reinterpret_cast<float4*>(h32 + (size_t)t * d + 4 * cq) = h;
          bf16x4 hb;
          hb.a = __floats2bfloat162_rn(h.x, h.y);
          hb.b = __floats2bfloat162_rn(h.z, h.w);
          *reinterpret_cast<bf16x4*>(h16 + (size_t)t * d + 4 * cq) = hb;
        }
      }
    }
  }
  if (c_last && t1 == T) *reinterpret_cast<float4*>(c_last + 4 * cq) = make_float4(c0r, c1r, c2r, c3r);
  if (bad) atomicOr(nonfinite, 1);  // reference raises NumericError (src/predictor.py:170-171)
#ifdef MP_DIAG
  if ((threadIdx.x & 31) == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    if (s_ticket < 1024) atomicMax(&g_scan_t[s_ticket][3], t_);
  }
#endif
}


// carry into shard `rank` of a token-sharded sequence: fold the shards' whole-range maps
// tots[g] = (A_g [d], B_g [d]) of shards g < rank onto c = c0 (or 0).
__global__ void k_sru_fold(const float* __restrict__ tots, int rank, int d, const float* __restrict__ c0,
                           float* __restrict__ out) {
  griddep_launch_dependents();
  griddep_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  float run = c0 ? c0[c] : 0.f;
  for (int g = 0; g < rank; ++g) run = fmaf(tots[(size_t)g * 2 * d + c], run, tots[(size_t)g * 2 * d + d + c]);
  out[c] = run;
}

// sparsemax rows (src/predictor.py:198-209) in float64, one thread per row:
// insertion-sort descending into local memory, sorted-threshold tau.
__global__ void k_sparsemax(const double* __restrict__ z, int n, int E, double* __restrict__ out) {
  griddep_launch_dependents();
  griddep_wait();
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
  const size_t sp_blocks = (size_t)cdiv(d, 128) * cdiv(T, kSpTokens);  // single-pass scan flags + ticket
  return al(sizeof(__nv_bfloat16) * (size_t)T * 3 * d) + 3 * al(sizeof(float) * (size_t)nch * d) +
         al(sizeof(int) * (sp_blocks + 1));
}

struct SruWs {
  __nv_bfloat16* ufr;
  float *aggA, *aggB, *carry;
  int* sp_flags;  // single-pass scan: per-block flags (+ ticket counter); block maps in aggA, carries in carry
  SruWs(void* ws, int T, int d) {
    const int nch = cdiv(T, kScanChunk);
    char* p = (char*)ws;
    ufr = (__nv_bfloat16*)p;
    p += al(sizeof(__nv_bfloat16) * (size_t)T * 3 * d);
    aggA = (float*)p;
    p += al(sizeof(float) * (size_t)nch * d);
    aggB = (float*)p;
    p += al(sizeof(float) * (size_t)nch * d);
    carry = (float*)p;
    p += al(sizeof(float) * (size_t)nch * d);
    sp_flags = (int*)p;
  }
};

#define SRU_CHECKS()                                                                                          \
  MP_REQUIRE(T >= 1, MP_ERR_CONFIG, "batch must contain at least one token");                                  \
  MP_REQUIRE(d >= 64 && d % 64 == 0, MP_ERR_CONFIG, "mp_sru: d=%d must be a multiple of 64 (pad)", d);           \
  MP_REQUIRE(ws_bytes >= mp_sru_workspace_bytes(T, d), MP_ERR_CONFIG, "mp_sru: workspace too small");

extern "C" int mp_sru_project(const void* x_bf16, const void* w_cat, const float* b_cat, int T, int d, void* ws,
                              size_t ws_bytes, void* stream) {
  SRU_CHECKS();
  // K1: [u | f | r] = x W_cat^T + b ; sigmoid on the f and r blocks
  return gemm_bf16(x_bf16, w_cat, SruWs(ws, T, d).ufr, T, 3 * d, d, 0, 3 * d, b_cat, 2, d, /*evict_last*/ 1, stream, pred_grid());
}

extern "C" int mp_sru_scan(const float* x_f32, int T, int d, const float* c0, float* h_f32, void* h_bf16,
                           float* c_last, int32_t* nonfinite, void* ws, size_t ws_bytes, void* stream) {
  SRU_CHECKS();
  cudaStream_t st = (cudaStream_t)stream;
  const SruWs w(ws, T, d);
  // K2: one launch -- chunk maps, decoupled look-back carries, replay + highway
  const int nblk = cdiv(T, kSpTokens), nstr = cdiv(d, 128);
  MP_CUDA_TRY(cudaMemsetAsync(w.sp_flags, 0, sizeof(int) * ((size_t)nstr * nblk + 1), st));
  MP_CUDA_TRY(launch_pdl(k_scan_fused, dim3(nstr * nblk), dim3(32 * kSpWarps), 0, st, w.ufr, x_f32, T, d, c0, h_f32,
                         (__nv_bfloat16*)h_bf16, c_last, nonfinite, w.sp_flags, w.aggA, w.carry, nblk));
  return MP_OK;
}

// Token-sharded SRU: every rank projects its own rows, then
//   mp_sru_scan_total   pass A + carries from 0; tot (2d) = the shard's whole-range map
//   (all-gather tot over ranks; mp_sru_fold_carry -> this shard's carry-in)
//   mp_sru_scan_finish  carries from carry-in + replay (pass A results reused from ws)
extern "C" int mp_sru_scan_total(int T, int d, float* tot, void* ws, size_t ws_bytes, void* stream) {
  SRU_CHECKS();
  cudaStream_t st = (cudaStream_t)stream;
  const SruWs w(ws, T, d);
  const int nch = cdiv(T, kScanChunk);
  const dim3 gq(cdiv(d / 4, 64), nch);
  MP_CUDA_TRY(launch_pdl(k_scan_aggregate, dim3(gq), dim3(64), 0, st, w.ufr, T, d, w.aggA, w.aggB));
  MP_CUDA_TRY(launch_pdl(k_scan_carry, dim3(cdiv(d, 32)), dim3(32 * kCarryGroups), 0, st, w.aggA, w.aggB, nch, d, nullptr, w.carry, tot));
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_sru_fold_carry(const float* tots, int rank, int d, const float* c0, float* carry_in, void* stream) {
  MP_REQUIRE(rank >= 0 && d >= 1, MP_ERR_CONFIG, "mp_sru_fold_carry: bad rank/d");
  k_sru_fold<<<cdiv(d, 256), 256, 0, (cudaStream_t)stream>>>(tots, rank, d, c0, carry_in);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_sru_scan_finish(const float* x_f32, int T, int d, const float* c0, float* h_f32, void* h_bf16,
                                  float* c_last, int32_t* nonfinite, void* ws, size_t ws_bytes, void* stream) {
  SRU_CHECKS();
  cudaStream_t st = (cudaStream_t)stream;
  const SruWs w(ws, T, d);
  const int nch = cdiv(T, kScanChunk);
  const dim3 gq(cdiv(d / 4, 64), nch);
  MP_CUDA_TRY(launch_pdl(k_scan_carry, dim3(cdiv(d, 32)), dim3(32 * kCarryGroups), 0, st, w.aggA, w.aggB, nch, d, c0, w.carry, nullptr));
  MP_CUDA_TRY(launch_pdl(k_scan_output, dim3(gq), dim3(64), 0, st, w.ufr, x_f32, T, d, w.carry, h_f32, (__nv_bfloat16*)h_bf16, c_last, nonfinite));
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_sru_layer(const void* x_bf16, const float* x_f32, const void* w_cat, const float* b_cat, int T,
                            int d, const float* c0, float* h_f32, void* h_bf16, float* c_last, int32_t* nonfinite,
                            void* ws, size_t ws_bytes, void* stream) {
  int rc = mp_sru_project(x_bf16, w_cat, b_cat, T, d, ws, ws_bytes, stream);
  if (rc) return rc;
  return mp_sru_scan(x_f32, T, d, c0, h_f32, h_bf16, c_last, nonfinite, ws, ws_bytes, stream);
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
  const int grid = units < pred_grid() ? units : pred_grid();
  if (bn == 256 && Eg <= 128) {  // one group per column half: both epilogue warpgroups work
    EpiGroupArgmaxT<true> es{assign, T, Eg, E, L};
    return launch_gemm<256, 4>(ta, tb, s, es, grid, st);
  }
  if (bn == 256) return launch_gemm<256, 4>(ta, tb, s, e, grid, st);
  if (bn == 128) return launch_gemm<128, 6>(ta, tb, s, e, grid, st);
  return launch_gemm<64, 8>(ta, tb, s, e, grid, st);
}

#ifdef MP_DIAG
extern "C" __attribute__((visibility("default"))) int mp_debug_scan_trace(unsigned long long* out) {
  MP_CUDA_TRY(cudaMemcpyFromSymbol(out, mp::g_scan_t, sizeof(mp::g_scan_t)));
  return MP_OK;
}
extern "C" __attribute__((visibility("default"))) int mp_debug_scan_trace_reset() {
  static unsigned long long zero[1024][4];
  MP_CUDA_TRY(cudaMemcpyToSymbol(mp::g_scan_t, zero, sizeof(zero)));
  return MP_OK;
}
#endif
