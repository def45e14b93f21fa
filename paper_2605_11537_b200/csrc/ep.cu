// Expert-parallel dispatch/combine planning.
//
// G ranks, tokens sharded contiguously by position, every rank routes its own
// tokens. After an all-gather of per-rank expert counts C[g][e], every rank
// computes the SAME plan from C and the (replicated) residency state:
//   * execution slots exactly as the single-device map (src/simulator.py:185-203):
//     cnt_e = res_e, or one corrective replica; slot (e, j) for j < cnt_e;
//   * a token's GLOBAL stable rank = its local rank + sum_{g < rank} C[g][e], so
//     slot(t) = off[e] + grank mod cnt_e is bit-identical to one device;
//   * replica -> GPU: the slot list (expert-major, ordinal-minor) is cut into G blocks of
//     equal rows -- slot s runs on GPU floor((rows before s + size_s / 2) * G / total rows).
//     Every GPU gets ~total/G rows and a hot expert's replicas stay on as few (consecutive)
//     GPUs as its rows need, so each expert's weights are streamed by as few GPUs as possible
//     (all expert weights are resident on every GPU);
//   * rows(g, s) = #tokens of rank g on slot s, in closed form:
//     #{y in [B_g, B_g + C_g) : y = j mod c} = F(B_g + C_g) - F(B_g),
//     F(x) = max(0, ceil((x - j) / c)).
// Sender packs rows by (destination, slot, position); receiver lays rows out by
// (slot, global position) -- the single-device order -- so the grouped GEMM and
// its results are bit-identical to the 1-GPU path.
//
// Fixed-split ("capacity") mode, peer_cap > 0: every (source, destination) block of the
// send / receive buffers has peer_cap rows, so the all-to-alls have equal, static splits
// and the whole step can be captured in a CUDA graph (no split sizes reach the host). A
// layer whose plan needs more than peer_cap rows for some peer sets *overflow and turns
// into a no-op on the device (no pieces, no sends); the caller checks the flag once per
// step and re-runs the step in the compact mode.
#include <cuda_bf16.h>

#include "common.cuh"

#include <algorithm>

namespace mp {

__device__ __forceinline__ int runs_before(int x, int j, int c) {  // F(x)
  return x > j ? (x - j + c - 1) / c : 0;
}

// grid 1, block 1024. ws layout given by EpPlanWs.
struct EpPlanWs {
  int32_t* off;        // E + 1 slot offsets
  int32_t* cnt;        // E
  int32_t* B;          // E: sum_{g < rank} C[g][e]
  int32_t* slot_gpu;   // S
  int32_t* slot_size;  // S
  int32_t* rows;       // G x S
  int32_t* send_base;  // S (this rank as sender)
  int32_t* recv_start; // G x S (this rank as receiver)
  int32_t* local_start;// G x S
};

__global__ void k_ep_plan(const int32_t* __restrict__ C, int G, int E, int rank, int max_slots, int split,
                          int32_t* __restrict__ res, EpPlanWs w, int32_t* __restrict__ send_counts,
                          int32_t* __restrict__ recv_counts, int32_t* __restrict__ num_local_rows,
                          int32_t* __restrict__ piece_row, int32_t* __restrict__ piece_rows,
                          int32_t* __restrict__ exp_begin, int32_t* __restrict__ err, int peer_cap,
                          int32_t* __restrict__ overflow) {
  griddep_launch_dependents();
  griddep_wait();
  extern __shared__ int sm[];
  __shared__ int red[40];
  __shared__ int s_over;
  if (threadIdx.x == 0) s_over = 0;
  int* s_off = sm;                   // E + 1
  int* s_lb = s_off + E + 1;         // max_slots + 1 : local base (hosted slots)
  int* s_pc = s_lb + max_slots + 1;  // max_slots + 1 : pieces per slot
  int* s_gpu = s_pc + max_slots + 1; // max_slots     : GPU of each slot
  int* s_rows = s_gpu + max_slots;   // G x max_slots : rows of (source, slot), for the per-peer scans
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int n = 0, b = 0;
    for (int g = 0; g < G; ++g) {
      const int c = C[(size_t)g * E + e];
      n += c;
      if (g < rank) b += c;
    }
    const int rp = res[e];
    const int c = rp > 0 ? rp : (n > 0 ? 1 : 0);
    res[e] = c;  // corrective replicas persist (src/simulator.py:190-192)
    w.cnt[e] = c;
    w.B[e] = b;
    s_off[e] = c;
  }
  __syncthreads();
  const int S = block_exclusive_scan(s_off, E, red);
  if (threadIdx.x == 0) s_off[E] = S;
  __syncthreads();
  if (S > max_slots) {  // report through the sizes the host reads anyway: no collective runs
    if (threadIdx.x == 0) {
      atomicExch(err, 1);
      *num_local_rows = -1;
      if (overflow) atomicOr(overflow, 1);  // fixed-split mode: the host re-runs the step compactly
    }
    for (int e = threadIdx.x; e <= E; e += blockDim.x) exp_begin[e] = 0;
    for (int g = threadIdx.x; g < G; g += blockDim.x) send_counts[g] = recv_counts[g] = 0;
    return;
  }
  for (int e = threadIdx.x; e <= E; e += blockDim.x) w.off[e] = s_off[e];
  // slots: expert, ordinal, size, GPU; per-rank row counts
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    int lo = 0, hi = E;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_off[mid] <= s) lo = mid; else hi = mid;
    }
    const int e = lo, j = s - s_off[e], c = s_off[e + 1] - s_off[e];
    int size = 0, acc = 0;
    for (int g = 0; g < G; ++g) {
      const int cg = C[(size_t)g * E + e];
      const int r = runs_before(acc + cg, j, c) - runs_before(acc, j, c);
      w.rows[(size_t)g * max_slots + s] = r;
      s_rows[(size_t)g * max_slots + s] = r;
      size += r;
      acc += cg;
    }
    w.slot_size[s] = size;
    s_lb[s] = size;  // scanned below into the rows before each slot
  }
  __syncthreads();
  const int total = block_exclusive_scan(s_lb, S, red);
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    const int size = w.slot_size[s];
    const long long mid2 = 2LL * s_lb[s] + size;  // twice the slot's row midpoint
    const int gpu = total > 0 ? (int)min((long long)G - 1, (mid2 * G) / (2LL * total)) : 0;
    w.slot_gpu[s] = gpu;
    s_gpu[s] = gpu;
  }
  __syncthreads();
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    const int size = w.slot_size[s], gpu = s_gpu[s];
    s_lb[s] = (gpu == rank) ? size : 0;
    s_pc[s] = (gpu == rank) ? (split ? cdiv(size, kBlockMRows) : (size > 0 ? 1 : 0)) : 0;
  }
  __syncthreads();
  const int nloc = block_exclusive_scan(s_lb, S, red);  // local row base of hosted slots
  const int P = block_exclusive_scan(s_pc, S, red);
  if (threadIdx.x == 0) {
    s_lb[S] = nloc;
    s_pc[S] = P;
    *num_local_rows = nloc;
  }
  __syncthreads();
  if (peer_cap > 0) {  // every (source, destination) block against the fixed split: all ranks hold
                       // the same counts and plan, so all reach the same decision
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int pair = warp; pair < G * G; pair += blockDim.x >> 5) {
      const int src = pair / G, dst = pair - src * G;
      int sum = 0;
      for (int s = lane; s < S; s += 32) sum += s_gpu[s] == dst ? s_rows[(size_t)src * max_slots + s] : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (lane == 0 && sum > peer_cap) s_over = 1;
    }
  }
  __syncthreads();
  if (s_over) {  // fixed splits too small: the layer becomes a no-op on every rank, the step is flagged
    if (threadIdx.x == 0) {
      atomicExch(err, 1);
      if (overflow) atomicOr(overflow, 1);
    }
    for (int e = threadIdx.x; e <= E; e += blockDim.x) exp_begin[e] = 0;
    return;
  }
  // sender tables (this rank) and receiver tables, one thread per peer
  {  // per peer d (one warp each, G <= 32): exclusive scans over the slots, 32 slots per step
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < G) {
      const int d = warp;
      int acc_s = 0, acc_r = 0;
      for (int base = 0; base < S; base += 32) {
        const int s = base + lane;
        const int gpu = s < S ? s_gpu[s] : -1;
        const int vs = gpu == d ? s_rows[(size_t)rank * max_slots + s] : 0;  // this rank sends slot s to d
        const int vr = gpu == rank ? s_rows[(size_t)d * max_slots + s] : 0;  // d sends slot s here
        int is = vs, ir = vr;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int ys = __shfl_up_sync(0xffffffffu, is, o), yr = __shfl_up_sync(0xffffffffu, ir, o);
          if (lane >= o) {
            is += ys;
            ir += yr;
          }
        }
        if (gpu == d) w.send_base[s] = acc_s + is - vs;                              // within d's block
        if (gpu == rank) w.recv_start[(size_t)d * max_slots + s] = acc_r + ir - vr;  // within d's block
        acc_s += __shfl_sync(0xffffffffu, is, 31);
        acc_r += __shfl_sync(0xffffffffu, ir, 31);
      }
      if (lane == 0) {
        send_counts[d] = acc_s;
        recv_counts[d] = acc_r;

      }
    }
  }
  __syncthreads();
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    const int gpu = s_gpu[s];
    int displ = 0;
    if (peer_cap > 0)
      displ = gpu * peer_cap;
    else
      for (int g = 0; g < gpu; ++g) displ += send_counts[g];
    w.send_base[s] += displ;
    if (gpu == rank) {
      int acc = s_lb[s], rdispl = 0;
      for (int g = 0; g < G; ++g) {
        w.local_start[(size_t)g * max_slots + s] = acc;
        acc += s_rows[(size_t)g * max_slots + s];
        w.recv_start[(size_t)g * max_slots + s] += rdispl;
        rdispl += peer_cap > 0 ? peer_cap : recv_counts[g];
      }
      const int row0 = s_lb[s], size = w.slot_size[s];
      const int p0 = s_pc[s], np = s_pc[s + 1] - p0;
      for (int p = 0; p < np; ++p) {
        piece_row[p0 + p] = split ? row0 + p * kBlockMRows : row0;
        piece_rows[p0 + p] = split ? min(kBlockMRows, size - p * kBlockMRows) : size;
      }
    }
  }
  for (int e = threadIdx.x; e <= E; e += blockDim.x) exp_begin[e] = s_pc[s_off[e]];
}

// Sender: global rank -> slot -> send position; one thread per token (chunked stable rank).
__global__ void k_ep_send_pos(const int32_t* __restrict__ route, int T, int E, int nch, const int32_t* __restrict__ cc,
                              EpPlanWs w, int32_t* __restrict__ send_pos, const int32_t* __restrict__ err) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ int se[kChunk];
  const int ch = blockIdx.x;
  const int t = ch * kChunk + threadIdx.x;
  if (*err) {  // the plan overflowed (max_slots or the fixed split): nothing is sent or combined
    if (t < T) send_pos[t] = -1;
    return;
  }
  const int e = (t < T) ? __ldg(&route[t]) : -1;
  se[threadIdx.x] = e;
  __syncthreads();
  int rin = 0;
  for (int k = 0; k < (int)threadIdx.x; ++k) rin += (se[k] == e);
  if (t >= T) return;
  const int b = w.B[e], c = w.cnt[e];
  const int grank = b + cc[(size_t)ch * E + e] + rin;
  const int j = grank % c;
  const int s = w.off[e] + j;
  send_pos[t] = w.send_base[s] + (grank / c - runs_before(b, j, c));
}

// sendbuf[send_pos[t]] = bf16(x[t]); one warp per token.
__global__ void k_ep_pack(const float* __restrict__ x, int T, int d, const int32_t* __restrict__ send_pos,
                          __nv_bfloat16* __restrict__ sendbuf) {
  griddep_launch_dependents();
  griddep_wait();
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (t >= T || send_pos[t] < 0) return;
  const float4* src = reinterpret_cast<const float4*>(x + (size_t)t * d);
  uint2* dst = reinterpret_cast<uint2*>(sendbuf + (size_t)send_pos[t] * d);
  for (int k = lane; k < d / 4; k += 32) {
    const float4 v = __ldg(&src[k]);
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    dst[k] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  }
}

// Expert parallelism over peer memory (NVLink P2P, fixed-split layout): source rank `rank`
// writes token t straight into destination g's receive block for it, row rank * peer_cap + j
// (send_pos[t] = g * peer_cap + j), and the token index beside it, so g's GEMM2 can add the
// result back into this rank's stream (EpiScatterAdd peer mode). One warp per token.
__global__ void k_ep_pack_peer(const float* __restrict__ x, int T, int d, const int32_t* __restrict__ send_pos,
                               int peer_cap, int rank, __nv_bfloat16* const* __restrict__ recv_rows,
                               int32_t* const* __restrict__ recv_tok) {
  griddep_launch_dependents();
  griddep_wait();
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int sp = t < T ? send_pos[t] : -1;
  if (sp >= 0) {
    const int g = sp / peer_cap, row = rank * peer_cap + (sp - g * peer_cap);
    const float4* src = reinterpret_cast<const float4*>(x + (size_t)t * d);
    uint2* dst = reinterpret_cast<uint2*>(recv_rows[g] + (size_t)row * d);
    for (int k = lane; k < d / 4; k += 32) {
      const float4 v = __ldg(&src[k]);
      __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
      dst[k] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
    }
    if (lane == 0) recv_tok[g][row] = t;
  }
  // no fence here: the barrier kernel that follows waits for this grid's completion (memory
  // flushed) and fences at system scope before it signals -- an on-stream barrier
}

// dst[g][row * dst_row_stride + rank * n + i] = src[row * n + i] for every rank g (peer stores):
// an all-gather of rows x n 32-bit words per rank (e.g. expert counts, SRU carry maps, predicted
// assignments); a device barrier completes it.
__global__ void k_peer_allgather_i32(const int32_t* __restrict__ src, int rows, int n, int rank, int G,
                                     int32_t* const* __restrict__ dst, int dst_row_stride) {
  griddep_launch_dependents();
  griddep_wait();
  const size_t total = (size_t)rows * n;
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < total; k += (size_t)gridDim.x * blockDim.x) {
    const int row = (int)(k / n), i = (int)(k - (size_t)row * n);
    const int32_t v = src[k];
    const size_t o = (size_t)row * dst_row_stride + (size_t)rank * n + i;
    for (int g = 0; g < G; ++g) dst[g][o] = v;
  }
}

// Receiver side of the peer-memory path: xperm[row] = recvbuf[idx[row]] and the destination
// code of the row's result, home * T_home + t (home = idx / peer_cap, t from recv_tok).
__global__ void k_ep_gather_peer(const __nv_bfloat16* __restrict__ buf, int n, int d, const int32_t* __restrict__ idx,
                                 const int32_t* __restrict__ n_dev, const int32_t* __restrict__ recv_tok, int peer_cap,
                                 int T_home, int32_t* __restrict__ dst_of_row, __nv_bfloat16* __restrict__ out) {
  griddep_launch_dependents();
  griddep_wait();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n || (n_dev != nullptr && row >= *n_dev)) return;
  const int ri = __ldg(&idx[row]);
  const uint4* src = reinterpret_cast<const uint4*>(buf + (size_t)ri * d);
  uint4* dst = reinterpret_cast<uint4*>(out + (size_t)row * d);
  for (int k = lane; k < d / 8; k += 32) dst[k] = __ldg(&src[k]);
  if (lane == 0) dst_of_row[row] = (ri / peer_cap) * T_home + recv_tok[ri];
}

// Device-side barrier over G ranks' flag arrays in peer memory (G <= 32, one warp): epoch e
// = ++*epoch; lane g publishes e into rank g's slot for this rank (release, system scope),
// lane s waits until rank s's e has arrived here (acquire). The kernels before it on the
// stream -- the peer stores and reductions it hands over -- have completed before it starts
// (stream order; griddepcontrol.wait covers a programmatic launch too), and the system-scope
// fence orders them before the flags (an on-stream barrier: no fence in the producers).
__global__ void k_peer_barrier(int32_t* const* __restrict__ flags, int rank, int G, int32_t* __restrict__ epoch,
                               int32_t* __restrict__ err) {
  griddep_wait();
  const int lane = threadIdx.x;
  int e = 0;
  if (lane == 0) {
    e = *epoch + 1;
    *epoch = e;
  }
  e = __shfl_sync(0xffffffffu, e, 0);
  __threadfence_system();
  if (lane < G) {
    int32_t* f = flags[lane] + rank;
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(f), "r"(e) : "memory");
  }
  if (lane < G) {
    const int32_t* f = flags[rank] + lane;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    int v;
    for (int it = 0;; ++it) {
      asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if (v >= e) break;
      __nanosleep(64);
      if ((it & 1023) == 1023) {  // a rank that never arrives: flag it instead of hanging the GPU
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 5000000000ull) {
          atomicOr(err, 1);
          break;
        }
      }
    }
  }
  __syncwarp();
  griddep_launch_dependents();
}

// Receiver: local row of every received row, per (source, hosted slot) run.
// grid (max_slots, G): one block per (slot, source); slots beyond the plan's count exit.
__global__ void k_ep_recv_map(int G, int max_slots, const int32_t* __restrict__ num_slots_p, int rank, EpPlanWs w,
                              int32_t* __restrict__ recv_of_local, const int32_t* __restrict__ err) {
  griddep_launch_dependents();
  griddep_wait();
  if (*err) return;
  const int s = blockIdx.x, g = blockIdx.y;
  if (s >= *num_slots_p || w.slot_gpu[s] != rank) return;
  const int n = w.rows[(size_t)g * max_slots + s];
  const int r0 = w.recv_start[(size_t)g * max_slots + s], l0 = w.local_start[(size_t)g * max_slots + s];
  for (int k = threadIdx.x; k < n; k += blockDim.x) recv_of_local[l0 + k] = r0 + k;
}

// xperm[row] = buf[idx[row]] for bf16 rows; one warp per row. n_dev (optional): the row
// count lives on the device (fixed-split EP: n is the buffer's capacity).
__global__ void k_gather_bf16(const __nv_bfloat16* __restrict__ buf, int n, int d, const int32_t* __restrict__ idx,
                              __nv_bfloat16* __restrict__ out, const int32_t* __restrict__ n_dev) {
  griddep_launch_dependents();
  griddep_wait();
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n || (n_dev != nullptr && row >= *n_dev)) return;
  const uint4* src = reinterpret_cast<const uint4*>(buf + (size_t)__ldg(&idx[row]) * d);
  uint4* dst = reinterpret_cast<uint4*>(out + (size_t)row * d);
  for (int k = lane; k < d / 8; k += 32) dst[k] = __ldg(&src[k]);
}

// x[t] += yback[send_pos[t]] (fp32; each token owns one row -> no atomics). one warp per token.
__global__ void k_ep_combine(float* __restrict__ x, int T, int d, const float* __restrict__ yback,
                             const int32_t* __restrict__ send_pos) {
  griddep_launch_dependents();
  griddep_wait();
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (t >= T || send_pos[t] < 0) return;
  float4* dst = reinterpret_cast<float4*>(x + (size_t)t * d);
  const float4* src = reinterpret_cast<const float4*>(yback + (size_t)send_pos[t] * d);
  for (int k = lane; k < d / 4; k += 32) {
    float4 o = dst[k];
    const float4 v = __ldg(&src[k]);
    o.x += v.x;
    o.y += v.y;
    o.z += v.z;
    o.w += v.w;
    dst[k] = o;
  }
}

static inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

static EpPlanWs carve(void* ws, int G, int E, int max_slots, int32_t** cc, int nch, int32_t** err, int32_t** nslots) {
  char* p = (char*)ws;
  auto take = [&](size_t n) {
    int32_t* r = (int32_t*)p;
    p += al(sizeof(int32_t) * n);
    return r;
  };
  EpPlanWs w;
  w.off = take(E + 1);
  w.cnt = take(E);
  w.B = take(E);
  w.slot_gpu = take(max_slots);
  w.slot_size = take(max_slots);
  w.rows = take((size_t)G * max_slots);
  w.send_base = take(max_slots);
  w.recv_start = take((size_t)G * max_slots);
  w.local_start = take((size_t)G * max_slots);
  *cc = take((size_t)nch * E + E);
  *err = take(1);
  *nslots = take(1);
  return w;
}

}  // namespace mp

using namespace mp;

extern "C" int mp_ep_plan_cap(const int32_t* route, int T, const int32_t* C, int G, int E, int rank, int max_slots,
                              int split_m, int peer_cap, int32_t* overflow, int32_t* res, int32_t* send_counts,
                              int32_t* recv_counts, int32_t* num_local_rows, int32_t* send_pos, int32_t* piece_row,
                              int32_t* piece_rows, int32_t* exp_begin, void* ws, size_t ws_bytes, void* stream);
extern "C" int mp_gather_rows_bf16_dn(const void* buf, int n_max, int d, const int32_t* idx, const int32_t* n_dev,
                                      void* out, void* stream);

extern "C" size_t mp_ep_workspace_bytes(int G, int T, int E, int max_slots) {
  const int nch = cdiv(T > 0 ? T : 1, kChunk);
  return al(4 * (size_t)(E + 1)) + 2 * al(4 * (size_t)E) + 3 * al(4 * (size_t)max_slots) +
         3 * al(4 * (size_t)G * max_slots) + al(4 * ((size_t)nch * E + E)) + 2 * al(4);
}

extern "C" int mp_ep_plan(const int32_t* route, int T, const int32_t* C, int G, int E, int rank, int max_slots,
                          int split_m, int32_t* res, int32_t* send_counts, int32_t* recv_counts,
                          int32_t* num_local_rows, int32_t* send_pos, int32_t* piece_row, int32_t* piece_rows,
                          int32_t* exp_begin, void* ws, size_t ws_bytes, void* stream) {
  return mp_ep_plan_cap(route, T, C, G, E, rank, max_slots, split_m, 0, nullptr, res, send_counts, recv_counts,
                        num_local_rows, send_pos, piece_row, piece_rows, exp_begin, ws, ws_bytes, stream);
}

extern "C" int mp_ep_plan_cap(const int32_t* route, int T, const int32_t* C, int G, int E, int rank, int max_slots,
                              int split_m, int peer_cap, int32_t* overflow, int32_t* res, int32_t* send_counts,
                              int32_t* recv_counts, int32_t* num_local_rows, int32_t* send_pos, int32_t* piece_row,
                              int32_t* piece_rows, int32_t* exp_begin, void* ws, size_t ws_bytes, void* stream) {
  MP_REQUIRE(G >= 1 && G <= 32 && rank >= 0 && rank < G && E >= 1 && max_slots >= E && T >= 0 && peer_cap >= 0,
             MP_ERR_CONFIG, "mp_ep_plan: bad sizes G=%d rank=%d E=%d peer_cap=%d", G, rank, E, peer_cap);
  MP_REQUIRE(ws_bytes >= mp_ep_workspace_bytes(G, T, E, max_slots), MP_ERR_CONFIG, "mp_ep_plan: workspace");
  cudaStream_t st = (cudaStream_t)stream;
  const int nch = cdiv(T > 0 ? T : 1, kChunk);
  int32_t *cc, *err, *nslots;
  EpPlanWs w = carve(ws, G, E, max_slots, &cc, nch, &err, &nslots);
  const size_t sm = sizeof(int) * ((size_t)E + 1 + 2 * ((size_t)max_slots + 1) + (size_t)(G + 1) * max_slots);
  MP_REQUIRE(sm <= 200 * 1024, MP_ERR_CONFIG, "mp_ep_plan: G x max_slots too large for shared memory");
  static bool configured = false;
  if (!configured) {
    MP_CUDA_TRY(cudaFuncSetAttribute(k_ep_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(200 * 1024)));
    configured = true;
  }
  MP_CUDA_TRY(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
  k_ep_plan<<<1, 1024, sm, st>>>(C, G, E, rank, max_slots, split_m & 1, res, w, send_counts, recv_counts,
                                 num_local_rows, piece_row, piece_rows, exp_begin, err, peer_cap, overflow);
  if (T > 0) {
    // local stable ranks (chunk histograms + exclusive scan over chunks)
    int rc = mp_histogram_ws(route, 1, T, E, cc + (size_t)nch * E, cc, (size_t)nch * E * 4, stream);
    if (rc) return rc;
    k_ep_send_pos<<<nch, kChunk, 0, st>>>(route, T, E, nch, cc, w, send_pos, err);
  }
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_ep_pack(const float* x, int T, int d, const int32_t* send_pos, void* sendbuf, void* stream) {
  MP_REQUIRE(d % 8 == 0, MP_ERR_CONFIG, "mp_ep_pack: d %% 8 != 0");
  if (T > 0) k_ep_pack<<<cdiv(T * 32, 256), 256, 0, (cudaStream_t)stream>>>(x, T, d, send_pos, (__nv_bfloat16*)sendbuf);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_ep_recv_layout(int G, int T, int E, int rank, int max_slots, const int32_t* recvbuf_rows_unused,
                                 int32_t* recv_of_local, void* ws, size_t ws_bytes, void* stream) {
  (void)recvbuf_rows_unused;
  const int nch = cdiv(T > 0 ? T : 1, kChunk);
  int32_t *cc, *err, *nslots;
  EpPlanWs w = carve(ws, G, E, max_slots, &cc, nch, &err, &nslots);
  MP_REQUIRE(ws_bytes >= mp_ep_workspace_bytes(G, T, E, max_slots), MP_ERR_CONFIG, "mp_ep_recv_layout: workspace");
  // number of slots = off[E]
  k_ep_recv_map<<<dim3(max_slots, G), 128, 0, (cudaStream_t)stream>>>(G, max_slots, w.off + E, rank, w,
                                                                       recv_of_local, err);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_gather_rows_bf16(const void* buf, int n, int d, const int32_t* idx, void* out, void* stream) {
  return mp_gather_rows_bf16_dn(buf, n, d, idx, nullptr, out, stream);
}

extern "C" int mp_gather_rows_bf16_dn(const void* buf, int n_max, int d, const int32_t* idx, const int32_t* n_dev,
                                      void* out, void* stream) {
  MP_REQUIRE(d % 8 == 0, MP_ERR_CONFIG, "mp_gather_rows_bf16: d %% 8 != 0");
  if (n_max > 0)
    k_gather_bf16<<<cdiv(n_max * 32, 256), 256, 0, (cudaStream_t)stream>>>((const __nv_bfloat16*)buf, n_max, d, idx,
                                                                             (__nv_bfloat16*)out, n_dev);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_ep_pack_peer(const float* x, int T, int d, const int32_t* send_pos, int peer_cap, int rank,
                               void* const* recv_rows, int32_t* const* recv_tok, void* stream) {
  MP_REQUIRE(T >= 0 && d % 4 == 0 && peer_cap >= 1 && rank >= 0, MP_ERR_CONFIG, "mp_ep_pack_peer: bad sizes");
  if (T == 0) return MP_OK;
  MP_CUDA_TRY(launch_pdl(k_ep_pack_peer, dim3(cdiv(T * 32, 256)), dim3(256), 0, (cudaStream_t)stream, x, T, d,
                         send_pos, peer_cap, rank, (__nv_bfloat16* const*)recv_rows, recv_tok));
  return MP_OK;
}

extern "C" int mp_ep_gather_peer(const void* buf, int n_max, int d, const int32_t* idx, const int32_t* n_dev,
                                 const int32_t* recv_tok, int peer_cap, int T_home, int32_t* dst_of_row, void* out,
                                 void* stream) {
  MP_REQUIRE(n_max >= 0 && d % 8 == 0 && peer_cap >= 1 && T_home >= 1, MP_ERR_CONFIG, "mp_ep_gather_peer: bad sizes");
  if (n_max == 0) return MP_OK;
  MP_CUDA_TRY(launch_pdl(k_ep_gather_peer, dim3(cdiv(n_max * 32, 256)), dim3(256), 0, (cudaStream_t)stream,
                         (const __nv_bfloat16*)buf, n_max, d, idx, n_dev, recv_tok, peer_cap, T_home, dst_of_row,
                         (__nv_bfloat16*)out));
  return MP_OK;
}

extern "C" int mp_peer_allgather_i32(const int32_t* src, int rows, int n, int rank, int G, int32_t* const* dst,
                                     int dst_row_stride, void* stream) {
  MP_REQUIRE(rows >= 0 && n >= 0 && G >= 1 && rank >= 0 && rank < G && (rows <= 1 || dst_row_stride >= G * n),
             MP_ERR_CONFIG, "mp_peer_allgather_i32: bad sizes");
  const size_t total = (size_t)rows * n;
  if (total == 0) return MP_OK;
  const int grid = (int)std::min<size_t>((total + 255) / 256, 4096);
  MP_CUDA_TRY(launch_pdl(k_peer_allgather_i32, dim3(grid), dim3(256), 0, (cudaStream_t)stream, src, rows, n, rank, G,
                         dst, dst_row_stride));
  return MP_OK;
}

extern "C" int mp_peer_barrier(int32_t* const* flags, int rank, int G, int32_t* epoch, int32_t* err, void* stream) {
  MP_REQUIRE(G >= 1 && G <= 32 && rank >= 0 && rank < G && err != nullptr, MP_ERR_CONFIG,
             "mp_peer_barrier: G in [1, 32], err required");
  MP_CUDA_TRY(launch_pdl(k_peer_barrier, dim3(1), dim3(32), 0, (cudaStream_t)stream, flags, rank, G, epoch, err));
  return MP_OK;
}

extern "C" int mp_ep_combine(float* x, int T, int d, const float* yback, const int32_t* send_pos, void* stream) {
  MP_REQUIRE(d % 4 == 0, MP_ERR_CONFIG, "mp_ep_combine: d %% 4 != 0");
  if (T > 0) k_ep_combine<<<cdiv(T * 32, 256), 256, 0, (cudaStream_t)stream>>>(x, T, d, yback, send_pos);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}
