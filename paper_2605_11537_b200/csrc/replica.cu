// K9: physical expert replicas (north_star: "a replica plan that physically copies overloaded
// experts"; reference token walk src/placement.py:143-160 emits LOAD / REPLICATE / OFFLOAD,
// PAPER.md:172-178 moves the expert weights).
//
// Each MoE layer owns a pool of P weight slots (U and V of one expert each, in the grouped
// GEMMs' pre-tiled layout). The residency state res[e] (replicas of expert e after placement
// and the execution map's corrective loads) is materialised in the pool:
//   pool_cnt[e]       ordinals of e that currently hold a copy
//   pool_of[e*R + j]  pool slot of replica (e, j)
//   free stack        unused pool slots
// mp_pool_update diffs res against pool_cnt: ordinals above res are OFFLOADed (their slots
// pushed on the free stack, experts ascending, ordinals descending -- the reference's reclaim
// order), missing ordinals pop a slot and get a copy job: REPLICATE from the expert's ordinal-0
// copy on the GPU when one exists, else LOAD from the master weights. mp_replica_copy runs the
// jobs (16-byte vector copies, one block column per job); mp_piece_pool gives every GEMM piece
// the pool slot of its replica, and the grouped GEMMs read their B operand from there
// (mp_ffn_up_pool / mp_ffn_down_pool). Everything stays on the device (graph-capturable).
#include "common.cuh"
#include "launch.cuh"

#include <algorithm>

namespace mp {

// single block of 1024 threads; E <= 1024
__global__ void k_pool_update(const int32_t* __restrict__ res, int E, int R, int P, int32_t* __restrict__ cnt,
                              int32_t* __restrict__ pool_of, int32_t* __restrict__ free_stack,
                              int32_t* __restrict__ free_top, int32_t* __restrict__ jobs, int32_t* __restrict__ njobs,
                              int32_t* __restrict__ stats, int32_t* __restrict__ err) {
  __shared__ int s_f[1025], s_a[1025], red[40];
  const int e = threadIdx.x;
  int o = 0, n = 0;
  if (e < E) {
    o = cnt[e];
    n = min(max(res[e], 0), R);
    s_f[e] = max(o - n, 0);
    s_a[e] = max(n - o, 0);
  } else {
    s_f[e] = s_a[e] = 0;
  }
  __syncthreads();
  const int nf = block_exclusive_scan(s_f, E, red);
  const int na = block_exclusive_scan(s_a, E, red);
  const int top0 = *free_top;
  if (top0 + nf - na < 0) {  // pool too small for the residency state
    if (threadIdx.x == 0) {
      *err = 1;
      *njobs = 0;
    }
    return;
  }
  // offloads: push ordinals o-1 .. n in that order
  if (e < E) {
    for (int k = 0; k < o - n; ++k) free_stack[top0 + s_f[e] + k] = pool_of[(size_t)e * R + (o - 1 - k)];
  }
  __syncthreads();
  const int top1 = top0 + nf;
  // allocations: job i = s_a[e] + k pops free_stack[top1 - 1 - i]
  if (e < E && n > o) {
    const int src0 = o > 0 ? pool_of[(size_t)e * R] : -1 - e;  // replicate from ordinal 0, else load the master
    int loads = 0;
    for (int k = 0; k < n - o; ++k) {
      const int i = s_a[e] + k;
      const int dst = free_stack[top1 - 1 - i];
      pool_of[(size_t)e * R + o + k] = dst;
      // the first new copy of an absent expert comes from the master; the rest replicate it
      const int src = (o == 0 && k > 0) ? pool_of[(size_t)e * R] : src0;
      jobs[2 * i] = dst;
      jobs[2 * i + 1] = src;
      loads += src < 0;
    }
    atomicAdd(&stats[0], loads);
    atomicAdd(&stats[1], n - o - loads);
  }
  if (e < E) {
    if (o > n) atomicAdd(&stats[2], o - n);
    cnt[e] = n;
  }
  if (threadIdx.x == 0) {
    *free_top = top1 - na;
    *njobs = na;
  }
}

// job j (grid.y) copies src -> dst for U and V; blocks of grid.x stride over the 16-byte words.
// Jobs are ordered so a replicate never reads a slot written in the same launch unless its
// source is the expert's ordinal 0 written by an earlier job: those are split into two passes.
__global__ void k_replica_copy(const uint4* __restrict__ mu, const uint4* __restrict__ mv, uint4* __restrict__ pu,
                               uint4* __restrict__ pv, size_t words, const int32_t* __restrict__ jobs,
                               const int32_t* __restrict__ njobs, int pass) {
  const int nj = *njobs;
  for (int j = blockIdx.y; j < nj; j += gridDim.y) {
  const int dst = jobs[2 * j], src = jobs[2 * j + 1];
  // pass 0: loads from the masters and replicates of copies that existed before this update;
  // pass 1: replicates whose source is a copy loaded in pass 0 (marked by a negative-source
  //         first job of the same expert -- identified as: source slot written by a pass-0 job)
  const bool from_master = src < 0;
  bool src_new = false;
  if (!from_master) {
    for (int k = 0; k < nj; ++k)
      if (jobs[2 * k] == src) {
        src_new = true;
        break;
      }
  }
  if ((pass == 0) == src_new) continue;
  const uint4* su = from_master ? mu + (size_t)(-1 - src) * words : pu + (size_t)src * words;
  const uint4* sv = from_master ? mv + (size_t)(-1 - src) * words : pv + (size_t)src * words;
  uint4* du = pu + (size_t)dst * words;
  uint4* dv = pv + (size_t)dst * words;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < words; i += (size_t)gridDim.x * blockDim.x) {
    du[i] = __ldg(&su[i]);
    dv[i] = __ldg(&sv[i]);
  }
  }
}

// piece p of expert e (exp_begin) -> pool slot of its replica: the slot of the piece's first row
// (token_to_slot[tok_of_row[row]]) minus the slot of the expert's first piece (ordinal 0 always
// holds the expert's first token) is the ordinal.
__global__ void k_piece_pool(const int32_t* __restrict__ piece_row, const int32_t* __restrict__ exp_begin, int E,
                             const int32_t* __restrict__ tok_of_row, const int32_t* __restrict__ token_to_slot,
                             const int32_t* __restrict__ pool_of, int R, int32_t* __restrict__ piece_wbase,
                             int max_pieces) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int np = exp_begin[E];
  if (p >= np || p >= max_pieces) return;
  int lo = 0, hi = E;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (exp_begin[mid] <= p) lo = mid; else hi = mid;
  }
  const int s = token_to_slot[tok_of_row[piece_row[p]]];
  const int s0 = token_to_slot[tok_of_row[piece_row[exp_begin[lo]]]];
  piece_wbase[p] = max(pool_of[(size_t)lo * R + (s - s0)], 0);  // -1 only if the pool overflowed (err)
}

__global__ void k_pool_init(int E, int R, int P, int32_t* cnt, int32_t* pool_of, int32_t* free_stack,
                            int32_t* free_top, int32_t* stats) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < E) cnt[i] = 0;
  if (i < P) free_stack[i] = P - 1 - i;  // pops hand out slots 0, 1, 2, ...
  for (size_t k = i; k < (size_t)E * R; k += (size_t)gridDim.x * blockDim.x) pool_of[k] = -1;
  if (i == 0) {
    *free_top = P;
    for (int k = 0; k < 4; ++k) stats[k] = 0;
  }
}

}  // namespace mp

using namespace mp;

// pool state: [cnt E][pool_of E*R][free_stack P][free_top 1][jobs 2P][njobs 1][stats 4][err 1]
static inline size_t al4(size_t n) { return (n * 4 + 255) & ~size_t(255); }
struct PoolWs {
  int32_t *cnt, *pool_of, *free_stack, *free_top, *jobs, *njobs, *stats, *err;
  PoolWs(void* ws, int E, int R, int P) {
    char* p = (char*)ws;
    auto take = [&](size_t n) {
      int32_t* r = (int32_t*)p;
      p += al4(n);
      return r;
    };
    cnt = take(E);
    pool_of = take((size_t)E * R);
    free_stack = take(P);
    free_top = take(1);
    jobs = take(2 * (size_t)P);
    njobs = take(1);
    stats = take(4);
    err = take(1);
  }
};

extern "C" size_t mp_pool_state_bytes(int E, int R, int P) {
  return al4(E) + al4((size_t)E * R) + al4(P) + al4(1) + al4(2 * (size_t)P) + al4(1) + al4(4) + al4(1);
}

extern "C" int mp_pool_init(int E, int R, int P, void* state, void* stream) {
  MP_REQUIRE(E >= 1 && E <= 1024 && R >= 1 && P >= 1, MP_ERR_CONFIG, "mp_pool_init: bad sizes E=%d R=%d P=%d", E, R, P);
  PoolWs w(state, E, R, P);
  const int n = std::max(E, P);
  k_pool_init<<<cdiv(n, 256), 256, 0, (cudaStream_t)stream>>>(E, R, P, w.cnt, w.pool_of, w.free_stack, w.free_top,
                                                              w.stats);
  MP_CUDA_TRY(cudaMemsetAsync(w.err, 0, 4, (cudaStream_t)stream));
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_pool_update(const int32_t* res, int E, int R, int P, void* state, void* stream) {
  MP_REQUIRE(E >= 1 && E <= 1024, MP_ERR_CONFIG, "mp_pool_update: E=%d", E);
  PoolWs w(state, E, R, P);
  k_pool_update<<<1, 1024, 0, (cudaStream_t)stream>>>(res, E, R, P, w.cnt, w.pool_of, w.free_stack, w.free_top, w.jobs,
                                                       w.njobs, w.stats, w.err);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_replica_copy(const void* master_u, const void* master_v, void* pool_u, void* pool_v,
                               size_t expert_bytes, int P, const void* state, int E, int R, void* stream) {
  MP_REQUIRE(expert_bytes % 16 == 0, MP_ERR_CONFIG, "mp_replica_copy: expert bytes %% 16 != 0");
  PoolWs w(const_cast<void*>(state), E, R, P);
  const size_t words = expert_bytes / 16;
  // 16 job lanes x 64 blocks: a step's handful of copies each get 64 blocks; empty lanes exit
  const dim3 grid((unsigned)std::min<size_t>(cdiv((int)std::min<size_t>(words, 1 << 30), 256 * 8), 64), 16);
  for (int pass = 0; pass < 2; ++pass)
    k_replica_copy<<<grid, 256, 0, (cudaStream_t)stream>>>((const uint4*)master_u, (const uint4*)master_v,
                                                           (uint4*)pool_u, (uint4*)pool_v, words, w.jobs, w.njobs,
                                                           pass);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_piece_pool(const int32_t* piece_row, const int32_t* exp_begin, int E, const int32_t* tok_of_row,
                             const int32_t* token_to_slot, const void* state, int R, int P, int32_t* piece_wbase,
                             int max_pieces, void* stream) {
  PoolWs w(const_cast<void*>(state), E, R, P);
  k_piece_pool<<<cdiv(max_pieces, 256), 256, 0, (cudaStream_t)stream>>>(piece_row, exp_begin, E, tok_of_row,
                                                                        token_to_slot, w.pool_of, R, piece_wbase,
                                                                        max_pieces);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

// stats[0..3] = loads, replicates, offloads (accumulated since mp_pool_init), err flag
extern "C" int mp_pool_stats(const void* state, int E, int R, int P, int32_t* out4, void* stream) {
  PoolWs w(const_cast<void*>(state), E, R, P);
  MP_CUDA_TRY(cudaMemcpyAsync(out4, w.stats, 3 * sizeof(int32_t), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  MP_CUDA_TRY(cudaMemcpyAsync(out4 + 3, w.err, sizeof(int32_t), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return MP_OK;
}
