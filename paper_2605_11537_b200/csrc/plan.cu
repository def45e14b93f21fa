// K4 (load histogram + capped replica plan) and K6 (placement token walk,
// execution map, replica-segment permutation) -- integer work, bit-exact with
// the reference.
//
// Reference semantics restated in closed form (verified
// against the reference in tests/):
//   cap_replicas  src/planner.py:36-72   water-fill: L* = max level with
//                 sum_e min(d_e, L*) <= C; +1 to the first C - sum experts with
//                 d_e > L* ordered by (d_e desc, e asc).
//   apply_layer   src/placement.py:109-165  slot(t) = off[e] + (rank_e(t) + r_e) mod cnt_e,
//                 r_e = min(res_prev_e, cap_e), cnt_e = min(cap_e, r_e + n_e); rank k < cnt_e - r_e gives
//                 LOAD (r_e = 0, k = 0) or REPLICATE ordinal r_e + k.
//   execution     src/simulator.py:185-203  cnt_e = res_e or 1 corrective LOAD,
//                 slot(t) = off'[e] + rank_e(t) mod cnt_e.
// rank_e(t) is the stable rank of token t among the tokens of expert e; it is
// built deterministically (no atomics decide order): per-128-token chunk
// counts -> per-expert exclusive scan over chunks -> in-chunk rank by a
// shared-memory broadcast compare.

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"


namespace mp {

int num_sms();

// counts per (layer, chunk, expert); grid (nch, L), block kChunk
__global__ void k_chunk_hist(const int32_t* __restrict__ assign, int T, int E, int nch, int32_t* __restrict__ cc) {
  griddep_launch_dependents();
  griddep_wait();
  extern __shared__ int hist[];
  const int l = blockIdx.y, ch = blockIdx.x;
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  const int t = ch * kChunk + threadIdx.x;
  if (t < T) {
    const int e = __ldg(&assign[(size_t)l * T + t]);
    atomicAdd(&hist[e], 1);
  }
  __syncthreads();
  int32_t* out = cc + ((size_t)l * nch + ch) * E;
  for (int e = threadIdx.x; e < E; e += blockDim.x) out[e] = hist[e];
}


// In place: cc[l][ch][e] <- sum_{ch' < ch} cc[l][ch'][e]; demand[l][e] <- total. Grid
// (ceil(E / 32), L), block 32 x 32 = (expert lane, chunk group); each thread scans
// a contiguous run of chunks for one expert (coalesced 128 B rows), group totals are
// scanned in shared memory, then every run adds its group offset.
__global__ void __launch_bounds__(1024) k_chunk_prefix_cols(int32_t* __restrict__ cc, int nch, int E,
                                                            int32_t* __restrict__ demand) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ int part[32][33];
  const int l = blockIdx.y;
  const int el = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + el;
  const int per = cdiv(nch, 32);
  const int ch0 = g * per, ch1 = min(nch, ch0 + per);
  int32_t* base = cc + (size_t)l * nch * E + e;
  int run = 0;
  if (e < E) {
    int ch = ch0;
    for (; ch + 4 <= ch1; ch += 4) {
      const int c0 = base[(size_t)(ch + 0) * E], c1 = base[(size_t)(ch + 1) * E];
      const int c2 = base[(size_t)(ch + 2) * E], c3 = base[(size_t)(ch + 3) * E];
      base[(size_t)(ch + 0) * E] = run;
      base[(size_t)(ch + 1) * E] = run + c0;
      base[(size_t)(ch + 2) * E] = run + c0 + c1;
      base[(size_t)(ch + 3) * E] = run + c0 + c1 + c2;
      run += c0 + c1 + c2 + c3;
    }
    for (; ch < ch1; ++ch) {
      const int c = base[(size_t)ch * E];
      base[(size_t)ch * E] = run;
      run += c;
    }
  }
  part[g][el] = run;
  __syncthreads();
  if (g == 0) {
    int acc = 0;
    for (int h = 0; h < 32; ++h) {
      const int v = part[h][el];
      part[h][el] = acc;
      acc += v;
    }
    if (e < E) demand[(size_t)l * E + e] = acc;
  }
  __syncthreads();
  const int off = part[g][el];
  if (e < E && off)
    for (int ch = ch0; ch < ch1; ++ch) base[(size_t)ch * E] += off;
}

// cap_replicas (src/planner.py:36-72) as a closed-form water-fill. grid L, block 1024.
__global__ void k_cap_replicas(const int32_t* __restrict__ demand, int E, int capacity, int unit,
                               int32_t* __restrict__ caps, int32_t* __restrict__ infeasible) {
  griddep_launch_dependents();
  griddep_wait();
  extern __shared__ int sd[];
  __shared__ int red[40];
  const int l = blockIdx.x;
  const int32_t* dl = demand + (size_t)l * E;
  int32_t* cl = caps + (size_t)l * E;
  int D = 0, tot = 0, mx = 0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int d = dl[e];
    if (unit > 1) d = (d + unit - 1) / unit;
    sd[e] = d;
    D += d > 0;
    tot += d;
    mx = max(mx, d);
  }
  D = block_sum(D, red);
  tot = block_sum(tot, red);
  mx = block_max(mx, red);
  if (threadIdx.x == 0) infeasible[l] = (D > 0 && tot > capacity && D > capacity) ? 1 : 0;
  if (D == 0 || tot <= capacity) {  // nothing to cap: caps == demand
    for (int e = threadIdx.x; e < E; e += blockDim.x) cl[e] = sd[e];
    return;
  }
  if (D > capacity) {  // InfeasibleCapacityError: caller decides (raise / distinct-only fallback)
    for (int e = threadIdx.x; e < E; e += blockDim.x) cl[e] = 0;
    return;
  }
  // largest level with sum_e min(d_e, level) <= capacity; level 1 always fits (D <= C)
  int lo = 1, hi = mx;
  while (hi - lo > 1) {
    const int mid = lo + (hi - lo) / 2;
    int s = 0;
    for (int e = threadIdx.x; e < E; e += blockDim.x) s += min(sd[e], mid);
    s = block_sum(s, red);
    if (s <= capacity) lo = mid; else hi = mid;
  }
  int s = 0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) s += min(sd[e], lo);
  s = block_sum(s, red);
  const int R = capacity - s;  // partial round: first R of {d > lo} by (d desc, e asc)
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int d = sd[e];
    int c = min(d, lo);
    if (d > lo && R > 0) {
      int rank = 0;
      for (int f = 0; f < E; ++f) {
        const int df = sd[f];
        rank += (df > d) || (df == d && f < e);
      }
      c += rank < R;
    }
    cl[e] = c;
  }
}

// apply_layer residency update (src/placement.py:116-141). grid L, block 1024.
// Writes per-layer cap_eff / r_eff / off to ws, offloads, res (new), fallback, num_slots.
__global__ void k_place_layer(const int32_t* __restrict__ demand, int E, const int32_t* __restrict__ caps_in,
                              int plan_capacity, int state_capacity, int32_t* __restrict__ res,
                              int32_t* __restrict__ cap_eff, int32_t* __restrict__ r_eff,
                              int32_t* __restrict__ off_g, int32_t* __restrict__ offloads,
                              int32_t* __restrict__ fallback, int32_t* __restrict__ num_slots) {
  griddep_launch_dependents();
  griddep_wait();
  extern __shared__ int s_cnt[];  // E
  __shared__ int red[40];
  const int l = blockIdx.x;
  const size_t b = (size_t)l * E;
  int bad = 0, sumcap = 0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int n = demand[b + e], c = caps_in[b + e];
    bad += (n > 0 && c < 1);
    sumcap += min(c, state_capacity + 1);  // exact whenever the sum can still fit
  }
  bad = block_sum(bad, red);
  const int sc = block_sum(sumcap, red);
  const bool fb = !(bad == 0 && sc <= state_capacity && plan_capacity <= state_capacity);
  if (threadIdx.x == 0) fallback[l] = fb ? 1 : 0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int n = demand[b + e];
    const int cap = fb ? (n > 0 ? 1 : 0) : caps_in[b + e];
    const int rp = res[b + e];
    int r, off, rn;
    if (n > 0) {
      r = min(rp, cap);
      off = max(rp - cap, 0);  // reclaim above the new cap
      rn = min(cap, r + n);    // replicas are created only as tokens arrive
    } else {
      r = 0;
      off = rp;  // offload every replica of an unmentioned expert
      rn = 0;
    }
    cap_eff[b + e] = rn;
    r_eff[b + e] = r;
    offloads[b + e] = off;
    res[b + e] = rn;
    s_cnt[e] = rn;
  }
  __syncthreads();
  const int total = block_exclusive_scan(s_cnt, E, red);
  for (int e = threadIdx.x; e < E; e += blockDim.x) off_g[(size_t)l * (E + 1) + e] = s_cnt[e];
  if (threadIdx.x == 0) {
    off_g[(size_t)l * (E + 1) + E] = total;
    num_slots[l] = total;
  }
}

// stable rank of token t among same-expert tokens; grid (nch, L), block kChunk
__device__ __forceinline__ int chunk_rank(const int32_t* __restrict__ route, int T, int l, int ch, int* se, int* e_out) {
  const int t = ch * kChunk + threadIdx.x;
  const int e = (t < T) ? __ldg(&route[(size_t)l * T + t]) : -1;
  se[threadIdx.x] = e;
  __syncthreads();
  int r = 0;
  for (int j = 0; j < (int)threadIdx.x; ++j) r += (se[j] == e);
  *e_out = e;
  return r;
}

__global__ void k_place_rank(const int32_t* __restrict__ assign, int T, int E, int nch, const int32_t* __restrict__ cc,
                             const int32_t* __restrict__ cap_eff, const int32_t* __restrict__ r_eff,
                             const int32_t* __restrict__ off_g, int32_t* __restrict__ token_to_slot,
                             int32_t* __restrict__ token_event) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ int se[kChunk];
  const int l = blockIdx.y, ch = blockIdx.x;
  int e;
  const int rin = chunk_rank(assign, T, l, ch, se, &e);
  const int t = ch * kChunk + threadIdx.x;
  if (t >= T) return;
  const size_t b = (size_t)l * E + e;
  const int rank = cc[((size_t)l * nch + ch) * E + e] + rin;
  const int cap = cap_eff[b], r = r_eff[b];
  const int off = off_g[(size_t)l * (E + 1) + e];
  token_to_slot[(size_t)l * T + t] = off + (rank + r) % cap;
  int ev = MP_EVENT_NONE;
  if (rank < cap - r)
    ev = (r == 0 && rank == 0) ? (MP_EVENT_LOAD << MP_EVENT_KIND_SHIFT)
                               : ((MP_EVENT_REPLICATE << MP_EVENT_KIND_SHIFT) | (r + rank));
  token_event[(size_t)l * T + t] = ev;
}

__device__ __forceinline__ int lower_bound_i32(const int32_t* a, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Pad each expert's piece count to even (the CTA-pair GEMM computes pieces 2p, 2p+1
// of one expert per cluster). s_off: exclusive slot offsets (E + 1), s_pc: pieces per slot.
__device__ inline void pad_pieces_even(const int* s_off, int E, int* s_pc) {
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int tot = 0;
    for (int s = s_off[e]; s < s_off[e + 1]; ++s) tot += s_pc[s];
    if (tot & 1) s_pc[s_off[e + 1] - 1] += 1;
  }
  __syncthreads();
}

// Pieces of one slot: M-tiles (split) or the whole slot; extra pieces beyond the
// real ones are empty padding (0 rows, a valid row address).
__device__ inline void emit_pieces(int32_t* pr, int32_t* pn, int p0, int np, int row0, int size, int split) {
  for (int p = 0; p < np; ++p) {
    const int rows = split ? min(kBlockMRows, size - p * kBlockMRows) : (p == 0 ? size : 0);
    pr[p0 + p] = (split && rows > 0) ? row0 + p * kBlockMRows : row0;
    pn[p0 + p] = max(rows, 0);
  }
}

// Execution map per layer (src/simulator.py:185-203) + slot rows + GEMM pieces.
// grid L, block 1024. smem: s_off[E+1] s_n[E] s_row[MS+1] s_pc[MS+1]
// Slot / row / piece layout of one layer into shared memory (sm: s_off[E+1] s_n[E]
// s_row[max_slots+1] s_pc[max_slots+1]); global outputs only when `write`. demand and
// res_in may live in global or shared memory.
__device__ void exec_layer_core(int l, int* sm, int* red, const int32_t* demand, const int32_t* res_in, bool write,
                                int E, int max_slots, int split_m, int32_t* res, int32_t* __restrict__ corrective,
                                int32_t* __restrict__ num_slots, int32_t* __restrict__ off_g,
                                int32_t* __restrict__ slot_row_g, int32_t* __restrict__ piece_row,
                                int32_t* __restrict__ piece_rows, int32_t* __restrict__ exp_begin, int pieces_stride,
                                int32_t* __restrict__ err) {
  int* s_off = sm;              // E + 1
  int* s_n = s_off + E + 1;     // E
  int* s_row = s_n + E;         // max_slots + 1
  int* s_pc = s_row + max_slots + 1;
  const size_t b = (size_t)l * E;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int n = demand[b + e], rp = res_in[b + e];
    const int cnt = rp > 0 ? rp : (n > 0 ? 1 : 0);
    if (write) {
      corrective[b + e] = (rp == 0 && n > 0) ? 1 : 0;
      res[b + e] = cnt;
    }
    s_off[e] = cnt;
    s_n[e] = n;
  }
  __syncthreads();
  const int ns = block_exclusive_scan(s_off, E, red);
  if (threadIdx.x == 0) {
    s_off[E] = ns;
    if (write) num_slots[l] = ns;
  }
  __syncthreads();
  if (ns > max_slots) {
    if (write && threadIdx.x == 0) atomicExch(err, 1);
    return;
  }
  for (int s = threadIdx.x; s < ns; s += blockDim.x) {
    // expert of slot s: largest e with s_off[e] <= s (experts with zero slots are skipped)
    int lo = 0, hi = E;  // invariant s_off[lo] <= s < s_off[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_off[mid] <= s) lo = mid; else hi = mid;
    }
    const int j = s - s_off[lo], c = s_off[lo + 1] - s_off[lo], n = s_n[lo];
    const int size = n > j ? (n - j + c - 1) / c : 0;
    s_row[s] = size;
    s_pc[s] = (split_m & 1) ? cdiv(size, kBlockMRows) : (size > 0 ? 1 : 0);
  }
  __syncthreads();
  if (split_m & 2) pad_pieces_even(s_off, E, s_pc);  // CTA-pair GEMM: even piece count per expert
  block_exclusive_scan(s_row, ns, red);
  const int P = block_exclusive_scan(s_pc, ns, red);
  if (threadIdx.x == 0) {
    s_pc[ns] = P;
  }
  __syncthreads();
  if (!write) return;
  int32_t* pr = piece_row + (size_t)l * pieces_stride;
  int32_t* pn = piece_rows + (size_t)l * pieces_stride;
  for (int s = threadIdx.x; s < ns; s += blockDim.x) slot_row_g[(size_t)l * (max_slots + 1) + s] = s_row[s];
  // sizes again from the scanned rows (total rows = sum of demand)
  int total_rows = 0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) total_rows += s_n[e];
  total_rows = block_sum(total_rows, red);
  for (int s = threadIdx.x; s < ns; s += blockDim.x) {
    const int row0 = s_row[s];
    const int size = (s + 1 < ns ? s_row[s + 1] : total_rows) - row0;
    const int p0 = s_pc[s], np = s_pc[s + 1] - p0;
    emit_pieces(pr, pn, p0, np, row0, size, split_m & 1);
  }
  for (int e = threadIdx.x; e <= E; e += blockDim.x) {
    off_g[(size_t)l * (E + 1) + e] = s_off[e];
    exp_begin[(size_t)l * (E + 1) + e] = s_pc[s_off[e]];
  }
}

__device__ void exec_layer_body(int l, int* sm, int* red, const int32_t* demand, int E, int max_slots, int split_m,
                                int32_t* res, int32_t* __restrict__ corrective, int32_t* __restrict__ num_slots,
                                int32_t* __restrict__ off_g, int32_t* __restrict__ slot_row_g,
                                int32_t* __restrict__ piece_row, int32_t* __restrict__ piece_rows,
                                int32_t* __restrict__ exp_begin, int pieces_stride, int32_t* __restrict__ err) {
  exec_layer_core(l, sm, red, demand, res, true, E, max_slots, split_m, res, corrective, num_slots, off_g, slot_row_g,
                  piece_row, piece_rows, exp_begin, pieces_stride, err);
}

__global__ void k_exec_layer(const int32_t* __restrict__ demand, int E, int max_slots, int split_m,
                             int32_t* __restrict__ res, int32_t* __restrict__ corrective,
                             int32_t* __restrict__ num_slots, int32_t* __restrict__ off_g,
                             int32_t* __restrict__ slot_row_g, int32_t* __restrict__ piece_row,
                             int32_t* __restrict__ piece_rows, int32_t* __restrict__ exp_begin, int pieces_stride,
                             int32_t* __restrict__ err) {
  griddep_launch_dependents();
  griddep_wait();
  extern __shared__ int sm[];
  __shared__ int red[40];
  exec_layer_body(blockIdx.x, sm, red, demand, E, max_slots, split_m, res, corrective, num_slots, off_g, slot_row_g,
                  piece_row, piece_rows, exp_begin, pieces_stride, err);
}


__device__ void exec_rank_body(int l, int ch, int* se, const int32_t* __restrict__ route, int T, int E, int nch,
                               int max_slots, const int32_t* __restrict__ cc, const int32_t* __restrict__ off_g,
                               const int32_t* __restrict__ slot_row_g, int32_t* __restrict__ token_to_slot,
                               int32_t* __restrict__ row_of_token, int32_t* __restrict__ tok_of_row) {
  int e;
  const int rin = chunk_rank(route, T, l, ch, se, &e);
  const int t = ch * kChunk + threadIdx.x;
  if (t >= T) return;
  const int rank = cc[((size_t)l * nch + ch) * E + e] + rin;
  const int32_t* off = off_g + (size_t)l * (E + 1);
  const int o = off[e], c = off[e + 1] - o;
  const int s = o + rank % c;
  const int row = slot_row_g[(size_t)l * (max_slots + 1) + s] + rank / c;
  token_to_slot[(size_t)l * T + t] = s;
  if (row_of_token) row_of_token[(size_t)l * T + t] = row;
  tok_of_row[(size_t)l * T + row] = t;
}

__global__ void k_exec_rank(const int32_t* __restrict__ route, int T, int E, int nch, int max_slots,
                            const int32_t* __restrict__ cc, const int32_t* __restrict__ off_g,
                            const int32_t* __restrict__ slot_row_g, int32_t* __restrict__ token_to_slot,
                            int32_t* __restrict__ row_of_token, int32_t* __restrict__ tok_of_row) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ int se[kChunk];
  exec_rank_body(blockIdx.y, blockIdx.x, se, route, T, E, nch, max_slots, cc, off_g, slot_row_g, token_to_slot,
                 row_of_token, tok_of_row);
}

// k_exec_rank (one layer) fused with the FFN permute: block = one 128-token chunk and 32
// warps; threads < 128 compute their token's stable rank, slot and row (k_exec_rank), then
// all 32 warps copy the chunk's rows x[t] (fp32) -> xperm[row] (bf16, round to nearest:
// the rows of mp_ffn_gather), four rows per warp.
template <int KQ>  // d / 4 float4 per row
__global__ void __launch_bounds__(1024) k_exec_rank_gather(const int32_t* __restrict__ route, int T, int E, int nch,
                                                           int max_slots, const int32_t* __restrict__ cc,
                                                           const int32_t* __restrict__ off_g,
                                                           const int32_t* __restrict__ slot_row_g,
                                                           int32_t* __restrict__ token_to_slot,
                                                           int32_t* __restrict__ row_of_token,
                                                           int32_t* __restrict__ tok_of_row, const float* __restrict__ x,
                                                           __nv_bfloat16* __restrict__ xperm) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ int se[kChunk], srow[kChunk];
  const int ch = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t = ch * kChunk + tid;
  int e = -1;
  if (tid < kChunk) {
    e = t < T ? __ldg(&route[t]) : -1;
    se[tid] = e;
  }
  __syncthreads();
  if (tid < kChunk) {
    int row = -1;
    if (t < T) {
      int r = 0;
      for (int j = 0; j < tid; ++j) r += (se[j] == e);
      const int rank = cc[(size_t)ch * E + e] + r;
      const int o = off_g[e], c = off_g[e + 1] - o;
      const int s = o + rank % c;
      row = slot_row_g[s] + rank / c;
      token_to_slot[t] = s;
      if (row_of_token) row_of_token[t] = row;
      tok_of_row[row] = t;
    }
    srow[tid] = row;
  }
  __syncthreads();
  constexpr int N = (KQ + 31) / 32;
  for (int k = warp; k < kChunk; k += 32) {
    const int row = srow[k];
    if (row < 0) continue;
    const float4* src = reinterpret_cast<const float4*>(x + (size_t)(ch * kChunk + k) * (KQ * 4));
    uint2* dst = reinterpret_cast<uint2*>(xperm + (size_t)row * (KQ * 4));
    float4 v[N];
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (lane + 32 * i < KQ) v[i] = __ldg(&src[lane + 32 * i]);
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (lane + 32 * i < KQ) dst[lane + 32 * i] = make_uint2(pack_bf16x2(v[i].x, v[i].y), pack_bf16x2(v[i].z, v[i].w));
  }
}


// Segments from an explicit token -> slot map. grid 1, block 1024.
// size[s] (from the chunk histogram) -> slot_row (scan) -> pieces (scan).
__global__ void k_seg_layer(const int32_t* __restrict__ size, const int32_t* __restrict__ slot_expert, int S, int E,
                            int split_m, int32_t* __restrict__ slot_row_g, int32_t* __restrict__ piece_row,
                            int32_t* __restrict__ piece_rows, int32_t* __restrict__ exp_begin) {
  griddep_launch_dependents();
  griddep_wait();
  extern __shared__ int sm[];
  __shared__ int red[40];
  int* s_row = sm;          // S + 1
  int* s_pc = s_row + S + 1;  // S + 1
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    const int n = size[s];
    s_row[s] = n;
    s_pc[s] = (split_m & 1) ? cdiv(n, kBlockMRows) : (n > 0 ? 1 : 0);
  }
  __syncthreads();
  if (split_m & 2) {  // even piece count per expert (slots grouped by expert)
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      const int a = lower_bound_i32(slot_expert, S, e), b = lower_bound_i32(slot_expert, S, e + 1);
      int tot = 0;
      for (int s = a; s < b; ++s) tot += s_pc[s];
      if (tot & 1) s_pc[b - 1] += 1;
    }
    __syncthreads();
  }
  const int total = block_exclusive_scan(s_row, S, red);
  const int P = block_exclusive_scan(s_pc, S, red);
  if (threadIdx.x == 0) {
    s_row[S] = total;
    s_pc[S] = P;
  }
  __syncthreads();
  for (int s = threadIdx.x; s < S; s += blockDim.x) {
    slot_row_g[s] = s_row[s];
    const int row0 = s_row[s], n = s_row[s + 1] - row0;
    const int p0 = s_pc[s], np = s_pc[s + 1] - p0;
    emit_pieces(piece_row, piece_rows, p0, np, row0, n, split_m & 1);
  }
  for (int e = threadIdx.x; e <= E; e += blockDim.x) {
    int lo = 0, hi = S;  // first slot with slot_expert >= e
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (slot_expert[mid] < e) lo = mid + 1; else hi = mid;
    }
    exp_begin[e] = s_pc[lo];
  }
}

__global__ void k_seg_rank(const int32_t* __restrict__ key, int T, int S, int nch, const int32_t* __restrict__ cc,
                           const int32_t* __restrict__ slot_row_g, int32_t* __restrict__ tok_of_row) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ int se[kChunk];
  const int ch = blockIdx.x;
  int s;
  const int rin = chunk_rank(key, T, 0, ch, se, &s);
  const int t = ch * kChunk + threadIdx.x;
  if (t >= T) return;
  tok_of_row[slot_row_g[s] + cc[(size_t)ch * S + s] + rin] = t;
}

static inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

static cudaError_t set_smem(const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace mp

using namespace mp;

extern "C" int mp_histogram(const int32_t* assign, int L, int T, int E, int32_t* demand, void* stream) {
  MP_REQUIRE(L >= 1 && T >= 0 && E >= 1, MP_ERR_CONFIG, "mp_histogram: bad sizes L=%d T=%d E=%d", L, T, E);
  cudaStream_t st = (cudaStream_t)stream;
  if (T == 0) {
    MP_CUDA_TRY(cudaMemsetAsync(demand, 0, sizeof(int32_t) * (size_t)L * E, st));
    return MP_OK;
  }
  const int nch = cdiv(T, kChunk);
  int32_t* cc = nullptr;
  // small scratch from the stream-ordered allocator: histogram is a utility entry point
  MP_CUDA_TRY(cudaMallocAsync((void**)&cc, sizeof(int32_t) * (size_t)L * nch * E, st));
  const size_t sm = sizeof(int) * (size_t)E;
  MP_REQUIRE(sm <= 200 * 1024, MP_ERR_CONFIG, "mp_histogram: E=%d too large", E);
  MP_CUDA_TRY(set_smem((const void*)k_chunk_hist, sm));
  MP_CUDA_TRY(launch_pdl(k_chunk_hist, dim3(dim3(nch, L)), dim3(kChunk), sm, st, assign, T, E, nch, cc));
  MP_CUDA_TRY(launch_pdl(k_chunk_prefix_cols, dim3(dim3(cdiv(E, 32), L)), dim3(1024), 0, st, cc, nch, E, demand));
  MP_CUDA_TRY(cudaGetLastError());
  MP_CUDA_TRY(cudaFreeAsync(cc, st));
  return MP_OK;
}

extern "C" size_t mp_histogram_workspace_bytes(int L, int T, int E) {
  return (size_t)L * cdiv(T > 0 ? T : 1, kChunk) * E * sizeof(int32_t);
}

// Same as mp_histogram with a caller-provided workspace (graph-capturable, no allocation).
extern "C" int mp_histogram_ws(const int32_t* assign, int L, int T, int E, int32_t* demand, void* ws, size_t ws_bytes,
                               void* stream) {
  MP_REQUIRE(L >= 1 && T >= 1 && E >= 1, MP_ERR_CONFIG, "mp_histogram_ws: bad sizes L=%d T=%d E=%d", L, T, E);
  MP_REQUIRE(ws_bytes >= mp_histogram_workspace_bytes(L, T, E), MP_ERR_CONFIG, "mp_histogram_ws: workspace");
  cudaStream_t st = (cudaStream_t)stream;
  const int nch = cdiv(T, kChunk);
  const size_t sm = sizeof(int) * (size_t)E;
  MP_REQUIRE(sm <= 200 * 1024, MP_ERR_CONFIG, "mp_histogram_ws: E=%d too large", E);
  MP_CUDA_TRY(set_smem((const void*)k_chunk_hist, sm));
  MP_CUDA_TRY(launch_pdl(k_chunk_hist, dim3(dim3(nch, L)), dim3(kChunk), sm, st, assign, T, E, nch, (int32_t*)ws));
  MP_CUDA_TRY(launch_pdl(k_chunk_prefix_cols, dim3(dim3(cdiv(E, 32), L)), dim3(1024), 0, st, (int32_t*)ws, nch, E, demand));
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_cap_replicas(const int32_t* demand, int L, int E, int capacity, int unit_rows, int32_t* caps,
                               int32_t* infeasible, void* stream) {
  MP_REQUIRE(capacity >= 1, MP_ERR_CONFIG, "capacity must be >= 1, got %d", capacity);
  MP_REQUIRE(L >= 1 && E >= 1 && unit_rows >= 1, MP_ERR_CONFIG, "mp_cap_replicas: bad sizes");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t sm = sizeof(int) * (size_t)E;
  MP_REQUIRE(sm <= 200 * 1024, MP_ERR_CONFIG, "mp_cap_replicas: E=%d too large", E);
  MP_CUDA_TRY(set_smem((const void*)k_cap_replicas, sm));
  MP_CUDA_TRY(launch_pdl(k_cap_replicas, dim3(L), dim3(1024), sm, st, demand, E, capacity, unit_rows, caps, infeasible));
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" size_t mp_place_workspace_bytes(int L, int T, int E) {
  const int nch = cdiv(T > 0 ? T : 1, kChunk);
  return align_up(sizeof(int32_t) * (size_t)L * nch * E) + align_up(sizeof(int32_t) * (size_t)L * E) * 3 +
         align_up(sizeof(int32_t) * (size_t)L * (E + 1));
}

extern "C" int mp_place(const int32_t* assign, int L, int T, int E, const int32_t* caps, int plan_capacity,
                        int state_capacity, int32_t* res, int32_t* token_to_slot, int32_t* token_event,
                        int32_t* offloads, int32_t* fallback, int32_t* num_slots, void* ws, size_t ws_bytes,
                        void* stream) {
  MP_REQUIRE(L >= 1 && T >= 0 && E >= 1, MP_ERR_CONFIG, "mp_place: bad sizes L=%d T=%d E=%d", L, T, E);
  MP_REQUIRE(ws_bytes >= mp_place_workspace_bytes(L, T, E), MP_ERR_CONFIG, "mp_place: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int nch = cdiv(T > 0 ? T : 1, kChunk);
  char* p = (char*)ws;
  int32_t* cc = (int32_t*)p;
  p += align_up(sizeof(int32_t) * (size_t)L * nch * E);
  int32_t* dem = (int32_t*)p;
  p += align_up(sizeof(int32_t) * (size_t)L * E);
  int32_t* cap_eff = (int32_t*)p;
  p += align_up(sizeof(int32_t) * (size_t)L * E);
  int32_t* r_eff = (int32_t*)p;
  p += align_up(sizeof(int32_t) * (size_t)L * E);
  int32_t* off_g = (int32_t*)p;
  const size_t sm = sizeof(int) * (size_t)E;
  MP_REQUIRE(sm <= 200 * 1024, MP_ERR_CONFIG, "mp_place: E=%d too large", E);
  MP_CUDA_TRY(set_smem((const void*)k_chunk_hist, sm));
  MP_CUDA_TRY(set_smem((const void*)k_place_layer, sm));
  if (T > 0) {
    MP_CUDA_TRY(launch_pdl(k_chunk_hist, dim3(dim3(nch, L)), dim3(kChunk), sm, st, assign, T, E, nch, cc));
  } else {
    MP_CUDA_TRY(cudaMemsetAsync(cc, 0, sizeof(int32_t) * (size_t)L * nch * E, st));
  }
  MP_CUDA_TRY(launch_pdl(k_chunk_prefix_cols, dim3(dim3(cdiv(E, 32), L)), dim3(1024), 0, st, cc, nch, E, dem));
  MP_CUDA_TRY(launch_pdl(k_place_layer, dim3(L), dim3(1024), sm, st, dem, E, caps, plan_capacity, state_capacity, res, cap_eff, r_eff, off_g,
                                     offloads, fallback, num_slots));
  if (T > 0)
    MP_CUDA_TRY(launch_pdl(k_place_rank, dim3(dim3(nch, L)), dim3(kChunk), 0, st, assign, T, E, nch, cc, cap_eff, r_eff, off_g, token_to_slot,
                                                  token_event));
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" size_t mp_exec_workspace_bytes(int L, int T, int E, int max_slots) {
  const int nch = cdiv(T > 0 ? T : 1, kChunk);
  return align_up(sizeof(int32_t) * (size_t)L * nch * E) + align_up(sizeof(int32_t) * (size_t)L * E) +
         align_up(sizeof(int32_t) * (size_t)L * (E + 1)) + align_up(sizeof(int32_t) * (size_t)L * (max_slots + 1)) +
         align_up(sizeof(int32_t) * 4);
}

extern "C" int mp_exec_map(const int32_t* route, int L, int T, int E, int max_slots, int split_m, int32_t* res,
                           int32_t* token_to_slot, int32_t* corrective, int32_t* num_slots, int32_t* row_of_token,
                           int32_t* tok_of_row, int32_t* piece_row, int32_t* piece_rows, int32_t* exp_begin,
                           void* ws, size_t ws_bytes, void* stream) {
  MP_REQUIRE(L >= 1 && T >= 1 && E >= 1 && max_slots >= 1, MP_ERR_CONFIG, "mp_exec_map: bad sizes L=%d T=%d E=%d",
             L, T, E);
  MP_REQUIRE(ws_bytes >= mp_exec_workspace_bytes(L, T, E, max_slots), MP_ERR_CONFIG,
             "mp_exec_map: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int nch = cdiv(T, kChunk);
  char* p = (char*)ws;
  int32_t* cc = (int32_t*)p;
  p += align_up(sizeof(int32_t) * (size_t)L * nch * E);
  int32_t* dem = (int32_t*)p;
  p += align_up(sizeof(int32_t) * (size_t)L * E);
  int32_t* off_g = (int32_t*)p;
  p += align_up(sizeof(int32_t) * (size_t)L * (E + 1));
  int32_t* slot_row = (int32_t*)p;
  p += align_up(sizeof(int32_t) * (size_t)L * (max_slots + 1));
  int32_t* err = (int32_t*)p;
  const size_t sm_h = sizeof(int) * (size_t)E;
  const size_t sm_x = sizeof(int) * ((size_t)2 * E + 1 + 2 * ((size_t)max_slots + 1));
  MP_REQUIRE(sm_h <= 200 * 1024 && sm_x <= 200 * 1024, MP_ERR_CONFIG, "mp_exec_map: E/max_slots too large");
  const int pieces_stride = max_slots + cdiv(T, kChunk);
  MP_CUDA_TRY(set_smem((const void*)k_chunk_hist, sm_h));
  MP_CUDA_TRY(set_smem((const void*)k_exec_layer, sm_x));
  MP_CUDA_TRY(launch_pdl(k_chunk_hist, dim3(dim3(nch, L)), dim3(kChunk), sm_h, st, route, T, E, nch, cc));
  MP_CUDA_TRY(launch_pdl(k_chunk_prefix_cols, dim3(dim3(cdiv(E, 32), L)), dim3(1024), 0, st, cc, nch, E, dem));
  MP_CUDA_TRY(launch_pdl(k_exec_layer, dim3(L), dim3(1024), sm_x, st, dem, E, max_slots, split_m, res, corrective, num_slots, off_g, slot_row,
                                      piece_row, piece_rows, exp_begin, pieces_stride, err));
  MP_CUDA_TRY(launch_pdl(k_exec_rank, dim3(dim3(nch, L)), dim3(kChunk), 0, st, route, T, E, nch, max_slots, cc, off_g, slot_row, token_to_slot,
                                               row_of_token, tok_of_row));
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}


// mp_exec_map (one layer) after mp_route_top1_hist wrote the chunk histograms into the
// first cdiv(T, 128) x E ints of ws: chunk prefixes, slot/row/piece layout, ranks (+ the FFN
// permute into xperm when given, ldx == d in {768, 1024}).
extern "C" int mp_exec_map_hist(const int32_t* route, int T, int E, int max_slots, int split_m, int32_t* res,
                                int32_t* token_to_slot, int32_t* corrective, int32_t* num_slots, int32_t* row_of_token,
                                int32_t* tok_of_row, int32_t* piece_row, int32_t* piece_rows, int32_t* exp_begin,
                                const float* x, int d, void* xperm, void* ws, size_t ws_bytes, void* stream) {
  MP_REQUIRE(T >= 1 && E >= 1 && max_slots >= 1 && d >= 1, MP_ERR_CONFIG, "mp_exec_map_hist: bad sizes T=%d E=%d", T,
             E);
  MP_REQUIRE(ws_bytes >= mp_exec_workspace_bytes(1, T, E, max_slots), MP_ERR_CONFIG,
             "mp_exec_map_hist: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int nch = cdiv(T, kChunk);
  char* p = (char*)ws;
  int32_t* cc = (int32_t*)p;
  p += align_up(sizeof(int32_t) * (size_t)nch * E);
  int32_t* dem = (int32_t*)p;
  p += align_up(sizeof(int32_t) * (size_t)E);
  int32_t* off_g = (int32_t*)p;
  p += align_up(sizeof(int32_t) * (size_t)(E + 1));
  int32_t* slot_row = (int32_t*)p;
  p += align_up(sizeof(int32_t) * (size_t)(max_slots + 1));
  int32_t* err = (int32_t*)p;
  const size_t sm_x = sizeof(int) * ((size_t)2 * E + 1 + 2 * ((size_t)max_slots + 1));
  MP_REQUIRE(sm_x <= 200 * 1024, MP_ERR_CONFIG, "mp_exec_map_hist: E/max_slots too large");
  const int pieces_stride = max_slots + nch;
  MP_CUDA_TRY(set_smem((const void*)k_exec_layer, sm_x));
  MP_CUDA_TRY(launch_pdl(k_chunk_prefix_cols, dim3(dim3(cdiv(E, 32), 1)), dim3(1024), 0, st, cc, nch, E, dem));
  MP_CUDA_TRY(launch_pdl(k_exec_layer, dim3(1), dim3(1024), sm_x, st, dem, E, max_slots, split_m, res, corrective,
                         num_slots, off_g, slot_row, piece_row, piece_rows, exp_begin, pieces_stride, err));
  if (xperm != nullptr) {
    MP_REQUIRE(d == 768 || d == 1024, MP_ERR_CONFIG, "mp_exec_map_hist: the fused permute needs d in {768, 1024}");
    auto kern = d == 768 ? k_exec_rank_gather<192> : k_exec_rank_gather<256>;
    MP_CUDA_TRY(launch_pdl(kern, dim3(nch), dim3(1024), 0, st, route, T, E, nch, max_slots, cc, off_g, slot_row,
                           token_to_slot, row_of_token, tok_of_row, x, (__nv_bfloat16*)xperm));
  } else {
    MP_CUDA_TRY(launch_pdl(k_exec_rank, dim3(dim3(nch, 1)), dim3(kChunk), 0, st, route, T, E, nch, max_slots, cc,
                           off_g, slot_row, token_to_slot, row_of_token, tok_of_row));
  }
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" size_t mp_segments_workspace_bytes(int T, int S) {
  const int nch = cdiv(T > 0 ? T : 1, kChunk);
  return align_up(sizeof(int32_t) * (size_t)nch * S) + 2 * align_up(sizeof(int32_t) * ((size_t)S + 1));
}

extern "C" int mp_segments_from_slots(const int32_t* token_to_slot, const int32_t* slot_expert, int T, int S, int E,
                                      int split_m, int32_t* tok_of_row, int32_t* piece_row, int32_t* piece_rows,
                                      int32_t* exp_begin, void* ws, size_t ws_bytes, void* stream) {
  MP_REQUIRE(T >= 1 && S >= 1 && E >= 1, MP_ERR_CONFIG, "mp_segments_from_slots: bad sizes T=%d S=%d E=%d", T, S, E);
  MP_REQUIRE(ws_bytes >= mp_segments_workspace_bytes(T, S), MP_ERR_CONFIG, "mp_segments_from_slots: workspace");
  cudaStream_t st = (cudaStream_t)stream;
  const int nch = cdiv(T, kChunk);
  char* p = (char*)ws;
  int32_t* cc = (int32_t*)p;
  p += align_up(sizeof(int32_t) * (size_t)nch * S);
  int32_t* size = (int32_t*)p;
  p += align_up(sizeof(int32_t) * ((size_t)S + 1));
  int32_t* slot_row = (int32_t*)p;
  const size_t sm_h = sizeof(int) * (size_t)S, sm_s = sizeof(int) * 2 * ((size_t)S + 1);
  MP_REQUIRE(sm_h <= 200 * 1024 && sm_s <= 200 * 1024, MP_ERR_CONFIG, "mp_segments_from_slots: S too large");
  MP_CUDA_TRY(set_smem((const void*)k_chunk_hist, sm_h));
  MP_CUDA_TRY(set_smem((const void*)k_seg_layer, sm_s));
  MP_CUDA_TRY(launch_pdl(k_chunk_hist, dim3(dim3(nch, 1)), dim3(kChunk), sm_h, st, token_to_slot, T, S, nch, cc));
  MP_CUDA_TRY(launch_pdl(k_chunk_prefix_cols, dim3(dim3(cdiv(S, 32), 1)), dim3(1024), 0, st, cc, nch, S, size));
  k_seg_layer<<<1, 1024, sm_s, st>>>(size, slot_expert, S, E, split_m, slot_row, piece_row, piece_rows, exp_begin);
  k_seg_rank<<<nch, kChunk, 0, st>>>(token_to_slot, T, S, nch, cc, slot_row, tok_of_row);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}
