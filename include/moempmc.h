/*
 * moempmc.h -- C ABI of the B200 (sm_100a) MoE-MPMC inference hot path.
 *
 * The reference (arXiv 2605.11537, package `moesim`, pure Python/numpy) has no
 * FFI: its boundary is the Python module API. Each entry point below replaces
 * the reference function cited next to it; the Python host layer
 * (paper_2605_11537_b200/*.py) keeps the reference signatures and calls these
 * through ctypes. INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Every pointer is a DEVICE pointer unless stated otherwise; buffers are
 *    caller-owned; `ws` is a caller-provided device workspace.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream). Calls are
 *    asynchronous on that stream and never synchronise the device.
 *  - int32 indices; bf16 = IEEE bfloat16 stored as uint16; row-major arrays.
 *  - Return value: MP_OK or an error code mapped 1:1 onto the reference
 *    exception classes (src/errors.py); mp_last_error() returns the message.
 */
#ifndef MOEMPMC_H
#define MOEMPMC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define MP_API __attribute__((visibility("default")))
#else
#define MP_API
#endif

#define MP_ABI_VERSION 1

#define MP_OK 0
#define MP_ERR_CONFIG 1     /* ConfigurationError       src/errors.py:8-9   */
#define MP_ERR_NUMERIC 2    /* NumericError             src/errors.py:26-27 */
#define MP_ERR_PLACEMENT 3  /* PlacementError           src/errors.py:30-31 */
#define MP_ERR_INFEASIBLE 4 /* InfeasibleCapacityError  src/errors.py:34-41 */
#define MP_ERR_CUDA 5       /* CUDA runtime failure (no reference analogue)  */

/* token_event encoding (src/placement.py:22-24 LOAD / REPLICATE) */
#define MP_EVENT_NONE (-1)
#define MP_EVENT_KIND_SHIFT 24
#define MP_EVENT_LOAD 1
#define MP_EVENT_REPLICATE 2

MP_API int mp_abi_version(void);
MP_API const char* mp_last_error(void);
MP_API int mp_device_info(int* sm_count, int* cc_major, int* cc_minor); /* host out-params */

/* ------------------------------------------------------------------ K4
 * Load histogram. demand[l*E+e] = #{t : assign[l*T+t] == e}.
 * Replaces HashTable._histograms (src/predictor.py:122-127) and
 * demand_counts (src/planner.py:27-33). assign values must lie in [0,E).
 */
MP_API int mp_histogram(const int32_t* assign, int L, int T, int E, int32_t* demand, void* stream);
/* Allocation-free form (CUDA-graph capturable). */
MP_API size_t mp_histogram_workspace_bytes(int L, int T, int E);
MP_API int mp_histogram_ws(const int32_t* assign, int L, int T, int E, int32_t* demand, void* ws, size_t ws_bytes,
                           void* stream);

/* Capped replica plan per layer, bit-exact with cap_replicas
 * (src/planner.py:36-72) via its closed-form water-fill; plan_all_layers
 * (src/planner.py:75-85) is the L>1 case. Demand may be expressed in tokens
 * (unit_rows = 1, reference semantics) or in M-tiles (unit_rows = 128:
 * ceil(n/128) per expert). caps[l*E+e] = 0 for undemanded experts.
 * infeasible[l] = 1 when #distinct > capacity (caps row left 0). */
MP_API int mp_cap_replicas(const int32_t* demand, int L, int E, int capacity, int unit_rows, int32_t* caps,
                    int32_t* infeasible, void* stream);

/* ------------------------------------------------------------------ K4+K6
 * Residency update + token walk of apply_layer (src/placement.py:109-165),
 * folded over L layers like apply_batch (src/placement.py:168-180).
 *   caps[l*E+e]       planned replica caps (0 = not in plan)          (in)
 *   res[l*E+e]        resident replica count per expert            (in/out)
 *   token_to_slot     index into the sorted (expert, ordinal) slot list (out)
 *   token_event       MP_EVENT_NONE or kind<<24 | ordinal per token    (out)
 *   offloads[l*E+e]   OFFLOAD pops for expert e (reclaim or full offload)(out)
 *   fallback[l]       1 when the layer fell back to distinct-only      (out)
 *   num_slots[l]      resident slots after placement                   (out)
 */
MP_API size_t mp_place_workspace_bytes(int L, int T, int E);
MP_API int mp_place(const int32_t* assign, int L, int T, int E, const int32_t* caps, int plan_capacity, int state_capacity,
             int32_t* res, int32_t* token_to_slot, int32_t* token_event, int32_t* offloads, int32_t* fallback,
             int32_t* num_slots, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------ K6
 * Execution map of BatchRunner._run_predicted (src/simulator.py:185-203):
 * tokens run on their TRUE expert, round-robin over the resident replicas;
 * an expert with no resident replica gets one corrective LOAD (persisted in
 * res). Also emits the replica-segment permutation consumed by the grouped
 * GEMM: rows are grouped by slot (expert-major, replica-minor), a slot's rows
 * in token order; pieces are the GEMM work units (one per slot, or per 128-row
 * M-tile of a slot when split_m bit 0 is set). split_m bit 1: pad every expert to an
 * even piece count (empty pieces have 0 rows) for the CTA-pair grouped GEMM.
 *   max_slots  >= max over layers of resident slots + corrective loads
 *   per layer l (strides): token_to_slot/row_of_token/tok_of_row: T;
 *   piece_row/piece_rows: max_slots + ceil(T/128); exp_begin: E + 1.
 */
MP_API size_t mp_exec_workspace_bytes(int L, int T, int E, int max_slots);
MP_API int mp_exec_map(const int32_t* route, int L, int T, int E, int max_slots, int split_m, int32_t* res,
                int32_t* token_to_slot, int32_t* corrective, int32_t* num_slots, int32_t* row_of_token,
                int32_t* tok_of_row, int32_t* piece_row, int32_t* piece_rows, int32_t* exp_begin, void* ws,
                size_t ws_bytes, void* stream);
/* mp_exec_map for one layer whose chunk histograms mp_route_top1_hist already wrote into the
 * first cdiv(T, 128) x E ints of ws (pass that region as its chunk_hist): chunk prefixes,
 * layout, ranks -- and with xperm (d in {768, 1024}) the permuted bf16 rows of
 * mp_ffn_gather. */
MP_API int mp_exec_map_hist(const int32_t* route, int T, int E, int max_slots, int split_m, int32_t* res,
                            int32_t* token_to_slot, int32_t* corrective, int32_t* num_slots, int32_t* row_of_token,
                            int32_t* tok_of_row, int32_t* piece_row, int32_t* piece_rows, int32_t* exp_begin,
                            const float* x, int d, void* xperm, void* ws, size_t ws_bytes, void* stream);

/* Per-layer cost-model inputs of one batch (src/simulator.py:210-235 over simulate_layer
 * :62-81 and the TransferLog, src/placement.py:35-63), counted on the device. One block per
 * layer; for layer l, counts[l*5 + {0..4}] = {LOAD events (token_event kind LOAD +
 * sum_e corrective[l,e]), REPLICATE events, OFFLOAD events (sum_e offloads[l,e]), longest
 * slot queue (max_s #{t : token_to_slot[l,t] == s}), num_slots[l]}. token_event (L x T,
 * mp_place), offloads (L x E_off, mp_place) and corrective (L x E_corr, mp_exec_map) may be
 * NULL (counted as 0). *err |= 1 when a token maps outside [0, num_slots[l]).
 * max_slots <= 49152. */
MP_API int mp_layer_counts(const int32_t* token_event, const int32_t* offloads, const int32_t* corrective,
                           const int32_t* token_to_slot, const int32_t* num_slots, int L, int T, int E_off,
                           int E_corr, int max_slots, int32_t* counts, int32_t* err, void* stream);

/* Replica segments from an explicit token -> slot map (a reference Placement,
 * src/router_oracle.py:64-74, as consumed by moe_forward :160-175): rows are
 * grouped by slot (stable in token order); slot_expert[s] must be
 * non-decreasing (slots sorted by (expert, ordinal)). Outputs as mp_exec_map
 * for one layer; piece arrays hold S + ceil(T/128) entries, exp_begin E + 1. */
MP_API size_t mp_segments_workspace_bytes(int T, int S);
MP_API int mp_segments_from_slots(const int32_t* token_to_slot, const int32_t* slot_expert, int T, int S, int E,
                                  int split_m, int32_t* tok_of_row, int32_t* piece_row, int32_t* piece_rows,
                                  int32_t* exp_begin, void* ws, size_t ws_bytes, void* stream);

/* SM partition for the two-stream schedule of the paper's pipeline (reference
 * src/pipeline.py:70-139: the hash-table builder for batch i+1 runs while batch i is
 * forwarded): persistent grids of the grouped expert GEMMs and of the predictor GEMMs
 * (SRU projection, heads). 0 = all SMs (default). Host-side setting, applies to launches
 * issued (or captured) after the call. */
MP_API int mp_set_sm_partition(int ffn_sms, int predictor_sms);

/* ------------------------------------------------------------------ K1 / generic
 * C[M x ldc] = epi(A[M x K] * B[N x K]^T) on tcgen05 (bf16 in, fp32 acc).
 * K % 64 == 0, N % 64 == 0 (pad with zero rows), 16-byte aligned rows.
 * c_dtype: 0 = bf16, 1 = fp32.  act: 0 none, 1 relu, 2 sigmoid(v+bias[n])
 * for n >= sig_from (columns below sig_from get +bias only when bias != NULL).
 */
MP_API int mp_gemm_bf16(const void* A, const void* B, void* C, int M, int N, int K, int c_dtype, int ldc,
                 const float* bias, int act, int sig_from, void* stream);

/* ------------------------------------------------------------------ K1+K2
 * One SRU layer over a token sequence (src/predictor.py:157-195):
 *   [u | f | r] = x W_cat^T (+ b), f,r = sigmoid   (tcgen05 GEMM, fused epilogue)
 *   c_t = f c_{t-1} + (1-f) u ;  h_t = r tanh(c_t) + (1-r) x_t   (chunked scan)
 * x_bf16/x_f32: T x d (d % 64 == 0), w_cat: 3d x d bf16, b_cat: 3d fp32
 * (zeros for the u block). Outputs h_f32 and h_bf16 (T x d).
 * ws >= mp_sru_workspace_bytes(T, d).
 */
MP_API size_t mp_sru_workspace_bytes(int T, int d);
MP_API int mp_sru_layer(const void* x_bf16, const float* x_f32, const void* w_cat, const float* b_cat, int T, int d,
                        const float* c0, float* h_f32, void* h_bf16, float* c_last, int32_t* nonfinite, void* ws,
                        size_t ws_bytes, void* stream);
/* The same layer in two parts, for callers that pipeline token ranges over streams
 * (the scan of rows [0, T/2) overlapping the projection of rows [T/2, T), carried by
 * c_last -> c0): mp_sru_project writes [u | f | r] into ws, mp_sru_scan runs the
 * recurrence + highway from it. Same ws for both; results equal mp_sru_layer. */
MP_API int mp_sru_project(const void* x_bf16, const void* w_cat, const float* b_cat, int T, int d, void* ws,
                          size_t ws_bytes, void* stream);
MP_API int mp_sru_scan(const float* x_f32, int T, int d, const float* c0, float* h_f32, void* h_bf16, float* c_last,
                       int32_t* nonfinite, void* ws, size_t ws_bytes, void* stream);
/* Token-sharded SRU (one sequence split over G ranks): each rank runs
 * mp_sru_project on its rows, mp_sru_scan_total (chunk maps + carries from 0; tot =
 * [A (d) | B (d)], the shard's whole-range affine map c_end = A c_start + B), all-gathers
 * tot (2d fp32 per rank), folds the lower ranks' maps with mp_sru_fold_carry
 * (tots: G x 2d, c0 = the sequence's initial state or NULL) and finishes with
 * mp_sru_scan_finish from that carry. Equals the unsharded layer up to fp32
 * re-association of the carry. */
MP_API int mp_sru_scan_total(int T, int d, float* tot, void* ws, size_t ws_bytes, void* stream);
MP_API int mp_sru_fold_carry(const float* tots, int rank, int d, const float* c0, float* carry_in, void* stream);
MP_API int mp_sru_scan_finish(const float* x_f32, int T, int d, const float* c0, float* h_f32, void* h_bf16,
                              float* c_last, int32_t* nonfinite, void* ws, size_t ws_bytes, void* stream);
/* c0 (d floats, NULL = zeros, src/predictor.py:190) is the cell state entering token 0 --
 * sru_cell's c_prev, or the carry of a preceding token shard; c_last (nullable) receives the
 * cell state after the last token. nonfinite (1 int) is OR-ed with 1 on NaN/inf state
 * (reference raises NumericError, src/predictor.py:170-171). */

/* sparsemax of n rows of E float64 logits (src/predictor.py:198-209), E <= 256. */
MP_API int mp_sparsemax_rows(const double* z, int n, int E, double* out, void* stream);

/* ------------------------------------------------------------------ K3
 * Predicted expert per (layer, token) = argmax_e h_t . heads[l,e]
 * (= argmax(sparsemax(.)), src/predictor.py:212-223). heads: ceil64(L*Eg) x d bf16 (zero rows pad),
 * layer l in rows [l*Eg, l*Eg+E), Eg = E rounded up to a power of two >= 32.
 */
MP_API int mp_heads_argmax(const void* h_bf16, const void* heads, int T, int d, int L, int E, int Eg, int32_t* assign,
                    void* stream);

/* ------------------------------------------------------------------ K5
 * True top-1 routing route_top1 (src/router_oracle.py:90-98) for a token
 * stream: fp64-faithful argmax of W_r x. The tensor-core pass uses split-bf16
 * (x_hi.w_hi + x_hi.w_lo + x_lo.w_hi, fp32 acc); tokens whose top-2 gap is
 * inside the error bound are re-decided in fp64 from the fp32 inputs.
 *   x: T x ldx fp32 (d valid columns); w_hl: Eg x 2d bf16 [w_hi | w_lo];
 *   w_f32: E x d fp32. ws >= mp_router_workspace_bytes(T, d).
 */
MP_API size_t mp_router_workspace_bytes(int T, int d);
MP_API int mp_route_top1(const float* x, int ldx, int T, int d, const void* w_hl, const float* w_f32, int E, int Eg,
                         float w_norm_max, int32_t* route, void* ws, size_t ws_bytes, void* stream);
/* Same with a precomputed per-column bound w_abs[k] = max_e |w_ek| (mp_router_weight_absmax),
 * the form the device-resident engine uses (weights are static). */
MP_API int mp_router_weight_absmax(const float* w_f32, int E, int d, float* w_abs, void* stream);
MP_API int mp_route_top1_ex(const float* x, int ldx, int T, int d, const void* w_hl, const float* w_f32,
                            const float* w_abs, int E, int Eg, int32_t* route, void* ws, size_t ws_bytes,
                            void* stream);
/* Exact routing (near ties re-decided in float64 inside the router, the arithmetic of the
 * recheck kernel) plus every 128-token tile's expert histogram in chunk_hist[tile][e]
 * (cdiv(T, 128) x E ints): the first stage of the execution map, for mp_exec_map_hist.
 * Eg in {64, 128}, ldx % 4 == 0, 16-byte aligned x. */
MP_API int mp_route_top1_hist(const float* x, int ldx, int T, int d, const void* w_hl, const float* w_f32,
                              const float* w_abs, int E, int Eg, int32_t* route, int32_t* chunk_hist, void* ws,
                              size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------ predictor training
 * SRU training on the GPU (reference src/predictor.py:238-379), float64 like the
 * reference. Layouts: (S sequences, T tokens, d) row-major.
 *   mp_sru_train_fwd   f = sigma(fpre + b_f), r = sigma(rpre + b_r), c_t = f c_{t-1} + (1 - f) u,
 *                      g = tanh(c), h = r g + (1 - r) x (caches f, r, c, g)
 *   mp_sru_train_bwd   reverse-time BPTT of one layer: du, dfp (d f_pre), drp (d r_pre),
 *                      dh_out = dh (1 - r), per-sequence bias-gradient sums (S x d)
 *   mp_train_ce        softmax cross-entropy of one MoE layer's head logits (S*T x E):
 *                      row losses and dlogits = (p - onehot) / S; labels (S, L, T) int64
 *   mp_train_colsum / mp_train_sum  deterministic reductions; mp_train_axpy y += alpha x;
 *   mp_train_nonfinite flag |= any non-finite. The dense products are host-issued GEMMs. */
MP_API int mp_sru_train_fwd(const double* u, const double* fpre, const double* rpre, const double* b_f,
                            const double* b_r, const double* x, int S, int T, int d, double* f, double* r, double* c,
                            double* g, double* h, void* stream);
MP_API int mp_sru_train_bwd(const double* dh, const double* x, const double* u, const double* f, const double* r,
                            const double* c, const double* g, int S, int T, int d, double* du, double* dfp,
                            double* drp, double* dh_out, double* bsum_f, double* bsum_r, void* stream);
MP_API int mp_train_colsum(const double* in, int R, int n, double* out, void* stream);
MP_API int mp_train_ce(const double* logits, const int64_t* labels, int S, int T, int L, int layer, int E,
                       double* dlogits, double* row_loss, void* stream);
MP_API int mp_train_sum(const double* in, int n, double* out, void* stream);
MP_API int mp_train_axpy(double* y, const double* x, size_t n, double alpha, void* stream);
/* Float64 GEMM of the trainer's dense products (the reference's numpy float64 matmuls,
 * src/predictor.py:238-334): C[MxN] = op(A) op(B) + beta C, row-major with leading dimensions
 * lda / ldb / ldc; op(A) = A (ta = 0, M x K) or A^T (ta = 1, A stored K x M); op(B) = B
 * (tb = 0, K x N) or B^T (tb = 1, B stored N x K). */
MP_API int mp_dgemm(int ta, int tb, int M, int N, int K, const double* A, int lda, const double* B, int ldb,
                    double beta, double* C, int ldc, void* stream);
MP_API int mp_train_nonfinite(const double* x, size_t n, int32_t* flag, void* stream);

/* ------------------------------------------------------------------ K6 gather + K7 + K8
 * One MoE layer's expert FFNs over replica segments, fused with the ungated
 * residual combine (src/router_oracle.py:101-111, 127-134):
 *   xperm[row]   = bf16(x[tok_of_row[row]])                       (gather)
 *   hid[row]     = relu(xperm[row] . U_e^T)                        (GEMM1)
 *   y[tok][:]   += hid[row] . V_e^T                                (GEMM2, scatter epilogue)
 * u: (E*Fp) x dp bf16, v: (E*dp) x Fp bf16 (zero padded, dp%64==0, Fp%256==0),
 * x, y: T x dp fp32; y == x gives the in-place residual stream update,
 * y = zeros gives expert_forward alone. Pieces from mp_exec_map /
 * mp_segments_from_slots (one layer). ws >= mp_ffn_workspace_bytes(T, dp, Fp).
 */
MP_API size_t mp_ffn_workspace_bytes(int T, int dp, int Fp);
MP_API int mp_moe_ffn(const float* x, float* y, int T, int dp, int Fp, int E, const void* u, const void* v,
                      const int32_t* tok_of_row, const int32_t* piece_row, const int32_t* piece_rows,
                      const int32_t* exp_begin, void* ws, size_t ws_bytes, void* stream);
/* The same layer as three launches (gather | GEMM1 | GEMM2) sharing `ws`, for callers that
 * time or overlap the grouped GEMMs separately. flags bit 0: u / v are in the pre-tiled
 * layout of mp_tile_kmajor (BN mp_ffn_up_bn(Fp) for u; mp_ffn_down_bn(dp) for v, or 256 with
 * bit 1 or bit 6); bit 1: CTA-pair (tcgen05 cta_group::2, M = 256) kernels over piece pairs --
 * pieces must come from a builder called with split_m bit 1 (even piece count per expert),
 * dp % 256 == 0; bit 5 (mp_ffn_down): store y[tok_of_row[row]] = result instead of adding it
 * (every target row has exactly one writer; the expert-parallel receive buffer then needs
 * no zeroing); bit 6 (mp_ffn_down, single-CTA kernel): v is tiled with 256-column slices
 * (the CTA-pair layout), so the same weights serve both kernels. Every mode gives bitwise
 * identical results.
 */
MP_API int mp_ffn_gather(const float* x, int T, int dp, int Fp, int E, const int32_t* tok_of_row, void* ws,
                         size_t ws_bytes, void* stream);
MP_API int mp_ffn_up(int T, int dp, int Fp, int E, const void* u, int flags, const int32_t* piece_row,
                     const int32_t* piece_rows, const int32_t* exp_begin, void* ws, size_t ws_bytes, void* stream);
MP_API int mp_ffn_down(float* y, int T, int dp, int Fp, int E, const void* v, int flags, const int32_t* tok_of_row,
                       const int32_t* piece_row, const int32_t* piece_rows, const int32_t* exp_begin, void* ws,
                       size_t ws_bytes, void* stream);
MP_API int mp_ffn_down_bn(int dp);
/* column-tile width (and mp_tile_kmajor BN) of the pre-tiled expert U weights for GEMM1 */
MP_API int mp_ffn_up_bn(int Fp);
/* K9 physical replicas (north_star; src/placement.py:143-160 LOAD / REPLICATE / OFFLOAD, PAPER.md
 * :172-178). A layer's pool of P expert-sized weight slots (pre-tiled U and V of one expert each)
 * materialises the residency state res[e] (replicas per expert, after placement and the
 * execution map): state = mp_pool_state_bytes(E, R, P) device bytes, R = max replicas of one
 * expert, set up by mp_pool_init. mp_pool_update diffs res against the materialised counts:
 * surplus ordinals are OFFLOADed (slots freed), missing ones get a slot and a copy job --
 * REPLICATE from the expert's ordinal-0 copy, or LOAD from the master weights when the expert
 * had no copy; mp_replica_copy runs the jobs (expert_bytes per tensor), mp_piece_pool maps every
 * GEMM piece (mp_exec_map outputs) to the weight slot of its replica, and mp_ffn_up_pool /
 * mp_ffn_down_pool run the grouped GEMMs on the pool (same flags as mp_ffn_up/down, single-CTA
 * pre-tiled only). mp_pool_stats copies {loads, replicates, offloads since init, overflow flag}
 * into 4 device ints. All device-side (no host sync). */
MP_API size_t mp_pool_state_bytes(int E, int R, int P);
MP_API int mp_pool_init(int E, int R, int P, void* state, void* stream);
MP_API int mp_pool_update(const int32_t* res, int E, int R, int P, void* state, void* stream);
MP_API int mp_replica_copy(const void* master_u, const void* master_v, void* pool_u, void* pool_v, size_t expert_bytes,
                           int P, const void* state, int E, int R, void* stream);
MP_API int mp_piece_pool(const int32_t* piece_row, const int32_t* exp_begin, int E, const int32_t* tok_of_row,
                         const int32_t* token_to_slot, const void* state, int R, int P, int32_t* piece_wbase,
                         int max_pieces, void* stream);
MP_API int mp_pool_stats(const void* state, int E, int R, int P, int32_t* out4, void* stream);
MP_API int mp_ffn_up_pool(int T, int dp, int Fp, int E, int W, const void* pool_u, int flags, const int32_t* piece_row,
                          const int32_t* piece_rows, const int32_t* exp_begin, const int32_t* piece_wbase, void* ws,
                          size_t ws_bytes, void* stream);
MP_API int mp_ffn_down_pool(float* y, int T, int dp, int Fp, int E, int W, const void* pool_v, int flags,
                            const int32_t* tok_of_row, const int32_t* piece_row, const int32_t* piece_rows,
                            const int32_t* exp_begin, const int32_t* piece_wbase, void* ws, size_t ws_bytes,
                            void* stream);
/* Diagnostics: per-CTA %globaltimer start / end (ns) of the last grouped-GEMM launch
 * (host arrays of n <= 1024). */
MP_API int mp_debug_cta_times(unsigned long long* t0, unsigned long long* t1, int n);
/* Weight layout transform for the grouped GEMM B operand:
 * dst[g][n / BN][k / 64][n % BN][k % 64] = src[g * N + n][k]   (bf16, G groups of N x K). */
MP_API int mp_tile_kmajor(const void* src, void* dst, int G, int N, int K, int BN, void* stream);

/* ------------------------------------------------------------------ C1/C2: expert parallelism
 * (SURVEY.md §8(e)). G ranks, tokens sharded by position, all expert weights resident on
 * every GPU, the slot list cut into G blocks of equal rows (a slot runs on the GPU its row
 * midpoint falls in). Per layer, after the caller all-gathers per-rank expert counts C
 * (G x E int32, from mp_histogram_ws):
 *   mp_ep_plan         same residency/corrective update and global stable ranks as the
 *                      single-device execution map; send/recv row counts per peer; this
 *                      rank's send position per token; local pieces of hosted replicas.
 *                      More slots than max_slots (>= G * capacity + E): num_local_rows = -1
 *                      and zero counts, so the caller raises before any collective
 *   mp_ep_pack         bf16 rows into the send buffer (destination-major)
 *   (caller: variable all-to-all of the rows, e.g. NCCL)
 *   mp_ep_recv_layout  local row (slot-major, global token order) of every received row
 *   mp_gather_rows_bf16 + mp_ffn_up/down (tok_of_row = recv_of_local: results land in
 *                      receive order)  (caller: reverse all-to-all of fp32 results)
 *   mp_ep_combine      x[t] += yback[send_pos[t]]
 * Results are bit-identical to the single-GPU path. ws >= mp_ep_workspace_bytes. */
MP_API size_t mp_ep_workspace_bytes(int G, int T, int E, int max_slots);
MP_API int mp_ep_plan(const int32_t* route, int T, const int32_t* C, int G, int E, int rank, int max_slots,
                      int split_m, int32_t* res, int32_t* send_counts, int32_t* recv_counts, int32_t* num_local_rows,
                      int32_t* send_pos, int32_t* piece_row, int32_t* piece_rows, int32_t* exp_begin, void* ws,
                      size_t ws_bytes, void* stream);
MP_API int mp_ep_pack(const float* x, int T, int d, const int32_t* send_pos, void* sendbuf, void* stream);
MP_API int mp_ep_recv_layout(int G, int T, int E, int rank, int max_slots, const int32_t* recvbuf_rows_unused,
                             int32_t* recv_of_local, void* ws, size_t ws_bytes, void* stream);
MP_API int mp_gather_rows_bf16(const void* buf, int n, int d, const int32_t* idx, void* out, void* stream);
MP_API int mp_ep_combine(float* x, int T, int d, const float* yback, const int32_t* send_pos, void* stream);
/* Fixed-split form (graph-capturable dispatch, no split sizes on the host): every (source,
 * destination) block of the send / receive buffers holds peer_cap rows, so the caller's
 * all-to-alls use equal static splits of peer_cap * d elements. If the layer needs more
 * than peer_cap rows for some peer, *overflow |= 1 and the layer does nothing on the device
 * (no pieces, no sends): check the flag once per step and re-run the step with
 * mp_ep_plan. peer_cap = 0 is mp_ep_plan. mp_gather_rows_bf16_dn gathers min(n_max,
 * *n_dev) rows (n_dev = the plan's num_local_rows, on the device). */
MP_API int mp_ep_plan_cap(const int32_t* route, int T, const int32_t* C, int G, int E, int rank, int max_slots,
                          int split_m, int peer_cap, int32_t* overflow, int32_t* res, int32_t* send_counts,
                          int32_t* recv_counts, int32_t* num_local_rows, int32_t* send_pos, int32_t* piece_row,
                          int32_t* piece_rows, int32_t* exp_begin, void* ws, size_t ws_bytes, void* stream);
MP_API int mp_gather_rows_bf16_dn(const void* buf, int n_max, int d, const int32_t* idx, const int32_t* n_dev,
                                  void* out, void* stream);
/* Peer-memory form of the fixed-split dispatch / combine (NVLink P2P; no all-to-all):
 * recv_rows / recv_tok / flags / peer_x are DEVICE arrays of G pointers, entry g = rank g's
 * receive rows (G * peer_cap x d bf16), receive token indices (G * peer_cap int32), barrier
 * flags (G int32, zero-initialised) and residual stream (T_home x d fp32), mapped into this
 * process (CUDA IPC; entry `rank` is the local buffer).
 *   mp_ep_pack_peer    token t -> rank g = send_pos[t] / peer_cap, row rank * peer_cap + j
 *                      of g's receive rows, and t into g's recv_tok at the same row
 *   mp_peer_barrier    device barrier of the G ranks (epoch counter in *epoch, one per rank);
 *                      orders the peer-memory writes before it for every rank after it; a rank
 *                      missing for 5 s sets *err |= 1 instead of hanging (check it per step)
 *   mp_peer_allgather_i32  dst[g][row * dst_row_stride + rank * n + i] = src[row * n + i] for
 *                      every rank g: all-gather of rows x n 32-bit words (expert counts, SRU
 *                      carry maps, predicted assignments) completed by the next barrier
 *   mp_ep_gather_peer  mp_gather_rows_bf16_dn + dst_of_row[r] = home * T_home + t of the row
 *   mp_ffn_down_peer   GEMM2 whose epilogue ADDS row r into peer_x[home][t] (the combine)
 * Per layer: counts -> allgather_i32 -> barrier -> plan_cap -> pack_peer -> barrier ->
 * recv_layout -> gather_peer -> ffn_up -> ffn_down_peer -> barrier. Bit-identical to the all-to-all form (one addend per element). */
MP_API int mp_ep_pack_peer(const float* x, int T, int d, const int32_t* send_pos, int peer_cap, int rank,
                           void* const* recv_rows, int32_t* const* recv_tok, void* stream);
MP_API int mp_peer_barrier(int32_t* const* flags, int rank, int G, int32_t* epoch, int32_t* err, void* stream);
MP_API int mp_peer_allgather_i32(const int32_t* src, int rows, int n, int rank, int G, int32_t* const* dst,
                                 int dst_row_stride, void* stream);
MP_API int mp_ep_gather_peer(const void* buf, int n_max, int d, const int32_t* idx, const int32_t* n_dev,
                             const int32_t* recv_tok, int peer_cap, int T_home, int32_t* dst_of_row, void* out,
                             void* stream);
MP_API int mp_ffn_down_peer(float* const* peer_x, int T_home, int T, int dp, int Fp, int E, const void* v, int flags,
                            const int32_t* dst_of_row, const int32_t* piece_row, const int32_t* piece_rows,
                            const int32_t* exp_begin, void* ws, size_t ws_bytes, void* stream);


/* Whole-step CUDA graphs (capture on `stream`, replay) and timing events that remain
 * valid inside a captured graph (recorded as external event nodes). Host plumbing. */
MP_API int mp_graph_begin(void* stream);
MP_API int mp_graph_end(void* stream, void** graph_exec);
/* As mp_graph_end; *kernel_nodes = kernel nodes in the captured graph (launches per replay). */
MP_API int mp_graph_end_counted(void* stream, void** graph_exec, int32_t* kernel_nodes);
MP_API int mp_graph_launch(void* graph_exec, void* stream);
MP_API int mp_graph_destroy(void* graph_exec);
MP_API int mp_event_create(void** ev);
MP_API int mp_event_record(void* ev, void* stream);
MP_API int mp_event_elapsed_ms(void* a, void* b, float* ms); /* host out-param */
MP_API int mp_event_destroy(void* ev);

/* L2 residency hint: persisting access-policy window over [ptr, ptr + bytes) for kernels
 * launched on `stream` (bytes = 0 clears). Host plumbing. */
MP_API int mp_l2_persist(void* ptr, size_t bytes, float hit_ratio, void* stream);
/* Host plumbing for peer memory: let kernels on the current device access memory of
 * `peer_device` (cudaDeviceEnablePeerAccess; already enabled is OK). MP_ERR_CONFIG when the
 * pair has no peer access (e.g. no NVLink / P2P between them). */
MP_API int mp_enable_peer_access(int peer_device);

/* Operand staging: y[i] = bf16(x[i]) (round to nearest even), n % 4 == 0. */
MP_API int mp_f32_to_bf16(const float* x, void* y, size_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MOEMPMC_H */
