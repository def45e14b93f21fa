// Per-layer transfer-event and queue counts of one batch, on the device: the inputs of the
// reference cost model (BatchRunner._metrics_from, src/simulator.py:210-235, over
// simulate_layer :62-81 and the TransferLog of src/placement.py:35-63).
//
// For every layer l (one block each):
//   counts[l*5 + 0]  LOAD events       placement loads (token events of kind LOAD) + corrective loads
//   counts[l*5 + 1]  REPLICATE events  token events of kind REPLICATE
//   counts[l*5 + 2]  OFFLOAD events    sum_e offloads[l, e]   (offloads: L x E_off, corrective: L x E_corr)
//   counts[l*5 + 3]  longest queue     max_s #{t : token_to_slot[l, t] == s}
//   counts[l*5 + 4]  slots             num_slots[l] (the execution map's slot count)
// The host turns these into the reference's Metrics (paper_2605_11537_b200/simulator.py).
#include "common.cuh"

namespace mp {

__global__ void k_layer_counts(const int32_t* __restrict__ token_event, const int32_t* __restrict__ offloads,
                               const int32_t* __restrict__ corrective, const int32_t* __restrict__ token_to_slot,
                               const int32_t* __restrict__ num_slots, int T, int E_off, int E_corr, int max_slots,
                               int32_t* __restrict__ counts, int32_t* __restrict__ err) {
  extern __shared__ int s_q[];  // max_slots queue lengths
  __shared__ int s_red[5];
  const int l = blockIdx.x;
  const int ns = num_slots[l];
  for (int s = threadIdx.x; s < max_slots; s += blockDim.x) s_q[s] = 0;
  if (threadIdx.x < 5) s_red[threadIdx.x] = 0;
  __syncthreads();
  int loads = 0, reps = 0, offl = 0, bad = 0;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const int s = token_to_slot[(size_t)l * T + t];
    if (s < 0 || s >= ns || s >= max_slots) {
      bad = 1;
    } else {
      atomicAdd(&s_q[s], 1);
    }
    if (token_event != nullptr) {
      const int ev = token_event[(size_t)l * T + t];
      if (ev >= 0) {
        const int kind = ev >> MP_EVENT_KIND_SHIFT;
        loads += kind == MP_EVENT_LOAD;
        reps += kind == MP_EVENT_REPLICATE;
      }
    }
  }
  if (offloads != nullptr)
    for (int e = threadIdx.x; e < E_off; e += blockDim.x) offl += offloads[(size_t)l * E_off + e];
  if (corrective != nullptr)
    for (int e = threadIdx.x; e < E_corr; e += blockDim.x) loads += corrective[(size_t)l * E_corr + e];
  __syncthreads();
  int qmax = 0;
  for (int s = threadIdx.x; s < max_slots; s += blockDim.x) qmax = max(qmax, s_q[s]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    loads += __shfl_xor_sync(0xffffffffu, loads, o);
    reps += __shfl_xor_sync(0xffffffffu, reps, o);
    offl += __shfl_xor_sync(0xffffffffu, offl, o);
    qmax = max(qmax, __shfl_xor_sync(0xffffffffu, qmax, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s_red[0], loads);
    atomicAdd(&s_red[1], reps);
    atomicAdd(&s_red[2], offl);
    atomicMax(&s_red[3], qmax);
    atomicOr(&s_red[4], bad);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    counts[l * 5 + 0] = s_red[0];
    counts[l * 5 + 1] = s_red[1];
    counts[l * 5 + 2] = s_red[2];
    counts[l * 5 + 3] = s_red[3];
    counts[l * 5 + 4] = ns;
    if (s_red[4]) atomicOr(err, 1);
  }
}

}  // namespace mp

using namespace mp;

extern "C" int mp_layer_counts(const int32_t* token_event, const int32_t* offloads, const int32_t* corrective,
                               const int32_t* token_to_slot, const int32_t* num_slots, int L, int T, int E_off,
                               int E_corr, int max_slots, int32_t* counts, int32_t* err, void* stream) {
  MP_REQUIRE(L >= 1 && T >= 1 && E_off >= 0 && E_corr >= 0 && max_slots >= 1 && max_slots <= 49152, MP_ERR_CONFIG,
             "mp_layer_counts: bad sizes (L=%d T=%d max_slots=%d)", L, T, max_slots);
  MP_REQUIRE(token_to_slot != nullptr && num_slots != nullptr && counts != nullptr && err != nullptr, MP_ERR_CONFIG,
             "mp_layer_counts: token_to_slot, num_slots, counts and err are required");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = sizeof(int) * (size_t)max_slots;
  if (smem > 48 * 1024) {
    static bool configured = false;
    if (!configured) {
      MP_CUDA_TRY(cudaFuncSetAttribute(k_layer_counts, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152 * 4));
      configured = true;
    }
  }
  k_layer_counts<<<L, 1024, smem, st>>>(token_event, offloads, corrective, token_to_slot, num_slots, T, E_off, E_corr, max_slots,
                                        counts, err);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}
