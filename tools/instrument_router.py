"""Inserts %globaltimer probes into csrc/router.cu (k_router_fused_tx phases, for tools/rt_probe.py).
Usage: python tools/instrument_router.py && python -c 'from paper_2605_11537_b200 import build; build.build()'
then run tools/rt_probe.py on the GPU; restore the file with git checkout afterwards."""
import pathlib
p = str(pathlib.Path(__file__).resolve().parents[1] / 'paper_2605_11537_b200/csrc/router.cu')
s=open(p).read()
s=s.replace('''template <int EG>
__global__ void __launch_bounds__(kRouterThreads, 1)
    k_router_fused_tx(''','''static __device__ unsigned long long g_rt[256][8];
static __device__ __forceinline__ unsigned long long rtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
template <int EG>
__global__ void __launch_bounds__(kRouterThreads, 1)
    k_router_fused_tx(''',1)
s=s.replace('''  if (warp == 2) tmem_alloc(tmem_slot, 2 * EG < 32 ? 32 : 2 * EG);
  griddep_wait();  // x is the previous layer's output
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
''','''  if (threadIdx.x == 0) g_rt[blockIdx.x][0] = rtime();
  if (warp == 2) tmem_alloc(tmem_slot, 2 * EG < 32 ? 32 : 2 * EG);
  griddep_wait();  // x is the previous layer's output
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) g_rt[blockIdx.x][1] = rtime();
''',1)
s=s.replace('''          mbar_wait(&full[stage], phase);
          mbar_wait(&conv[xstage], xphase);
          tc_fence_after();''','''          if (kb == 6) g_rt[blockIdx.x + 128][3] = rtime();
          mbar_wait(&full[stage], phase);
          if (kb == 6) g_rt[blockIdx.x + 128][4] = rtime();
          mbar_wait(&conv[xstage], xphase);
          tc_fence_after();
          if (kb == 0) g_rt[blockIdx.x][2] = rtime();
          if (kb == 6) g_rt[blockIdx.x][3] = rtime();''',1)
s=s.replace('''        umma_commit(tfull);''','''        umma_commit(tfull);
        g_rt[blockIdx.x][4] = rtime();''',1)
s=s.replace('''        mbar_wait(tfull, tile & 1);
        tc_fence_after();''','''        mbar_wait(tfull, tile & 1);
        tc_fence_after();
        if (threadIdx.x == 128) g_rt[blockIdx.x][5] = rtime();''',1)
s=s.replace('''      named_bar_sync(1, kRfConvThreads);
      if (hist_cc != nullptr) {  // the tile is one 128-token chunk of the execution map''','''      named_bar_sync(1, kRfConvThreads);
      if (threadIdx.x == 128) g_rt[blockIdx.x][6] = rtime();
      if (hist_cc != nullptr) {  // the tile is one 128-token chunk of the execution map''',1)
s=s.replace('''      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&xfull[xstage], xphase);
        uint8_t* sxs = smem + L::kXOffset + xstage * L::kXs;''','''      for (int kb = 0; kb < nkb; ++kb) {
        if (kb == 6 && threadIdx.x == 128) g_rt[blockIdx.x][7] = rtime();
        mbar_wait(&xfull[xstage], xphase);
        if (kb == 6 && threadIdx.x == 128) g_rt[blockIdx.x + 128][0] = rtime();
        uint8_t* sxs = smem + L::kXOffset + xstage * L::kXs;''',1)
s=s.replace('''        named_bar_sync(2, kRfConvThreads);
        uint8_t* shi = sxs;''','''        named_bar_sync(2, kRfConvThreads);
        if (kb == 6 && threadIdx.x == 128) g_rt[blockIdx.x + 128][1] = rtime();
        uint8_t* shi = sxs;''',1)
s=s.replace('''        if (lane == 0) mbar_arrive(&conv[xstage]);
        if (++xstage == kRxXStages) {''','''        if (lane == 0) mbar_arrive(&conv[xstage]);
        if (kb == 6 && threadIdx.x == 128) g_rt[blockIdx.x + 128][2] = rtime();
        if (++xstage == kRxXStages) {''',1)
s+='''
extern "C" __attribute__((visibility("default"))) int mp_debug_router_times(unsigned long long* out, int n) {
  MP_CUDA_TRY(cudaMemcpyFromSymbol(out, mp::g_rt, sizeof(unsigned long long) * 8 * n));
  return MP_OK;
}
'''
print(s.count('g_rt'))
open(p,'w').write(s)
