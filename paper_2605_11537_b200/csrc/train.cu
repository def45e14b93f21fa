// SRU predictor training on the GPU: the float64
// recurrences of the forward-with-caches and of back-propagation through time,
// the softmax cross-entropy of the head logits, and deterministic reductions.
// The dense products (x W^T, dU^T x, dz @ heads, ...) are plain float64 library
// GEMMs issued by the host (training/inference precision: the reference trains in
// float64, src/predictor.py:238-379).
//
// Elementwise arithmetic uses explicit round-to-nearest intrinsics so nothing is
// contracted into FMAs: every cell update rounds exactly like the reference's
// numpy expressions (only exp / tanh / log may differ in the last ulp).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"

namespace mp {

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }

// 1 / (1 + exp(-clip(z, -60, 60)))  (src/predictor.py:24-25)
__device__ __forceinline__ double sigmoid64(double z) {
  z = fmin(fmax(z, -60.0), 60.0);
  return __ddiv_rn(1.0, add(1.0, exp(-z)));
}

// Forward of one SRU layer over S sequences x T tokens (src/predictor.py:238-254):
//   f = sigma(x W_f^T + b_f), r = sigma(x W_r^T + b_r) (products from the host GEMMs),
//   c_t = f c_{t-1} + (1 - f) u, g = tanh(c),
//   h = r g + (1 - r) x. One thread per (sequence, channel), tokens in order.
__global__ void k_sru_train_fwd(const double* __restrict__ u, const double* __restrict__ fpre,
                                const double* __restrict__ rpre, const double* __restrict__ bf,
                                const double* __restrict__ br, const double* __restrict__ x, int S, int T, int d,
                                double* __restrict__ f, double* __restrict__ r, double* __restrict__ c,
                                double* __restrict__ g, double* __restrict__ h) {
  griddep_launch_dependents();
  griddep_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S * d) return;
  const int s = i / d, ch = i - s * d;
  double ct = 0.0;
  const double bft = bf[ch], brt = br[ch];
  for (int t = 0; t < T; ++t) {
    const size_t o = ((size_t)s * T + t) * d + ch;
    const double ft = sigmoid64(add(fpre[o], bft)), rt = sigmoid64(add(rpre[o], brt));
    ct = add(mul(ft, ct), mul(sub(1.0, ft), u[o]));
    const double gt = tanh(ct);
    f[o] = ft;
    r[o] = rt;
    c[o] = ct;
    g[o] = gt;
    h[o] = add(mul(rt, gt), mul(sub(1.0, rt), x[o]));
  }
}

// Back-propagation through one SRU layer (src/predictor.py:257-294), reverse time:
//   drp = dh (g - x) r (1 - r); dc = dh r (1 - g^2); dct = dc + next;
//   df = dct (c_{t-1} - u); du = dct (1 - f); next = dct f; dfp = df f (1 - f).
// Also dh_out = dh (1 - r) (the highway part of d_hidden) and per-sequence bias-gradient
// partial sums over tokens (summed over sequences by mp_train_colsum).
__global__ void k_sru_train_bwd(const double* __restrict__ dh, const double* __restrict__ x,
                                const double* __restrict__ u, const double* __restrict__ f,
                                const double* __restrict__ r, const double* __restrict__ c,
                                const double* __restrict__ g, int S, int T, int d, double* __restrict__ du,
                                double* __restrict__ dfp, double* __restrict__ drp, double* __restrict__ dh_out,
                                double* __restrict__ bsum_f, double* __restrict__ bsum_r) {
  griddep_launch_dependents();
  griddep_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S * d) return;
  const int s = i / d, ch = i - s * d;
  double nxt = 0.0, sf = 0.0, sr = 0.0;
  for (int t = T - 1; t >= 0; --t) {
    const size_t o = ((size_t)s * T + t) * d + ch;
    const double dht = dh[o], gt = g[o], rt = r[o], ft = f[o], ut = u[o], xt = x[o];
    const double dr = mul(mul(mul(dht, sub(gt, xt)), rt), sub(1.0, rt));
    const double dc = mul(mul(dht, rt), sub(1.0, mul(gt, gt)));
    const double dct = add(dc, nxt);
    const double cp = t > 0 ? c[o - d] : 0.0;
    const double df = mul(dct, sub(cp, ut));
    du[o] = mul(dct, sub(1.0, ft));
    nxt = mul(dct, ft);
    const double dfpt = mul(mul(df, ft), sub(1.0, ft));
    dfp[o] = dfpt;
    drp[o] = dr;
    dh_out[o] = mul(dht, sub(1.0, rt));
    sf = add(sf, dfpt);
    sr = add(sr, dr);
  }
  bsum_f[(size_t)s * d + ch] = sf;
  bsum_r[(size_t)s * d + ch] = sr;
}

// out[j] = sum_i in[i][j] in row order (deterministic).
__global__ void k_train_colsum(const double* __restrict__ in, int R, int n, double* __restrict__ out) {
  griddep_launch_dependents();
  griddep_wait();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double s = 0.0;
  for (int i = 0; i < R; ++i) s = add(s, in[(size_t)i * n + j]);
  out[j] = s;
}

// Softmax cross-entropy per row of N x E logits (src/predictor.py:312-325):
// row_loss = -log(max(p[label], 1e-300)); dz = (p - onehot(label)) * inv_S.
// labels: element (row) at labels[row * lstride] (one MoE layer of the (S, L, T) array).
__global__ void k_train_ce(const double* __restrict__ z, const int64_t* __restrict__ labels, int S, int T, int L,
                           int layer, int E, double inv_S, double* __restrict__ dz, double* __restrict__ row_loss) {
  griddep_launch_dependents();
  griddep_wait();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= S * T) return;
  const int s = row / T, t = row - s * T;
  const int lab = (int)labels[((size_t)s * L + layer) * T + t];
  const double* zr = z + (size_t)row * E;
  double m = zr[0];
  for (int e = 1; e < E; ++e) m = fmax(m, zr[e]);
  double sum = 0.0;
  for (int e = 0; e < E; ++e) sum = add(sum, exp(sub(zr[e], m)));
  double* dr = dz + (size_t)row * E;
  double picked = 0.0;
  for (int e = 0; e < E; ++e) {
    const double p = __ddiv_rn(exp(sub(zr[e], m)), sum);
    if (e == lab) picked = p;
    dr[e] = mul(e == lab ? sub(p, 1.0) : p, inv_S);
  }
  row_loss[row] = -log(fmax(picked, 1e-300));
}

// Single-block deterministic sum of n doubles (fixed tree over a fixed thread layout).
__global__ void k_train_sum(const double* __restrict__ in, int n, double* __restrict__ out) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ double sh[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s = add(s, in[i]);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] = add(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sh[0];
}

// y += alpha * x (SGD step), elementwise without contraction.
__global__ void k_train_axpy(double* __restrict__ y, const double* __restrict__ x, size_t n, double alpha) {
  griddep_launch_dependents();
  griddep_wait();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    y[i] = sub(y[i], mul(-alpha, x[i]));
}

// flag |= any non-finite among n values
__global__ void k_train_nonfinite(const double* __restrict__ x, size_t n, int32_t* __restrict__ flag) {
  griddep_launch_dependents();
  griddep_wait();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) {
      atomicOr(flag, 1);
      return;
    }
}

}  // namespace mp

using namespace mp;

extern "C" int mp_sru_train_fwd(const double* u, const double* fpre, const double* rpre, const double* b_f,
                                const double* b_r, const double* x, int S, int T, int d, double* f, double* r, double* c,
                                double* g, double* h, void* stream) {
  MP_REQUIRE(S >= 1 && T >= 1 && d >= 1, MP_ERR_CONFIG, "mp_sru_train_fwd: bad S/T/d");
  k_sru_train_fwd<<<cdiv(S * d, 128), 128, 0, (cudaStream_t)stream>>>(u, fpre, rpre, b_f, b_r, x, S, T, d, f, r, c, g,
                                                                       h);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_sru_train_bwd(const double* dh, const double* x, const double* u, const double* f, const double* r,
                                const double* c, const double* g, int S, int T, int d, double* du, double* dfp,
                                double* drp, double* dh_out, double* bsum_f, double* bsum_r, void* stream) {
  MP_REQUIRE(S >= 1 && T >= 1 && d >= 1, MP_ERR_CONFIG, "mp_sru_train_bwd: bad S/T/d");
  k_sru_train_bwd<<<cdiv(S * d, 128), 128, 0, (cudaStream_t)stream>>>(dh, x, u, f, r, c, g, S, T, d, du, dfp, drp,
                                                                       dh_out, bsum_f, bsum_r);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_train_colsum(const double* in, int R, int n, double* out, void* stream) {
  MP_REQUIRE(R >= 1 && n >= 1, MP_ERR_CONFIG, "mp_train_colsum: bad sizes");
  k_train_colsum<<<cdiv(n, 128), 128, 0, (cudaStream_t)stream>>>(in, R, n, out);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_train_ce(const double* logits, const int64_t* labels, int S, int T, int L, int layer, int E,
                           double* dlogits, double* row_loss, void* stream) {
  MP_REQUIRE(S >= 1 && T >= 1 && E >= 1 && layer >= 0 && layer < L, MP_ERR_CONFIG, "mp_train_ce: bad sizes");
  k_train_ce<<<cdiv(S * T, 128), 128, 0, (cudaStream_t)stream>>>(logits, labels, S, T, L, layer, E, 1.0 / S, dlogits,
                                                                   row_loss);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_train_sum(const double* in, int n, double* out, void* stream) {
  MP_REQUIRE(n >= 1, MP_ERR_CONFIG, "mp_train_sum: n < 1");
  k_train_sum<<<1, 256, 0, (cudaStream_t)stream>>>(in, n, out);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_train_axpy(double* y, const double* x, size_t n, double alpha, void* stream) {
  if (n == 0) return MP_OK;
  const int grid = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  k_train_axpy<<<grid, 256, 0, (cudaStream_t)stream>>>(y, x, n, alpha);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}

extern "C" int mp_train_nonfinite(const double* x, size_t n, int32_t* flag, void* stream) {
  if (n == 0) return MP_OK;
  const int grid = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  k_train_nonfinite<<<grid, 256, 0, (cudaStream_t)stream>>>(x, n, flag);
  MP_CUDA_TRY(cudaGetLastError());
  return MP_OK;
}
