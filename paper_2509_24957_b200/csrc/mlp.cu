// General frozen-MLP forward in fp64 (reference predictor.py:126-151), one CTA
// per input row: LayerNorm (population variance, eps 1e-5) -> [W x + b ->
// optional inference batch-norm -> ReLU | erf-GeLU]* -> head -> clipped
// sigmoid (1-dim head) or softmax. Each output neuron is one warp-wide dot
// product (coalesced weight rows). This is the drop-in for `mlp_forward` with
// hidden layers and for the 5-way complexity head of predict_difficulty("mlp");
// the linear probe on the hot path is K1 (score.cu).
#include "common.cuh"
#include "../../include/duchess_b200.h"

namespace duchess {

constexpr int kMlpThreads = 256;

__device__ double block_sum_d(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < kMlpThreads / 32; ++w) s += red[w];
  __syncthreads();
  return s;
}

__device__ double block_max_d(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = red[0];
  for (int w = 1; w < kMlpThreads / 32; ++w) s = fmax(s, red[w]);
  __syncthreads();
  return s;
}

// y[j] = b[j] + W[j, :] . x  (warp per output)
__device__ void dense(const double* W, const double* b, const double* x, double* y, int n_in,
                      int n_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = warp; j < n_out; j += kMlpThreads / 32) {
    const double* row = W + int64_t(j) * n_in;
    double acc = 0.0;
    for (int k = lane; k < n_in; k += 32) acc = fma(row[k], x[k], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y[j] = acc + b[j];
  }
  __syncthreads();
}

constexpr int kMaxHidden = 64;
struct MlpShape {
  int32_t dims[kMaxHidden + 2];
  int32_t act[kMaxHidden];
};

__global__ void __launch_bounds__(kMlpThreads)
mlp_kernel(const double* params, MlpShape shape, int n_hidden, int head, int has_ln, int has_bn,
           const double* xin, int max_dim, double* logits, double* probs) {
  const int32_t* dims = shape.dims;
  const int32_t* act = shape.act;
  extern __shared__ double sm[];
  __shared__ double red[kMlpThreads / 32];
  double* a = sm;
  double* bbuf = sm + max_dim;
  const int64_t row = blockIdx.x;
  const int H = dims[0];
  const double* x = xin + row * H;
  for (int h = threadIdx.x; h < H; h += kMlpThreads) a[h] = x[h];
  __syncthreads();
  double s = 0.0;
  for (int h = threadIdx.x; h < H; h += kMlpThreads) s += a[h];
  const double mean = block_sum_d(s, red) / double(H);
  double q = 0.0;
  for (int h = threadIdx.x; h < H; h += kMlpThreads) q += (a[h] - mean) * (a[h] - mean);
  const double var = block_sum_d(q, red) / double(H);
  const double inv = 1.0 / sqrt(var + 1e-5);
  const double* p = params;
  const double* g = has_ln ? p : nullptr;
  const double* bl = has_ln ? p + H : nullptr;
  if (has_ln) p += 2 * H;
  for (int h = threadIdx.x; h < H; h += kMlpThreads) {
    double z = (a[h] - mean) * inv;
    if (has_ln) z = z * g[h] + bl[h];
    a[h] = z;
  }
  __syncthreads();
  for (int k = 0; k < n_hidden; ++k) {
    const int din = dims[k], dout = dims[k + 1];
    const double* W = p;
    const double* b = p + int64_t(din) * dout;
    p = b + dout;
    dense(W, b, a, bbuf, din, dout);
    const double *bm = nullptr, *bv = nullptr, *bg = nullptr, *bb = nullptr;
    if (has_bn) {
      bm = p; bv = p + dout; bg = p + 2 * dout; bb = p + 3 * dout;
      p += 4 * dout;
    }
    for (int j = threadIdx.x; j < dout; j += kMlpThreads) {
      double v = bbuf[j];
      if (has_bn) v = (v - bm[j]) / sqrt(bv[j] + 1e-5) * bg[j] + bb[j];
      v = act[k] == 0 ? fmax(v, 0.0) : v * 0.5 * (1.0 + erf(v / sqrt(2.0)));
      bbuf[j] = v;
    }
    __syncthreads();
    double* t = a; a = bbuf; bbuf = t;
  }
  const int dl = dims[n_hidden];
  dense(p, p + int64_t(dl) * head, a, bbuf, dl, head);
  double* lg = logits + row * head;
  double* pr = probs + row * head;
  if (head == 1) {
    if (threadIdx.x == 0) {
      const double z = bbuf[0];
      lg[0] = z;
      pr[0] = fmin(fmax(1.0 / (1.0 + exp(-z)), kProbClip), 1.0 - kProbClip);
    }
    return;
  }
  double m = -INFINITY;
  for (int j = threadIdx.x; j < head; j += kMlpThreads) m = fmax(m, bbuf[j]);
  m = block_max_d(m, red);
  double e = 0.0;
  for (int j = threadIdx.x; j < head; j += kMlpThreads) e += exp(bbuf[j] - m);
  const double tot = block_sum_d(e, red);
  for (int j = threadIdx.x; j < head; j += kMlpThreads) {
    lg[j] = bbuf[j];
    pr[j] = exp(bbuf[j] - m) / tot;
  }
}

}  // namespace duchess

using namespace duchess;

extern "C" int duchess_mlp_forward(const double* params, const int32_t* dims, int32_t n_hidden,
                                   int32_t head_dim, const int32_t* act, int32_t has_ln,
                                   int32_t has_bn, const double* x, int64_t n_rows,
                                   double* logits, double* probs, void* stream) {
  // dims (n_hidden + 1 entries) / act (n_hidden) are HOST arrays, passed by value.
  if (!params || !dims || n_hidden < 0 || head_dim < 1 || !x || !logits || !probs) return DUCHESS_EINVAL;
  if (n_rows == 0) return DUCHESS_OK;
  if (n_hidden > kMaxHidden) return DUCHESS_EINVAL;
  MlpShape shape{};
  int max_dim = head_dim;
  for (int k = 0; k <= n_hidden; ++k) {
    shape.dims[k] = dims[k];
    max_dim = dims[k] > max_dim ? dims[k] : max_dim;
  }
  shape.dims[n_hidden + 1] = head_dim;
  for (int k = 0; k < n_hidden; ++k) shape.act[k] = act ? act[k] : 0;
  const size_t smem = size_t(2) * max_dim * sizeof(double);
  if (smem > 200 * 1024) return DUCHESS_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaFuncSetAttribute(mlp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  mlp_kernel<<<unsigned(n_rows), kMlpThreads, smem, s>>>(params, shape, n_hidden, head_dim, has_ln,
                                                         has_bn, x, max_dim, logits, probs);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DUCHESS_OK : DUCHESS_ECUDA;
}
