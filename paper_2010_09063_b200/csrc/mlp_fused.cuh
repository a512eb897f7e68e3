// Fused per-example pass of small dense models (logistic regression, FCNN
// 104-50-10 / 104-50-2): one warp per example runs the forward pass
// (models.cpp:182-196, relu fused), the softmax / sigmoid cross-entropy and
// its gradient (kernels.hpp:516-566), the input-gradient chain
// (autodiff.cpp:121-124,155-159) and the ghost-norm factors of every dense
// block (strategies.cpp:140-148: ||a (x) d||^2 = ||a||^2 ||d||^2, bias ||d||^2)
// in fp64. It writes exactly what the layer-wise schedule writes (activations,
// output cotangents, losses, per-block squared norms), so the aggregation
// kernel consumes it unchanged. These models are launch-latency bound: the
// layer-wise schedule spends ~6 dependent launches per step on ~1 MFLOP.
#pragma once

#include "kernels.cuh"

namespace pgb {
namespace mlp {

constexpr int kMaxLayers = 4;
constexpr int kMaxWidth = 128;
constexpr int kMaxClasses = 32;
constexpr int kWarps = 8;  // examples per CTA

constexpr int kMaxParams = 40 * 1024;  // staged in shared memory

struct DenseLayer {
  int in, out, relu;
  int pW, pb;          // parameter block ordinals (norm partial columns)
  int offW, offb;      // offsets of W (in, out) row-major and b (out) in the flat parameters
  float* act;          // (B, out) output after the fused relu
  float* gout;         // (B, out) cotangent of the output
};

struct Params {
  int n;  // dense layers
  DenseLayer L[kMaxLayers];
  const float* params;  // flat parameters; [stage_off, stage_off + P) staged into shared memory
  int P, stage_off;     // (offW / offb are relative to stage_off)
  float* gin;           // optional (B, L[0].in): cotangent of the input (an embedding head)
  const float* x;  // (B, L[0].in)
  const float* y;  // (B) labels as float
  float* xin;      // (B, L[0].in): the inputs again, the ghost factor a of layer 0
  // multi-step graphs over a device-resident ring of batches (as mnist::Params):
  // step s = *step_base + step_off reads batch (s - ring_origin) mod ring_n
  const long long* step_base;
  int step_off;
  const float* xring;
  const float* yring;
  long long ring_origin;
  int ring_n;
  float* loss;     // (B)
  double* parts;   // (B, nparts) squared norm per parameter block
  int nparts, B, classes;
  DevError* err;
  // the step's Gaussian noise drawn by extra CTAs while the examples run
  // (kernels.hpp:597-614), so the aggregation's epilogue only loads it:
  // blocks nb_first .. nb_first + nnb - 1 of the parameter vector
  StepArgs a;
  float* noise;  // (P_total) or null
  int noise_ctas, nb_first, nnb;
  long long nb_off[2 * kMaxLayers], nb_size[2 * kMaxLayers], nb_pair[2 * kMaxLayers + 1];
};

// extra CTA k of mlp_kernel: one Box-Muller pair per thread
__device__ __forceinline__ void draw_noise(const Params& P, int k) {
  const long long q = (long long)k * blockDim.x + threadIdx.x;
  if (!P.a.add_noise || q >= P.nb_pair[P.nnb]) return;
  int b = 0;
  while (b + 1 < P.nnb && P.nb_pair[b + 1] <= q) ++b;
  const long long jp = q - P.nb_pair[b];
  const long long st = P.step_base ? *P.step_base + P.step_off : P.a.step;
  float n0, n1;
  gauss_pair(stream_key(P.a.seed, noise_stream(st, P.nb_first + b)), jp, &n0, &n1);
  float* dst = P.noise + P.nb_off[b] + 2 * jp;
  dst[0] = n0;
  if (2 * jp + 1 < P.nb_size[b]) dst[1] = n1;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(32 * kWarps) mlp_kernel(const Params P) {
  // per warp: the input and every layer's output (kept for the relu masks)
  __shared__ float act[kWarps][kMaxLayers + 1][kMaxWidth];
  __shared__ float grad[kWarps][2][kMaxWidth];
  extern __shared__ float wsm[];  // all parameters (a few K floats)
  asm volatile("griddepcontrol.launch_dependents;");
  const int ex_ctas = (int)gridDim.x - P.noise_ctas;
  if ((int)blockIdx.x >= ex_ctas) {
    draw_noise(P, (int)blockIdx.x - ex_ctas);
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * kWarps + warp;
  // stage the parameters: every load in flight at once instead of one cold
  // L1 miss per weight row in the dependent FMA chains below
  for (int j = threadIdx.x; j < P.P; j += 32 * kWarps) wsm[j] = __ldg(P.params + P.stage_off + j);
  __syncthreads();
  if (i >= P.B) return;  // warp-level work only: no CTA barriers below
  float(*A)[kMaxWidth] = act[warp];
  const int in0 = P.L[0].in;
  const float* X = P.x;
  const float* Y = P.y;
  if (P.xring) {
    const long long st = *P.step_base + P.step_off - P.ring_origin;
    long long bi = st % P.ring_n;
    if (bi < 0) bi += P.ring_n;
    X = P.xring + bi * P.B * in0;
    Y = P.yring + bi * P.B;
  }
  for (int k = lane; k < in0; k += 32) {
    const float v = __ldg(X + (size_t)i * in0 + k);
    A[0][k] = v;
    if (P.xin) P.xin[(size_t)i * in0 + k] = v;
  }
  __syncwarp();

  // ---- forward: z = a W + b (ascending k), relu fused ----------------------
  double asq[kMaxLayers];
#pragma unroll
  for (int l = 0; l < kMaxLayers; ++l) {
    if (l >= P.n) break;
    const DenseLayer& L = P.L[l];
    double s = 0.0;
    for (int k = lane; k < L.in; k += 32) s += (double)A[l][k] * A[l][k];
    asq[l] = warp_sum_d(s);
    const float* W = wsm + L.offW;
    for (int c = lane; c < L.out; c += 32) {
      float acc = 0.0f;
#pragma unroll 8
      for (int k = 0; k < L.in; ++k) acc = fmaf(A[l][k], W[k * L.out + c], acc);
      float v = acc + wsm[L.offb + c];
      if (L.relu) v = fmaxf(v, 0.0f);
      A[l + 1][c] = v;
      L.act[(size_t)i * L.out + c] = v;
    }
    __syncwarp();
  }

  // ---- loss and dlogits (xent_kernel semantics) ---------------------------
  const DenseLayer& T = P.L[P.n - 1];
  const int K = P.classes;
  const float* z = A[P.n];
  float* g = grad[warp][0];
  const float raw = __ldg(Y + i);
  const int Kc = K == 1 ? 2 : K;
  if (!valid_id(raw, Kc)) {
    if (lane == 0) {
      raise_index(P.err, 0, i, raw, Kc);
      P.loss[i] = 0.0f;
    }
    for (int c = lane; c < K; c += 32) g[c] = 0.0f;
  } else {
    const int yv = (int)raw;
    if (K == 1) {
      if (lane == 0) {
        const float zz = z[0], az = fabsf(zz);
        P.loss[i] = (zz > 0.0f ? zz : 0.0f) - zz * float(yv) + log1pf(expf(-az));
        g[0] = 1.0f / (1.0f + expf(-zz)) - float(yv);
      }
    } else {
      const float zl = lane < K ? z[lane] : -INFINITY;
      float m = zl;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      const float e = lane < K ? expf(zl - m) : 0.0f;
      float se = e;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
      if (lane == 0) P.loss[i] = m + logf(se) - z[yv];
      if (lane < K) g[lane] = e * (1.0f / se) - (lane == yv ? 1.0f : 0.0f);
    }
  }
  __syncwarp();
  for (int c = lane; c < K; c += 32) T.gout[(size_t)i * K + c] = g[c];

  // ---- backward: dX = G W^T (ascending c), relu mask of the layer below;
  // ghost norms of each dense block on the way ------------------------------
  int cur = 0;
#pragma unroll
  for (int l = kMaxLayers - 1; l >= 0; --l) {
    if (l >= P.n) continue;
    const DenseLayer& L = P.L[l];
    const float* gl = grad[warp][cur];
    double s = 0.0;
    for (int c = lane; c < L.out; c += 32) s += (double)gl[c] * gl[c];
    const double dsq = warp_sum_d(s);
    if (lane == 0) {
      P.parts[(size_t)i * P.nparts + L.pW] = asq[l] * dsq;
      P.parts[(size_t)i * P.nparts + L.pb] = dsq;
    }
    if (l == 0 && !P.gin) break;
    float* gn = grad[warp][cur ^ 1];
    const bool relu_below = l > 0 && P.L[l > 0 ? l - 1 : 0].relu;
    float* gdst = l > 0 ? P.L[l > 0 ? l - 1 : 0].gout : P.gin;
    for (int k = lane; k < L.in; k += 32) {
      const float* w = wsm + L.offW + k * L.out;
      float acc = 0.0f;
#pragma unroll 8
      for (int c = 0; c < L.out; ++c) acc = fmaf(gl[c], w[c], acc);
      const float v = (relu_below && !(A[l][k] > 0.0f)) ? 0.0f : acc;
      gn[k] = v;
      gdst[(size_t)i * L.in + k] = v;
    }
    if (l == 0) break;
    __syncwarp();
    cur ^= 1;
  }
}

}  // namespace mlp
}  // namespace pgb
