// sm_100a kernels of the DPSGD step (fp32 CUDA-core path).
//
// Each kernel names the reference computation it replaces. Layout is the
// reference's: NCHW activations, (in,out) dense weights, (D,C,k,k) conv
// weights, block-major per-example stacks (block p is (B, |p|)).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pgb_internal.h"
#include "trace.cuh"

namespace pgb {

constexpr int kMaxBlocks = PGB_MAX_PARAMS;

// Device-side index errors (checked_id, kernels.hpp:475-489). The reference
// throws at the first bad value in its own loop order -- the embedding gather
// of the forward before the loss's labels, each in ascending position -- so
// the device keeps the error with the smallest (kind, position) key, whatever
// order the threads find them in: one 64-bit atomicMax on the complemented
// key (order bit, position, value bits), which also carries the offending
// value. The step's update kernel refuses to write parameters once code is
// set (the reference throws before apply_update).
struct DevError {
  int code;        // pgb_status, 0 = none
  int limit_label; // classes of the softmax_xent label check
  int limit_id;    // rows of the embedding gather
  int pad;
  unsigned long long inv_key;  // ~((label ? 1 : 0) << 62 | pos << 32 | value bits)
};

__device__ __forceinline__ void raise_index(DevError* e, int what, long long pos, float v,
                                            int limit) {
  const unsigned long long p = (unsigned long long)min(max(pos, 0ll), (1ll << 30) - 1);
  const unsigned long long key =
      ((unsigned long long)(what == 0 ? 1 : 0) << 62) | (p << 32) | __float_as_uint(v);
  atomicMax(&e->inv_key, ~key);
  if (what == 0) e->limit_label = limit;
  else e->limit_id = limit;
  atomicExch(&e->code, PGB_ERR_INDEX);
}

// Packed fp32 FMA (sm_100 FFMA2): {a0, a1} += w * {x0, x1}, each lane of the
// pair rounded exactly like fmaf. ptxas folds the scalar w into a broadcast
// operand, so one instruction does two fused multiply-adds.
__device__ __forceinline__ void ffma2(float& a0, float& a1, float w, float x0, float x1) {
  unsigned long long acc, xx, ww;
  asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(xx) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(ww) : "f"(w));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(ww), "l"(xx));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(acc));
}
// {a0, a1} += {w0, w1} * x
__device__ __forceinline__ void ffma2v(float& a0, float& a1, float w0, float w1, float x) {
  ffma2(a0, a1, x, w0, w1);
}
// {a0, a1} += {x0, x1} * {y0, y1} (element-wise)
__device__ __forceinline__ void ffma2pp(float& a0, float& a1, float x0, float x1, float y0,
                                        float y1) {
  unsigned long long acc, xx, yy;
  asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(xx) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(yy) : "f"(y0), "f"(y1));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(xx), "l"(yy));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(acc));
}

// checked_id (kernels.hpp:475-489): integral and within [0, V).
__device__ __forceinline__ bool valid_id(float raw, int V) {
  return raw == rintf(raw) && raw >= 0.0f && raw < float(V);
}

// ---------------------------------------------------------------------------
// Generic register-tiled SGEMM: C[z][m][n] = sum_k A(z,m,k) B(z,k,n).
// Operand gathers and the epilogue are supplied by Op, which is how the
// implicit-im2col convolutions, the transposed convolution (backward data)
// and the per-example weight-gradient GEMMs share one tile engine.
// ---------------------------------------------------------------------------
template <class Op, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    tile_gemm_kernel(Op op) {
  constexpr int NT = (BM / TM) * (BN / TN);
  __shared__ __align__(16) float As[BK][BM];
  __shared__ __align__(16) float Bs[BK][BN];
  const int z = blockIdx.z;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  const int M = op.M, N = op.N, K = op.K;
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

  for (int k0 = 0; k0 < K; k0 += BK) {
    for (int e = tid; e < BM * BK; e += NT) {
      const int mm = e / BK, kk = e % BK;
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? op.a(z, m, k) : 0.0f;
    }
    for (int e = tid; e < BK * BN; e += NT) {
      const int kk = e / BN, nn = e % BN;
      const int n = n0 + nn, k = k0 + kk;
      Bs[kk][nn] = (n < N && k < K) ? op.b(z, k, n) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[kk][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[kk][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + ty * TM + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + tx * TN + j;
      if (n < N) op.store(z, m, n, acc[i][j]);
    }
  }
}

// ---- operand adapters -----------------------------------------------------

// dense forward (models.cpp:182-196): z = x W + b, optional fused relu.
struct DenseFwdOp {
  int M, N, K;  // M = B, N = out, K = in
  const float* x;
  const float* W;
  const float* bias;
  float* out;
  int relu;
  __device__ float a(int, int m, int k) const { return x[(size_t)m * K + k]; }
  __device__ float b(int, int k, int n) const { return W[(size_t)k * N + n]; }
  __device__ void store(int, int m, int n, float v) const {
    v += bias[n];
    out[(size_t)m * N + n] = relu ? fmaxf(v, 0.0f) : v;
  }
};

// dense input gradient (autodiff.cpp:155-159): dX = G W^T; the relu VJP of an
// upstream relu (gt-mask on its output, autodiff.cpp:121-124) is fused.
struct DenseBwdXOp {
  int M, N, K;  // M = B, N = in, K = out
  const float* g;
  const float* W;
  const float* mask;  // relu output, or null
  float* gx;
  __device__ float a(int, int m, int k) const { return g[(size_t)m * K + k]; }
  __device__ float b(int, int k, int n) const { return W[(size_t)n * K + k]; }
  __device__ void store(int, int m, int n, float v) const {
    const size_t i = (size_t)m * N + n;
    gx[i] = (mask && !(mask[i] > 0.0f)) ? 0.0f : v;
  }
};

struct ConvGeom {
  int C, H, W, D, Ho, Wo, k, stride, pad;
};

// conv forward as implicit-im2col GEMM (models.cpp:197-220; im2col rows
// ordered (c,u,v), kernels.hpp:412-440): M = D, N = B*Ho*Wo, K = C*k*k.
struct ConvFwdOp {
  int M, N, K;
  ConvGeom g;
  const float* x;
  const float* W;
  const float* bias;
  float* out;
  int relu;
  __device__ float a(int, int m, int k) const { return W[(size_t)m * K + k]; }
  __device__ float b(int, int k, int n) const {
    const int P = g.Ho * g.Wo;
    const int bb = n / P, p = n - bb * P;
    const int oy = p / g.Wo, ox = p - oy * g.Wo;
    const int kk2 = g.k * g.k;
    const int c = k / kk2, r = k - c * kk2;
    const int u = r / g.k, v = r - u * g.k;
    const int iy = oy * g.stride + u - g.pad, ix = ox * g.stride + v - g.pad;
    if (iy < 0 || iy >= g.H || ix < 0 || ix >= g.W) return 0.0f;
    return x[(((size_t)bb * g.C + c) * g.H + iy) * g.W + ix];
  }
  __device__ void store(int, int m, int n, float v) const {
    const int P = g.Ho * g.Wo;
    const int bb = n / P, p = n - bb * P;
    v += bias[m];
    out[((size_t)bb * g.D + m) * P + p] = relu ? fmaxf(v, 0.0f) : v;
  }
};

// conv input gradient (im2col VJP = col2im of W^T G, autodiff.cpp:186-192),
// written as a gather so no output element is accumulated by two threads:
// M = C, N = B*H*W, K = D*k*k.
struct ConvBwdXOp {
  int M, N, K;
  ConvGeom g;
  const float* gout;  // (B, D, Ho, Wo)
  const float* W;
  const float* mask;  // relu output of the input activation, or null
  float* gx;
  __device__ float a(int, int m, int k) const {
    const int kk2 = g.k * g.k;
    const int d = k / kk2, r = k - d * kk2;
    return W[((size_t)d * g.C + m) * kk2 + r];
  }
  __device__ float b(int, int k, int n) const {
    const int HW = g.H * g.W;
    const int bb = n / HW, q = n - bb * HW;
    const int iy = q / g.W, ix = q - iy * g.W;
    const int kk2 = g.k * g.k;
    const int d = k / kk2, r = k - d * kk2;
    const int u = r / g.k, v = r - u * g.k;
    const int ny = iy + g.pad - u, nx = ix + g.pad - v;
    if (ny < 0 || nx < 0) return 0.0f;
    const int oy = ny / g.stride, ox = nx / g.stride;
    if (oy * g.stride != ny || ox * g.stride != nx || oy >= g.Ho || ox >= g.Wo) return 0.0f;
    return gout[(((size_t)bb * g.D + d) * g.Ho + oy) * g.Wo + ox];
  }
  __device__ void store(int, int m, int n, float v) const {
    const int HW = g.H * g.W;
    const int bb = n / HW, q = n - bb * HW;
    const size_t i = ((size_t)bb * g.C + m) * HW + q;
    gx[i] = (mask && !(mask[i] > 0.0f)) ? 0.0f : v;
  }
};

// per-example conv weight gradient (strategies.cpp:156-170):
// dW_z = dz_z (D x P) . patches_z^T (P x CKK), one GEMM per example z.
struct ConvDWOp {
  int M, N, K;  // M = D, N = C*k*k, K = Ho*Wo
  ConvGeom g;
  const float* gout;  // (B, D, Ho, Wo)
  const float* x;     // (B, C, H, W)
  float* stack;       // (B, D*C*k*k)
  __device__ float a(int z, int m, int k) const {
    return gout[((size_t)z * g.D + m) * K + k];
  }
  __device__ float b(int z, int k, int n) const {
    const int oy = k / g.Wo, ox = k - oy * g.Wo;
    const int kk2 = g.k * g.k;
    const int c = n / kk2, r = n - c * kk2;
    const int u = r / g.k, v = r - u * g.k;
    const int iy = oy * g.stride + u - g.pad, ix = ox * g.stride + v - g.pad;
    if (iy < 0 || iy >= g.H || ix < 0 || ix >= g.W) return 0.0f;
    return x[(((size_t)z * g.C + c) * g.H + iy) * g.W + ix];
  }
  __device__ void store(int z, int m, int n, float v) const {
    stack[(size_t)z * M * N + (size_t)m * N + n] = v;
  }
};

// ---- per-example dense gradients (strategies.cpp:149-154) -----------------
// dW_i = a_i (x) d_i into stack (B, in*out); db_i = d_i into (B, out).
__global__ void dense_pex_kernel(const float* __restrict__ act, const float* __restrict__ g,
                                 int B, int in, int out, float* __restrict__ sW,
                                 float* __restrict__ sb) {
  const size_t per = (size_t)in * out;
  const size_t total = (size_t)B * per;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
       e += (size_t)gridDim.x * blockDim.x) {
    const size_t b = e / per, r = e - b * per;
    const int i = (int)(r / out), o = (int)(r - (size_t)i * out);
    sW[e] = act[b * in + i] * g[b * out + o];
  }
  if (sb)
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < (size_t)B * out;
         e += (size_t)gridDim.x * blockDim.x)
      sb[e] = g[e];
}

// per-example conv bias gradient: db_i[d] = sum_P dz_i[d, :] (strategies.cpp:168)
__global__ void conv_db_pex_kernel(const float* __restrict__ g, int BD, int P,
                                   float* __restrict__ sb) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= BD) return;
  const float* row = g + (size_t)warp * P;
  float s = 0.0f;
  for (int p = lane; p < P; p += 32) s += row[p];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) sb[warp] = s;
}

// ---- parameter-free layers ----------------------------------------------------

// flat index e of a (BC, H, W) tensor -> (bc, y, x); 32-bit divisions when
// the tensor allows (64-bit division is a long instruction sequence and was
// the bound of the pooling kernels)
__device__ __forceinline__ void split_bchw(size_t e, int H, int W, size_t& bc, int& y, int& x,
                                           bool small) {
  if (small) {
    const unsigned ee = (unsigned)e, hw = (unsigned)(H * W);
    const unsigned b = ee / hw, r = ee - b * hw;
    const unsigned yy = r / (unsigned)W;
    bc = b;
    y = (int)yy;
    x = (int)(r - yy * (unsigned)W);
  } else {
    x = (int)(e % W);
    y = (int)((e / W) % H);
    bc = e / ((size_t)W * H);
  }
}

// max/avg pooling via window reduction (tape.cpp:269-282): avg = sum * 1/k^2.
__global__ void pool_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, int BC,
                                int H, int W, int Ho, int Wo, int k, int s, int is_max) {
  const size_t total = (size_t)BC * Ho * Wo;
  const bool small = total < (1ull << 31);
  const float inv = 1.0f / float(k * k);
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
       e += (size_t)gridDim.x * blockDim.x) {
    size_t bc;
    int oy, ox;
    split_bchw(e, Ho, Wo, bc, oy, ox, small);
    const float* xp = x + bc * H * W;
    float m = 0.0f, sum = 0.0f;
    bool first = true;
    for (int u = 0; u < k; ++u)
      for (int v = 0; v < k; ++v) {
        const float val = xp[(oy * s + u) * W + ox * s + v];
        sum += val;
        if (first || val > m) m = val;
        first = false;
      }
    y[e] = is_max ? m : sum * inv;
  }
}

// pool backward as a gather over the windows containing each input element;
// max routes to the FIRST maximum in window order (kernels.hpp:377-396).
__global__ void pool_bwd_kernel(const float* __restrict__ x, const float* __restrict__ g,
                                const float* __restrict__ mask, float* __restrict__ gx,
                                int BC, int H, int W, int Ho, int Wo, int k, int s,
                                int is_max) {
  const size_t total = (size_t)BC * H * W;
  const bool small = total < (1ull << 31);
  const float inv = 1.0f / float(k * k);
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
       e += (size_t)gridDim.x * blockDim.x) {
    size_t bc;
    int iy, ix;
    split_bchw(e, H, W, bc, iy, ix, small);
    const float* xp = x + bc * H * W;
    const float* gp = g + bc * Ho * Wo;
    float acc = 0.0f;
    const int oy_lo = iy >= k ? (iy - k) / s + 1 : 0, oy_hi = min(iy / s, Ho - 1);
    const int ox_lo = ix >= k ? (ix - k) / s + 1 : 0, ox_hi = min(ix / s, Wo - 1);
    for (int oy = oy_lo; oy <= oy_hi; ++oy)
      for (int ox = ox_lo; ox <= ox_hi; ++ox) {
        if (oy * s > iy || iy >= oy * s + k || ox * s > ix || ix >= ox * s + k) continue;
        if (is_max) {
          int best_u = 0, best_v = 0;
          float bv = xp[(oy * s) * W + ox * s];
          for (int u = 0; u < k; ++u)
            for (int v = 0; v < k; ++v) {
              const float val = xp[(oy * s + u) * W + ox * s + v];
              if (val > bv) {
                bv = val;
                best_u = u;
                best_v = v;
              }
            }
          if (oy * s + best_u == iy && ox * s + best_v == ix) acc += gp[oy * Wo + ox];
        } else {
          acc += gp[oy * Wo + ox] * inv;
        }
      }
    gx[e] = (mask && !(mask[e] > 0.0f)) ? 0.0f : acc;
  }
}

// 3x3 / stride 1 / pad 1 convolution of a few-channel input (the CIFAR
// first layer, C = 3) directly on the CUDA cores in fp32
// (models.cpp:197-220 computes the same sum as an im2col GEMM): a 27-tap
// sum per output is too short for the tensor cores to pay for the im2col
// gather. One thread = 4 consecutive outputs of a row, all D channels in
// groups of 16 (64 accumulators); its 3 x 6 input window per channel sits in
// registers, the weights ([tap][d], 16-byte broadcast loads) in shared memory.
// Bias and ReLU fused; out NCHW, float4 stores.
template <int C>
__global__ void __launch_bounds__(256) conv3x3_smallc_fwd_kernel(
    const float* __restrict__ x, const float* __restrict__ Wt, const float* __restrict__ bias,
    float* __restrict__ out, int B, int D, int H, int W, int relu) {
  extern __shared__ float sw[];  // [C * 9][D] then bias[D]
  for (int e = threadIdx.x; e < C * 9 * D; e += blockDim.x) {
    const int d = e / (C * 9), k = e - d * (C * 9);
    sw[k * D + d] = Wt[e];
  }
  for (int d = threadIdx.x; d < D; d += blockDim.x) sw[C * 9 * D + d] = bias[d];
  __syncthreads();
  const int W4 = W >> 2;
  const long long total = (long long)B * H * W4;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int xq = (int)(t % W4);
    const long long r = t / W4;
    const int y = (int)(r % H), n = (int)(r / H);
    const int x0 = xq * 4;
    float xw[C][3][6];
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int yy = y + u - 1;
        const bool rowok = yy >= 0 && yy < H;
        const float* row = x + (((size_t)n * C + c) * H + (rowok ? yy : 0)) * W;
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          const int xx = x0 - 1 + j;
          xw[c][u][j] = (rowok && xx >= 0 && xx < W) ? __ldg(row + xx) : 0.0f;
        }
      }
    for (int d0 = 0; d0 < D; d0 += 16) {
      float acc[16][4];
#pragma unroll
      for (int dd = 0; dd < 16; ++dd) {
        const float b = sw[C * 9 * D + d0 + dd];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[dd][i] = b;
      }
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int u = 0; u < 3; ++u)
#pragma unroll
          for (int v = 0; v < 3; ++v) {
            const float4* wk = reinterpret_cast<const float4*>(sw + (c * 9 + u * 3 + v) * D + d0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 w4 = wk[q];
              const float wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
              for (int e = 0; e < 4; ++e)
#pragma unroll
                for (int i = 0; i < 4; ++i)
                  acc[q * 4 + e][i] = fmaf(wv[e], xw[c][u][i + v], acc[q * 4 + e][i]);
            }
          }
#pragma unroll
      for (int dd = 0; dd < 16; ++dd) {
        float4 o = make_float4(acc[dd][0], acc[dd][1], acc[dd][2], acc[dd][3]);
        if (relu) {
          o.x = fmaxf(o.x, 0.0f);
          o.y = fmaxf(o.y, 0.0f);
          o.z = fmaxf(o.z, 0.0f);
          o.w = fmaxf(o.w, 0.0f);
        }
        *reinterpret_cast<float4*>(out + (((size_t)n * D + d0 + dd) * H + y) * W + x0) = o;
      }
    }
  }
}

// 2x2 windows with stride 2 tiling the input (H = 2 Ho, W = 2 Wo: every input
// element in exactly one window) -- the CIFAR pools. One thread per window,
// 8-byte row loads/stores; the same fp32 operations as pool_fwd_kernel /
// pool_bwd_kernel (window order (0,0), (0,1), (1,0), (1,1); first max).
__global__ void pool2_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, int BC,
                                 int Ho, int Wo, int is_max) {
  const unsigned total = (unsigned)BC * Ho * Wo;
  const int W = 2 * Wo;
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += gridDim.x * blockDim.x) {
    const unsigned ox = e % Wo, t = e / Wo, oy = t % Ho, bc = t / Ho;
    const size_t base = ((size_t)bc * 2 * Ho + 2 * oy) * W + 2 * ox;
    const float2 r0 = *reinterpret_cast<const float2*>(x + base);
    const float2 r1 = *reinterpret_cast<const float2*>(x + base + W);
    float out;
    if (is_max) {
      float m = r0.x;
      if (r0.y > m) m = r0.y;
      if (r1.x > m) m = r1.x;
      if (r1.y > m) m = r1.y;
      out = m;
    } else {
      float s = __fadd_rn(0.0f, r0.x);
      s = __fadd_rn(s, r0.y);
      s = __fadd_rn(s, r1.x);
      s = __fadd_rn(s, r1.y);
      out = __fmul_rn(s, 0.25f);
    }
    y[e] = out;
  }
}

__global__ void pool2_bwd_kernel(const float* __restrict__ x, const float* __restrict__ g,
                                 const float* __restrict__ mask, float* __restrict__ gx, int BC,
                                 int Ho, int Wo, int is_max) {
  const unsigned total = (unsigned)BC * Ho * Wo;
  const int W = 2 * Wo;
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += gridDim.x * blockDim.x) {
    const unsigned ox = e % Wo, t = e / Wo, oy = t % Ho, bc = t / Ho;
    const size_t base = ((size_t)bc * 2 * Ho + 2 * oy) * W + 2 * ox;
    const float gv = g[e];
    float o[4];
    if (is_max) {
      const float2 r0 = *reinterpret_cast<const float2*>(x + base);
      const float2 r1 = *reinterpret_cast<const float2*>(x + base + W);
      const float v[4] = {r0.x, r0.y, r1.x, r1.y};
      int best = 0;
      float bv = v[0];
#pragma unroll
      for (int q = 1; q < 4; ++q)
        if (v[q] > bv) {
          bv = v[q];
          best = q;
        }
#pragma unroll
      for (int q = 0; q < 4; ++q) o[q] = q == best ? __fadd_rn(0.0f, gv) : 0.0f;
    } else {
      const float a = __fadd_rn(0.0f, __fmul_rn(gv, 0.25f));
#pragma unroll
      for (int q = 0; q < 4; ++q) o[q] = a;
    }
    if (mask) {
      const float2 m0 = *reinterpret_cast<const float2*>(mask + base);
      const float2 m1 = *reinterpret_cast<const float2*>(mask + base + W);
      if (!(m0.x > 0.0f)) o[0] = 0.0f;
      if (!(m0.y > 0.0f)) o[1] = 0.0f;
      if (!(m1.x > 0.0f)) o[2] = 0.0f;
      if (!(m1.y > 0.0f)) o[3] = 0.0f;
    }
    *reinterpret_cast<float2*>(gx + base) = make_float2(o[0], o[1]);
    *reinterpret_cast<float2*>(gx + base + W) = make_float2(o[2], o[3]);
  }
}

// global average pool (models.cpp:227-232): sum over H,W then * 1/(H*W)
__global__ void gap_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, int BC,
                               int HW) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= BC) return;
  float s = 0.0f;
  for (int j = lane; j < HW; j += 32) s += x[(size_t)warp * HW + j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[warp] = s * (1.0f / float(HW));
}

__global__ void gap_bwd_kernel(const float* __restrict__ g, const float* __restrict__ mask,
                               float* __restrict__ gx, int BC, int HW) {
  const size_t total = (size_t)BC * HW;
  const float inv = 1.0f / float(HW);
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
       e += (size_t)gridDim.x * blockDim.x) {
    const float v = g[e / HW] * inv;
    gx[e] = (mask && !(mask[e] > 0.0f)) ? 0.0f : v;
  }
}

__global__ void relu_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, size_t n) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x)
    y[e] = fmaxf(x[e], 0.0f);
}

__global__ void mask_kernel(const float* __restrict__ g, const float* __restrict__ mask,
                            float* __restrict__ gx, size_t n) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x)
    gx[e] = mask[e] > 0.0f ? g[e] : 0.0f;
}

// embedding gather fused with the sequence mean-pool (models.cpp:241-262):
// y[b,e] = (sum_t table[id_bt, e]) * 1/L. Ids validated (checked_id).
constexpr int kPoolMaxL = 2048;
constexpr int kPoolGroups = 4;   // token groups per example (partial sums)
constexpr int kPoolMaxE = 1024;  // widths whose partial sums are staged in shared memory

__global__ void embed_pool_fwd_kernel(const float* __restrict__ ids,
                                      const float* __restrict__ table, float* __restrict__ y,
                                      int B, int L, int E, int V, DevError* err) {
  const int b = blockIdx.x;
  if (L > kPoolMaxL) {  // long sequences: the plain loop
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      float s = 0.0f;
      for (int t = 0; t < L; ++t) {
        const float raw = ids[(size_t)b * L + t];
        if (!valid_id(raw, V)) {
          if (e == 0) raise_index(err, 1, (long long)b * L + t, raw, V);
          continue;
        }
        s += table[(size_t)(int)raw * E + e];
      }
      y[(size_t)b * E + e] = s * (1.0f / float(L));
    }
    return;
  }
  // the example's ids once (validated); then the threads split into G groups
  // of ew (>= E) lanes, group g summing tokens [g L / G, (g + 1) L / G) in
  // order with 16 row gathers in flight, the G partial sums added in group
  // order (fp32 re-association of the reference's single chain,
  // models.cpp:241-262: within the parity tolerance)
  __shared__ int sid[kPoolMaxL];
  __shared__ float part[kPoolGroups][kPoolMaxE];
  for (int t = threadIdx.x; t < L; t += blockDim.x) {
    const float raw = ids[(size_t)b * L + t];
    const bool ok = valid_id(raw, V);
    if (!ok) raise_index(err, 1, (long long)b * L + t, raw, V);
    sid[t] = ok ? (int)raw : -1;
  }
  __syncthreads();
  const int ew = ((E + 31) / 32) * 32;
  const int G = E <= kPoolMaxE ? max(1, min(kPoolGroups, (int)blockDim.x / ew)) : 1;
  const int g = threadIdx.x / ew, e = threadIdx.x - g * ew;
  if (g < G && e < E) {
    const int t0 = (int)((long long)L * g / G), t1 = (int)((long long)L * (g + 1) / G);
    float s = 0.0f;
    int t = t0;
    for (; t + 16 <= t1; t += 16) {
      float v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int r = sid[t + q];
        v[q] = r >= 0 ? __ldg(table + (size_t)r * E + e) : 0.0f;
      }
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (sid[t + q] >= 0) s += v[q];
    }
    for (; t < t1; ++t)
      if (sid[t] >= 0) s += __ldg(table + (size_t)sid[t] * E + e);
    if (G > 1) part[g][e] = s;
    else y[(size_t)b * E + e] = s * (1.0f / float(L));
  }
  if (G > 1) {
    __syncthreads();
    for (int e2 = threadIdx.x; e2 < E; e2 += blockDim.x) {
      float s = part[0][e2];
      for (int q = 1; q < G; ++q) s += part[q][e2];
      y[(size_t)b * E + e2] = s * (1.0f / float(L));
    }
  }
}

// embed_pool_fwd_kernel for E % 4 == 0, E <= 128 and a 16-byte aligned
// table: one warp per token group, lane l holding elements 4l..4l+3 (one
// 16-byte gather per token), 16 groups of L/16 tokens, the group partials
// added in group order (the same fp32
// re-association class as embed_pool_fwd_kernel's four groups).
constexpr int kPool4Groups = 16;
__global__ void __launch_bounds__(32 * kPool4Groups, 3) embed_pool4_fwd_kernel(
    const float* __restrict__ ids, const float* __restrict__ table, float* __restrict__ y,
    int B, int L, int E, int V, DevError* err) {
  __shared__ int sid[kPoolMaxL];
  __shared__ float4 part[kPool4Groups][32];
  const int b = blockIdx.x, t = threadIdx.x, g = t >> 5, lane = t & 31;
  for (int k = t; k < L; k += blockDim.x) {
    const float raw = ids[(size_t)b * L + k];
    const bool ok = valid_id(raw, V);
    if (!ok) raise_index(err, 1, (long long)b * L + k, raw, V);
    sid[k] = ok ? (int)raw : -1;
  }
  __syncthreads();
  const int e0 = 4 * lane;
  const bool act = e0 < E;
  const int t0 = (int)((long long)L * g / kPool4Groups), t1 = (int)((long long)L * (g + 1) / kPool4Groups);
  float4 s = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  // 8 gathers in flight per lane keeps the kernel at <= 40 registers: three
  // 512-thread CTAs per SM (one wave for B = 512; 16 in flight at ~100
  // registers allowed one CTA per SM and 3.5 waves)
  for (int k = t0; k < t1; k += 8) {
    float4 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = k + q < t1 ? sid[k + q] : -1;
      v[q] = (act && r >= 0) ? __ldg(reinterpret_cast<const float4*>(table + (size_t)r * E + e0))
                             : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (k + q < t1 && sid[k + q] >= 0) {
        s.x += v[q].x;
        s.y += v[q].y;
        s.z += v[q].z;
        s.w += v[q].w;
      }
  }
  part[g][lane] = s;
  __syncthreads();
  if (g == 0 && act) {
    float4 a = part[0][lane];
#pragma unroll
    for (int q = 1; q < kPool4Groups; ++q) {
      const float4 c = part[q][lane];
      a.x += c.x;
      a.y += c.y;
      a.z += c.z;
      a.w += c.w;
    }
    const float inv = 1.0f / float(L);
    *reinterpret_cast<float4*>(y + (size_t)b * E + e0) =
        make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv);
  }
}

// per-example dense table gradient (strategies.cpp:171-188): the pooled
// cotangent times 1/L scattered to each token's row, tokens in order.
__global__ void embed_pex_kernel(const float* __restrict__ ids, const float* __restrict__ g,
                                 int B, int L, int E, int V, float* __restrict__ stack) {
  const int b = blockIdx.x;
  float* tb = stack + (size_t)b * V * E;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const float v = g[(size_t)b * E + e] * (1.0f / float(L));
    for (int t = 0; t < L; ++t) {
      const float raw = ids[(size_t)b * L + t];
      if (!valid_id(raw, V)) continue;
      tb[(size_t)(int)raw * E + e] += v;
    }
  }
}

// softmax cross-entropy + its gradient per example (kernels.hpp:516-566);
// the loss is a SUM over examples so the cotangent of each loss_i is 1.
__global__ void xent_kernel(const float* __restrict__ logits, const float* __restrict__ labels,
                            int B, int K, float* __restrict__ loss, float* __restrict__ dlogits,
                            DevError* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  const float raw = labels[i];
  const int Kc = K == 1 ? 2 : K;
  const float* z = logits + (size_t)i * K;
  float* d = dlogits + (size_t)i * K;
  if (!valid_id(raw, Kc)) {
    raise_index(err, 0, i, raw, Kc);
    for (int k = 0; k < K; ++k) d[k] = 0.0f;
    loss[i] = 0.0f;
    return;
  }
  const int y = (int)raw;
  if (K == 1) {
    const float zz = z[0], az = fabsf(zz);
    loss[i] = (zz > 0.0f ? zz : 0.0f) - zz * float(y) + log1pf(expf(-az));
    d[0] = 1.0f / (1.0f + expf(-zz)) - float(y);
    return;
  }
  float m = z[0];
  for (int k = 1; k < K; ++k) m = fmaxf(m, z[k]);
  float s = 0.0f;
  for (int k = 0; k < K; ++k) s += expf(z[k] - m);
  loss[i] = m + logf(s) - z[y];
  const float inv = 1.0f / s;
  for (int k = 0; k < K; ++k) d[k] = expf(z[k] - m) * inv - (k == y ? 1.0f : 0.0f);
}

// ---- norms, clip, clipped sum, noise, update ---------------------------------

// Where each parameter block's per-example gradient rows live. kind 0: a
// materialised row g_i = base[i*stride + j]; kind 1: a dense-layer weight
// block kept factored (ghost representation, strategies.cpp:140-154):
// g_i[r*out + c] = fl(a[i*a_stride + r] * base[i*stride + c]) -- exactly the
// fp32 element of the reference's per-example outer-product stack.
struct BlockTable {
  int n;
  long long size[kMaxBlocks];       // |p|
  long long param_off[kMaxBlocks];  // offset in the flat parameter vector
  long long pair_off[kMaxBlocks + 1];  // prefix sum of ceil(|p|/2)
  int kind[kMaxBlocks];
  const float* base[kMaxBlocks];
  long long stride[kMaxBlocks];
  const float* a[kMaxBlocks];
  long long a_stride[kMaxBlocks];
  int out[kMaxBlocks];
  // optional transposed copy of the parameter block kept in step with the
  // update (row-major (rows, cols) block -> shadow[c * rows + r])
  float* shadow[kMaxBlocks];
  int shadow_rows[kMaxBlocks];
  int shadow_swz[kMaxBlocks];  // XOR swizzle mask (0: plain transpose)
  // optional hi/lo tensor-core operand copies (mnist_tc.cuh): 1 conv1 W, 2 conv2 W
  float* tcw[kMaxBlocks];
  int tcw_kind[kMaxBlocks];
  // kind-0 blocks whose rows are already clipped sums of unit groups (the
  // MNIST kernel's conv2 pair rows): row count (0: one row per unit, scaled
  // by the unit's clip factor in the aggregation)
  int rows[kMaxBlocks];
  int norm_pre[kMaxBlocks];  // 1: per-example squared norm already in parts (sumsq skips)
};

// Per-example dW of a few-channel 3x3 / stride 1 / pad 1 convolution on a
// 32-wide map (the CIFAR first layer) on the CUDA cores in fp32: one block per
// example, lane = output column x, warp w = DPW output channels (more
// warps loop over channel groups); each thread sums its column over all rows
// into 4 x C x 9 accumulators, then a fixed xor-shuffle tree adds the 32
// columns. Input rows are staged zero-padded in shared memory and walked as a
// three-row register window (one new padded row, C x 3 loads, per output row
// instead of C x 9); each warp stages its DPW cotangent channels (DPW x H x 32
// floats, contiguous in g) in its own shared slice with every 16-byte load in
// flight at once, so no row waits on a global round trip. Writes the
// reference's stack row (D, C, 3, 3) (strategies.cpp:156-170) and the block's
// squared norm (fp64) into parts.
// per-warp slice: the staged cotangent rows, later the column-sum transpose
template <int C, int DPW>
__host__ __device__ constexpr size_t smallc_dw_slice_floats(int H) {
  return (((size_t)DPW * H * 32 > (size_t)DPW * C * 9 * 33 ? (size_t)DPW * H * 32
                                                            : (size_t)DPW * C * 9 * 33) + 3) &
         ~(size_t)3;
}
template <int C, int DPW>
__host__ __device__ constexpr size_t smallc_dw_smem_floats(int H, int nw) {
  return (((size_t)C * (H + 2) * 34 + 3) & ~(size_t)3) + (size_t)nw * smallc_dw_slice_floats<C, DPW>(H);
}

template <int C, int DPW>
__global__ void __launch_bounds__(256, 2) conv3x3_smallc_dw_kernel(
    const float* __restrict__ x, const float* __restrict__ g, float* __restrict__ stack, int D,
    int H, double* __restrict__ parts, int nparts, int pb, float* __restrict__ sb) {
  constexpr int W = 32, WP = 34, K = C * 9;
  extern __shared__ __align__(16) float xs[];  // [C][H + 2][34], zero border; then the g slices
  __shared__ double wsq[16];
  const int z = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const float* xz = x + (size_t)z * C * H * W;
  // staged in batches with every load of a batch in flight before its stores
  // (a plain copy loop would wait one global round trip per element)
  constexpr int kXB = 8;
  for (int e0 = threadIdx.x; e0 < C * (H + 2) * WP; e0 += kXB * blockDim.x) {
    float v[kXB];
#pragma unroll
    for (int q = 0; q < kXB; ++q) {
      const int e = e0 + q * blockDim.x;
      const int c = e / ((H + 2) * WP), r = e - c * (H + 2) * WP;
      const int yy = r / WP - 1, xx = r % WP - 1;
      v[q] = (e < C * (H + 2) * WP && yy >= 0 && yy < H && xx >= 0 && xx < W)
                 ? __ldg(xz + ((size_t)c * H + yy) * W + xx) : 0.0f;
    }
#pragma unroll
    for (int q = 0; q < kXB; ++q)
      if (e0 + q * blockDim.x < C * (H + 2) * WP) xs[e0 + q * blockDim.x] = v[q];
  }
  float* gs = xs + ((C * (H + 2) * WP + 3) & ~3) + (size_t)warp * smallc_dw_slice_floats<C, DPW>(H);
  __syncthreads();
  double sq = 0.0;
  for (int d0 = warp * DPW; d0 < D; d0 += nw * DPW) {
    {  // this warp's cotangent channels d0 .. d0 + DPW - 1 (zero past D)
      const int nch = min(DPW, D - d0);
      const float* src = g + ((size_t)z * D + d0) * H * W;
      const int n = nch * H * W;
      constexpr int kGB = 8;
      if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        const float4* s4 = reinterpret_cast<const float4*>(src);
        float4* d4 = reinterpret_cast<float4*>(gs);
        for (int e0 = lane; e0 < n / 4; e0 += 32 * kGB) {
          float4 r[kGB];
#pragma unroll
          for (int q = 0; q < kGB; ++q)
            if (e0 + 32 * q < n / 4) r[q] = __ldg(s4 + e0 + 32 * q);
#pragma unroll
          for (int q = 0; q < kGB; ++q)
            if (e0 + 32 * q < n / 4) d4[e0 + 32 * q] = r[q];
        }
      } else {
        for (int e = lane; e < n; e += 32) gs[e] = __ldg(src + e);
      }
      for (int e = n + lane; e < DPW * H * W; e += 32) gs[e] = 0.0f;
      __syncwarp();
      // the example's bias gradient of these channels from the staged rows,
      // with conv_db_pex_kernel's arithmetic (lane-strided partials, xor
      // butterfly): bitwise the same, and the cotangent is not read again
      for (int dd = 0; dd < nch; ++dd) {
        float sbv = 0.0f;
        for (int p = lane; p < H * W; p += 32) sbv += gs[dd * H * W + p];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sbv += __shfl_xor_sync(0xffffffffu, sbv, o);
        if (lane == 0) sb[(size_t)z * D + d0 + dd] = sbv;
      }
    }
    float acc[DPW][K];
#pragma unroll
    for (int dd = 0; dd < DPW; ++dd)
#pragma unroll
      for (int k = 0; k < K; ++k) acc[dd][k] = 0.0f;
    // padded rows y, y + 1, y + 2 of every input channel at columns lane .. lane + 2
    float xw[3][C][3];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int v = 0; v < 3; ++v) xw[u][c][v] = xs[(c * (H + 2) + u) * WP + lane + v];
    for (int y = 0; y < H; ++y) {
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int v = 0; v < 3; ++v) xw[2][c][v] = xs[(c * (H + 2) + y + 2) * WP + lane + v];
      float gv[DPW];
#pragma unroll
      for (int dd = 0; dd < DPW; ++dd) gv[dd] = gs[(dd * H + y) * W + lane];
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int u = 0; u < 3; ++u)
#pragma unroll
          for (int v = 0; v < 3; ++v) {
            const float xv = xw[u][c][v];
#pragma unroll
            for (int dd = 0; dd < DPW; ++dd)
              acc[dd][c * 9 + u * 3 + v] = fmaf(gv[dd], xv, acc[dd][c * 9 + u * 3 + v]);
          }
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int v = 0; v < 3; ++v) {
          xw[0][c][v] = xw[1][c][v];
          xw[1][c][v] = xw[2][c][v];
        }
    }
    // the 32 columns: transposed through the warp's slice (rows of 33 floats,
    // conflict-free), lane l then sums outputs l, l + 32, ... in column order
    __syncwarp();  // every lane is done reading the cotangent rows
#pragma unroll
    for (int dd = 0; dd < DPW; ++dd)
#pragma unroll
      for (int k = 0; k < K; ++k) gs[(dd * K + k) * 33 + lane] = acc[dd][k];
    __syncwarp();
    float* st = stack + ((size_t)z * D + d0) * K;
    for (int o = lane; o < DPW * K; o += 32) {
      const float* row = gs + o * 33;
      float a = 0.0f;
#pragma unroll
      for (int j = 0; j < 32; ++j) a += row[j];
      if (d0 + o / K < D) {
        st[o] = a;
        sq = fma((double)a, (double)a, sq);
      }
    }
    __syncwarp();  // every lane is done with the slice before the next group overwrites it
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if (lane == 0) wsq[warp] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += wsq[w];
    parts[(size_t)z * nparts + pb] = t;
  }
}

// parts[i * nparts + p] = the fixed-order sum of example i's tile sums
__global__ void tile_sq_reduce_kernel(const double* __restrict__ tile_sq, int tiles, int B,
                                      double* __restrict__ parts, int nparts, int p) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  double acc = 0.0;
  for (int q = 0; q < tiles; ++q) acc += tile_sq[(size_t)i * tiles + q];
  parts[(size_t)i * nparts + p] = acc;
}

// ---- hi/lo UMMA operand shadows of the MNIST conv weights (mnist_tc.cuh) ---
// float layout of one shadow buffer (hi and lo stacked along the M/N rows so
// one MMA multiplies both halves; tf32 MMAs cost a fixed ~50 cycles below
// N ~ 100, so wider instructions are nearly free):
//   [0,2048)       conv1 W: rows hl*16 + d (32), K = tap,    kmaj(., tap, 128, 512)
//   [2048,+16384)  conv2 W: rows hl*32 + d (64), K = k2,     kmaj(., k2, 128, 1024)
//   [18432,+8192)  conv2 W^T hi, then lo: rows k2 (256), K = d, kmaj(k2, d, 128, 4096)
constexpr int kTcwW1C = 0, kTcwW2C = 2048, kTcwW2T = 2048 + 2 * 8192;
constexpr int kTcwFloats = kTcwW2T + 2 * 8192;

__host__ __device__ __forceinline__ int kmaj_f(int r, int k, int sbo, int lbo) {
  return ((r & 7) * 16 + (k & 3) * 4 + (r >> 3) * sbo + (k >> 2) * lbo) >> 2;
}

// x = hi + lo with hi = rna_tf32(x) (3xTF32 operands)
__device__ __forceinline__ void tf32_split(float x, float& hi, float& lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  lo = x - hi;
}

__device__ __forceinline__ void tcw_write(float* tcw, int which, long long j, float v) {
  float hi, lo;
  tf32_split(v, hi, lo);
  if (which == 1) {  // conv1 W (16, 64)
    const int d = (int)(j >> 6), k = (int)(j & 63);
    tcw[kTcwW1C + kmaj_f(d, k, 128, 512)] = hi;
    tcw[kTcwW1C + kmaj_f(16 + d, k, 128, 512)] = lo;
  } else {  // conv2 W (32, 256)
    const int d = (int)(j >> 8), k = (int)(j & 255);
    tcw[kTcwW2C + kmaj_f(d, k, 128, 1024)] = hi;
    tcw[kTcwW2C + kmaj_f(32 + d, k, 128, 1024)] = lo;
    const int o2 = kTcwW2T + kmaj_f(k, d, 128, 4096);
    tcw[o2] = hi;
    tcw[o2 + 8192] = lo;
  }
}

// Transposed shadow of a (rows, cols) parameter block, rows a power of two:
// element (r, c) at dst[c * rows + (r ^ (c & (rows - 1)))]. The XOR swizzle
// makes both a row of the shadow (fixed c) and a column across consecutive c
// (fixed r) bank-conflict-free once the shadow is bulk-copied to shared memory.
__host__ __device__ __forceinline__ long long shadow_index(long long r, long long c, int rows,
                                                           int swz) {
  return c * rows + (r ^ (c & swz));
}

__device__ __forceinline__ void write_param(const BlockTable& bt, int p, long long j,
                                            float* params, float v) {
  params[bt.param_off[p] + j] = v;
  if (bt.shadow[p]) {
    const long long cols = bt.size[p] / bt.shadow_rows[p];
    const long long r = j / cols, c = j - r * cols;
    bt.shadow[p][shadow_index(r, c, bt.shadow_rows[p], bt.shadow_swz[p])] = v;
  }
  if (bt.tcw[p]) tcw_write(bt.tcw[p], bt.tcw_kind[p], j, v);
}

// write_param split in two: the destinations (dependent reads of the block
// table) resolved early, the stores later
struct ParamDst {
  float* p;
  float* sh;
  float* tcw;
  int tcw_kind;
};

__device__ __forceinline__ ParamDst param_dst(const BlockTable& bt, int p, long long j,
                                              float* params) {
  ParamDst d;
  d.p = params + bt.param_off[p] + j;
  d.sh = nullptr;
  if (bt.shadow[p]) {
    const long long cols = bt.size[p] / bt.shadow_rows[p];
    const long long r = j / cols, c = j - r * cols;
    d.sh = bt.shadow[p] + shadow_index(r, c, bt.shadow_rows[p], bt.shadow_swz[p]);
  }
  d.tcw = bt.tcw[p];
  d.tcw_kind = bt.tcw_kind[p];
  return d;
}

__device__ __forceinline__ void param_store(const ParamDst& d, long long j, float v) {
  *d.p = v;
  if (d.sh) *d.sh = v;
  if (d.tcw) tcw_write(d.tcw, d.tcw_kind, j, v);
}

__device__ __forceinline__ float grad_at(const BlockTable& bt, int p, long long i, long long j) {
  if (bt.kind[p] == 0) return bt.base[p][i * bt.stride[p] + j];
  const long long r = j / bt.out[p], c = j - r * bt.out[p];
  return __fmul_rn(bt.a[p][i * bt.a_stride[p] + r], bt.base[p][i * bt.stride[p] + c]);
}

__device__ __forceinline__ double block_reduce_sum(double acc, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  double v = 0.0;
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  __syncthreads();
  return v;
}

// Squared per-example norm of one parameter block, fp64 accumulation
// (sumsq_lanes, kernels.hpp:573-589) in a fixed order (deterministic). Ghost
// blocks use ||a (x) d||^2 = ||a||^2 ||d||^2. grid (n_blocks, B).
__global__ void sumsq_kernel(BlockTable bt, int B, double* __restrict__ parts) {
  __shared__ double red[32];
  const int p = blockIdx.x;
  const long long i = blockIdx.y;
  // sparse embedding (embed_index_kernel) and conv dW blocks (the dW GEMM's
  // tile sums) have their norms written elsewhere
  if (bt.kind[p] == 2 || bt.norm_pre[p]) return;
  if (bt.kind[p] == 0) {
    const long long per = bt.size[p];
    const float* row = bt.base[p] + i * bt.stride[p];
    double acc = 0.0;
    for (long long j = threadIdx.x; j < per; j += blockDim.x) {
      const double v = row[j];
      acc += v * v;
    }
    acc = block_reduce_sum(acc, red);
    if (threadIdx.x == 0) parts[i * bt.n + p] = acc;
  } else {
    const long long in = bt.size[p] / bt.out[p];
    const float* ar = bt.a[p] + i * bt.a_stride[p];
    const float* dr = bt.base[p] + i * bt.stride[p];
    double sa = 0.0, sd = 0.0;
    for (long long r = threadIdx.x; r < in; r += blockDim.x) sa += (double)ar[r] * ar[r];
    for (long long c = threadIdx.x; c < bt.out[p]; c += blockDim.x) sd += (double)dr[c] * dr[c];
    sa = block_reduce_sum(sa, red);
    sd = block_reduce_sum(sd, red);
    if (threadIdx.x == 0) parts[i * bt.n + p] = sa * sd;
  }
}

// Device step parameters, refreshed before every launch/graph replay.
struct StepArgs {
  float clip, sigma, lr;
  float inv_units;   // (float)1 / units, dpsgd.cpp:357
  unsigned long long seed;
  long long step;
  int units;         // clipped units in this step (B/m)
  int add_noise;     // sigma > 0
};

__global__ void finalize_norms_kernel(const double* __restrict__ parts, int nb, int units,
                                      float* __restrict__ norms) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= units) return;
  double acc = 0.0;
  for (int p = 0; p < nb; ++p) acc += parts[(size_t)i * nb + p];
  norms[i] = (float)sqrt(acc);
}

// Box-Muller normal pair (kernels.hpp:597-614): double precision, then cast.
__device__ __forceinline__ void gauss_pair(uint64_t key, long long pair, float* c, float* s) {
  const double two_pi = 6.283185307179586476925286766559;
  const double u1 = double((value_at(key, 2ull * pair) >> 11) + 1) * 0x1.0p-53;
  const double u2 = double((value_at(key, 2ull * pair + 1) >> 11) + 1) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  double sn, cs;
  sincos(two_pi * u2, &sn, &cs);
  *c = (float)(r * cs);
  *s = (float)(r * sn);
}

// Locate the block of a global pair index (table cached in shared memory).
__device__ __forceinline__ int find_block(const long long* pair_off, int n, long long q) {
  int p = 0;
  while (p + 1 < n && pair_off[p + 1] <= q) ++p;
  return p;
}

// Clipped sum over the units (dpsgd.cpp:287-307), then noise / mean / SGD
// update (dpsgd.cpp:308-317, apply_update :173-183) with the reference's fp32
// operation order per element: acc += fl(g_ij * s_i), acc += fl((sigma*C) * n_j),
// acc = fl(acc * (1/units)), p = fl(p - fl(lr * acc)).
//
// Work unit = one tile of one parameter block (tile table built once per
// engine and block-kind signature, see Engine::tiles_for):
//   materialised rows (kind 0): kAggCols consecutive columns; lane l owns
//     columns 4l..4l+3 (one 16-byte load per unit when aligned);
//   factored dense rows (kind 1, g_i = a_i (x) d_i): kAggRows weight rows r x
//     32 columns c; lane l owns column c0+l of every row, so one coalesced
//     load of d_i and kAggRows broadcast values of a_i feed kAggRows FMAs
//     a_ir * fl(d_ic * s_i) -- the outer-product stack is never written to
//     memory (one rounding per element fewer than the reference's order).
// A CTA of kAggWarps warps owns one tile; warp w sums a contiguous slice of
// the units (ascending), with the first batch of loads issued before the clip
// factors are computed; slices are combined in warp order through shared
// memory. Fixed order: run-to-run deterministic; differs from the reference's
// single ascending chain only by fp32 re-association. No float atomics.
//
// mode 0: fused single-GPU step (noise, mean, update); mode 1: write the
// clipped sum only (multi-GPU before the all-reduce, and the parity probe).
constexpr int kAggWarps = 16;
constexpr int kAggCols = 128;
constexpr int kAggRows = 8;       // kind-1 rows per tile of the in-kernel aggregation
constexpr int kAggRowsSep = 8;    // ... and of the separate aggregation kernel (16: fewer,
                                  // taller tiles re-reading d_i less, measured 2.5% slower)
constexpr int kAggBatch = 16; // units per load batch (materialised)
constexpr int kAggChunk = 16; // units per load batch (factored)

// Tile plan of one launch: tile_start[p] = first CTA of parameter block p
// (prefix sums over the blocks' tile counts, built on the host from the block
// kinds of the launch's BlockTable; Engine::agg_plan). Passed by value so a
// CTA locates its tile without a memory round trip.
struct AggPlan {
  int n;
  int rows1;  // kind-1 weight rows per tile (kAggRows or kAggRowsSep)
  int tile_start[kMaxBlocks + 1];
};

struct AggTile {
  int p;   // parameter block
  int j0;  // kind 0: first column; kind 1: first weight row r0
  int n;   // kind 0: columns (<= kAggCols); kind 1: rows (<= kAggRows)
  int c0;  // kind 1: first column c0 (32 per tile)
};

__device__ __forceinline__ AggTile agg_tile(const BlockTable& bt, const AggPlan& plan, int bid) {
  // the block holding tile bid: binary search of the prefix sums (dependent
  // reads of the launch's constant bank; log2(n) of them instead of n)
  int p = 0, hi = plan.n - 1;
  while (p < hi) {
    const int mid = (p + hi + 1) >> 1;
    if (plan.tile_start[mid] <= bid) p = mid;
    else hi = mid - 1;
  }
  const int q = bid - plan.tile_start[p];
  AggTile t;
  t.p = p;
  if (bt.kind[p] == 0) {
    t.j0 = q * kAggCols;
    t.n = (int)min((long long)kAggCols, bt.size[p] - t.j0);
    t.c0 = 0;
  } else {
    const int out = bt.out[p], in = (int)(bt.size[p] / out);
    const int ctiles = (out + 31) / 32;
    t.j0 = (q / ctiles) * plan.rows1;
    t.c0 = (q % ctiles) * 32;
    t.n = min(plan.rows1, in - t.j0);
  }
  return t;
}

__device__ __forceinline__ void agg_scales(const double* __restrict__ parts, int nparts, int U,
                                           float clip, float* s_sh, float* norms_out,
                                           int* cnt_sh, int tid) {
  int local_clipped = 0;
  for (int i = tid; i < U; i += 32 * kAggWarps) {
    double acc = 0.0;
    for (int q = 0; q < nparts; ++q) acc += parts[(size_t)i * nparts + q];
    const float nrm = (float)sqrt(acc);
    s_sh[i] = nrm > clip ? __fdiv_rn(clip, nrm) : 1.0f;
    if (norms_out) norms_out[i] = nrm;
    local_clipped += nrm > clip;
  }
  local_clipped = __reduce_add_sync(0xffffffffu, local_clipped);
  if ((tid & 31) == 0) cnt_sh[tid >> 5] = local_clipped;
}


// Everything one aggregation launch needs, passed by value as the kernel's
// single parameter: a CUDA-graph replay swaps in the step's arguments with
// one kernel-node parameter update (no host-to-device copy on the stream).
struct AggLaunch {
  BlockTable bt;
  AggPlan plan;
  StepArgs a;
  const double* parts;  // fp64 squared-norm partials, (U, nparts)
  float* params;
  float* sum_out;       // mode 1
  float* norms_out;     // (U), written by CTA 0
  int* clipped_out;     // written (not accumulated) by CTA 0
  const DevError* err;
  // set when the per-example kernel already finalised the step's tail
  // inputs (fused MNIST): clip factors, clip flags and the noise vector
  const float* scales;      // (U) or null: computed from parts
  const int* clip_flags;    // (U)
  const float* noise;       // (P) or null: drawn here
  // multi-step graphs: the step index of the noise streams is read on the
  // device (*step_base + step_off) instead of a.step
  const long long* step_base;
  int step_off;
  int U, nparts, mode;
};

// Loads of per-example data: through the read-only path for a separate
// aggregation kernel; L2-coherent (ld.global.cg) when the aggregation runs
// inside the kernel that wrote the data (after a grid barrier).
template <bool kCoherent, class T>
__device__ __forceinline__ T agg_ld(const T* p) {
  if constexpr (kCoherent) return __ldcg(p);
  else return __ldg(p);
}

// Clip factors into shared memory: copied when the per-example kernel
// finalised them, else computed from the fp64 norm partials.
template <bool kCoherent>
__device__ __forceinline__ void agg_prologue(const AggLaunch& L, float* s_sh, float* norms_cta,
                                             int* cnt_sh, int tid) {
  if (L.scales) {
    int local = 0;
    for (int i = tid; i < L.U; i += 32 * kAggWarps) {
      s_sh[i] = agg_ld<kCoherent>(L.scales + i);
      if (norms_cta) local += agg_ld<kCoherent>(L.clip_flags + i);
    }
    local = __reduce_add_sync(0xffffffffu, local);
    if ((tid & 31) == 0) cnt_sh[tid >> 5] = local;
  } else {
    agg_scales(L.parts, L.nparts, L.U, L.a.clip, s_sh, norms_cta, cnt_sh, tid);
  }
}

// Synchronises the 32 * kAggWarps threads running one aggregation tile: the
// whole CTA (separate kernel) or one named-barrier group of a larger CTA.
__device__ __forceinline__ void agg_sync(int bar_id) {
  if (bar_id < 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;" :: "r"(bar_id), "r"(32 * kAggWarps) : "memory");
}

// One tile of the aggregation, run by 32 * kAggWarps threads (tid) that
// synchronise with agg_sync(bar_id); s_sh holds the clip factors (U floats,
// then the factored-row staging), part_sh the per-warp partial sums.
template <bool kCoherent, int kBatch = kAggBatch, int kRows = kAggRows>
__device__ __forceinline__ void agg_tile_run(const AggLaunch& L, int tile_id, int tid, int bar_id,
                                             float* s_sh, float (*part_sh)[kRows * 32],
                                             int* cnt_sh) {
  const BlockTable& bt = L.bt;
  const StepArgs& a = L.a;
  float* __restrict__ params = L.params;
  const int U = L.U, mode = L.mode;
  const AggTile tile = agg_tile(bt, L.plan, tile_id);
  const int p = tile.p;
  const int lane = tid & 31, warp = tid >> 5;
  // this thread's epilogue column, and its current parameter / the step
  // arguments / the error flag, fetched now so they are not on the tail
  long long j;
  bool has_col;
  if (bt.kind[p] == 0) {
    has_col = tid < tile.n;
    j = (long long)tile.j0 + tid;
  } else {
    const int rr = tid >> 5, c = tile.c0 + (tid & 31);
    has_col = rr < tile.n && c < bt.out[p];
    j = (long long)(tile.j0 + rr) * bt.out[p] + c;
  }
  // the addresses of the parameter and its copies, resolved before the wait
  // (the parameter itself only after it: with the next step's per-example
  // kernel a programmatic dependent of this one, this grid can start while
  // the previous step's aggregation is still updating these columns)
  ParamDst dst{nullptr, nullptr, nullptr, 0};
  if (has_col && mode == 0) dst = param_dst(bt, p, j, params);
  asm volatile("" : "+l"(dst.p), "+l"(dst.sh), "+l"(dst.tcw), "+r"(dst.tcw_kind));
  // pre-clipped row groups (bt.rows) are summed with unit factors
  const bool pre = bt.kind[p] == 0 && bt.rows[p] > 0;
  const int nrow = pre ? bt.rows[p] : U;
  const int rows = (nrow + kAggWarps - 1) / kAggWarps;
  const int i0 = min(nrow, warp * rows), i1 = min(nrow, i0 + rows);
  float* norms_cta = tile_id == 0 ? L.norms_out : nullptr;
  // the block's row sources, materialised before the wait
  const float* rbase = bt.base[p];
  const float* abase = bt.a[p];
  long long rstride = bt.stride[p], astride = bt.a_stride[p];
  int outp = bt.out[p];
  asm volatile("" : "+l"(rbase), "+l"(abase), "+l"(rstride), "+l"(astride), "+r"(outp));
  if constexpr (!kCoherent) {
    // address translation of the first rows ahead of the wait (L2 prefetch:
    // no data enters L1 before the producer is done)
    if (i0 < i1) {
      const float* r0 = bt.kind[p] == 0 ? rbase + tile.j0 + (long long)i0 * rstride
                                        : rbase + (long long)i0 * rstride;
      asm volatile("prefetch.global.L2 [%0];" :: "l"(r0));
    }
    // Programmatic dependent launch: the tile decode above (dependent reads of
    // the launch's constant bank, cold at every replay) overlaps the
    // per-example kernel's tail; everything below reads its outputs.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    PGB_MARK(PGB_TRACE_AGG + 8 * tile_id + 5);
  }
  const float cur = dst.p ? __ldcg(dst.p) : 0.0f;
  const float pre_noise =
      (has_col && mode == 0 && L.noise && a.add_noise) ? agg_ld<kCoherent>(L.noise + bt.param_off[p] + j)
                                                       : 0.0f;
  const bool failed = L.err && agg_ld<kCoherent>(&L.err->code) != 0;

  if (bt.kind[p] == 0) {
    // ---- materialised rows: 4 columns per lane ----
    const int c0 = 4 * lane;
    const int ncol = max(0, min(4, tile.n - c0));
    const long long stride = rstride;
    const float* base = rbase + tile.j0 + c0;
    const bool vec = ncol == 4 && (stride & 3) == 0 &&
                     (reinterpret_cast<uintptr_t>(base) & 15) == 0;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    float v[kBatch][4];
    auto load = [&](int ib) {
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int i = ib + u;
        if (i < i1 && ncol > 0) {
          const float* src = base + (long long)i * stride;
          if (vec) {
            const float4 q = agg_ld<kCoherent>(reinterpret_cast<const float4*>(src));
            v[u][0] = q.x; v[u][1] = q.y; v[u][2] = q.z; v[u][3] = q.w;
          } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) v[u][c] = c < ncol ? agg_ld<kCoherent>(src + c) : 0.0f;
          }
        }
      }
    };
    load(i0);  // in flight while the clip factors are computed
#ifdef PGB_TRACE
    if (!kCoherent && tid == 0) {  // timestamp once the first rows have arrived
      if (__float_as_uint(v[0][0]) == 0x7fc00001u) asm volatile("trap;");
      PGB_MARK_T(PGB_TRACE_AGG + 8 * tile_id + 6, 0);
    }
#endif
    agg_prologue<kCoherent>(L, s_sh, norms_cta, cnt_sh, tid);
    if (!kCoherent) PGB_MARK_T(PGB_TRACE_AGG + 8 * tile_id + 7, 0);
    agg_sync(bar_id);
    if (!kCoherent) PGB_MARK_T(PGB_TRACE_AGG + 8 * tile_id + 1, 0);
    for (int ib = i0; ib < i1; ib += kBatch) {
      if (ib != i0) load(ib);
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        if (ib + u < i1) {
          const float s = pre ? 1.0f : s_sh[ib + u];
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[c] = __fadd_rn(acc[c], __fmul_rn(v[u][c], s));
        }
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) part_sh[warp][c0 + c] = acc[c];
  } else {
    // ---- factored dense rows: kRows weight rows x 32 columns ----
    // Per chunk of kAggChunk units the warp issues every load at once: d_ic
    // into registers (lane = c), the a_i[r0 .. r0+15] rows through a
    // per-warp shared staging area (read back as broadcasts).
    const int out = outp;
    const int c = tile.c0 + lane;
    const bool cok = c < out;
    const int nr = tile.n;
    const float* A = abase + tile.j0;
    const float* D = rbase + (cok ? c : 0);
    const long long as = astride, ds = rstride;
    float* a_st = s_sh + ((U + 3) & ~3) + warp * (kAggChunk * kRows);
    float acc[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) acc[r] = 0.0f;
    float dv[kAggChunk], ar[kAggChunk * kRows / 32];
    auto load = [&](int ib) {
#pragma unroll
      for (int u = 0; u < kAggChunk; ++u)
        dv[u] = (cok && ib + u < i1) ? agg_ld<kCoherent>(D + (long long)(ib + u) * ds) : 0.0f;
#pragma unroll
      for (int q = 0; q < kAggChunk * kRows / 32; ++q) {
        const int e = q * 32 + lane, u = e / kRows, r = e % kRows;
        ar[q] = (ib + u < i1 && r < nr) ? agg_ld<kCoherent>(A + (long long)(ib + u) * as + r) : 0.0f;
      }
    };
    load(i0);
    agg_prologue<kCoherent>(L, s_sh, norms_cta, cnt_sh, tid);
    agg_sync(bar_id);
    if (!kCoherent) PGB_MARK_T(PGB_TRACE_AGG + 8 * tile_id + 2, 0);
    for (int ib = i0; ib < i1; ib += kAggChunk) {
      if (ib != i0) load(ib);
#pragma unroll
      for (int q = 0; q < kAggChunk * kRows / 32; ++q) a_st[q * 32 + lane] = ar[q];
      __syncwarp();
#pragma unroll
      for (int u = 0; u < kAggChunk; ++u) {
        if (ib + u < i1) {
          // acc_r += a_ir * fl(d_ic * s_i) as one FMA per element (the
          // reference's fl(fl(a * d) * s) + acc costs three rounded ops; the
          // clipped sum is the issue-bound tail of the step, and the product
          // differs from it by at most one rounding, SURVEY 8(d) tolerance)
          const float ds = __fmul_rn(dv[u], s_sh[ib + u]);
          const float4* a4 = reinterpret_cast<const float4*>(a_st + u * kRows);
#pragma unroll
          for (int q = 0; q < kRows / 4; ++q) {
            const float4 x = a4[q];
            acc[4 * q] = __fmaf_rn(x.x, ds, acc[4 * q]);
            acc[4 * q + 1] = __fmaf_rn(x.y, ds, acc[4 * q + 1]);
            acc[4 * q + 2] = __fmaf_rn(x.z, ds, acc[4 * q + 2]);
            acc[4 * q + 3] = __fmaf_rn(x.w, ds, acc[4 * q + 3]);
          }
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r) part_sh[warp][r * 32 + lane] = acc[r];
  }
  agg_sync(bar_id);
  if (!kCoherent) PGB_MARK_T(PGB_TRACE_AGG + 8 * tile_id + 3, 0);

  // ---- epilogue: one thread per column of the tile ----
  if (tile_id == 0 && tid == 0 && L.clipped_out) {
    int n = 0;
#pragma unroll
    for (int w = 0; w < kAggWarps; ++w) n += cnt_sh[w];
    *L.clipped_out = n;
  }
  if (!has_col) return;
  const int t = tid;
  float sum = part_sh[0][t];
#pragma unroll
  for (int w = 1; w < kAggWarps; ++w) sum = __fadd_rn(sum, part_sh[w][t]);
  if (mode == 1) {
    L.sum_out[bt.param_off[p] + j] = sum;
    return;
  }
  if (a.add_noise) {
    float n = pre_noise;
    if (!L.noise) {
      // the pair's two normals come from one Box-Muller draw (kernels.hpp:597-614)
      float n0, n1;
      const long long stp = L.step_base ? *L.step_base + L.step_off : a.step;
      gauss_pair(stream_key(a.seed, noise_stream(stp, p)), j >> 1, &n0, &n1);
      n = (j & 1) ? n1 : n0;
    }
    sum = __fadd_rn(sum, __fmul_rn(__fmul_rn(a.sigma, a.clip), n));
  }
  sum = __fmul_rn(sum, a.inv_units);
  if (failed) return;
  param_store(dst, j, __fsub_rn(cur, __fmul_rn(a.lr, sum)));
}

__global__ void __launch_bounds__(32 * kAggWarps) aggregate_kernel(const AggLaunch L) {
  extern __shared__ float s_sh[];  // clip factors, one per unit
  __shared__ float part_sh[kAggWarps][kAggRowsSep * 32];
  __shared__ int cnt_sh[kAggWarps];
  PGB_MARK(PGB_TRACE_AGG + 8 * blockIdx.x + 0);
  // the next step's per-example kernel may start its input-only prologue
  asm volatile("griddepcontrol.launch_dependents;");
  // programmatic dependent launch: this grid may be resident before the
  // per-example kernel has finished; agg_tile_run waits for it
  agg_tile_run<false, kAggBatch, kAggRowsSep>(L, blockIdx.x, threadIdx.x, -1, s_sh, part_sh,
                                              cnt_sh);
  PGB_MARK(PGB_TRACE_AGG + 8 * blockIdx.x + 4);
}

// ---- sparse per-example embedding gradients (embedding -> seq_avgpool) ----
// The reference materialises the per-example table gradient as a dense
// (B, V, E) stack (strategies.cpp:171-188): row r of example i is v_i = u_i/L
// (u_i the pooled cotangent) added once per occurrence of token r, in token
// order. Here each example keeps only its distinct tokens and counts; the
// element value is the same fp32 chain acc = fl(acc + v) repeated c times.
constexpr int kEmbMaxL = 1024;
constexpr int kEmbMaxE = 1024;
constexpr int kEmbHist = 64;  // token counts per example handled by the count histogram  // pooled-cotangent rows staged in shared memory up to this width

__device__ __forceinline__ float emb_chain(float v, int c) {
  if (c == 1) return v;  // fl(0 + v) = v, the common case
  float acc = 0.0f;
  for (int k = 0; k < c; ++k) acc = __fadd_rn(acc, v);
  return acc;
}

// Per example (one CTA): sort the L token ids, keep distinct tokens and their
// counts (tok/cnt rows of length L, n_distinct), mark example i in each
// token's row bitmap (bit i of bits[r * words]), and the example's squared
// norm of the embedding block in fp64 (dpsgd.cpp:254-270) into
// parts[i * nparts + p].
__global__ void __launch_bounds__(256) embed_index_kernel(
    const float* __restrict__ ids, const float* __restrict__ u, int L, int E, int V, int words,
    int* __restrict__ tok, int* __restrict__ cnt, int* __restrict__ nd,
    unsigned* __restrict__ bits, double* __restrict__ parts, int nparts, int p) {
  __shared__ int key[kEmbMaxL];
  __shared__ int seg[kEmbMaxL + 1];
  __shared__ int nseg;
  __shared__ double red[32];
  const int i = blockIdx.x, t = threadIdx.x;
  int Lp = 1;
  while (Lp < L) Lp <<= 1;
  if (Lp <= (int)blockDim.x && blockDim.x == 256) {
    // one key per thread (sentinels past L), bitonic network over 256 keys in
    // registers: exchanges with stride < 32 by warp shuffles, the 6 with
    // stride >= 32 through shared memory
    int v = 0x7fffffff;
    if (t < L) {
      const float raw = ids[(size_t)i * L + t];
      if (valid_id(raw, V)) v = (int)raw;  // invalid ids raised by the forward
    }
#pragma unroll
    for (int size = 2; size <= 256; size <<= 1)
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        int other;
        if (stride >= 32) {
          key[t] = v;
          __syncthreads();
          other = key[t ^ stride];
          __syncthreads();
        } else {
          other = __shfl_xor_sync(0xffffffffu, v, stride);
        }
        const bool up = (t & size) == 0, lower = (t & stride) == 0;
        v = (lower == up) ? min(v, other) : max(v, other);
      }
    key[t] = v;
    Lp = 256;
    __syncthreads();
  } else {
    for (int k = t; k < Lp; k += blockDim.x) {
      int v = 0x7fffffff;
      if (k < L) {
        const float raw = ids[(size_t)i * L + k];
        if (valid_id(raw, V)) v = (int)raw;  // invalid ids raised by the forward
      }
      key[k] = v;
    }
    __syncthreads();
    // bitonic sort (ascending)
    for (int size = 2; size <= Lp; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int k = t; k < Lp / 2; k += blockDim.x) {
          const int a = 2 * k - (k & (stride - 1));
          const int b = a + stride;
          const bool up = (a & size) == 0;
          const int x = key[a], y = key[b];
          if ((x > y) == up) {
            key[a] = y;
            key[b] = x;
          }
        }
        __syncthreads();
      }
  }
  // segment starts (distinct tokens) in order: first occurrences flagged in
  // parallel, compacted with warp ballots and a per-chunk warp prefix
  {
    __shared__ int wtot[32];
    const int lane = t & 31, wp = t >> 5, nw = blockDim.x >> 5;
    int base = 0, end = 0;
    for (int k0 = 0; k0 < Lp; k0 += blockDim.x) {
      const int k = k0 + t;
      const bool valid = k < L && key[k] != 0x7fffffff;
      const bool f = valid && (k == 0 || key[k] != key[k - 1]);
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (lane == 0) wtot[wp] = __popc(bal);
      end += __syncthreads_count(valid);
      int off = base, tot = 0;
      for (int q = 0; q < nw; ++q) {
        off += q < wp ? wtot[q] : 0;
        tot += wtot[q];
      }
      if (f) seg[off + __popc(bal & ((1u << lane) - 1u))] = k;
      base += tot;
      __syncthreads();
    }
    if (t == 0) {
      seg[base] = end;
      nseg = base;
      nd[i] = base;
    }
  }
  __syncthreads();
  const int n = nseg;
  for (int k = t; k < n; k += blockDim.x) {
    const int r = key[seg[k]];
    tok[(size_t)i * L + k] = r;
    cnt[(size_t)i * L + k] = seg[k + 1] - seg[k];
    const int c = seg[k + 1] - seg[k];
    atomicOr(&bits[(size_t)r * words + (i >> 5)], 1u << (i & 31));
    // the second bitmap (bits + V * words) marks the rows this example holds
    // more than once: only those look their count up in the aggregation
    if (c > 1) atomicOr(&bits[((size_t)V + r) * words + (i >> 5)], 1u << (i & 31));
  }
  // ||G_i||^2 = sum over distinct tokens and e of chain(u_ie / L, c)^2 (the
  // pooled cotangent row staged in shared memory once)
  __shared__ float urow[kEmbMaxE];
  const bool staged = E <= kEmbMaxE;
  if (staged)
    for (int e = t; e < E; e += blockDim.x) urow[e] = u[(size_t)i * E + e];
  __syncthreads();
  const float* ur = staged ? urow : u + (size_t)i * E;
  const float invL = 1.0f / float(L);
  // every token with count c contributes the same sum_e chain(u_e / L, c)^2:
  // one pass over e per distinct count (fp64, any order)
  __shared__ int hist[kEmbHist];
  for (int c = t; c < kEmbHist; c += blockDim.x) hist[c] = 0;
  __syncthreads();
  for (int k = t; k < n; k += blockDim.x) {
    const int c = seg[k + 1] - seg[k];
    if (c < kEmbHist) atomicAdd(&hist[c], 1);
  }
  __syncthreads();
  double acc = 0.0;
  const int lane = t & 31, wp = t >> 5, nw = blockDim.x >> 5;
  for (int c = 1 + wp; c < kEmbHist; c += nw) {
    const int m = hist[c];
    if (!m) continue;
    double sc = 0.0;
    for (int e = lane; e < E; e += 32) {
      const float g = emb_chain(ur[e] * invL, c);
      sc += (double)g * g;
    }
    acc += sc * m;
  }
  for (int k = t; k < n; k += blockDim.x) {  // counts beyond the histogram
    const int c = seg[k + 1] - seg[k];
    if (c < kEmbHist) continue;
    for (int e = 0; e < E; ++e) {
      const float g = emb_chain(ur[e] * invL, c);
      acc += (double)g * g;
    }
  }
  acc = block_reduce_sum(acc, red);
  if (t == 0) parts[(size_t)i * nparts + p] = acc;
}

// Clipped sum of the embedding block over the examples containing each row,
// then noise / mean / update (mode 0) or the sum alone (mode 1), one warp per
// table row, every row (inactive rows get noise only). Examples are visited in
// ascending order (the reference's views-path order, dpsgd.cpp:287-307); each
// term is fl(g * s_i). The row's bitmap is cleared for the next step.
struct EmbAggLaunch {
  BlockTable bt;
  StepArgs a;
  const double* parts;
  const float* norms;  // (B) per-example norms (finalize_norms_kernel), once per step
  const float* u;      // (B, E) pooled cotangent
  const int* tok;      // (B, L)
  const int* cnt;
  const int* nd;       // (B)
  unsigned* bits;      // (V, words)
  float* params;
  float* sum_out;      // mode 1
  const DevError* err;
  const long long* step_base;  // multi-step graphs: the noise step on the device
  int step_off;
  int p, B, L, E, V, words, nparts, mode;
};

__global__ void __launch_bounds__(256, 4) embed_agg_kernel(const EmbAggLaunch A) {
  extern __shared__ float s_emb[];  // clip factors (B)
  __shared__ unsigned wsh[8][32];   // the current row's bitmap words, per warp
  __shared__ unsigned msh[8][32];   // ... and its multi-occurrence words
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  for (int i = t; i < A.B; i += blockDim.x) {
    const float nrm = A.norms[i];
    s_emb[i] = nrm > A.a.clip ? __fdiv_rn(A.a.clip, nrm) : 1.0f;
  }
  __syncthreads();
  const BlockTable& bt = A.bt;
  const StepArgs& a = A.a;
  const float invL = 1.0f / float(A.L);
  const bool failed = A.err && A.err->code != 0;
  const uint64_t key =
      stream_key(a.seed, noise_stream(A.step_base ? *A.step_base + A.step_off : a.step, A.p));
  const long long E = A.E;
  __shared__ int lst_i[8][32], lst_c[8][32];
  __shared__ float lst_s[8][32];
  for (int r = blockIdx.x * 8 + w; r < A.V; r += gridDim.x * 8) {
    const unsigned word = lane < A.words ? A.bits[(size_t)r * A.words + lane] : 0u;
    const unsigned mword =
        lane < A.words ? A.bits[((size_t)A.V + r) * A.words + lane] : 0u;
    const unsigned active = __ballot_sync(0xffffffffu, word != 0u);
    wsh[w][lane] = word;
    msh[w][lane] = mword;
    __syncwarp();
    // this lane's element pairs of the row: jb + lane + 32 q, in blocks of 64
    // pairs (one block for E <= 126)
    const long long j0 = (long long)r * E, jp1 = (j0 + E - 1) >> 1;
    for (long long jb = j0 >> 1; jb <= jp1; jb += 64) {
    float acc[2][2] = {{0.0f, 0.0f}, {0.0f, 0.0f}};
    long long e0q[2];
    bool okq[2][2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const long long jp = jb + lane + 32 * q;
      e0q[q] = 2 * jp - j0;
      okq[q][0] = jp <= jp1 && e0q[q] >= 0 && e0q[q] < E;
      okq[q][1] = jp <= jp1 && e0q[q] + 1 >= 0 && e0q[q] + 1 < E;
    }
    // the row's examples in ascending order, 32 at a time: the count of token
    // r in example i is found once per example (one lane each, binary search
    // of its distinct tokens), then every lane adds fl(chain(u_ie / L, c) s_i)
    int fill = 0;
    auto flush = [&]() {
      if (lane < fill) {
        const int i = lst_i[w][lane];
        int c = 1;  // the common case: the token once in the example
        if ((msh[w][i >> 5] >> (i & 31)) & 1u) {
          // its count: binary search of the example's distinct tokens
          const int* tk = A.tok + (size_t)i * A.L;
          int lo = 0, hi = A.nd[i] - 1;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (tk[mid] < r) lo = mid + 1;
            else hi = mid;
          }
          c = A.cnt[(size_t)i * A.L + lo];
        }
        lst_c[w][lane] = c;
        lst_s[w][lane] = s_emb[i];
      }
      __syncwarp();
      // four examples' u values in flight at a time, added in example order
      for (int k0 = 0; k0 < fill; k0 += 4) {
        float uv[4][2][2];
#pragma unroll
        for (int d = 0; d < 4; ++d) {
          const int k = min(k0 + d, fill - 1);
          const float* ui = A.u + (size_t)lst_i[w][k] * E;
#pragma unroll
          for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int h = 0; h < 2; ++h) uv[d][q][h] = okq[q][h] ? __ldg(ui + e0q[q] + h) : 0.0f;
        }
#pragma unroll
        for (int d = 0; d < 4; ++d) {
          if (k0 + d >= fill) break;
          const int c = lst_c[w][k0 + d];
          const float s = lst_s[w][k0 + d];
#pragma unroll
          for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (okq[q][h])
                acc[q][h] = __fadd_rn(acc[q][h], __fmul_rn(emb_chain(uv[d][q][h] * invL, c), s));
        }
      }
      __syncwarp();
      fill = 0;
    };
    unsigned am = active;
    unsigned bw = 0;
    int wd = 0;
    while (true) {
      // next example of the row in ascending order, or the end
      while (!bw && am) {
        wd = __ffs(am) - 1;
        am &= am - 1;
        bw = wsh[w][wd];
      }
      const bool more = bw != 0;
      if (more) {
        const int bb = __ffs(bw) - 1;
        bw &= bw - 1;
        if (lane == 0) lst_i[w][fill] = wd * 32 + bb;
        ++fill;
      }
      if (fill == 32 || (!more && fill)) {
        __syncwarp();
        flush();
      }
      if (!more) break;
    }
    const float scale = __fmul_rn(a.sigma, a.clip);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const long long jp = jb + lane + 32 * q;
      if (jp > jp1) continue;
      float n0 = 0.0f, n1 = 0.0f;
      if (A.mode == 0 && a.add_noise) gauss_pair(key, jp, &n0, &n1);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!okq[q][h]) continue;
        const long long j = j0 + e0q[q] + h;
        float sum = acc[q][h];
        if (A.mode == 1) {
          A.sum_out[bt.param_off[A.p] + j] = sum;
          continue;
        }
        if (a.add_noise) sum = __fadd_rn(sum, __fmul_rn(scale, h ? n1 : n0));
        sum = __fmul_rn(sum, a.inv_units);
        if (failed) continue;
        const float cur = A.params[bt.param_off[A.p] + j];
        write_param(bt, A.p, j, A.params, __fsub_rn(cur, __fmul_rn(a.lr, sum)));
      }
    }
    }  // pair blocks
    if (lane < A.words && word) A.bits[(size_t)r * A.words + lane] = 0u;
    if (lane < A.words && mword) A.bits[((size_t)A.V + r) * A.words + lane] = 0u;
    __syncwarp();
  }
}

// embed_agg_kernel with four consecutive elements per lane (E % 4 == 0, the
// table 16-byte aligned, no shadow copies): the row's example list is built
// in parallel (one bitmap word per lane, a warp scan for the offsets; the
// count looked up by the lane that owns the example), then every example of
// the row costs one 16-byte load of its pooled cotangent per lane. Same
// arithmetic per element and the same ascending example order as
// embed_agg_kernel, so the two are bitwise equal (tests/test_embed_gpu.py).
constexpr int kEmbAggWarps = 8;
__global__ void __launch_bounds__(32 * kEmbAggWarps) embed_agg4_kernel(const EmbAggLaunch A) {
  extern __shared__ float s_emb[];                 // clip factors (B)
  __shared__ int lst[kEmbAggWarps][1024];          // (count << 10) | example, ascending
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  for (int i = t; i < A.B; i += blockDim.x) {
    // the norm from the fp64 partials, as finalize_norms_kernel computes it
    double acc = 0.0;
    for (int q = 0; q < A.nparts; ++q) acc += A.parts[(size_t)i * A.nparts + q];
    const float nrm = (float)sqrt(acc);
    s_emb[i] = nrm > A.a.clip ? __fdiv_rn(A.a.clip, nrm) : 1.0f;
  }
  __syncthreads();
  const StepArgs& a = A.a;
  const float invL = 1.0f / float(A.L);
  const bool failed = A.err && A.err->code != 0;
  const uint64_t key =
      stream_key(a.seed, noise_stream(A.step_base ? *A.step_base + A.step_off : a.step, A.p));
  const int E = A.E;
  const float scale = __fmul_rn(a.sigma, a.clip);
  float* tab = A.params + A.bt.param_off[A.p];
  float* sum_out = A.sum_out ? A.sum_out + A.bt.param_off[A.p] : nullptr;
  int* L = lst[w];
  for (int r = blockIdx.x * kEmbAggWarps + w; r < A.V; r += gridDim.x * kEmbAggWarps) {
    const bool hasw = lane < A.words;
    const unsigned word = hasw ? A.bits[(size_t)r * A.words + lane] : 0u;
    const unsigned mword = hasw ? A.bits[((size_t)A.V + r) * A.words + lane] : 0u;
    // this lane's examples go to list slots [off, off + popc(word))
    const int cntw = __popc(word);
    int off = cntw;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, off, o);
      if (lane >= o) off += v;
    }
    const int n = __shfl_sync(0xffffffffu, off, 31);
    off -= cntw;
    for (unsigned bw = word; bw; bw &= bw - 1) {
      const int bb = __ffs(bw) - 1, i = lane * 32 + bb;
      int c = 1;  // the common case: the token once in the example
      if ((mword >> bb) & 1u) {
        const int* tk = A.tok + (size_t)i * A.L;
        int lo = 0, hi = A.nd[i] - 1;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (tk[mid] < r) lo = mid + 1;
          else hi = mid;
        }
        c = A.cnt[(size_t)i * A.L + lo];
      }
      L[off++] = (c << 10) | i;
    }
    __syncwarp();
    const long long j0 = (long long)r * E;
    for (int eb = 0; eb < E; eb += 128) {  // warp-uniform trip count
      const int e0 = eb + 4 * lane;
      const bool ok = e0 < E;
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      for (int k0 = 0; k0 < n; k0 += 8) {
        float4 uv[8];
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          const int k = min(k0 + d, n - 1);
          const int i = L[k] & 1023;
          uv[d] = ok ? __ldg(reinterpret_cast<const float4*>(A.u + (size_t)i * E + e0))
                     : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        }
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          if (k0 + d >= n) break;
          const int pk = L[k0 + d];
          const int c = pk >> 10;
          const float s = s_emb[pk & 1023];
          float g[4] = {uv[d].x * invL, uv[d].y * invL, uv[d].z * invL, uv[d].w * invL};
          if (c != 1) {  // warp-uniform: emb_chain once per example, not per element
            float ch[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 1
            for (int k = 0; k < c; ++k)
#pragma unroll
              for (int h = 0; h < 4; ++h) ch[h] = __fadd_rn(ch[h], g[h]);
#pragma unroll
            for (int h = 0; h < 4; ++h) g[h] = ch[h];
          }
#pragma unroll
          for (int h = 0; h < 4; ++h) acc[h] = __fadd_rn(acc[h], __fmul_rn(g[h], s));
        }
      }
      if (ok) {
        const long long j = j0 + e0;  // even: two whole normal pairs
        if (A.mode == 1) {
          *reinterpret_cast<float4*>(sum_out + j) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        } else {
          float nz[4] = {0.0f, 0.0f, 0.0f, 0.0f};
          if (a.add_noise) {
            gauss_pair(key, j >> 1, &nz[0], &nz[1]);
            gauss_pair(key, (j >> 1) + 1, &nz[2], &nz[3]);
          }
          if (!failed) {
            float4 cur = *reinterpret_cast<const float4*>(tab + j);
            float* cv = reinterpret_cast<float*>(&cur);
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              float sm = acc[h];
              if (a.add_noise) sm = __fadd_rn(sm, __fmul_rn(scale, nz[h]));
              sm = __fmul_rn(sm, a.inv_units);
              cv[h] = __fsub_rn(cv[h], __fmul_rn(a.lr, sm));
            }
            *reinterpret_cast<float4*>(tab + j) = cur;
          }
        }
      }
    }
    if (hasw && word) A.bits[(size_t)r * A.words + lane] = 0u;
    if (hasw && mword) A.bits[((size_t)A.V + r) * A.words + lane] = 0u;
    __syncwarp();
  }
}

// ---- ghost norms of 3x3 / stride-1 / pad-1 conv weight blocks --------------
// ||dW_i||^2 = sum_{p,q} (g_p . g_q) (a_p . a_q) with a_p the im2col patch at
// output position p and g_p the output cotangent there (the ghost-norm
// identity, generalised from dense layers to convolutions): the patch Gram is
// a sum of shifted input Grams, a_p . a_q = sum_taps x~_{p+t} . x~_{q+t} (x~ the
// zero-padded input). For the 8x8 and 4x4 layers (HW <= 64) this is far less
// work than the per-example dW GEMM, and no (B, D, C, 3, 3) stack is written.
// One CTA of 256 threads per example; Grams in fp32 (dots of length C, D),
// the weighted sum over (p, q) in fp64, into parts[i * nparts + pb]
// (dpsgd.cpp:254-270 accumulates the block's squares in double).
template <int HW>
__global__ void __launch_bounds__(256) conv_gram_norm_kernel(
    const float* __restrict__ x, const float* __restrict__ g, int C, int D, int W,
    double* __restrict__ parts, int nparts, int pb, float* __restrict__ sb) {
  static_assert(HW == 16 || HW == 64, "ghost norms for 4x4 and 8x8 maps");
  constexpr int R = HW == 64 ? 4 : 1;  // (p, q) block per thread: R x R
  extern __shared__ float gsm[];
  float* xs = gsm;               // [C][HW]
  float* gs = xs + C * HW;       // [D][HW]
  float* gx = gs + D * HW;       // [HW][HW]
  __shared__ double red[8];
  const int i = blockIdx.x, t = threadIdx.x;
  const float* xi = x + (size_t)i * C * HW;
  const float* gi = g + (size_t)i * D * HW;
  // 16-byte loads, four in flight per thread (HW is 16 or 64: rows stay aligned)
  {
    const float4* xi4 = reinterpret_cast<const float4*>(xi);
    const float4* gi4 = reinterpret_cast<const float4*>(gi);
    float4* xs4 = reinterpret_cast<float4*>(xs);
    float4* gs4 = reinterpret_cast<float4*>(gs);
#pragma unroll 4
    for (int e = t; e < C * HW / 4; e += 256) xs4[e] = __ldg(xi4 + e);
#pragma unroll 4
    for (int e = t; e < D * HW / 4; e += 256) gs4[e] = __ldg(gi4 + e);
  }
  __syncthreads();
  if (sb) {
    // the example's conv bias gradient (D), with conv_db_pex_kernel's
    // arithmetic (lane-strided partials, xor butterfly): bitwise the same
    const int w = t >> 5, lane = t & 31;
    for (int d = w; d < D; d += 8) {
      float s = 0.0f;
      for (int p = lane; p < HW; p += 32) s += gs[d * HW + p];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) sb[(size_t)i * D + d] = s;
    }
  }
  const int tp = t / (HW / R), tq = t % (HW / R);
  float ax[R][R], ag[R][R];
#pragma unroll
  for (int j = 0; j < R; ++j)
#pragma unroll
    for (int k = 0; k < R; ++k) ax[j][k] = ag[j][k] = 0.0f;
  auto gram = [&](const float* src, int n, float (*acc)[R]) {
    for (int c = 0; c < n; ++c) {
      float a[R], b[R];
      if constexpr (R == 4) {
        const float4 va = reinterpret_cast<const float4*>(src + c * HW)[tp];
        const float4 vb = reinterpret_cast<const float4*>(src + c * HW)[tq];
        a[0] = va.x; a[1] = va.y; a[2] = va.z; a[3] = va.w;
        b[0] = vb.x; b[1] = vb.y; b[2] = vb.z; b[3] = vb.w;
      } else {
        a[0] = src[c * HW + tp];
        b[0] = src[c * HW + tq];
      }
#pragma unroll
      for (int j = 0; j < R; ++j)
#pragma unroll
        for (int k = 0; k < R; ++k) acc[j][k] = fmaf(a[j], b[k], acc[j][k]);
    }
  };
  gram(xs, C, ax);
  gram(gs, D, ag);
#pragma unroll
  for (int j = 0; j < R; ++j)
#pragma unroll
    for (int k = 0; k < R; ++k) gx[(tp * R + j) * HW + tq * R + k] = ax[j][k];
  __syncthreads();
  const int H = HW / W;
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < R; ++j)
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int pp = tp * R + j, qq = tq * R + k;
      const int py = pp / W, px = pp - py * W, qy = qq / W, qx = qq - qy * W;
      float ga = 0.0f;
#pragma unroll
      for (int u = -1; u <= 1; ++u)
#pragma unroll
        for (int v = -1; v <= 1; ++v) {
          const int a0 = py + u, a1 = px + v, b0 = qy + u, b1 = qx + v;
          if (a0 >= 0 && a0 < H && a1 >= 0 && a1 < W && b0 >= 0 && b0 < H && b1 >= 0 && b1 < W)
            ga += gx[(a0 * W + a1) * HW + b0 * W + b1];
        }
      acc = fma((double)ag[j][k], (double)ga, acc);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((t & 31) == 0) red[t >> 5] = acc;
  __syncthreads();
  if (t == 0) {
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += red[w];
    parts[(size_t)i * nparts + pb] = tot;
  }
}

// Per-example norms, clip factors and clip flags from the fp64 partials (the
// same arithmetic as agg_scales), once per step, for the steps whose conv
// weight gradients are summed by a clip-scaled GEMM.
struct ScalesLaunch {
  const double* parts;
  int nparts, U;
  StepArgs a;
  float* scale;
  int* flags;
  float* norms;  // the step's result slot (a per-launch node argument)
};

__global__ void step_scales_kernel(const ScalesLaunch L) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L.U) return;
  double acc = 0.0;
  for (int q = 0; q < L.nparts; ++q) acc += L.parts[(size_t)i * L.nparts + q];
  const float nrm = (float)sqrt(acc);
  const float clip = L.a.clip;
  L.scale[i] = nrm > clip ? __fdiv_rn(clip, nrm) : 1.0f;
  L.flags[i] = nrm > clip ? 1 : 0;
  if (L.norms) L.norms[i] = nrm;
}

// After the all-reduce of the clipped sums: noise (one shared draw from the
// common seed, so every rank adds the same vector), mean over the global
// units, update (dpsgd.cpp:308-317, apply_update :173-183). One thread per
// normal PAIR: each Box-Muller draw (kernels.hpp:597-614) feeds both of its
// elements, and the pair's two sums / parameters are adjacent.
struct NoiseLaunch {
  BlockTable bt;
  StepArgs a;
  const float* sum;  // the all-reduced clipped sum
  float* params;
  const DevError* err;
  const float* noise;          // (P) the step's normals drawn by the fused kernel, or null
  const long long* step_base;  // multi-step graphs: the noise step on the device
  int step_off;
  // the step's clip counts (local, all-reduced) copied from the all-reduce's
  // fixed buffer into the step's result slot (a per-launch node argument,
  // where the all-reduce's pointers are fixed at capture)
  const int* cnt_in;
  int* clipped_out;
  int only_kind;  // >= 0: update only the blocks of this kind (the others are done)
};

__global__ void __launch_bounds__(256) noise_update_kernel(const NoiseLaunch L) {
  const BlockTable& bt = L.bt;
  const StepArgs& a = L.a;
  const float* __restrict__ sum = L.sum;
  float* __restrict__ params = L.params;
  __shared__ long long pair_sh[kMaxBlocks + 1];
  if (threadIdx.x == 0) {
    long long o = 0;
    for (int p = 0; p < bt.n; ++p) {
      pair_sh[p] = o;
      o += (bt.size[p] + 1) / 2;
    }
    pair_sh[bt.n] = o;
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0 && L.clipped_out && L.clipped_out != L.cnt_in) {
    L.clipped_out[0] = L.cnt_in[0];
    L.clipped_out[1] = L.cnt_in[1];
  }
  if (L.err && L.err->code != 0) return;
  const long long total = pair_sh[bt.n];
  const long long stp = L.step_base ? *L.step_base + L.step_off : a.step;
  const float scale = __fmul_rn(a.sigma, a.clip);
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    int lo = 0, hi = bt.n - 1;  // the block holding pair q (binary search)
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pair_sh[mid] <= q) lo = mid;
      else hi = mid - 1;
    }
    const int p = lo;
    if (L.only_kind >= 0 && bt.kind[p] != L.only_kind) continue;
    const long long jp = q - pair_sh[p], j0 = 2 * jp;
    const long long off = bt.param_off[p];
    float nv[2] = {0.0f, 0.0f};
    if (a.add_noise) {
      if (L.noise) {
        nv[0] = L.noise[off + j0];
        if (j0 + 1 < bt.size[p]) nv[1] = L.noise[off + j0 + 1];
      } else {
        gauss_pair(stream_key(a.seed, noise_stream(stp, p)), jp, &nv[0], &nv[1]);
      }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const long long j = j0 + e;
      if (j >= bt.size[p]) break;
      float acc = sum[off + j];
      if (a.add_noise) acc = __fadd_rn(acc, __fmul_rn(scale, nv[e]));
      acc = __fmul_rn(acc, a.inv_units);
      const float cur = params[off + j];
      write_param(bt, p, j, params, __fsub_rn(cur, __fmul_rn(a.lr, acc)));
    }
  }
}

// Materialise every block's per-example rows into block-major stacks
// (B, |p|): the compute_views probe and the microbatch path.
__global__ void materialize_kernel(BlockTable bt, int B, float* __restrict__ stacks) {
  long long total = 0;
  for (int p = 0; p < bt.n; ++p) total += bt.size[p];
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total * B;
       e += (long long)gridDim.x * blockDim.x) {
    long long j = e;
    int p = 0;
    long long off = 0;
    while (j >= bt.size[p] * B) {
      j -= bt.size[p] * B;
      off += bt.size[p] * B;
      ++p;
    }
    const long long per = bt.size[p];
    const long long i = j / per, c = j - i * per;
    float* dst = stacks + off + j;
    const float v = grad_at(bt, p, i, c);
    if (bt.kind[p] != 0 || bt.base[p] + i * bt.stride[p] + c != dst) *dst = v;
  }
}

// microbatch means (dpsgd.cpp:102-132) over materialised stacks: unit u =
// mean of m consecutive rows, summed in order from zero then * (float)1/m.
__global__ void microbatch_kernel(const float* __restrict__ stacks, BlockTable bt, int B,
                                  int m, float* __restrict__ units_out) {
  const int U = B / m;
  const float inv = 1.0f / float(m);
  long long total = 0;
  for (int p = 0; p < bt.n; ++p) total += bt.size[p];
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total * U;
       e += (long long)gridDim.x * blockDim.x) {
    const int u = (int)(e / total);
    long long j = e - (long long)u * total;
    int p = 0;
    while (j >= bt.size[p]) j -= bt.size[p++];
    const long long per = bt.size[p];
    const float* src = stacks + bt.param_off[p] * B;
    float acc = 0.0f;
    for (int r = 0; r < m; ++r) acc = __fadd_rn(acc, src[((long long)u * m + r) * per + j]);
    units_out[bt.param_off[p] * U + (long long)u * per + j] = __fmul_rn(acc, inv);
  }
}

// plain SGD (dpsgd.cpp:334-346): p -= lr * (sum_i g_i) * 1/B
__global__ void sgd_kernel(BlockTable bt, int B, float lr, float* __restrict__ params) {
  long long total = 0;
  for (int p = 0; p < bt.n; ++p) total += bt.size[p];
  const float inv = 1.0f / float(B);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    long long j = e;
    int p = 0;
    while (j >= bt.size[p]) j -= bt.size[p++];
    float acc = 0.0f;
    for (int i = 0; i < B; ++i) acc = __fadd_rn(acc, grad_at(bt, p, i, j));
    const float cur = params[bt.param_off[p] + j];
    write_param(bt, p, j, params, __fsub_rn(cur, __fmul_rn(lr, __fmul_rn(acc, inv))));
  }
}

// shadow[c * rows + r] = block[r * cols + c] (after a host parameter upload)
__global__ void transpose_kernel(const float* __restrict__ src, int rows, int cols, int swz,
                                 float* __restrict__ dst) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += gridDim.x * blockDim.x) {
    const int r = e / cols, c = e - r * cols;
    dst[shadow_index(r, c, rows, swz)] = src[e];
  }
}

// Grid-wide barrier for a grid whose CTAs are all co-resident (one per SM,
// checked by the host). The counter only grows: each launch adds gridDim.x,
// and a CTA waits for the next multiple of gridDim.x, so no reset is needed
// between launches. Writes before the barrier are visible after it (CTA
// barrier + gpu-scope fence by the arriving thread, acquire on the wait).
__device__ __forceinline__ void grid_barrier(unsigned long long* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long old = atomicAdd(ctr, 1ull);
    const unsigned long long target = (old / gridDim.x + 1) * gridDim.x;
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
      __nanosleep(32);
    }
  }
  __syncthreads();
}

// IDX payload bytes -> fp32 (io::load_idx + load_mnist's / 255,
// proj/core/src/dataset.cpp:77-80,98-103): float(b), divided when scale > 0
__global__ void decode_u8_kernel(const unsigned char* __restrict__ b, long long n, float scale,
                                 float* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float v = (float)b[i];
    out[i] = scale > 0.0f ? __fdiv_rn(v, scale) : v;
  }
}

// device-side step counter of the multi-step graphs
__global__ void set_counter_kernel(long long* v, long long value) { *v = value; }
__global__ void advance_counter_kernel(long long* v, long long by) { *v += by; }

// Holds the stream for `ns` nanoseconds (profiling: lets the host queue a
// whole instrumented step before the GPU starts it).
__global__ void spin_kernel(long long ns) {
  long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 >= ns) break;
    __nanosleep(10000);
  }
}

__global__ void gaussian_kernel(uint64_t key, long long n, float* __restrict__ out) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; 2 * q < n;
       q += (long long)gridDim.x * blockDim.x) {
    float c, s;
    gauss_pair(key, q, &c, &s);
    out[2 * q] = c;
    if (2 * q + 1 < n) out[2 * q + 1] = s;
  }
}

}  // namespace pgb
