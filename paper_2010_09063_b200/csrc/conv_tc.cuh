// Convolution GEMMs of the layer-wise engine on tcgen05 (3xTF32, TMEM
// accumulators) through tc::tc_gemm_kernel: implicit im2col, no patch
// matrix in HBM. Rows/columns follow the reference's im2col order (c,u,v)
// (kernels.hpp:412-440) and its NCHW layouts.
//
//   forward        C[(b,pos)][d]   = sum_(c,u,v) x[b,c,iy,ix] W[d,(c,u,v)]   (+bias, relu)
//   per-example dW C_b[(c,u,v)][d] = sum_pos   x[b,c,iy,ix] dz[b,d,pos]     (strategies.cpp:156-170)
//   input grad     C[(b,iy,ix)][c] = sum_(d,u',v') dz[b,d,iy+u'-(k-1-p),..] W[d,c,k-1-u',k-1-v']
//                  (stride 1: the im2col VJP col2im as a flipped "full" convolution;
//                   other strides use the divisibility-checked gather)
#pragma once

#include "kernels.cuh"
#include "tc.cuh"

namespace pgb {
namespace tc {

struct TcConvFwdOp {
  static constexpr bool kTableA = true;
  int M, N, K;  // M = B*Ho*Wo, N = D, K = C*k*k
  ConvGeom g;
  const float* x;
  const float* W;
  const float* bias;
  float* out;
  int relu;
  __device__ const float* img(int) const { return x; }
  __device__ int img_h() const { return g.H; }
  __device__ int img_w() const { return g.W; }
  __device__ int4 row_info(int, int m) const {
    if (m >= M) return make_int4(0, 0, 0, 0);
    const int P = g.Ho * g.Wo;
    const int bb = m / P, p = m - bb * P;
    const int oy = p / g.Wo, ox = p - oy * g.Wo;
    return make_int4(bb * g.C * g.H * g.W, oy * g.stride - g.pad, ox * g.stride - g.pad, 1);
  }
  __device__ int4 k_info(int, int k) const {
    if (k >= K) return make_int4(0, 0, 0, 0);
    const int kk2 = g.k * g.k;
    const int c = k / kk2, r = k - c * kk2;
    const int u = r / g.k, v = r - u * g.k;
    return make_int4(c * g.H * g.W, u, v, 1);
  }
  __device__ float b(int, int n, int k) const { return __ldg(W + (size_t)n * K + k); }
  __device__ void store(int, int m, int n, float v) const {
    const int P = g.Ho * g.Wo;
    const int bb = m / P, p = m - bb * P;
    v += bias[n];
    out[((size_t)bb * g.D + n) * P + p] = relu ? fmaxf(v, 0.0f) : v;
  }
};

struct TcConvDWOp {
  static constexpr bool kTableA = true;
  int M, N, K;  // M = C*k*k, N = D, K = Ho*Wo; one GEMM per example z
  ConvGeom g;
  const float* x;     // (B, C, H, W)
  const float* gout;  // (B, D, Ho, Wo)
  float* stack;       // (B, D*C*k*k)
  double* tile_sq;    // (B, tiles): each tile's squared sum (the block's per-example norm)
  __device__ const float* img(int z) const { return x + (size_t)z * g.C * g.H * g.W; }
  __device__ int img_h() const { return g.H; }
  __device__ int img_w() const { return g.W; }
  __device__ int4 row_info(int, int m) const {
    if (m >= M) return make_int4(0, 0, 0, 0);
    const int kk2 = g.k * g.k;
    const int c = m / kk2, r = m - c * kk2;
    const int u = r / g.k, v = r - u * g.k;
    return make_int4(c * g.H * g.W, u - g.pad, v - g.pad, 1);
  }
  __device__ int4 k_info(int, int k) const {
    if (k >= K) return make_int4(0, 0, 0, 0);
    const int oy = k / g.Wo, ox = k - oy * g.Wo;
    return make_int4(0, oy * g.stride, ox * g.stride, 1);
  }
  __device__ float b(int z, int n, int k) const {
    return __ldg(gout + ((size_t)z * g.D + n) * K + k);
  }
  // four consecutive positions k..k+3 (k % 4 == 0) of one output row: one
  // index computation, the zero padding only at the row's ends
  __device__ bool vec_ok() const { return g.stride == 1 && g.Wo % 4 == 0 && K % 4 == 0; }
  __device__ float4 a4(int z, const int4& ri, int k) const {
    float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    if (!ri.w || k >= K) return v;
    const int oy = k / g.Wo, ox = k - oy * g.Wo;
    const int iy = ri.y + oy;
    if ((unsigned)iy >= (unsigned)g.H) return v;
    const float* row = img(z) + ri.x + (size_t)iy * g.W;
    const int ix = ri.z + ox;
    v.x = (unsigned)(ix) < (unsigned)g.W ? __ldg(row + ix) : 0.0f;
    v.y = (unsigned)(ix + 1) < (unsigned)g.W ? __ldg(row + ix + 1) : 0.0f;
    v.z = (unsigned)(ix + 2) < (unsigned)g.W ? __ldg(row + ix + 2) : 0.0f;
    v.w = (unsigned)(ix + 3) < (unsigned)g.W ? __ldg(row + ix + 3) : 0.0f;
    return v;
  }
  __device__ float4 b4(int z, int n, int k) const {
    if (n >= N || k >= K) return make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    return __ldg(reinterpret_cast<const float4*>(gout + ((size_t)z * g.D + n) * K + k));
  }
  __device__ void store(int z, int m, int n, float v) const {
    stack[(size_t)z * M * N + (size_t)n * M + m] = v;
  }
};

// stride-1 input gradient as a full convolution of dz with the flipped W
struct TcConvBwdXS1Op {
  static constexpr bool kTableA = true;
  int M, N, K;  // M = B*H*W, N = C, K = D*k*k (d, u', v')
  ConvGeom g;
  const float* gout;  // (B, D, Ho, Wo)
  const float* W;
  const float* mask;  // relu output of the input activation, or null
  float* gx;
  __device__ const float* img(int) const { return gout; }
  __device__ int img_h() const { return g.Ho; }
  __device__ int img_w() const { return g.Wo; }
  __device__ int4 row_info(int, int m) const {
    if (m >= M) return make_int4(0, 0, 0, 0);
    const int HW = g.H * g.W;
    const int bb = m / HW, q = m - bb * HW;
    const int iy = q / g.W, ix = q - iy * g.W;
    const int sh = g.k - 1 - g.pad;
    return make_int4(bb * g.D * g.Ho * g.Wo, iy - sh, ix - sh, 1);
  }
  __device__ int4 k_info(int, int k) const {
    if (k >= K) return make_int4(0, 0, 0, 0);
    const int kk2 = g.k * g.k;
    const int d = k / kk2, r = k - d * kk2;
    const int u = r / g.k, v = r - u * g.k;
    return make_int4(d * g.Ho * g.Wo, u, v, 1);
  }
  __device__ float b(int, int n, int k) const {
    const int kk2 = g.k * g.k;
    const int d = k / kk2, r = k - d * kk2;
    const int u = r / g.k, v = r - u * g.k;
    return __ldg(W + (((size_t)d * g.C + n) * g.k + (g.k - 1 - u)) * g.k + (g.k - 1 - v));
  }
  __device__ size_t gx_index(int m, int n) const {
    const int HW = g.H * g.W;
    const int bb = m / HW, q = m - bb * HW;
    return ((size_t)bb * g.C + n) * HW + q;
  }
  // the relu mask of an output element, loaded before any store of its
  // column group (tc_gemm_kernel: HasPre)
  __device__ float pre(int, int m, int n) const {
    return mask ? __ldg(mask + gx_index(m, n)) : 1.0f;
  }
  __device__ void store_pre(int, int m, int n, float v, float mk) const {
    gx[gx_index(m, n)] = !(mk > 0.0f) ? 0.0f : v;
  }
  __device__ void store(int z, int m, int n, float v) const { store_pre(z, m, n, v, pre(z, m, n)); }
};

// general stride: per-element gather with the divisibility check
struct TcConvBwdXOp {
  static constexpr bool kTableA = false;
  int M, N, K;  // M = B*H*W, N = C, K = D*k*k
  ConvGeom g;
  const float* gout;
  const float* W;
  const float* mask;
  float* gx;
  __device__ float a(int, int m, int k) const {
    const int HW = g.H * g.W;
    const int bb = m / HW, q = m - bb * HW;
    const int iy = q / g.W, ix = q - iy * g.W;
    const int kk2 = g.k * g.k;
    const int d = k / kk2, r = k - d * kk2;
    const int u = r / g.k, v = r - u * g.k;
    const int ny = iy + g.pad - u, nx = ix + g.pad - v;
    if (ny < 0 || nx < 0) return 0.0f;
    const int oy = ny / g.stride, ox = nx / g.stride;
    if (oy * g.stride != ny || ox * g.stride != nx || oy >= g.Ho || ox >= g.Wo) return 0.0f;
    return __ldg(gout + (((size_t)bb * g.D + d) * g.Ho + oy) * g.Wo + ox);
  }
  __device__ float b(int, int n, int k) const {
    const int kk2 = g.k * g.k;
    const int d = k / kk2, r = k - d * kk2;
    return __ldg(W + ((size_t)d * g.C + n) * kk2 + r);
  }
  __device__ size_t gx_index(int m, int n) const {
    const int HW = g.H * g.W;
    const int bb = m / HW, q = m - bb * HW;
    return ((size_t)bb * g.C + n) * HW + q;
  }
  // the relu mask of an output element, loaded before any store of its
  // column group (tc_gemm_kernel: HasPre)
  __device__ float pre(int, int m, int n) const {
    return mask ? __ldg(mask + gx_index(m, n)) : 1.0f;
  }
  __device__ void store_pre(int, int m, int n, float v, float mk) const {
    gx[gx_index(m, n)] = !(mk > 0.0f) ? 0.0f : v;
  }
  __device__ void store(int z, int m, int n, float v) const { store_pre(z, m, n, v, pre(z, m, n)); }
};

constexpr int kConvThreads = 256;

template <class Op, int BN>
inline void launch_bn(const Op& op, int batch, cudaStream_t s) {
  const size_t smem = sizeof(TcSmem<BN>);
  static unsigned long long attr_devs = 0;  // per instantiation, per device (bit = device)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 64 || !(attr_devs >> dev & 1ull)) {
    cudaFuncSetAttribute(tc_gemm_kernel<Op, BN, kConvThreads>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (dev < 64) attr_devs |= 1ull << dev;
  }
  dim3 grid((op.N + BN - 1) / BN, (op.M + kBM - 1) / kBM, batch);
  tc_gemm_kernel<Op, BN, kConvThreads><<<grid, kConvThreads, smem, s>>>(op);
}

// Output tiles of one GEMM launch() makes for (M, N) (tile_sq row length).
inline int tile_count(int M, int N) {
  const int bn = N <= 32 ? 32 : N <= 64 ? 64 : 128;
  return ((N + bn - 1) / bn) * ((M + kBM - 1) / kBM);
}

// Pick the column tile from N (TMEM holds 3 accumulators of BN columns).
template <class Op>
inline void launch(const Op& op, int batch, cudaStream_t s) {
  if (op.N <= 32)
    launch_bn<Op, 32>(op, batch, s);
  else if (op.N <= 64)
    launch_bn<Op, 64>(op, batch, s);
  else
    launch_bn<Op, 128>(op, batch, s);
}

}  // namespace tc
}  // namespace pgb
