// Fused per-example DPSGD kernel for the reference MNIST CNN
// (proj/core/src/models.cpp:107-121):
//   conv(1->16, 8x8, s2, p3) relu maxpool(2,2) conv(16->32, 4x4) relu flatten
//   dense(512->32) relu dense(32->10), softmax cross-entropy.
// One CTA owns one example end to end: forward, loss, backward, the
// per-example weight gradients of both convolutions (written to the stacks,
// strategies.cpp:156-170), the dense-layer factors a_i / delta_i for the
// ghost-norm representation of the dense blocks (strategies.cpp:140-154),
// and the example's squared global gradient norm in fp64 (dpsgd.cpp:254-270).
// Every activation stays in shared memory; HBM sees the input image, the
// parameters (L2-resident, shared by all CTAs) and the gradient outputs.
#pragma once

#include "kernels.cuh"

namespace pgb {
namespace mnist {

constexpr int H0 = 28, XP = 34;            // input, padded input (pad 3)
constexpr int D1 = 16, K1 = 8, O1 = 14;    // conv1 out 16x14x14
constexpr int PO = 7;                      // pooled 16x7x7
constexpr int C2 = 16, D2 = 32, K2 = 4, O2 = 4;
constexpr int KC2 = C2 * K2 * K2;          // 256 = im2col rows of conv2
constexpr int NP2 = O2 * O2;               // 16 conv2 output positions
constexpr int F1 = 512, H1 = 32, NC = 10;
constexpr int NT = 256;
constexpr int W2S = 33;                    // padded stride of the transposed conv2 weights

struct Smem {
  float xs[XP * XP];                 // padded input
  float w1[D1 * K1 * K1];            // conv1 weights [d][u][v]
  float b1[D1];
  float b2[D2];
  float a1[D1 * O1 * O1];            // relu(conv1)
  union {
    float p1[D1 * PO * PO];          // maxpool output
    float dp1[D1 * PO * PO];         // its cotangent (p1 is dead by then)
  } up;
  float w2t[KC2 * W2S];              // conv2 weights [c,u,v][d] (padded)
  float buf[KC2 * NP2];              // conv2 im2col [k][pos] -> [pos][k] -> dcols [pos][k]
  union {
    float part[8 * NP2 * D2];        // split-K partials of conv2 fwd [w][pos][d]
    float z1[8 * H1];                // fc1 split partials
    float d1[O1 * O1 * D1];          // d conv1-linear [pos][d]
  } u1;
  float a2[F1];                      // relu(conv2) = fc1 input (flatten order)
  float dc2[NP2 * D2];               // d conv2-linear [pos][d]
  float h[H1], dz1[H1], dz2[16], logits[16];
  double red[NT / 32];
  unsigned char pidx[D1 * PO * PO];  // first-max window slot
};

struct Params {
  const float* x;       // (B, 1, 28, 28) or null: read from args
  const float* y;       // (B)
  const float* w;       // flat parameters
  long long off[8];     // parameter block offsets
  float* st_c1w;        // (B, 1024)   per-example conv1 dW
  float* st_c1b;        // (B, 16)
  float* st_c2w;        // (B, 8192)
  float* st_c2b;        // (B, 32)
  float* a2;            // (B, 512)    fc1 input
  float* dz1;           // (B, 32)     fc1 output cotangent (= fc1 bias grad)
  float* h;             // (B, 32)     fc2 input
  float* dz2;           // (B, 10)     dlogits (= fc2 bias grad)
  float* loss;          // (B)
  double* normsq;       // (B)         squared global per-example norm
  DevError* err;
  int B;
};

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < NT / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  __syncthreads();
  return t;  // valid in thread 0
}

__global__ void __launch_bounds__(NT, 2) fused_kernel(Params prm) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int b = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const float* W = prm.w;
  const float* gW1 = W + prm.off[0];
  const float* gb1 = W + prm.off[1];
  const float* gW2 = W + prm.off[2];
  const float* gb2 = W + prm.off[3];
  const float* gW3 = W + prm.off[4];
  const float* gb3 = W + prm.off[5];
  const float* gW4 = W + prm.off[6];
  const float* gb4 = W + prm.off[7];
  const float* x = prm.x + (size_t)b * H0 * H0;

  // ---- stage input (zero-padded) and the conv weights ---------------------
  for (int i = t; i < XP * XP; i += NT) {
    const int r = i / XP - 3, c = i % XP - 3;
    S.xs[i] = (r >= 0 && r < H0 && c >= 0 && c < H0) ? __ldg(x + r * H0 + c) : 0.0f;
  }
  for (int i = t; i < D1 * K1 * K1; i += NT) S.w1[i] = __ldg(gW1 + i);
  if (t < D1) S.b1[t] = __ldg(gb1 + t);
  if (t < D2) S.b2[t] = __ldg(gb2 + t);
  for (int i = t; i < D2 * KC2; i += NT) {  // coalesced read, [k][d] write
    const int d = i / KC2, k = i % KC2;
    S.w2t[k * W2S + d] = __ldg(gW2 + i);
  }
  __syncthreads();

  // ---- conv1 + relu: one output position per thread, window in registers --
  if (t < O1 * O1) {
    const int oy = t / O1, ox = t % O1;
    float win[K1 * K1];
#pragma unroll
    for (int u = 0; u < K1; ++u)
#pragma unroll
      for (int v = 0; v < K1; ++v) win[u * K1 + v] = S.xs[(2 * oy + u) * XP + 2 * ox + v];
#pragma unroll 1
    for (int d = 0; d < D1; ++d) {
      const float4* w4 = reinterpret_cast<const float4*>(S.w1 + d * K1 * K1);
      float acc = 0.0f;
#pragma unroll
      for (int q = 0; q < K1 * K1 / 4; ++q) {
        const float4 wv = w4[q];
        acc = fmaf(wv.x, win[4 * q], acc);
        acc = fmaf(wv.y, win[4 * q + 1], acc);
        acc = fmaf(wv.z, win[4 * q + 2], acc);
        acc = fmaf(wv.w, win[4 * q + 3], acc);
      }
      S.a1[d * O1 * O1 + t] = fmaxf(acc + S.b1[d], 0.0f);
    }
  }
  __syncthreads();

  // ---- maxpool 2x2/2 (first max in window order, kernels.hpp:377-396) -------
  for (int i = t; i < D1 * PO * PO; i += NT) {
    const int c = i / (PO * PO), r = i % (PO * PO), py = r / PO, px = r % PO;
    const float* src = S.a1 + c * O1 * O1 + (2 * py) * O1 + 2 * px;
    float m = src[0];
    int slot = 0;
    if (src[1] > m) { m = src[1]; slot = 1; }
    if (src[O1] > m) { m = src[O1]; slot = 2; }
    if (src[O1 + 1] > m) { m = src[O1 + 1]; slot = 3; }
    S.up.p1[i] = m;
    S.pidx[i] = (unsigned char)slot;
  }
  __syncthreads();

  // ---- conv2 im2col: buf[k][pos], k = (c,u,v), pos = (oy,ox) -------------
  for (int i = t; i < KC2 * NP2; i += NT) {
    const int k = i / NP2, pos = i % NP2;
    const int c = k / 16, u = (k / 4) % 4, v = k % 4, oy = pos / 4, ox = pos % 4;
    S.buf[i] = S.up.p1[c * PO * PO + (oy + u) * PO + ox + v];
  }
  __syncthreads();

  // ---- conv2 + relu: lane = out channel, warp = K slice of 32, split-K ----
  {
    const int d = lane;
    float acc[NP2];
#pragma unroll
    for (int p = 0; p < NP2; ++p) acc[p] = 0.0f;
    for (int kk = 0; kk < 32; ++kk) {
      const int k = warp * 32 + kk;
      const float w = S.w2t[k * W2S + d];
      const float4* cr = reinterpret_cast<const float4*>(S.buf + k * NP2);
#pragma unroll
      for (int q = 0; q < NP2 / 4; ++q) {
        const float4 c4 = cr[q];
        acc[4 * q] = fmaf(w, c4.x, acc[4 * q]);
        acc[4 * q + 1] = fmaf(w, c4.y, acc[4 * q + 1]);
        acc[4 * q + 2] = fmaf(w, c4.z, acc[4 * q + 2]);
        acc[4 * q + 3] = fmaf(w, c4.w, acc[4 * q + 3]);
      }
    }
#pragma unroll
    for (int p = 0; p < NP2; ++p) S.u1.part[(warp * NP2 + p) * D2 + d] = acc[p];
  }
  __syncthreads();
  for (int i = t; i < D2 * NP2; i += NT) {  // i = pos*32 + d
    const int d = i % D2, p = i / D2;
    float s = 0.0f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += S.u1.part[w * D2 * NP2 + i];
    S.a2[d * NP2 + p] = fmaxf(s + S.b2[d], 0.0f);
  }
  // the patches again, transposed, for the per-example dW: buf[pos][k]
  for (int i = t; i < KC2 * NP2; i += NT) {
    const int pos = i / KC2, k = i % KC2;
    const int c = k / 16, u = (k / 4) % 4, v = k % 4, oy = pos / 4, ox = pos % 4;
    S.buf[i] = S.up.p1[c * PO * PO + (oy + u) * PO + ox + v];
  }
  __syncthreads();

  // ---- fc1 (512->32) + relu: lane = unit, warp = 64-row slice --------------
  {
    float s = 0.0f;
    #pragma unroll 16
    for (int i = warp * 64; i < warp * 64 + 64; ++i) s = fmaf(S.a2[i], __ldg(gW3 + i * H1 + lane), s);
    S.u1.z1[warp * H1 + lane] = s;
  }
  __syncthreads();
  if (warp == 0) {
    float z = __ldg(gb3 + lane);
#pragma unroll
    for (int w = 0; w < 8; ++w) z += S.u1.z1[w * H1 + lane];
    const float hv = fmaxf(z, 0.0f);
    S.h[lane] = hv;
    __syncwarp();
    // fc2 (32->10) + softmax cross-entropy (kernels.hpp:516-566)
    float lg = 0.0f;
    if (lane < NC) {
      lg = __ldg(gb4 + lane);
      for (int j = 0; j < H1; ++j) lg = fmaf(S.h[j], __ldg(gW4 + j * NC + lane), lg);
      S.logits[lane] = lg;
    }
    __syncwarp();
    const float raw = prm.y[b];
    const bool ok = valid_id(raw, NC);
    if (!ok && lane == 0) raise_index(prm.err, 0, b, raw, NC);
    const int y = ok ? (int)raw : 0;
    float m = S.logits[0];
    for (int c = 1; c < NC; ++c) m = fmaxf(m, S.logits[c]);
    float se = 0.0f;
    for (int c = 0; c < NC; ++c) se += expf(S.logits[c] - m);
    if (lane < NC) {
      const float g = ok ? expf(lg - m) / se - (lane == y ? 1.0f : 0.0f) : 0.0f;
      S.dz2[lane] = g;
    }
    if (lane == 0) prm.loss[b] = ok ? m + logf(se) - S.logits[y] : 0.0f;
    __syncwarp();
    // dz1 = (W4 dz2) * [h > 0]
    float g1 = 0.0f;
    for (int c = 0; c < NC; ++c) g1 = fmaf(__ldg(gW4 + lane * NC + c), S.dz2[c], g1);
    S.dz1[lane] = hv > 0.0f ? g1 : 0.0f;
  }
  __syncthreads();

  // ---- fc1 backward data: da2[i] = W3[i,:] . dz1, relu mask -> dc2 --------
  for (int i = warp; i < F1; i += NT / 32) {
    float v = __ldg(gW3 + i * H1 + lane) * S.dz1[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) {
      const int d = i / NP2, pos = i % NP2;
      S.dc2[pos * D2 + d] = S.a2[i] > 0.0f ? v : 0.0f;
    }
  }
  __syncthreads();

  double sq = 0.0;  // this thread's share of ||g_i||^2
  const size_t bo = (size_t)b;

  // ---- conv2 per-example dW: thread = k (c,u,v), loop d ---------------------
  {
    const int k = t;  // NT == KC2
    float cv[NP2];
#pragma unroll
    for (int p = 0; p < NP2; ++p) cv[p] = S.buf[p * KC2 + k];
    float* out = prm.st_c2w + bo * (D2 * KC2);
#pragma unroll 2
    for (int d = 0; d < D2; ++d) {
      float acc = 0.0f;
#pragma unroll
      for (int p = 0; p < NP2; ++p) acc = fmaf(S.dc2[p * D2 + d], cv[p], acc);
      out[d * KC2 + k] = acc;
      sq += (double)acc * acc;
    }
  }
  if (t < D2) {  // conv2 bias
    float s = 0.0f;
    for (int p = 0; p < NP2; ++p) s += S.dc2[p * D2 + t];
    prm.st_c2b[bo * D2 + t] = s;
    sq += (double)s * s;
  }

  __syncthreads();  // buf (patches) is overwritten with dcols below

  // ---- conv2 backward data: dcols[pos][k] = sum_d W2[d][k] dc2[d][pos] ------
  {
    const int k = t;
    float wr[D2];
#pragma unroll
    for (int d = 0; d < D2; ++d) wr[d] = S.w2t[k * W2S + d];
#pragma unroll 1
    for (int p = 0; p < NP2; ++p) {
      const float4* g4 = reinterpret_cast<const float4*>(S.dc2 + p * D2);
      float acc = 0.0f;
#pragma unroll
      for (int q = 0; q < D2 / 4; ++q) {
        const float4 g = g4[q];
        acc = fmaf(wr[4 * q], g.x, acc);
        acc = fmaf(wr[4 * q + 1], g.y, acc);
        acc = fmaf(wr[4 * q + 2], g.z, acc);
        acc = fmaf(wr[4 * q + 3], g.w, acc);
      }
      S.buf[p * KC2 + k] = acc;
    }
  }
  __syncthreads();
  // col2im as a gather: dp1[c][iy][ix] = sum_{u,v} dcols[(c,u,v)][(iy-u, ix-v)]
  for (int i = t; i < D1 * PO * PO; i += NT) {
    const int c = i / (PO * PO), r = i % (PO * PO), iy = r / PO, ix = r % PO;
    float s = 0.0f;
    for (int u = 0; u < K2; ++u) {
      const int oy = iy - u;
      if (oy < 0 || oy >= O2) continue;
      for (int v = 0; v < K2; ++v) {
        const int ox = ix - v;
        if (ox < 0 || ox >= O2) continue;
        s += S.buf[(oy * O2 + ox) * KC2 + c * 16 + u * 4 + v];
      }
    }
    S.up.dp1[i] = s;
  }
  __syncthreads();
  // maxpool backward (route to the first max) + relu mask on a1 -> d1 [pos][d]
  for (int i = t; i < D1 * O1 * O1; i += NT) {  // i = pos*16 + d
    const int d = i % D1, r = i / D1, oy = r / O1, ox = r % O1;
    const int pi = d * PO * PO + (oy / 2) * PO + ox / 2;
    const int slot = (oy & 1) * 2 + (ox & 1);
    const float g = (S.pidx[pi] == slot && S.a1[d * O1 * O1 + r] > 0.0f) ? S.up.dp1[pi] : 0.0f;
    S.u1.d1[i] = g;
  }
  __syncthreads();

  // ---- conv1 per-example dW: thread = (tap, group of 4 channels) ------------
  {
    const int k = t % (K1 * K1), dg = t / (K1 * K1);
    const int u = k / K1, v = k % K1;
    float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
    for (int oy = 0; oy < O1; ++oy) {
      const float* xr = S.xs + (2 * oy + u) * XP + v;
#pragma unroll 2
      for (int ox = 0; ox < O1; ++ox) {
        const float xv = xr[2 * ox];
        const float4 g = reinterpret_cast<const float4*>(S.u1.d1 + (oy * O1 + ox) * D1)[dg];
        acc0 = fmaf(g.x, xv, acc0);
        acc1 = fmaf(g.y, xv, acc1);
        acc2 = fmaf(g.z, xv, acc2);
        acc3 = fmaf(g.w, xv, acc3);
      }
    }
    float* out = prm.st_c1w + bo * (D1 * K1 * K1);
    out[(4 * dg + 0) * 64 + k] = acc0;
    out[(4 * dg + 1) * 64 + k] = acc1;
    out[(4 * dg + 2) * 64 + k] = acc2;
    out[(4 * dg + 3) * 64 + k] = acc3;
    sq += (double)acc0 * acc0 + (double)acc1 * acc1 + (double)acc2 * acc2 + (double)acc3 * acc3;
  }
  if (t < D1) {  // conv1 bias
    float s = 0.0f;
    for (int p = 0; p < O1 * O1; ++p) s += S.u1.d1[p * D1 + t];
    prm.st_c1b[bo * D1 + t] = s;
    sq += (double)s * s;
  }

  // ---- dense factors for the ghost-norm blocks + their norm terms ----------
  double a2sq = 0.0;
  for (int i = t; i < F1; i += NT) {
    const float v = S.a2[i];
    prm.a2[bo * F1 + i] = v;
    a2sq += (double)v * v;
  }
  double hsq = 0.0, dz1sq = 0.0, dz2sq = 0.0;
  if (t < H1) {
    const float hv = S.h[t], g = S.dz1[t];
    prm.h[bo * H1 + t] = hv;
    prm.dz1[bo * H1 + t] = g;
    hsq = (double)hv * hv;
    dz1sq = (double)g * g;
  }
  if (t < NC) {
    const float g = S.dz2[t];
    prm.dz2[bo * NC + t] = g;
    dz2sq = (double)g * g;
  }
  const double tot = block_sum(sq, S.red);
  const double A2 = block_sum(a2sq, S.red);
  const double Hs = block_sum(hsq, S.red);
  const double G1 = block_sum(dz1sq, S.red);
  const double G2 = block_sum(dz2sq, S.red);
  if (t == 0) {
    // ||a (x) d||^2 = ||a||^2 ||d||^2 (weight) + ||d||^2 (bias), strategies.cpp:140-148
    prm.normsq[b] = tot + G1 * (A2 + 1.0) + G2 * (Hs + 1.0);
  }
}

}  // namespace mnist
}  // namespace pgb
