// Fused per-example DPSGD kernel for the reference MNIST CNN
// (proj/core/src/models.cpp:107-121):
//   conv(1->16, 8x8, s2, p3) relu maxpool(2,2) conv(16->32, 4x4) relu flatten
//   dense(512->32) relu dense(32->10), softmax cross-entropy.
// One CTA owns one example end to end: forward, loss, backward, the
// per-example weight gradients of both convolutions (written to the stacks,
// strategies.cpp:156-170), the dense-layer factors a_i / delta_i for the
// ghost-norm representation of the dense blocks (strategies.cpp:140-154),
// and the example's squared global gradient norm in fp64 (dpsgd.cpp:254-270).
// Every activation stays in shared memory. The image and the conv weights
// arrive by TMA bulk copies (cp.async.bulk + mbarrier); the conv2 weights
// are read from a transposed copy the update kernel keeps in step.
#pragma once

#include "kernels.cuh"

namespace pgb {
namespace mnist {

constexpr int H0 = 28, XP = 34;            // input, padded input (pad 3)
constexpr int XS = 40;                     // xs row stride (bank-conflict-free taps)
constexpr int D1 = 16, K1 = 8, O1 = 14;    // conv1 out 16x14x14
constexpr int PO = 7;                      // pooled 16x7x7
constexpr int C2 = 16, D2 = 32, K2 = 4, O2 = 4;
constexpr int KC2 = C2 * K2 * K2;          // 256 = im2col rows of conv2
constexpr int NP2 = O2 * O2;               // 16 conv2 output positions
constexpr int F1 = 512, H1 = 32, NC = 10;
constexpr int NT = 256;

struct Smem {
  float w2t[KC2 * D2];               // conv2 weights [k=(c,u,v)][d]   (TMA)
  float w1[D1 * K1 * K1];            // conv1 weights [d][u][v]        (TMA)
  float b1[D1];                      //                                (TMA)
  float b2[D2];                      //                                (TMA)
  float xs[XP * XS];                 // padded input, row stride XS
  float a1[D1 * O1 * O1];            // relu(conv1)
  union {
    float p1[D1 * PO * PO];          // maxpool output
    float dp1[D1 * PO * PO];         // its cotangent (p1 is dead by then)
  } up;
  float buf[KC2 * NP2];              // conv2 im2col [k][pos] -> [pos][k] -> dcols [pos][k]
  union {
    float xstage[H0 * H0];           // raw image (TMA), padded into xs
    float part[8 * NP2 * D2];        // split-K partials of conv2 fwd [w][pos][d]
    float z1[8 * H1];                // fc1 split partials
    float d1[O1 * O1 * D1];          // d conv1-linear [pos][d]
  } u1;
  float a2[F1];                      // relu(conv2) = fc1 input (flatten order)
  float dc2[NP2 * D2];               // d conv2-linear [pos][d]
  float dc2t[D2 * NP2];              // the same, [d][pos]
  float h[H1], dz1[H1], dz2[16], logits[16];
  double red5[5][NT / 32];
  unsigned long long bar;            // mbarrier of the bulk copies
  unsigned char pidx[D1 * PO * PO];  // first-max window slot
};

struct Params {
  const float* x;       // (B, 1, 28, 28)
  const float* y;       // (B)
  const float* w;       // flat parameters
  const float* w2t;     // conv2 weights transposed, (256, 32)
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

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// TMA bulk global->shared copy completing on an mbarrier (SASS: UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}

__global__ void __launch_bounds__(NT, 2) fused_kernel(Params prm) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int b = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const float* W = prm.w;
  const float* gW3 = W + prm.off[4];
  const float* gb3 = W + prm.off[5];
  const float* gW4 = W + prm.off[6];
  const float* gb4 = W + prm.off[7];

  // ---- TMA: image + conv weights + biases into shared memory --------------
  constexpr uint32_t kBytes = sizeof(float) * (H0 * H0 + D1 * K1 * K1 + D1 + D2 + KC2 * D2);
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(&S.bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_addr(&S.bar)), "r"(kBytes) : "memory");
    bulk_g2s(S.u1.xstage, prm.x + (size_t)b * H0 * H0, sizeof(float) * H0 * H0, &S.bar);
    bulk_g2s(S.w1, W + prm.off[0], sizeof(float) * D1 * K1 * K1, &S.bar);
    bulk_g2s(S.b1, W + prm.off[1], sizeof(float) * D1, &S.bar);
    bulk_g2s(S.b2, W + prm.off[3], sizeof(float) * D2, &S.bar);
    bulk_g2s(S.w2t, prm.w2t, sizeof(float) * KC2 * D2, &S.bar);
  }
  // zero the padding ring of xs while the copies fly
  for (int i = t; i < XP * XS; i += NT) {
    const int r = i / XS - 3, c = i % XS - 3;
    if (!(r >= 0 && r < H0 && c >= 0 && c < H0)) S.xs[i] = 0.0f;
  }
  __syncthreads();  // barrier initialised before anyone waits on it
  {
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; "
          "selp.u32 %0, 1, 0, p; }"
          : "=r"(done) : "r"(smem_addr(&S.bar)) : "memory");
  }
  for (int i = t; i < H0 * H0; i += NT) S.xs[(i / H0 + 3) * XS + i % H0 + 3] = S.u1.xstage[i];
  __syncthreads();

  // ---- conv1 + relu: one output position per thread, window in registers --
  if (t < O1 * O1) {
    const int oy = t / O1, ox = t % O1;
    float win[K1 * K1];
#pragma unroll
    for (int u = 0; u < K1; ++u)
#pragma unroll
      for (int v = 0; v < K1; ++v) win[u * K1 + v] = S.xs[(2 * oy + u) * XS + 2 * ox + v];
#pragma unroll 2
    for (int d = 0; d < D1; ++d) {
      const float4* w4 = reinterpret_cast<const float4*>(S.w1 + d * K1 * K1);
      float acc0 = 0.0f, acc1 = 0.0f;
#pragma unroll
      for (int q = 0; q < K1 * K1 / 4; ++q) {
        const float4 wv = w4[q];
        acc0 = fmaf(wv.x, win[4 * q], acc0);
        acc1 = fmaf(wv.y, win[4 * q + 1], acc1);
        acc0 = fmaf(wv.z, win[4 * q + 2], acc0);
        acc1 = fmaf(wv.w, win[4 * q + 3], acc1);
      }
      S.a1[d * O1 * O1 + t] = fmaxf(acc0 + acc1 + S.b1[d], 0.0f);
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
#pragma unroll 4
    for (int kk = 0; kk < 32; ++kk) {
      const int k = warp * 32 + kk;
      const float w = S.w2t[k * D2 + d];
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
    float wv[64];
#pragma unroll
    for (int r = 0; r < 64; ++r) wv[r] = __ldg(gW3 + (warp * 64 + r) * H1 + lane);
    float s0 = 0.0f, s1 = 0.0f;
#pragma unroll
    for (int r = 0; r < 64; r += 2) {
      s0 = fmaf(S.a2[warp * 64 + r], wv[r], s0);
      s1 = fmaf(S.a2[warp * 64 + r + 1], wv[r + 1], s1);
    }
    S.u1.z1[warp * H1 + lane] = s0 + s1;
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
#pragma unroll
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
#pragma unroll
    for (int c = 0; c < NC; ++c) g1 = fmaf(__ldg(gW4 + lane * NC + c), S.dz2[c], g1);
    S.dz1[lane] = hv > 0.0f ? g1 : 0.0f;
  }
  __syncthreads();

  // ---- fc1 backward data: da2[i] = W3[i,:] . dz1, relu mask -> dc2 --------
  {
    const float4* g4 = reinterpret_cast<const float4*>(S.dz1);
#pragma unroll
    for (int rr = 0; rr < F1 / NT; ++rr) {
      const int i = t + rr * NT;
      const float4* w4 = reinterpret_cast<const float4*>(gW3 + i * H1);
      float4 wv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) wv[q] = __ldg(w4 + q);
      float s0 = 0.0f, s1 = 0.0f;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 g = g4[q];
        s0 = fmaf(wv[q].x, g.x, s0);
        s1 = fmaf(wv[q].y, g.y, s1);
        s0 = fmaf(wv[q].z, g.z, s0);
        s1 = fmaf(wv[q].w, g.w, s1);
      }
      const float v = S.a2[i] > 0.0f ? s0 + s1 : 0.0f;
      const int d = i / NP2, pos = i % NP2;
      S.dc2[pos * D2 + d] = v;
      S.dc2t[i] = v;  // [d][pos] == flatten order
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
#pragma unroll 4
    for (int d = 0; d < D2; ++d) {
      const float4* g4 = reinterpret_cast<const float4*>(S.dc2t + d * NP2);
      float acc0 = 0.0f, acc1 = 0.0f;
#pragma unroll
      for (int q = 0; q < NP2 / 4; ++q) {
        const float4 g = g4[q];
        acc0 = fmaf(g.x, cv[4 * q], acc0);
        acc1 = fmaf(g.y, cv[4 * q + 1], acc1);
        acc0 = fmaf(g.z, cv[4 * q + 2], acc0);
        acc1 = fmaf(g.w, cv[4 * q + 3], acc1);
      }
      const float acc = acc0 + acc1;
      out[d * KC2 + k] = acc;
      sq = fma((double)acc, (double)acc, sq);
    }
  }
  if (t < D2) {  // conv2 bias
    float s = 0.0f;
    for (int p = 0; p < NP2; ++p) s += S.dc2t[t * NP2 + p];
    prm.st_c2b[bo * D2 + t] = s;
    sq = fma((double)s, (double)s, sq);
  }
  __syncthreads();  // buf (patches) is overwritten with dcols below

  // ---- conv2 backward data: dcols[pos][(u,v),c] = sum_d W2[d][c,u,v] dc2[d][pos]
  {
    const int c = t % C2, uv = t / C2, k = c * 16 + uv;  // lanes: consecutive c
    const float* gW2 = W + prm.off[2];
    float wr[D2];
#pragma unroll
    for (int d = 0; d < D2; ++d) wr[d] = __ldg(gW2 + d * KC2 + k);
#pragma unroll 2
    for (int p = 0; p < NP2; ++p) {
      const float4* g4 = reinterpret_cast<const float4*>(S.dc2 + p * D2);
      float acc0 = 0.0f, acc1 = 0.0f;
#pragma unroll
      for (int q = 0; q < D2 / 4; ++q) {
        const float4 g = g4[q];
        acc0 = fmaf(wr[4 * q], g.x, acc0);
        acc1 = fmaf(wr[4 * q + 1], g.y, acc1);
        acc0 = fmaf(wr[4 * q + 2], g.z, acc0);
        acc1 = fmaf(wr[4 * q + 3], g.w, acc1);
      }
      S.buf[p * KC2 + t] = acc0 + acc1;
    }
  }
  __syncthreads();
  // col2im as a gather: dp1[c][iy][ix] = sum_{u,v} dcols[(iy-u, ix-v)][(u,v),c]
  for (int i = t; i < D1 * PO * PO; i += NT) {  // i = (iy*7+ix)*16 + c
    const int c = i % C2, r = i / C2, iy = r / PO, ix = r % PO;
    float s = 0.0f;
#pragma unroll
    for (int u = 0; u < K2; ++u) {
      const int oy = iy - u;
      if (oy < 0 || oy >= O2) continue;
#pragma unroll
      for (int v = 0; v < K2; ++v) {
        const int ox = ix - v;
        if (ox < 0 || ox >= O2) continue;
        s += S.buf[(oy * O2 + ox) * KC2 + (u * 4 + v) * C2 + c];
      }
    }
    S.up.dp1[c * PO * PO + r] = s;
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

  // ---- conv1 per-example dW: thread = (tap, 8 channels, half of the rows) ---
  {
    const int k = t % (K1 * K1), dg = (t / (K1 * K1)) & 1, half = t / (2 * K1 * K1);
    const int u = k / K1, v = k % K1;
    float acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = 0.0f;
    for (int oy = half * 7; oy < half * 7 + 7; ++oy) {
      const float* xr = S.xs + (2 * oy + u) * XS + v;
      const float4* g4 = reinterpret_cast<const float4*>(S.u1.d1 + oy * O1 * D1) + 2 * dg;
#pragma unroll 7
      for (int ox = 0; ox < O1; ++ox) {
        const float xv = xr[2 * ox];
        const float4 ga = g4[ox * 4];
        const float4 gb = g4[ox * 4 + 1];
        acc[0] = fmaf(ga.x, xv, acc[0]);
        acc[1] = fmaf(ga.y, xv, acc[1]);
        acc[2] = fmaf(ga.z, xv, acc[2]);
        acc[3] = fmaf(ga.w, xv, acc[3]);
        acc[4] = fmaf(gb.x, xv, acc[4]);
        acc[5] = fmaf(gb.y, xv, acc[5]);
        acc[6] = fmaf(gb.z, xv, acc[6]);
        acc[7] = fmaf(gb.w, xv, acc[7]);
      }
    }
    // combine the two row halves through shared memory (buf is free)
    if (half == 1) {
#pragma unroll
      for (int c = 0; c < 8; ++c) S.buf[(dg * 8 + c) * 64 + k] = acc[c];
    }
    __syncthreads();
    if (half == 0) {
      float* out = prm.st_c1w + bo * (D1 * K1 * K1);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int d = dg * 8 + c;
        const float g = acc[c] + S.buf[d * 64 + k];
        out[d * 64 + k] = g;
        sq = fma((double)g, (double)g, sq);
      }
    }
  }
  if (t < D1) {  // conv1 bias
    float s = 0.0f;
    for (int p = 0; p < O1 * O1; ++p) s += S.u1.d1[p * D1 + t];
    prm.st_c1b[bo * D1 + t] = s;
    sq = fma((double)s, (double)s, sq);
  }

  // ---- dense factors for the ghost-norm blocks + their norm terms ----------
  double a2sq = 0.0;
  for (int i = t; i < F1; i += NT) {
    const float v = S.a2[i];
    prm.a2[bo * F1 + i] = v;
    a2sq = fma((double)v, (double)v, a2sq);
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
  // one block-wide reduction of the five fp64 norm terms
  double v5[5] = {sq, a2sq, hsq, dz1sq, dz2sq};
#pragma unroll
  for (int q = 0; q < 5; ++q)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v5[q] += __shfl_xor_sync(0xffffffffu, v5[q], o);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < 5; ++q) S.red5[q][warp] = v5[q];
  __syncthreads();
  if (t == 0) {
    double r5[5] = {0, 0, 0, 0, 0};
    for (int w = 0; w < NT / 32; ++w)
#pragma unroll
      for (int q = 0; q < 5; ++q) r5[q] += S.red5[q][w];
    // ||a (x) d||^2 = ||a||^2 ||d||^2 (weight) + ||d||^2 (bias), strategies.cpp:140-148
    prm.normsq[b] = r5[0] + r5[3] * (r5[1] + 1.0) + r5[4] * (r5[2] + 1.0);
  }
}

}  // namespace mnist
}  // namespace pgb
