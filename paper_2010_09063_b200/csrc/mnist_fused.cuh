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
//
// Shape of the launch: B = 256 examples on 148 SMs is at most two examples
// per SM, so per-SM throughput is set by how well two co-resident CTAs hide
// shared-memory and barrier latency. Each CTA therefore runs 16 warps (two
// CTAs = 32 warps per SM) with a 64-register budget; every phase is split so
// all 512 threads have work and per-thread state stays small.
#pragma once

#include "kernels.cuh"

namespace pgb {
namespace mnist {

constexpr int H0 = 28, XP = 34;            // input, padded input (pad 3)
constexpr int XS = 40;                     // xs row stride (bank-conflict-free taps)
constexpr int D1 = 16, K1 = 8, O1 = 14;    // conv1 out 16x14x14
constexpr int NP1 = O1 * O1;               // 196 conv1 output positions
constexpr int PO = 7;                      // pooled 16x7x7
constexpr int C2 = 16, D2 = 32, K2 = 4, O2 = 4;
constexpr int KC2 = C2 * K2 * K2;          // 256 = im2col rows of conv2
constexpr int NP2 = O2 * O2;               // 16 conv2 output positions
constexpr int F1 = 512, H1 = 32, NC = 10;
constexpr int DCP = K2 * K2 * 17;           // dcols row pitch: (u,v) rows of 16 c + 1 pad
constexpr int NT = 512;
constexpr int NW = NT / 32;

struct Smem {
  float w2t[KC2 * D2];               // conv2 weights, swizzled transpose (TMA):
                                     //   W2[d][k] at [k*32 + (d ^ (k & 31))]
  float w1t[K1 * K1 * D1];           // conv1 weights [(u,v)][d]       (TMA, transposed shadow)
  float b1[D1];                      //                                (TMA)
  float b2[D2];                      //                                (TMA)
  float xs[XP * XS];                 // padded input, row stride XS
  float a1[D1 * NP1];                // relu(conv1) [d][pos]
  union {
    float p1[D1 * PO * PO];          // maxpool output
    float dp1[D1 * PO * PO];         // its cotangent (p1 is dead by then)
  } up;
  float buf[NP2 * DCP];              // conv2 im2col (swizzled [k][pos]) -> dcols (padded
                                     // [pos][(u,v)][c]) -> conv1 dW partials
  union {
    float xstage[H0 * H0];           // raw image (TMA), padded into xs
    float part[8 * NP2 * D2];        // split-K partials of conv2 fwd [kslice][pos][d]
    float z1[NW * H1];               // fc1 split partials
    float d1[NP1 * D1];              // d conv1-linear [pos][d]
  } u1;
  float a2[F1];                      // relu(conv2) = fc1 input (flatten order [d][pos])
  float dc2[NP2 * D2];               // d conv2-linear [pos][d]
  float dc2t[D2 * NP2];              // the same, [d][pos]
  float h[H1], dz1[H1], dz2[16], logits[16];
  float w4[H1 * NC], b4[16], b3[H1];  // fc weights/biases needed by the loss tail
  float yb;                          // this example's label
  float b1red[NW][D1];               // per-warp partials of the conv1 bias gradient
  double red5[5][NW];
  unsigned long long bar[2];         // mbarriers: [0] image + conv1, [1] conv2
  unsigned char pidx[D1 * PO * PO];  // first-max window slot
};

struct Params {
  const float* x;       // (B, 1, 28, 28)
  const float* y;       // (B)
  const float* w;       // flat parameters
  const float* w2t;     // conv2 weights transposed, (256, 32), swizzled
  const float* w1t;     // conv1 weights transposed, (64, 16)
  long long off[8];     // parameter block offsets
  float* st_c1w;        // (B, 1024)   per-example conv1 dW
  float* st_c1b;        // (B, 16)
  float* st_c2w;        // (B, 8192)
  float* c2_pairs;      // tc_kernel, optional: ((B+1)/2, 8192) clipped pair rows of conv2 W
                        // written instead of st_c2w (the step's aggregation follows)
  float* st_c2b;        // (B, 32)
  float* a2;            // (B, 512)    fc1 input
  float* dz1;           // (B, 32)     fc1 output cotangent (= fc1 bias grad)
  float* h;             // (B, 32)     fc2 input
  float* dz2;           // (B, 10)     dlogits (= fc2 bias grad)
  float* loss;          // (B)
  double* normsq;       // (B)         squared global per-example norm
  DevError* err;
  int B;
  // step tail work done here so the aggregation kernel only streams:
  StepArgs a;           // the step's DP arguments
  float* norms;         // (B) pre-clip norms            (dpsgd.cpp:254-270)
  float* scale;         // (B) clip factors              (dpsgd.cpp:91-99)
  int* clipped;         // (B) 1 where norm > C
  float* noise;         // (P) the step's normals n_j    (dpsgd.cpp:308-316), or null
  long long size[8];    // parameter block sizes
  long long pair_off[9];  // prefix sums of ceil(|p| / 2)
  const float* tcw;       // hi/lo UMMA operand shadows of the conv weights (tc_kernel)
  // multi-step epoch graphs: the step index is *step_base + step_off (the
  // host writes step_base once per chunk of steps), else a.step
  const long long* step_base;
  int step_off;
  // ... and, for device-resident data, the batch is picked from a ring of
  // ring_n batches by the step index: batch (step - ring_origin) mod ring_n
  const float* xring;
  const float* yring;
  long long ring_origin;
  int ring_n;
  // tc_kernel only: run the step's aggregation (clipped sum, noise, update)
  // in-kernel after a grid barrier, agg_tiles tiles over the CTA halves
  unsigned long long* grid_ctr;
  int agg_tiles;
  // the next step's input batch (or null): its images are prefetched into L2
  // at kernel start so the next launch's TMA loads hit L2 instead of HBM
  const float* x_next;
};

__device__ __forceinline__ long long step_index(const Params& prm) {
  return prm.step_base ? *prm.step_base + prm.step_off : prm.a.step;
}

// the next step's images (resident ring: batch step+1 mod ring_n), or null
__device__ __forceinline__ const float* next_inputs(const Params& prm) {
  if (prm.xring) {
    long long bi = (step_index(prm) + 1 - prm.ring_origin) % prm.ring_n;
    if (bi < 0) bi += prm.ring_n;
    return prm.xring + bi * prm.B * (H0 * H0);
  }
  return prm.x_next;
}

// this step's input batch (x, y)
__device__ __forceinline__ void step_inputs(const Params& prm, const float*& x, const float*& y) {
  x = prm.x;
  y = prm.y;
  if (prm.xring) {
    long long bi = (step_index(prm) - prm.ring_origin) % prm.ring_n;
    if (bi < 0) bi += prm.ring_n;
    x = prm.xring + bi * prm.B * (H0 * H0);
    y = prm.yring + bi * prm.B;
  }
}

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

// swizzled slot of im2col element (k, pos)
__device__ __forceinline__ int im2col_at(int k, int pos) {
  return k * NP2 + ((((pos >> 2) ^ (k >> 1)) & 3) << 2) + (pos & 3);
}

__device__ __forceinline__ void mbar_wait0(unsigned long long* bar) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(smem_addr(bar)) : "memory");
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
  PGB_MARK(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 0);
  // let the aggregation grid be scheduled as SMs free up (it waits with
  // griddepcontrol.wait for this grid's results)
  asm volatile("griddepcontrol.launch_dependents;");

  // ---- TMA: image + conv weights + biases into shared memory --------------
  // Two transactions so conv1 starts as soon as its 7 KB have landed while the
  // 32 KB of conv2 weights are still in flight.
  constexpr uint32_t kBytes0 = sizeof(float) * (H0 * H0 + D1 * K1 * K1 + D1);
  constexpr uint32_t kBytes1 = sizeof(float) * (D2 + KC2 * D2);
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(&S.bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_addr(&S.bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_addr(&S.bar[0])), "r"(kBytes0) : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_addr(&S.bar[1])), "r"(kBytes1) : "memory");
    const float *gx, *gy;
    step_inputs(prm, gx, gy);
    bulk_g2s(S.u1.xstage, gx + (size_t)b * H0 * H0, sizeof(float) * H0 * H0, &S.bar[0]);
    bulk_g2s(S.w1t, prm.w1t, sizeof(float) * D1 * K1 * K1, &S.bar[0]);
    bulk_g2s(S.b1, W + prm.off[1], sizeof(float) * D1, &S.bar[0]);
    bulk_g2s(S.b2, W + prm.off[3], sizeof(float) * D2, &S.bar[1]);
    bulk_g2s(S.w2t, prm.w2t, sizeof(float) * KC2 * D2, &S.bar[1]);
  }
  // the loss tail's operands (fc2 weights/biases, fc1 bias, label), fetched
  // now so they are not a dependent chain later
  if (t < H1 * NC) S.w4[t] = __ldg(gW4 + t);
  else if (t < H1 * NC + NC) S.b4[t - H1 * NC] = __ldg(gb4 + t - H1 * NC);
  else if (t < H1 * NC + NC + H1) S.b3[t - H1 * NC - NC] = __ldg(gb3 + t - H1 * NC - NC);
  else if (t == H1 * NC + NC + H1) {
    const float *gx, *gy;
    step_inputs(prm, gx, gy);
    S.yb = gy[b];
  }
  // zero the padding ring of xs while the copies fly
  for (int i = t; i < XP * XS; i += NT) {
    const int r = i / XS - 3, c = i % XS - 3;
    if (!(r >= 0 && r < H0 && c >= 0 && c < H0)) S.xs[i] = 0.0f;
  }
  __syncthreads();  // barrier initialised before anyone waits on it
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 1);
  mbar_wait0(&S.bar[0]);
  for (int i = t; i < H0 * H0; i += NT) S.xs[(i / H0 + 3) * XS + i % H0 + 3] = S.u1.xstage[i];
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 2);

  // ---- conv1 + relu: thread = (two horizontally adjacent positions, 4 channels)
  // Per kernel row u the two 8-tap windows share one 10-value input segment;
  // each tap is one broadcast 16-byte load of 4 channel weights and two packed
  // FMAs (FFMA2) per position.
  if (t < 4 * (NP1 / 2)) {
    const int pp = t % (NP1 / 2), cq = t / (NP1 / 2);
    const int oy = pp / (O1 / 2), ox0 = 2 * (pp % (O1 / 2));
    float acc[2][4];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int d = 0; d < 4; ++d) acc[q][d] = 0.0f;
#pragma unroll 2
    for (int u = 0; u < K1; ++u) {
      float seg[K1 + 2];
      const float2* x2 = reinterpret_cast<const float2*>(S.xs + (2 * oy + u) * XS + 2 * ox0);
#pragma unroll
      for (int v = 0; v < (K1 + 2) / 2; ++v) {
        const float2 x = x2[v];
        seg[2 * v] = x.x;
        seg[2 * v + 1] = x.y;
      }
#pragma unroll
      for (int v = 0; v < K1; ++v) {
        const float4 w = *reinterpret_cast<const float4*>(S.w1t + (u * K1 + v) * D1 + cq * 4);
        ffma2v(acc[0][0], acc[0][1], w.x, w.y, seg[v]);
        ffma2v(acc[0][2], acc[0][3], w.z, w.w, seg[v]);
        ffma2v(acc[1][0], acc[1][1], w.x, w.y, seg[v + 2]);
        ffma2v(acc[1][2], acc[1][3], w.z, w.w, seg[v + 2]);
      }
    }
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const int dd = cq * 4 + d;
      S.a1[dd * NP1 + oy * O1 + ox0] = fmaxf(acc[0][d] + S.b1[dd], 0.0f);
      S.a1[dd * NP1 + oy * O1 + ox0 + 1] = fmaxf(acc[1][d] + S.b1[dd], 0.0f);
    }
  }
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 3);

  // ---- maxpool 2x2/2 (first max in window order, kernels.hpp:377-396) -------
  for (int i = t; i < D1 * PO * PO; i += NT) {
    const int c = i / (PO * PO), r = i % (PO * PO), py = r / PO, px = r % PO;
    const float* src = S.a1 + c * NP1 + (2 * py) * O1 + 2 * px;
    float m = src[0];
    int slot = 0;
    if (src[1] > m) { m = src[1]; slot = 1; }
    if (src[O1] > m) { m = src[O1]; slot = 2; }
    if (src[O1 + 1] > m) { m = src[O1 + 1]; slot = 3; }
    S.up.p1[i] = m;
    S.pidx[i] = (unsigned char)slot;
  }
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 4);

  // ---- conv2 im2col: buf[k][pos], k = (c,u,v), pos = (oy,ox) -------------
  // 16-byte chunks of a row are XOR-swizzled by (k >> 1) & 3 (im2col_at), so
  // the per-example dW reads below (lanes on consecutive k) are conflict-free.
  for (int i = t; i < KC2 * NP2; i += NT) {
    const int k = i / NP2, pos = i % NP2;
    const int c = k / 16, u = (k / 4) % 4, v = k % 4, oy = pos / 4, ox = pos % 4;
    S.buf[im2col_at(k, pos)] = S.up.p1[c * PO * PO + (oy + u) * PO + ox + v];
  }
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 5);

  // ---- conv2 + relu: lane = out channel, warp = (K slice of 32, 8 positions)
  mbar_wait0(&S.bar[1]);
  {
    const int d = lane, ks = warp & 7, ph = warp >> 3;
    float acc[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) acc[p] = 0.0f;
#pragma unroll 4
    for (int kk = 0; kk < 32; ++kk) {
      const int k = ks * 32 + kk;
      const float w = S.w2t[k * D2 + (d ^ (k & 31))];
      const float4 c0 = *reinterpret_cast<const float4*>(S.buf + im2col_at(k, ph * 8));
      const float4 c1 = *reinterpret_cast<const float4*>(S.buf + im2col_at(k, ph * 8 + 4));
      ffma2(acc[0], acc[1], w, c0.x, c0.y);
      ffma2(acc[2], acc[3], w, c0.z, c0.w);
      ffma2(acc[4], acc[5], w, c1.x, c1.y);
      ffma2(acc[6], acc[7], w, c1.z, c1.w);
    }
#pragma unroll
    for (int p = 0; p < 8; ++p) S.u1.part[(ks * NP2 + ph * 8 + p) * D2 + d] = acc[p];
  }
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 6);
  {  // i = pos*32 + d
    const int d = t % D2, p = t / D2;
    float s = 0.0f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += S.u1.part[w * D2 * NP2 + t];
    S.a2[d * NP2 + p] = fmaxf(s + S.b2[d], 0.0f);
  }
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 7);

  // ---- fc1 (512->32) + relu: lane = unit, warp = 32-row slice -------------
  // The warp's 32x32 slice of W3 (coalesced rows) stays in registers for the
  // backward pass below.
  float wv[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) wv[r] = __ldg(gW3 + (warp * 32 + r) * H1 + lane);
  {
    float s0 = 0.0f, s1 = 0.0f;
    const float2* a22 = reinterpret_cast<const float2*>(S.a2 + warp * 32);
#pragma unroll
    for (int r = 0; r < 32; r += 2) {
      const float2 av = a22[r / 2];
      ffma2pp(s0, s1, av.x, av.y, wv[r], wv[r + 1]);
    }
    S.u1.z1[warp * H1 + lane] = s0 + s1;
  }
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 8);
  if (warp == 0) {
    // fc1 bias + relu, fc2 (32->10), softmax cross-entropy (kernels.hpp:516-566)
    // and dz1 = (W4 dz2) * [h > 0]. Lane j holds h_j; the 10 logits are
    // butterfly sums (every lane ends with all of them), so the softmax, the
    // loss and dlogits are computed redundantly per lane without further
    // communication (the exp-sum in the reference's class order).
    float zp[4] = {S.b3[lane], 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int w = 0; w < NW; ++w) zp[w & 3] += S.u1.z1[w * H1 + lane];
    const float hv = fmaxf((zp[0] + zp[1]) + (zp[2] + zp[3]), 0.0f);
    S.h[lane] = hv;
    float pr[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) pr[c] = hv * S.w4[lane * NC + c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int c = 0; c < NC; ++c) pr[c] += __shfl_xor_sync(0xffffffffu, pr[c], o);
    const float raw = S.yb;
    const bool ok = valid_id(raw, NC);
    if (!ok && lane == 0) raise_index(prm.err, 0, b, raw, NC);
    const int y = ok ? (int)raw : 0;
    float m = -INFINITY, ly = 0.0f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      pr[c] += S.b4[c];
      m = fmaxf(m, pr[c]);
      ly = c == y ? pr[c] : ly;
    }
    float e[NC], se = 0.0f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      e[c] = expf(pr[c] - m);
      se += e[c];
    }
    float g1 = 0.0f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const float g = ok ? e[c] / se - (c == y ? 1.0f : 0.0f) : 0.0f;
      if (lane == c) S.dz2[c] = g;
      g1 = fmaf(S.w4[lane * NC + c], g, g1);
    }
    if (lane == 0) prm.loss[b] = ok ? m + logf(se) - ly : 0.0f;
    S.dz1[lane] = hv > 0.0f ? g1 : 0.0f;
  } else if (warp < 3 && prm.noise && prm.a.add_noise) {
    // meanwhile warps 1-2 draw this CTA's share of the step's Gaussian noise
    // (one Box-Muller pair per thread, kernels.hpp:597-614)
    const long long pairs = prm.pair_off[8];
    const long long per = (pairs + gridDim.x - 1) / gridDim.x;
    for (long long k = t - 32; k < per; k += 64) {
      const long long q = (long long)b * per + k;
      if (q >= pairs) break;
      int p = 0;
      while (p < 7 && prm.pair_off[p + 1] <= q) ++p;
      const long long jp = q - prm.pair_off[p];
      float n0, n1;
      gauss_pair(stream_key(prm.a.seed, noise_stream(step_index(prm), p)), jp, &n0, &n1);
      float* dst = prm.noise + prm.off[p] + 2 * jp;
      dst[0] = n0;
      if (2 * jp + 1 < prm.size[p]) dst[1] = n1;
    }
  }
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 9);

  // ---- fc1 backward data: da2[i] = W3[i,:] . dz1, relu mask -> dc2 --------
  // From the register-resident W3 slice: products W3[r][lane] * dz1[lane],
  // then a transpose-reduce across the lanes (recursive halving: after the
  // five exchange steps lane l holds the full sum of row 32*warp + l).
  {
    const float g = S.dz1[lane];
#pragma unroll
    for (int r = 0; r < 32; ++r) wv[r] *= g;
#pragma unroll
    for (int st = 0; st < 5; ++st) {
      const int half = 16 >> st, off = 16 >> st;
      const bool upper = (lane & off) != 0;
#pragma unroll
      for (int r = 0; r < half; ++r) {
        const float send = upper ? wv[r] : wv[r + half];
        const float keep = upper ? wv[r + half] : wv[r];
        wv[r] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    const int i = warp * 32 + lane;
    const float v = S.a2[i] > 0.0f ? wv[0] : 0.0f;
    const int d = i / NP2, pos = i % NP2;
    S.dc2[pos * D2 + d] = v;
    S.dc2t[i] = v;  // [d][pos] == flatten order
  }
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 10);

  double sq = 0.0;  // this thread's share of ||g_i||^2
  const size_t bo = (size_t)b;

  // ---- conv2 per-example dW: thread = (k (c,u,v), half of the channels) ----
  {
    const int k = t & (KC2 - 1), dh = t >> 8;
    float cv[NP2];
#pragma unroll
    for (int q = 0; q < NP2 / 4; ++q) {
      const float4 x = *reinterpret_cast<const float4*>(S.buf + im2col_at(k, 4 * q));
      cv[4 * q] = x.x; cv[4 * q + 1] = x.y; cv[4 * q + 2] = x.z; cv[4 * q + 3] = x.w;
    }
    float* out = prm.st_c2w + bo * (D2 * KC2);
#pragma unroll 4
    for (int dd = 0; dd < D2 / 2; ++dd) {
      const int d = dh * (D2 / 2) + dd;
      const float4* g4 = reinterpret_cast<const float4*>(S.dc2t + d * NP2);
      float acc0 = 0.0f, acc1 = 0.0f;
#pragma unroll
      for (int q = 0; q < NP2 / 4; ++q) {
        const float4 g = g4[q];
        ffma2pp(acc0, acc1, g.x, g.y, cv[4 * q], cv[4 * q + 1]);
        ffma2pp(acc0, acc1, g.z, g.w, cv[4 * q + 2], cv[4 * q + 3]);
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
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 11);

  // ---- conv2 backward data: dcols[pos][(u,v),c] = sum_d W2[d][c,u,v] dc2[pos][d]
  // thread = (k, half of the positions), lanes on consecutive k: column k of
  // W2 from the swizzled shared transpose (conflict-free), dc2 rows as
  // broadcasts.
  {
    const int k = t & (KC2 - 1), ph = t >> 8;
    const int c = k / 16, uv = k % 16;
    float wr[D2];
#pragma unroll
    for (int d = 0; d < D2; ++d) wr[d] = S.w2t[k * D2 + (d ^ (k & 31))];
#pragma unroll 2
    for (int pp = 0; pp < NP2 / 2; ++pp) {
      const int p = ph * (NP2 / 2) + pp;
      const float4* g4 = reinterpret_cast<const float4*>(S.dc2 + p * D2);
      float acc0 = 0.0f, acc1 = 0.0f;
#pragma unroll
      for (int q = 0; q < D2 / 4; ++q) {
        const float4 g = g4[q];
        ffma2pp(acc0, acc1, wr[4 * q], wr[4 * q + 1], g.x, g.y);
        ffma2pp(acc0, acc1, wr[4 * q + 2], wr[4 * q + 3], g.z, g.w);
      }
      S.buf[p * DCP + uv * 17 + c] = acc0 + acc1;
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
        s += S.buf[(oy * O2 + ox) * DCP + (u * 4 + v) * 17 + c];
      }
    }
    S.up.dp1[c * PO * PO + r] = s;
  }
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 13);
  // maxpool backward (route to the first max) + relu mask on a1 -> d1 [pos][d]
  // Thread t always has channel d = t % 16 (NT % 16 == 0), so it also keeps a
  // partial of the conv1 bias gradient sum_pos d1[pos][d].
  float b1part = 0.0f;
  for (int i = t; i < D1 * NP1; i += NT) {  // i = pos*16 + d
    const int d = i % D1, r = i / D1, oy = r / O1, ox = r % O1;
    const int pi = d * PO * PO + (oy / 2) * PO + ox / 2;
    const int slot = (oy & 1) * 2 + (ox & 1);
    const float g = (S.pidx[pi] == slot && S.a1[d * NP1 + r] > 0.0f) ? S.up.dp1[pi] : 0.0f;
    S.u1.d1[i] = g;
    b1part += g;
  }
  b1part += __shfl_xor_sync(0xffffffffu, b1part, 16);
  if (lane < D1) S.b1red[warp][lane] = b1part;
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 14);

  // ---- conv1 per-example dW: thread = (2 taps, 8 channels, 1/8 of the rows)
  // Taps (u, v) and (u + 4, v) share every d1 load; the 8 row groups are
  // combined by a 3-level tree through three free shared buffers (buf, a1,
  // then u1 once d1 is dead), each level halving the groups.
  {
    const int kp = t & 31, dg = (t >> 5) & 1, rg = t >> 6;
    const int u = kp / K1, v = kp % K1;  // taps kp and kp + 32
    const int oy0 = rg < 6 ? 2 * rg : 6 + rg, oy1 = rg < 6 ? oy0 + 2 : oy0 + 1;
    float acc0[8], acc1[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc0[c] = acc1[c] = 0.0f;
    for (int oy = oy0; oy < oy1; ++oy) {
      const float* xr0 = S.xs + (2 * oy + u) * XS + v;
      const float* xr1 = xr0 + 4 * XS;
      const float4* g4 = reinterpret_cast<const float4*>(S.u1.d1 + oy * O1 * D1) + 2 * dg;
#pragma unroll 7
      for (int ox = 0; ox < O1; ++ox) {
        const float x0 = xr0[2 * ox], x1 = xr1[2 * ox];
        const float4 ga = g4[ox * 4];
        const float4 gb = g4[ox * 4 + 1];
        ffma2v(acc0[0], acc0[1], ga.x, ga.y, x0);
        ffma2v(acc0[2], acc0[3], ga.z, ga.w, x0);
        ffma2v(acc0[4], acc0[5], gb.x, gb.y, x0);
        ffma2v(acc0[6], acc0[7], gb.z, gb.w, x0);
        ffma2v(acc1[0], acc1[1], ga.x, ga.y, x1);
        ffma2v(acc1[2], acc1[3], ga.z, ga.w, x1);
        ffma2v(acc1[4], acc1[5], gb.x, gb.y, x1);
        ffma2v(acc1[6], acc1[7], gb.z, gb.w, x1);
      }
    }
    // partial (group g, channel d, tap k) of a level lives at [g][d][k]
    auto put = [&](float* dst, int g) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        dst[(g * D1 + dg * 8 + c) * 64 + kp] = acc0[c];
        dst[(g * D1 + dg * 8 + c) * 64 + kp + 32] = acc1[c];
      }
    };
    auto add = [&](const float* src, int g) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        acc0[c] += src[(g * D1 + dg * 8 + c) * 64 + kp];
        acc1[c] += src[(g * D1 + dg * 8 + c) * 64 + kp + 32];
      }
    };
    if (rg >= 4) put(S.buf, rg - 4);
    __syncthreads();
    if (rg < 4) add(S.buf, rg);
    if (rg == 2 || rg == 3) put(S.a1, rg - 2);
    __syncthreads();
    if (rg < 2) add(S.a1, rg);
    if (rg == 1) put(S.u1.d1, 0);
    __syncthreads();
    PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 15);
    if (rg == 0) {
      add(S.u1.d1, 0);
      float* out = prm.st_c1w + bo * (D1 * K1 * K1);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int d = dg * 8 + c;
        out[d * 64 + kp] = acc0[c];
        out[d * 64 + kp + 32] = acc1[c];
        sq = fma((double)acc0[c], (double)acc0[c], sq);
        sq = fma((double)acc1[c], (double)acc1[c], sq);
      }
    }
  }
  if (t < D1) {  // conv1 bias: the per-warp partials of the pool-backward pass
    float s = 0.0f;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += S.b1red[w][t];
    prm.st_c1b[bo * D1 + t] = s;
    sq = fma((double)s, (double)s, sq);
  }

  // ---- dense factors for the ghost-norm blocks + their norm terms ----------
  double a2sq = 0.0;
  {
    const float v = S.a2[t];  // NT == F1
    prm.a2[bo * F1 + t] = v;
    a2sq = (double)v * v;
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
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 16);
  if (t == 0) {
    double r5[5] = {0, 0, 0, 0, 0};
    for (int w = 0; w < NW; ++w)
#pragma unroll
      for (int q = 0; q < 5; ++q) r5[q] += S.red5[q][w];
    // ||a (x) d||^2 = ||a||^2 ||d||^2 (weight) + ||d||^2 (bias), strategies.cpp:140-148
    const double nsq = r5[0] + r5[3] * (r5[1] + 1.0) + r5[4] * (r5[2] + 1.0);
    prm.normsq[b] = nsq;
    // norm and clip factor of this example (dpsgd.cpp:254-270, :91-99)
    const float nrm = (float)sqrt(nsq);
    const float C = prm.a.clip;
    prm.norms[b] = nrm;
    prm.scale[b] = nrm > C ? __fdiv_rn(C, nrm) : 1.0f;
    prm.clipped[b] = nrm > C ? 1 : 0;
    PGB_MARK(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 23);
  }
}

}  // namespace mnist
}  // namespace pgb
