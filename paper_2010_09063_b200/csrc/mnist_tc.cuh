// Per-example DPSGD kernel for the reference MNIST CNN (proj/core/src/models.cpp:107-121)
// with the convolution GEMMs on the 5th-generation tensor cores (tcgen05,
// kind::tf32, 3xTF32 split, fp32 accumulators in TMEM).
//
// One CTA of 1024 threads owns a PAIR of examples (examples 2c, 2c+1); each
// half of the CTA (512 threads) runs the element-wise / reduction phases of
// its example exactly like the SIMT kernel in mnist_fused.cuh, and one
// thread issues the tensor-core GEMMs for both examples:
//
//   conv1 forward  (per example, M = 128 rows (oy, e) x 2 column parities,
//                  N = 16 channels, K = 64 taps): implicit im2col straight
//                  from the padded image. The A operand is a K-major UMMA
//                  view of "Y" -- the padded image stored as rows of 32
//                  floats, with the two 4-column halves of every 8-tap kernel
//                  row interleaved as consecutive rows and one copy per
//                  output-column parity -- so each 8-row core matrix is
//                  eight output positions of one output row, and a K = 8 step
//                  is one kernel row u. No patch matrix is ever built.
//   conv2 forward  (pair-joint: M = 64 (32 channels + pad), N = 32 positions
//                  of the two examples, K = 256): A = conv2 weights, B = the
//                  pooled map's im2col.
//   conv2 dW       (per example, M = 256 im2col rows, N = 32 channels,
//                  K = 16 positions): the reference's dz_i . patches_i^T
//                  (strategies.cpp:156-170), straight to the stacks.
//   conv2 dX       (pair-joint: M = 256, N = 32 positions, K = 32 channels):
//                  the col2im VJP input (autodiff.cpp:155-196).
//
// All operands are K-major, no swizzle (tcgen05 accepts tf32 MN-major only in
// the 128B_BASE32B swizzle); fp32 values are split x = hi + lo with
// hi = rna_tf32(x). A kind::tf32 MMA costs a fixed ~50 cycles up to N ~ 100
// (measured, scripts/umma_rate.py), so the split is folded into the M/N
// dimensions instead of issuing three MMAs per K step: the hi and lo copies of
// one operand are stacked as extra rows (N = 2n or M = 2m) and both halves of
// the other accumulate into the same TMEM columns; the epilogue adds the
// quadrants (hi.hi + hi.lo + lo.hi + lo.lo). 128 MMAs per example pair. Weight operands (hi/lo, in UMMA layout) come from a
// shadow that the update kernel keeps in step with the parameters and arrive
// by TMA bulk copies; the conv2 dX weights (transposed) are fetched while the
// dense layers run.
//   conv1 dW       (per example, M = 128 = 8 kernel rows x hi/lo x 8 taps,
//                  N = 32 = d1 hi | lo, K = 224 positions): implicit im2col^T
//                  from "Z", the padded image cut into 16-byte chunks of four
//                  output columns per tap parity/offset (see below).
#pragma once

#include "mnist_fused.cuh"
#include "tc.cuh"

namespace pgb {
namespace mnist {

constexpr int TNT = 1024;                 // two examples x 512 threads
constexpr int YROWS = 68, YS = 32;        // Y rows per (example, hi/lo, parity), floats per row
constexpr int YBLK = YROWS * YS;          // 2176 floats
constexpr int OFF_W1C = 8 * YBLK;         // conv1 weight operand after the 8 Y blocks
constexpr int REGA = OFF_W1C + 2 * 1024;  // 19456 floats (76 KB)
constexpr int W2HL = 8192;                // one hi or lo copy of a conv2 weight operand
constexpr int DCOLS = NP2 * DCP;          // dcols floats per example

constexpr int TCW_W1C = kTcwW1C, TCW_W2C = kTcwW2C, TCW_W2T = kTcwW2T;

// rna-tf32 split of an fp32 value
__device__ __forceinline__ void split_hl(float x, float& hi, float& lo) { tf32_split(x, hi, lo); }

struct TcSmem {
  float regA[REGA];            // Y + conv1 W -> P2 -> P2^T -> dcols -> conv1 dW partials
  float w2[2 * W2HL + 128];    // conv2 W (hi, lo) -> conv2 W^T (hi, lo) -> d1, dp1 (+512 B slack)
  float xstage[2][H0 * H0];    // raw images (TMA)
  float p1[2][D1 * PO * PO];   // pooled maps
  float dc2c[64 * 32];         // conv2-output cotangent: rows hl*32 + pair position, K = d
  float dc2tc[2][64 * 16];     // [ex] rows hl*32 + d, K = position
  float c2lo[D2][32];          // conv2 forward: the lo-row half of the accumulator
  float dc2f[2][D2 * NP2];     // [ex] fp32 [d][pos]
  float a2[2][F1];
  float z1[2][NW][H1];
  float h[2][H1], dz1[2][H1], dz2[2][16];
  alignas(16) float w4[H1 * NC];  // TMA destinations (16-byte aligned)
  alignas(16) float b4[16];
  alignas(16) float b3[H1];
  alignas(16) float b1[D1];
  alignas(16) float b2[D2];
  float yb[2];
  float b1red[2][NW][D1];
  double red5[2][5][NW];
  float scl[2];  // the pair's clip factors (conv2 pair rows)
  // 0: images, 1: conv2 W, 2: conv2 W^T, 3: MMA commits, 4: conv1 W + small blocks
  uint64_t bar[5];
  uint32_t tmem;
  unsigned char pidx[2][D1 * PO * PO];
};

__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float* v) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}

// A single thread issues a tcgen05.mma only every ~120 cycles (the issuing
// warp stalls on each UTCHMMA), while the tensor core retires these small
// MMAs every ~35-50 cycles (scripts/umma_rate.py), so each GEMM phase is
// split into independent accumulator chains issued by lane 0 of warps 0..3.
constexpr int kIssuers = 4;

// kGridAgg: the in-kernel aggregation after a grid barrier (PGB_GRID_SYNC=1,
// opt-in); compiled out of the default instantiation, whose register
// allocation it would otherwise burden (measured: 340 B of spills vs none)
template <bool kGridAgg>
__global__ void __launch_bounds__(TNT, 1) tc_kernel(Params prm, const AggLaunch agg) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  TcSmem& S = *reinterpret_cast<TcSmem*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int ex = t >> 9, tt = t & (NT - 1), wh = tt >> 5;
  const int b0 = 2 * blockIdx.x, b = b0 + ex;
  const int nex = min(2, prm.B - b0);
  const bool has = ex < nex;
  const float* W = prm.w;
  const float* gW3 = W + prm.off[4];
  const float* tcw = prm.tcw;
  float* regA = S.regA;
  PGB_MARK(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 0);
  asm volatile("griddepcontrol.launch_dependents;");

  // Everything up to the griddepcontrol.wait below touches only this step's
  // inputs: when the kernel is a programmatic dependent of the previous
  // step's aggregation (multi-step graphs), the CTA's start, TMEM allocation
  // and image load overlap that kernel's tail. The weights it updates and the
  // buffers it reads are touched only after the wait. (Measured: letting the
  // other threads run ahead into the Y build, with one thread waiting and
  // fetching the weights after the first barrier, is ~1% slower.)
  if (warp == 0) tc::tmem_alloc(&S.tmem, 512);
  if (t == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) tc::mbar_init(&S.bar[i], 1);
    tc::mbar_init(&S.bar[3], kIssuers);  // every issuer commits once per GEMM phase
    tc::mbar_init(&S.bar[4], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t img = (uint32_t)(sizeof(float) * H0 * H0 * nex);
    // conv1 W operand and the small parameter blocks (biases, fc2 W; b4 as
    // 12 floats for the 16-byte granularity) on one barrier
    constexpr uint32_t kSmall = 4u * (D1 + D2 + H1 * NC + H1 + 12);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_addr(&S.bar[0])), "r"(img) : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_addr(&S.bar[4])), "r"(8192u + kSmall) : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_addr(&S.bar[1])), "r"(65536u) : "memory");
    const float *gx, *gy;
    step_inputs(prm, gx, gy);
    bulk_g2s(S.xstage[0], gx + (size_t)b0 * H0 * H0, img, reinterpret_cast<unsigned long long*>(&S.bar[0]));
    // warm L2 with the next step's images of this CTA's pair
    if (const float* xn = next_inputs(prm))
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                   :: "l"(xn + (size_t)b0 * H0 * H0), "r"(img) : "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    PGB_MARK(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 25);
    auto* b0bar = reinterpret_cast<unsigned long long*>(&S.bar[4]);
    bulk_g2s(regA + OFF_W1C, tcw + TCW_W1C, 8192u, b0bar);
    bulk_g2s(S.b1, W + prm.off[1], 4u * D1, b0bar);
    bulk_g2s(S.b2, W + prm.off[3], 4u * D2, b0bar);
    bulk_g2s(S.b3, W + prm.off[5], 4u * H1, b0bar);
    bulk_g2s(S.w4, W + prm.off[6], 4u * H1 * NC, b0bar);
    bulk_g2s(S.b4, W + prm.off[7], 4u * 12, b0bar);
    bulk_g2s(S.w2, tcw + TCW_W2C, 65536u, reinterpret_cast<unsigned long long*>(&S.bar[1]));
  }
  // the label: loaded now, first used by the loss tail (lane 0 of warp 0 of
  // the half holds it; no barrier waits on the load)
  float ylab = 0.0f;
  if (tt == 0 && has) {
    const float *gx, *gy;
    step_inputs(prm, gx, gy);
    ylab = gy[b];
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = S.tmem;
  PGB_MARK(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 21);
  tc::mbar_wait(&S.bar[0], 0);
  PGB_MARK(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 22);

  // ---- the Y operand of conv1 forward ----------------------------------------
  // Y[ex][hl][par][R = 2r + h][c] = xpad[r][c + 2 par + 4 h]
  // thread: column c = tt % 32, rows R = tt / 32 + 16 j (h = R % 2 fixed)
  if (has) {
    const int c = tt & 31, R0 = tt >> 5;
    const int ix0 = c + 4 * (R0 & 1) - 3;  // parity 0; parity 1 reads ix0 + 2
    const bool okx0 = ix0 >= 0 && ix0 < H0, okx1 = ix0 + 2 >= 0 && ix0 + 2 < H0;
    float* yb = regA + ex * 4 * YBLK + c;  // blocks (hl, par) at yb + (2 hl + par) YBLK
#pragma unroll
    for (int R = R0; R < YROWS; R += 16) {
      const int iy = (R >> 1) - 3;
      const bool oky = iy >= 0 && iy < H0;
      const int xi = (oky ? iy : 0) * H0 + ix0;
      const float v0 = (oky && okx0) ? S.xstage[ex][xi] : 0.0f;
      const float v1 = (oky && okx1) ? S.xstage[ex][xi + 2] : 0.0f;
      float h0, l0, h1, l1;
      split_hl(v0, h0, l0);
      split_hl(v1, h1, l1);
      yb[R * YS] = h0;
      yb[YBLK + R * YS] = h1;
      yb[2 * YBLK + R * YS] = l0;
      yb[3 * YBLK + R * YS] = l1;
    }
  }
  // every thread past this point may read the updated weights or write
  // buffers the previous step's aggregation reads
  asm volatile("griddepcontrol.wait;" ::: "memory");
  tc::fence_proxy_async();
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 1);

  // ---- conv1 forward on the tensor cores ------------------------------------
  // D[(oy, e)][n] for output column ox = 2e + par; K step u = kernel row u:
  // A rows at Y + 2u rows (SBO 512 B = one output row, LBO 128 B = the h
  // half); B = [W hi | W lo] (N = 32 rows hl*16 + d), K step u at 1024u bytes.
  // Yhi.[Whi|Wlo] and Ylo.[Whi|Wlo] accumulate into the same 32 columns, so
  // the result is D[:, d] + D[:, 16 + d] (the lo.lo term rides along).
  if (lane == 0 && warp < kIssuers) {
    // issuer w: example e = w / 2, parity par = w % 2
    tc::fence_after_sync();
    constexpr uint32_t idesc = tc::idesc_tf32(128, 32);
    const int e = warp >> 1, par = warp & 1;
    tc::mbar_wait(&S.bar[4], 0);
    if (e < nex) {
      const uint32_t wb = tc::smem_u32(regA + OFF_W1C);
      const uint32_t yh = tc::smem_u32(regA + ((e * 2 + 0) * 2 + par) * YBLK);
      const uint32_t yl = tc::smem_u32(regA + ((e * 2 + 1) * 2 + par) * YBLK);
      const uint32_t dm = tmem + (uint32_t)((2 * e + par) * 32);
#pragma unroll
      for (int u = 0; u < K1; ++u) {
        const uint64_t bw = tc::make_desc(wb + 1024u * u, 512, 128);
        tc::mma_tf32(dm, tc::make_desc(yh + 256u * u, 128, 512), bw, idesc, u > 0 ? 1u : 0u);
        tc::mma_tf32(dm, tc::make_desc(yl + 256u * u, 128, 512), bw, idesc, 1u);
      }
    }
    tc::commit(&S.bar[3]);
  } else if (wh == 4 || wh == 5) {
    // while the tensor core runs: this CTA's share of the step's Gaussian
    // noise (kernels.hpp:597-614), one Box-Muller pair per thread
    if (prm.noise && prm.a.add_noise) {
      const long long pairs = prm.pair_off[8];
      const long long per = (pairs + gridDim.x - 1) / gridDim.x;
      for (long long k = ex * 64 + tt - 128; k < per; k += 128) {
        const long long q = (long long)blockIdx.x * per + k;
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
    PGB_MARK_T(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 17, 128);
  }
  tc::mbar_wait(&S.bar[3], 0);
  tc::mbar_wait(&S.bar[4], 0);  // the small blocks (biases, fc2 W)
  tc::fence_after_sync();
  PGB_MARK(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 2);

  // ---- conv1 bias + relu + maxpool 2x2/2 straight from TMEM -----------------
  // Thread (quadrant q, lane) holds row m = 32q + lane = (oy = 4q + lane/8,
  // e = lane % 8) of both parities: ox = 2e and 2e + 1 are in-thread, oy + 1 is
  // lane ^ 8. First max in window order (kernels.hpp:377-396).
  {
    const int q = warp & 3, g = warp >> 2, e = g >> 2, dq = g & 3;
    if (e < nex) {
      float v[2][4];
#pragma unroll
      for (int par = 0; par < 2; ++par) {
        float m4[4], c4[4];
        const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((2 * e + par) * 32 + dq * 4);
        tmem_ld4(base, m4);
        tmem_ld4(base + 16, c4);
#pragma unroll
        for (int j = 0; j < 4; ++j) v[par][j] = fmaxf((m4[j] + c4[j]) + S.b1[dq * 4 + j], 0.0f);
      }
      const int oy = 4 * q + (lane >> 3), ee = lane & 7;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float a00 = v[0][j], a01 = v[1][j];
        const float a10 = __shfl_xor_sync(0xffffffffu, a00, 8);
        const float a11 = __shfl_xor_sync(0xffffffffu, a01, 8);
        if (!(lane & 8) && oy < O1 && ee < PO) {
          float m = a00;
          int slot = 0;
          if (a01 > m) { m = a01; slot = 1; }
          if (a10 > m) { m = a10; slot = 2; }
          if (a11 > m) { m = a11; slot = 3; }
          const int i = (dq * 4 + j) * PO * PO + (oy >> 1) * PO + ee;
          S.p1[e][i] = m;
          S.pidx[e][i] = (unsigned char)slot;
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 3);

  // ---- conv2 im2col as the B operand: rows hl*32 + pair position, K = (c,u,v)
  // regA[kmaj(32 hl + 16 ex + pos, k, 128, 1024)]; 32 lanes fill one core.
  // lane = (position % 8) * 4 + k % 4 (one core row each); warp wh takes the
  // (position-group pg, k-group kq) cores pg = wh & 1, kq = wh / 2 + 8 j
  if (has) {
    const int r8 = lane >> 2, kl = lane & 3;
    const int pg = wh & 1;
    const float* src = S.p1[ex] + (r8 >> 2) * PO + (r8 & 3) + kl + pg * 2 * PO;
    float* dst = regA + lane + (ex * 2 + pg) * 32;
#pragma unroll
    for (int kq = wh >> 1; kq < KC2 / 4; kq += NW / 2) {
      const float x = src[(kq >> 2) * PO * PO + (kq & 3) * PO];
      float hi, lo;
      split_hl(x, hi, lo);
      dst[kq * 256] = hi;
      dst[kq * 256 + 128] = lo;
    }
  }
  tc::fence_proxy_async();
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 4);

  // ---- conv2 forward: one MMA per K step computes all four products ------
  // D[hl_a*32 + d][hl_b*32 + pair position] = [Whi; Wlo] . [Phi | Plo]^T
  // (M = 64, N = 64); the result is the sum of the hi.hi, hi.lo, lo.hi (and
  // lo.lo) quadrants.
  // issuer w: K steps s = w (mod 4) into the accumulator at 256 + 64 w
  if (lane == 0 && warp < kIssuers) {
    tc::fence_after_sync();
    tc::mbar_wait(&S.bar[1], 0);
    constexpr uint32_t idesc = tc::idesc_tf32(64, 64);
    const uint32_t wa = tc::smem_u32(S.w2), pb = tc::smem_u32(regA);
#pragma unroll
    for (int s = warp; s < KC2 / 8; s += kIssuers)
      tc::mma_tf32(tmem + 256 + 64u * warp, tc::make_desc(wa + 2048u * s, 1024, 128),
                   tc::make_desc(pb + 2048u * s, 1024, 128), idesc, s >= kIssuers ? 1u : 0u);
    tc::commit(&S.bar[3]);
  }
  // fc1 weight slice into registers while the tensor core runs
  float wv[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) wv[r] = __ldg(gW3 + (wh * 32 + r) * H1 + lane);
  tc::mbar_wait(&S.bar[3], 1);
  tc::fence_after_sync();
  if (t == 0) {
    // conv2 W is dead: fetch its transpose for the input-gradient GEMM
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_addr(&S.bar[2])), "r"(65536u) : "memory");
    bulk_g2s(S.w2, tcw + TCW_W2T, 65536u, reinterpret_cast<unsigned long long*>(&S.bar[2]));
  }
  PGB_MARK(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 5);
  // M = 64 accumulator: row m at lane m % 16 + 32 (m / 16): quadrants 0, 1
  // hold the hi rows of d = 16q + lane, quadrants 2, 3 the lo rows. Warp
  // (q, g) reads columns 4g.. and 32 + 4g.. (the hi and lo halves of N).
  float c2acc[4];
  {
    const int q = warp & 3, g = warp >> 2;
    const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(256 + g * 4);
#pragma unroll
    for (int j = 0; j < 4; ++j) c2acc[j] = 0.0f;
#pragma unroll
    for (int sl = 0; sl < kIssuers; ++sl) {
      float m4[4], c4[4];
      tmem_ld4(base + 64 * sl, m4);
      tmem_ld4(base + 64 * sl + 32, c4);
#pragma unroll
      for (int j = 0; j < 4; ++j) c2acc[j] += m4[j] + c4[j];
    }
    if (q >= 2 && lane < 16)
#pragma unroll
      for (int j = 0; j < 4; ++j) S.c2lo[(q - 2) * 16 + lane][g * 4 + j] = c2acc[j];
  }
  tc::fence_before_sync();
  __syncthreads();
  {
    const int q = warp & 3, g = warp >> 2;
    if (q < 2 && lane < 16) {
      const int d = q * 16 + lane;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int col = g * 4 + j, e = col >> 4, pos = col & 15;
        if (e < nex) S.a2[e][d * NP2 + pos] = fmaxf((c2acc[j] + S.c2lo[d][col]) + S.b2[d], 0.0f);
      }
    }
  }
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 6);

  // ---- fc1 (512->32): lane = unit, warp = 32-row slice -------------------
  if (has) {
    float s0 = 0.0f, s1 = 0.0f;
    const float2* a22 = reinterpret_cast<const float2*>(S.a2[ex] + wh * 32);
#pragma unroll
    for (int r = 0; r < 32; r += 2) {
      const float2 av = a22[r / 2];
      ffma2pp(s0, s1, av.x, av.y, wv[r], wv[r + 1]);
    }
    S.z1[ex][wh][lane] = s0 + s1;
  }
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 7);

  if (wh == 0) {
    if (has) {
      // fc1 bias + relu, fc2, softmax cross-entropy (kernels.hpp:516-566), dz1
      float zp[4] = {S.b3[lane], 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int w = 0; w < NW; ++w) zp[w & 3] += S.z1[ex][w][lane];
      const float hv = fmaxf((zp[0] + zp[1]) + (zp[2] + zp[3]), 0.0f);
      S.h[ex][lane] = hv;
      // lane c < 10 owns logit c: sum_j h_j W4[j][c] in ascending j
      const int c = lane < NC ? lane : 0;
      float lg = 0.0f;
#pragma unroll
      for (int j = 0; j < H1; ++j) lg = fmaf(__shfl_sync(0xffffffffu, hv, j), S.w4[j * NC + c], lg);
      lg += S.b4[c];
      const float raw = __shfl_sync(0xffffffffu, ylab, 0);
      const bool ok = valid_id(raw, NC);
      if (!ok && lane == 0) raise_index(prm.err, 0, b, raw, NC);
      const int y = ok ? (int)raw : 0;
      float m = lane < NC ? lg : -INFINITY;
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      m = __shfl_sync(0xffffffffu, m, 0);
      const float e = lane < NC ? expf(lg - m) : 0.0f;
      float se = e;
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
      se = __shfl_sync(0xffffffffu, se, 0);
      const float ly = __shfl_sync(0xffffffffu, lg, y);
      const float g = (ok && lane < NC) ? e / se - (lane == y ? 1.0f : 0.0f) : 0.0f;
      if (lane < NC) S.dz2[ex][lane] = g;
      if (lane == 0) prm.loss[b] = ok ? m + logf(se) - ly : 0.0f;
      // dz1_j = (W4 dz2)_j * [h_j > 0]: lane j
      float g1 = 0.0f;
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) g1 = fmaf(S.w4[lane * NC + cc], __shfl_sync(0xffffffffu, g, cc), g1);
      S.dz1[ex][lane] = hv > 0.0f ? g1 : 0.0f;
    }
    PGB_MARK_T(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 16, 0);
  } else if (has) {
    // the im2col again, transposed (A of conv2 dW): rows k, K = position,
    // regA[(2 ex + hl) * 4096 + kmaj(k, pos, 128, 4096)]
    // lane = (k % 8) * 4 + position % 4; warps 1..15 take the cores
    // (k-group kg, position quad pq), combo = kg * 4 + pq
    const int r8 = lane >> 2, pl = lane & 3;
    const int l0 = (r8 >> 2) * PO + (r8 & 3) + pl;  // (u%2 half, v, ox) part of the gather
    float* dst = regA + (2 * ex) * 4096 + lane;
    for (int cb = wh - 1; cb < 32 * 4; cb += NW - 1) {
      const int kg = cb >> 2, pq = cb & 3;
      const float x = S.p1[ex][(kg >> 1) * PO * PO + pq * PO + (kg & 1) * 2 * PO + l0];
      float hi, lo;
      split_hl(x, hi, lo);
      dst[kg * 32 + pq * 1024] = hi;
      dst[4096 + kg * 32 + pq * 1024] = lo;
    }
    PGB_MARK_T(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 18, 32);
  }
  tc::fence_proxy_async();
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 8);

  // ---- fc1 backward data + relu mask -> dc2 (both UMMA layouts, hi/lo) ----
  if (has) {
    const float g = S.dz1[ex][lane];
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
    const int i = wh * 32 + lane;
    const float v = S.a2[ex][i] > 0.0f ? wv[0] : 0.0f;
    const int d = i / NP2, pos = i % NP2;
    float hi, lo;
    split_hl(v, hi, lo);
    S.dc2c[kmaj_f(ex * 16 + pos, d, 128, 1024)] = hi;
    S.dc2c[kmaj_f(32 + ex * 16 + pos, d, 128, 1024)] = lo;
    S.dc2tc[ex][kmaj_f(d, pos, 128, 1024)] = hi;
    S.dc2tc[ex][kmaj_f(32 + d, pos, 128, 1024)] = lo;
    S.dc2f[ex][i] = v;
  }
  tc::fence_proxy_async();
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 9);

  // ---- conv2 dW (per example) and conv2 dX (pair) on the tensor cores ------
  // issuers 0, 1: dX tile 0, 1 (pair: D[k2][pos], 4 K steps over d);
  // issuers 2, 3: dW of example 0, 1 (D[k2][d], 2 tiles x 2 K steps over pos).
  // B = [G hi | G lo] (N = 64): A hi and A lo accumulate into the same 64
  // columns, the result is D[:, n] + D[:, 32 + n].
  if (lane == 0 && warp < kIssuers) {
    tc::fence_after_sync();
    constexpr uint32_t idesc = tc::idesc_tf32(128, 64);
    if (warp < 2) {
      tc::mbar_wait(&S.bar[2], 0);
      const int tl = warp;
      const uint32_t wth = tc::smem_u32(S.w2), wtl = wth + 4u * W2HL;
      const uint32_t gb = tc::smem_u32(S.dc2c);
      const uint32_t dm = tmem + (uint32_t)(tl * 64);
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const uint64_t bd = tc::make_desc(gb + 2048u * s, 1024, 128);
        tc::mma_tf32(dm, tc::make_desc(wth + 2048u * tl + 8192u * s, 4096, 128), bd, idesc,
                     s > 0 ? 1u : 0u);
        tc::mma_tf32(dm, tc::make_desc(wtl + 2048u * tl + 8192u * s, 4096, 128), bd, idesc, 1u);
      }
    } else if (warp - 2 < nex) {
      const int e = warp - 2;
      const uint32_t ah = tc::smem_u32(regA + (2 * e) * 4096), al = ah + 16384u;
      const uint32_t bb = tc::smem_u32(S.dc2tc[e]);
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int tl = 0; tl < 2; ++tl) {
          const uint32_t dm = tmem + 128 + (uint32_t)((2 * e + tl) * 64);
          const uint64_t bd = tc::make_desc(bb + 2048u * s, 1024, 128);
          tc::mma_tf32(dm, tc::make_desc(ah + 2048u * tl + 8192u * s, 4096, 128), bd, idesc,
                       s > 0 ? 1u : 0u);
          tc::mma_tf32(dm, tc::make_desc(al + 2048u * tl + 8192u * s, 4096, 128), bd, idesc, 1u);
        }
    }
    tc::commit(&S.bar[3]);
  }
  double sq = 0.0;  // this thread's share of its example's ||g_i||^2
  const size_t bo = (size_t)b;
  if (tt < D2 && has) {  // conv2 bias
    float s = 0.0f;
    for (int p = 0; p < NP2; ++p) s += S.dc2f[ex][tt * NP2 + p];
    prm.st_c2b[bo * D2 + tt] = s;
    sq = fma((double)s, (double)s, sq);
  }
  tc::mbar_wait(&S.bar[3], 0);
  tc::fence_after_sync();
  PGB_MARK(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 10);

  // conv2 dW -> stacks: the half of example ex reads its own accumulators;
  // warp (q, tile, column half), row k = 128 tile + 32 q + lane
  {
    const int q = wh & 3, g = wh >> 2, tl = g >> 1, ch = g & 1;
    if (has) {
      const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + 128 + (uint32_t)((2 * ex + tl) * 64 + ch * 16);
      float m8[8], c8[8];
      const int k = tl * 128 + q * 32 + lane;
      float* out = prm.st_c2w + bo * (D2 * KC2);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        tc::tmem_ld8(base + hh * 8, m8);
        tc::tmem_ld8(base + 32 + hh * 8, c8);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float v = m8[j] + c8[j];
          if (!prm.c2_pairs) out[(ch * 16 + hh * 8 + j) * KC2 + k] = v;
          sq = fma((double)v, (double)v, sq);
        }
      }
    }
  }
  // conv2 dX -> dcols[ex][pos][(u,v) * 17 + c]: warp (q, tile, 8-column group)
  {
    const int q = warp & 3, g = warp >> 2, tl = g >> 2, cq = g & 3;
    const int e = cq >> 1;
    if (e < nex) {
      float m8[8], c8[8];
      const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(tl * 64 + cq * 8);
      tc::tmem_ld8(base, m8);
      tc::tmem_ld8(base + 32, c8);
      const int k = tl * 128 + q * 32 + lane, c = k >> 4, uv = k & 15;
      float* dcols = regA + e * DCOLS;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int pos = (cq & 1) * 8 + j;
        dcols[pos * DCP + uv * 17 + c] = m8[j] + c8[j];
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 11);

  // conv1-output cotangent as the B operand of conv1 dW: rows hl*16 + d,
  // K = oy*16 + ox (ox 14, 15 zero), kmaj(., ., 128, 512): 7168 floats/example
  float* d1c = S.w2 + ex * 7168;
  float* dp1 = S.w2 + 2 * 7168 + ex * (D1 * PO * PO);
  // col2im as a gather: dp1[c][iy][ix] = sum_{u,v} dcols[(iy-u, ix-v)][(u,v),c]
  if (has) {
    const float* dcols = regA + ex * DCOLS;
    for (int i = tt; i < D1 * PO * PO; i += NT) {  // i = (iy*7+ix)*16 + c
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
          s += dcols[(oy * O2 + ox) * DCP + (u * 4 + v) * 17 + c];
        }
      }
      dp1[c * PO * PO + r] = s;
    }
  }
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 12);
  // maxpool backward (first max) + relu mask (the routed element is the
  // pooled max, so relu' = [p1 > 0]) -> d1 as a UMMA operand; conv1 bias
  // partials. Meanwhile the image view Z for conv1 dW (below).
  float b1part = 0.0f;
  float* Z = regA + ex * 8704;
  if (has) {
    // element (oy*16 + ox)*16 + d: thread tt has d = tt % 16, ox = (tt / 16) % 16,
    // oy = tt / 256 + 2 j (so the pooled row is j and the window slot fixed)
    const int d = tt & 15, ox = (tt >> 4) & 15, oy0 = tt >> 8;
    const int slot = oy0 * 2 + (ox & 1);
    const int pb = d * PO * PO + (ox >> 1);
    float* dst = d1c + kmaj_f(d, (tt >> 4), 128, 512);
#pragma unroll
    for (int j = 0; j < PO; ++j) {
      float g = 0.0f;
      const int pi = pb + j * PO;
      if (ox < O1 && S.pidx[ex][pi] == slot && S.p1[ex][pi] > 0.0f) g = dp1[pi];
      float hi, lo;
      split_hl(g, hi, lo);
      dst[j * 1024] = hi;
      dst[j * 1024 + 64] = lo;
      b1part += g;
    }
    // Z[R' = 2R + hl][j4][c = 4p + s][i] = xpad[R][2 (4 j4 + s + i) + p]: for tap
    // (u, v = 2s + p) and output columns 4 j4 .. 4 j4 + 3 of output row oy, the
    // 16-byte chunk (R = 2 oy + u, j4, c) holds the four inputs, so a K-major
    // core matrix is eight taps of one kernel row (permuted v) x four
    // positions, rows 16 B apart; kernel row u and the hi/lo copy are the
    // rows R' (SBO 512 B), position quads the j4 chunks (LBO 128 B).
    {
      const int col = tt & 127, i4 = col & 3, c = (col >> 2) & 7, j4 = col >> 5;
      const int ix = 2 * (4 * j4 + (c & 3) + i4) + (c >> 2) - 3;
      const bool okx = ix >= 0 && ix < H0;
#pragma unroll
      for (int R = tt >> 7; R < 34; R += 4) {
        const int iy = R - 3;
        const float v = (okx && iy >= 0 && iy < H0) ? S.xstage[ex][iy * H0 + ix] : 0.0f;
        float hi, lo;
        split_hl(v, hi, lo);
        Z[(2 * R) * 128 + col] = hi;
        Z[(2 * R + 1) * 128 + col] = lo;
      }
    }
  }
  b1part += __shfl_xor_sync(0xffffffffu, b1part, 16);
  if (lane < D1) S.b1red[ex][wh][lane] = b1part;
  tc::fence_proxy_async();
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 13);

  // ---- conv1 per-example dW on the tensor cores ----------------------------
  // D[(u, hl, c)][n] = sum_pos Z . [d1 hi | d1 lo]^T (M = 128, N = 32); K step
  // = output row oy and an 8-column half jp. The result for tap (u, v = 2s+p),
  // channel d is the sum over the hl rows and the two N halves.
  // issuer w: example w / 2, output rows oy in [7 (w % 2), 7 (w % 2) + 7)
  // into the accumulator at 32 w (the two halves are added at readback)
  if (lane == 0 && warp < kIssuers) {
    tc::fence_after_sync();
    constexpr uint32_t idesc = tc::idesc_tf32(128, 32);
    const int e = warp >> 1, oy0 = 7 * (warp & 1);
    if (e < nex) {
      const uint32_t za = tc::smem_u32(regA + e * 8704), db = tc::smem_u32(S.w2 + e * 7168);
#pragma unroll
      for (int oy = oy0; oy < oy0 + 7; ++oy)
#pragma unroll
        for (int jp = 0; jp < 2; ++jp)
          tc::mma_tf32(tmem + (uint32_t)(warp * 32), tc::make_desc(za + 2048u * oy + 256u * jp, 128, 512),
                       tc::make_desc(db + 2048u * oy + 1024u * jp, 512, 128), idesc,
                       (oy > oy0 || jp) ? 1u : 0u);
    }
    tc::commit(&S.bar[3]);
  }
  // while the tensor core runs: conv1 bias, the dense factors and their norm terms
  if (tt < D1 && has) {  // conv1 bias
    float s = 0.0f;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += S.b1red[ex][w][tt];
    prm.st_c1b[bo * D1 + tt] = s;
    sq = fma((double)s, (double)s, sq);
  }

  // ---- dense factors for the ghost-norm blocks + their norm terms ----------
  double a2sq = 0.0, hsq = 0.0, dz1sq = 0.0, dz2sq = 0.0;
  if (has) {
    const float v = S.a2[ex][tt];
    prm.a2[bo * F1 + tt] = v;
    a2sq = (double)v * v;
    if (tt < H1) {
      const float hv = S.h[ex][tt], g = S.dz1[ex][tt];
      prm.h[bo * H1 + tt] = hv;
      prm.dz1[bo * H1 + tt] = g;
      hsq = (double)hv * hv;
      dz1sq = (double)g * g;
    }
    if (tt < NC) {
      const float g = S.dz2[ex][tt];
      prm.dz2[bo * NC + tt] = g;
      dz2sq = (double)g * g;
    }
  }
  {
    double v4[4] = {a2sq, hsq, dz1sq, dz2sq};
    const int nq = wh == 0 ? 4 : 1;  // the h / dz terms live in warp 0 of the half
    for (int q = 0; q < nq; ++q)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v4[q] += __shfl_xor_sync(0xffffffffu, v4[q], o);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 4; ++q) S.red5[ex][1 + q][wh] = v4[q];
  }
  tc::mbar_wait(&S.bar[3], 1);
  tc::fence_after_sync();
  PGB_MARK(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 14);
  {
    // warp (q, dq) of half ex: row m = 32q + lane = (u = m/16, hl = m/8 % 2,
    // c = m % 8); 4 channels d = 4dq.. from both N halves, hl rows via lane^8
    const int q = wh & 3, dq = wh >> 2;
    float m4[4], c4[4];
    const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ex * 64 + dq * 4);
    if (has) {
      float m4b[4], c4b[4];
      tmem_ld4(base, m4);
      tmem_ld4(base + 16, c4);
      tmem_ld4(base + 32, m4b);
      tmem_ld4(base + 48, c4b);
#pragma unroll
      for (int j = 0; j < 4; ++j) m4[j] += m4b[j] + c4b[j];
      const int m = q * 32 + lane, u = m >> 4, c = m & 7, v = 2 * (c & 3) + (c >> 2);
      float* out = prm.st_c1w + bo * (D1 * K1 * K1);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float val = m4[j] + c4[j];
        val += __shfl_xor_sync(0xffffffffu, val, 8);
        if (!(m & 8)) {
          out[(dq * 4 + j) * 64 + u * K1 + v] = val;
          sq = fma((double)val, (double)val, sq);
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if (lane == 0) S.red5[ex][0][wh] = sq;
  tc::fence_before_sync();
  __syncthreads();
  PGB_MARK_BAR(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 15);
  if (!prm.c2_pairs && warp == 0) tc::tmem_dealloc(tmem, 512);
  if (tt == 0 && has) {
    double r5[5] = {0, 0, 0, 0, 0};
    for (int w = 0; w < NW; ++w)
#pragma unroll
      for (int q = 0; q < 5; ++q) r5[q] += S.red5[ex][q][w];
    // ||a (x) d||^2 = ||a||^2 ||d||^2 (weight) + ||d||^2 (bias), strategies.cpp:140-148
    const double nsq = r5[0] + r5[3] * (r5[1] + 1.0) + r5[4] * (r5[2] + 1.0);
    prm.normsq[b] = nsq;
    const float nrm = (float)sqrt(nsq);
    const float C = prm.a.clip;
    prm.norms[b] = nrm;
    prm.scale[b] = nrm > C ? __fdiv_rn(C, nrm) : 1.0f;
    prm.clipped[b] = nrm > C ? 1 : 0;
    S.scl[ex] = prm.scale[b];
    PGB_MARK(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 23);
  }

  // ---- conv2 W as clipped pair rows ----------------------------------------
  // fl(g_2c s_2c) + fl(g_2c+1 s_2c+1) for the CTA's two examples, re-read from
  // the dW accumulators (untouched since): the aggregation then sums half as
  // many rows of the step's largest block. warp (q, tile, 8-channel group)
  if (prm.c2_pairs) {
    __syncthreads();
    const int q = warp & 3, g = warp >> 2, tl = g >> 2, cg = g & 3;
    const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + 128 + (uint32_t)(tl * 64 + cg * 8);
    float m0[8], c0[8], m1[8], c1[8];
    tc::tmem_ld8(base, m0);
    tc::tmem_ld8(base + 32, c0);
    const bool two = nex > 1;
    if (two) {
      tc::tmem_ld8(base + 128, m1);
      tc::tmem_ld8(base + 128 + 32, c1);
    }
    const float s0 = S.scl[0], s1 = two ? S.scl[1] : 0.0f;
    const int k = tl * 128 + q * 32 + lane;
    float* out = prm.c2_pairs + (size_t)blockIdx.x * (D2 * KC2);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float v = __fmul_rn(m0[j] + c0[j], s0);
      if (two) v = __fadd_rn(v, __fmul_rn(m1[j] + c1[j], s1));
      out[(cg * 8 + j) * KC2 + k] = v;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 512);
    PGB_MARK(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 24);
  }

  // ---- the step's aggregation, in-kernel ----------------------------------
  // Every CTA is resident (one per SM), so after a grid barrier the CTA
  // halves run the aggregation tiles of aggregate_kernel (clipped sum in a
  // fixed order, noise, mean, update) on the per-example outputs above.
  if (kGridAgg && prm.agg_tiles > 0) {
    PGB_MARK(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 19);
    grid_barrier(prm.grid_ctr);
    PGB_MARK(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 20);
    float* s_sh = regA + ex * 4096;  // clip factors + factored-row staging
    auto part_sh = reinterpret_cast<float(*)[kAggRows * 32]>(regA + 8192 + ex * 4096);
    int* cnt_sh = reinterpret_cast<int*>(regA + 16384) + ex * kAggWarps;
    // tile t on half t / gridDim of CTA t % gridDim: at most one tile per SM
    // until the halves' second round (the heavy factored fc1 tiles are
    // consecutive, so they land on different SMs)
    for (int tile = blockIdx.x + ex * gridDim.x; tile < prm.agg_tiles; tile += 2 * gridDim.x)
      agg_tile_run<true, 8>(agg, tile, tt, 1 + ex, s_sh, part_sh, cnt_sh);
    if (ex == 0) PGB_MARK(PGB_TRACE_FUSED + PGB_FUSED_SLOTS * blockIdx.x + 21);
  }
}

// conv weight blocks -> the hi/lo UMMA operands of tc_kernel (after a host
// upload; the update kernel keeps them in step through write_param)
__global__ void tc_shadow_kernel(const float* __restrict__ w1, const float* __restrict__ w2,
                                 float* __restrict__ tcw) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 1024 + 8192; e += gridDim.x * blockDim.x) {
    if (e < 1024) tcw_write(tcw, 1, e, w1[e]);
    else tcw_write(tcw, 2, e - 1024, w2[e - 1024]);
  }
}

}  // namespace mnist
}  // namespace pgb
