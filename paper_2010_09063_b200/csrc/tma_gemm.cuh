// Warp-specialised tcgen05 GEMM fed by tensor-map TMA (cp.async.bulk.tensor,
// SASS UTMALDG), for the convolution GEMMs of the layer-wise engine (CIFAR):
//
//   D[m][n] = sum_k A[m][k] * B[n][k]      fp32-accurate (3xTF32), TMEM accumulator
//
// Both operands are K-major with the 128-byte swizzle: a K chunk is 32 fp32
// (one 128-B row per operand row), loaded by TMA boxes straight from the
// activation / weight tensors -- the implicit im2col is the box coordinates
// (a tap of the 3x3 kernel is a shifted box; the zero padding is the TMA
// out-of-bounds fill), no patch matrix and no register gather.
//
// fp32 accuracy: every operand arrives pre-split as two tensors, hi =
// rna_tf32(x) and lo = rna_tf32(x - hi), written by the memory-bound layout
// kernels that produce the operand anyway (NHWC copy, weight permute, shifted
// copies); TMA loads both, so the GEMM itself does no CUDA-core work.
// D += Ahi.Bhi + Ahi.Blo + Alo.Bhi, each dropped or rounded term <= 2^-22
// relative. (tcgen05 kind::tf32 truncates fp32 operands to their top 19 bits,
// scripts/tf32_probe.py: feeding the raw tile as hi measured ~1e-5 normwise,
// and splitting in the GEMM on four warps made it split-bound.)
//
// The tensor core's fp32 accumulation is not round-to-nearest (a K = 1152
// chain in one accumulator measured ~8e-6 normwise, linear in K), so the hi.hi
// products rotate over NACC accumulators chunk by chunk and the two small
// correction products share one more; the epilogue adds them in fp32 on the
// CUDA cores (all of TMEM: one CTA per SM).
//
// Roles (256 threads): warp 0 lane 0 issues the four TMA boxes of a stage
// (A hi / lo, B hi / lo) into an S-stage ring; warp 1 lane 0 issues the 12
// MMAs of a stage and commits them to the stage's "empty" barrier, which hands
// the stage back to TMA; warps 4-7 run the epilogue from TMEM.
//
// Modes (im2col as box coordinates; conv 3x3, stride 1, pad 1):
//   kPlain   A[M][K], B[N][K] row-major (self-test)
//   kConvFwd A = input  NHWC (channels padded to Cp, a multiple of 32): m = position,
//            k = (tap, c); B = Wt[d][tap * Cp + c]; out NCHW + bias (+ relu)
//   kConvDx  A = output cotangent NHWC (Dp), m = input position, k = (tap, d),
//            shifted by the flipped tap; B = Wt2[c][tap * Dp + d];
//            out NCHW gx (* [mask > 0], the relu of the layer below)
//   kConvDw  per example z: A = input NCHW, m = (tap, c) (a box per tap),
//            k = position; B = output cotangent NCHW (n = d). The K chunk is
//            32 consecutive positions of the flattened H*W plane (one 128-B
//            swizzle row for any W); a tap's row shift is a shift of W
//            positions in that plane (OOB at the image border: zeros), its
//            column shift comes from three pre-shifted copies of the input
//            ([v][n][c][p] = x[n][c][p + v - 1] within the row), since TMA
//            boxes start on 16-byte boundaries of the innermost dimension;
//            out = the reference's per-example dW stack (B, D, C, 3, 3)
//            (strategies.cpp:156-170) + each tile's squared sum (fp64)
//   kConvDwSum the clipped weight gradient sum_i s_i dW_i as ONE GEMM over
//            K = (example, position): the kConvDw operands with the cotangent
//            pre-scaled by the example's clip factor (scale_split_kernel);
//            the examples are split over the grid (tile z = example range
//            [z * ex_per, (z+1) * ex_per)), each split's raw tile goes to a
//            workspace and dw_sum_reduce_kernel adds the splits in order
#pragma once

#include <cuda.h>

#include "kernels.cuh"
#include "tc.cuh"

namespace pgb {
namespace tg {

constexpr int kBM = 128, kBK = 32, kThreads = 256;
enum Mode { kPlain = 0, kConvFwd = 1, kConvDx = 2, kConvDw = 3, kConvDwSum = 4 };

struct alignas(64) Params {
  CUtensorMap ta, tb;        // the hi tensors
  CUtensorMap ta_lo, tb_lo;  // the lo tensors (same geometry)
  int mode;
  int M, N;          // GEMM rows / columns (valid extents)
  int nchunks;       // K chunks of 32
  // geometry (conv modes)
  int C, H, W, D;    // layer input channels, spatial, output channels
  int Cg;            // fwd: Cp / 32 (channel groups per tap); dx: Dp / 32
  int by, bn;        // fwd/dx A box: rows per image, images (box = 32 x W x by x bn)
  int Cr, T;         // dw: rows per tap slot (multiple of 8), tap slots per M tile
  int big_c;         // dw: C >= 128 -> M tile = 128 channels of one tap
  int bx, dw_by;     // dw boxes: x extent, rows per chunk
  int tiles;         // tiles per GEMM (ntn * ntm), tile_sq row length
  int ntn, ntm, nz;  // N tiles, M tiles, GEMMs (examples / example splits); set by launch()
  int ex_per, nex;   // dw-sum: examples per split, examples in total
  int ksplit;        // fwd / dx / plain: K splits (tile z); > 1: raw tiles to ws
  int halo;          // fwd / dx: halo stages (chunk = (kernel column v, 32 channels))
  int rot;           // dw halo: accumulators per kernel row (1: two TMEM buffers; 2: one)
  int narrow;        // folded tiles: the lo.(hi) MMA at N = BN (no lo.lo product)
  int raw;           // dw halo: plain fp32 operands, lo halves split in the kernel
  float* ws;         // dw-sum: split workspace [z][mt][n][128 rows]
  // epilogue
  float* out;
  const float* bias;
  const float* mask;
  double* tile_sq;
  int relu;
  int ldc;           // kPlain: row stride of out
};

// Halo mode (forward / input gradient on 16- and 32-wide maps, N <= 64): a
// stage holds the (rows + 2) x W input rows around a 128-position tile for
// one kernel column v and 32 channels, and the three kernel rows u read it at
// row offsets u * W -- UMMA descriptor start addresses, whole 1024-B swizzle
// atoms since W * 128 B is -- so each input element crosses L2 -> SMEM once
// per kernel column instead of once per tap.
constexpr int kHaloRows = 192;  // A rows of a halo stage: (128 / W + 2) * W <= 192
template <int BN, bool H = false>
constexpr int stages() {
  return H ? (BN >= 64 ? 2 : 3) : (BN >= 128 ? 3 : BN >= 64 ? 4 : 5);
}
// Narrow tiles (BN <= 64) fold the 3xTF32 split into N: the B stage holds the
// hi rows then the lo rows (2 BN rows, one operand), so a K step is two MMAs
// of width 2 BN -- Ahi.[Bhi;Blo] and Alo.[Bhi;Blo] -- instead of three of
// width BN (a single thread issues an MMA only every ~50-120 cycles and below
// N ~ 100 an MMA costs that fixed time, scripts/umma_rate.py); the epilogue
// adds column n and BN + n (the lo.lo product rides along, <= 2^-44 relative).
template <int BN>
constexpr bool folded() { return BN <= 64; }
// TMEM: two 256-column accumulator buffers (the epilogue of tile k overlaps
// the MMAs of tile k+1) except for BN = 128, whose hi.hi rotation needs the
// whole of TMEM (the tensor core's fp32 accumulation is not round-to-nearest:
// chains are kept short by rotating the hi.hi products over accumulators).
template <int BN>
constexpr int nbuf() { return BN >= 128 ? 1 : 2; }
template <int BN>
constexpr int acc_stride() { return folded<BN>() ? (2 * BN < 32 ? 32 : 2 * BN) : (BN < 32 ? 32 : BN); }
// accumulators per buffer: folded -- all of them rotate; unfolded -- the
// hi.hi rotation plus one for the two correction products
template <int BN>
constexpr int nacc() {
  return folded<BN>() ? (512 / nbuf<BN>()) / acc_stride<BN>()
                      : (512 / nbuf<BN>()) / acc_stride<BN>() - 1;
}

template <int BN, bool H = false>
struct Smem {
  static constexpr int S = stages<BN, H>();
  static constexpr int T = H ? 3 : 1;            // taps (kernel rows) per stage
  static constexpr int RA = H ? kHaloRows : kBM;  // A rows per stage
  float a_hi[S][RA * kBK];
  float a_lo[S][RA * kBK];
  float b[S][T][2][BN * kBK];  // per tap: hi rows, then lo rows (one 2 BN-row operand)
  uint64_t full[S], empty[S], split[S];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem;
  double sq[4];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA descriptor, K-major, SWIZZLE_128B: 8-row atoms of 128 B, SBO = 1024 B
// between atoms (LBO unused); the K step inside the atom advances the start
// address by 32 B (8 tf32). Tiles are 1024-B aligned.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* m, int c0, int c1,
                                       uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      :: "r"(dst), "l"(m), "r"(c0), "r"(c1), "r"(bar) : "memory");
}
__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2,
                                       uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      :: "r"(dst), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
}
__device__ __forceinline__ void tma_4d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2,
                                       int c3, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      :: "r"(dst), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar) : "memory");
}
__device__ __forceinline__ void tma_5d(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2,
                                       int c3, int c4, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      :: "r"(dst), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  return __uint_as_float(h);
}

// the lo half of a plain fp32 operand the tensor core reads as the truncated
// tf32 hi: x - trunc_tf32(x) (exact in fp32)
__device__ __forceinline__ float4 lo_of(float4 x) {
  const auto lo1 = [](float v) { return v - __uint_as_float(__float_as_uint(v) & 0xffffe000u); };
  return make_float4(lo1(x.x), lo1(x.y), lo1(x.z), lo1(x.w));
}

// the 3xTF32 pair of one value: hi = rna(x), lo = rna(x - hi)
__device__ __forceinline__ void split2(float x, float& hi, float& lo) {
  hi = rna_tf32(x);
  lo = rna_tf32(x - hi);
}

// Bytes TMA delivers per stage for operand A of M tile mt (full boxes, OOB
// included). A dW tile past the ninth tap leaves its slots unloaded: those
// accumulator rows are never stored.
__device__ __forceinline__ uint32_t a_bytes(const Params& p, int mt) {
  if (p.mode == kConvDw || p.mode == kConvDwSum)
    return (uint32_t)(p.big_c ? kBM : min(p.T, 9 - mt * p.T) * p.Cr) * kBK * 4;
  return kBM * kBK * 4;
}

// Issue the TMA boxes of K chunk q of tile (mt, nt) for example z: operand
// A from (ma, into da) and B from (mb, into db) -- once for the hi tensors,
// once for the lo tensors.
__device__ __forceinline__ void issue_boxes(const Params& p, const CUtensorMap* ma,
                                            const CUtensorMap* mb, uint32_t da, uint32_t db,
                                            int BN, int q, int mt, int nt, int z, uint32_t bar,
                                            bool load_a = true) {
  switch (p.mode) {
    case kPlain:
      if (load_a) tma_2d(da, ma, q * kBK, mt * kBM, bar);
      tma_2d(db, mb, q * kBK, nt * BN, bar);
      break;
    case kConvFwd:
    case kConvDx: {
      const int tap = q / p.Cg, cg = q - tap * p.Cg;
      const int u = tap / 3, v = tap - 3 * u;
      const int HW = p.H * p.W;
      const int m0 = mt * kBM, n0 = m0 / HW, y0 = (m0 - n0 * HW) / p.W;
      // forward: x + v - 1, y + u - 1; input gradient: the flipped tap
      const int dx = p.mode == kConvFwd ? v - 1 : 1 - v;
      const int dy = p.mode == kConvFwd ? u - 1 : 1 - u;
      if (load_a) tma_4d(da, ma, cg * kBK, dx, y0 + dy, n0, bar);
      tma_2d(db, mb, tap * p.Cg * kBK + cg * kBK, nt * BN, bar);
      break;
    }
    case kConvDw:
    case kConvDwSum: {
      const int p0 = q * kBK;  // first position of the chunk (flattened H*W)
      if (!load_a) {
      } else if (p.big_c) {
        const int cgs = p.C / kBM, tap = mt / cgs, c0 = (mt - tap * cgs) * kBM;
        const int u = tap / 3, v = tap - 3 * u;
        tma_4d(da, ma, p0 + (u - 1) * p.W, c0, z, v, bar);
      } else {
        for (int sl = 0; sl < p.T; ++sl) {
          const int tap = mt * p.T + sl;
          if (tap >= 9) break;
          const int u = tap / 3, v = tap - 3 * u;
          tma_4d(da + sl * p.Cr * kBK * 4, ma, p0 + (u - 1) * p.W, 0, z, v, bar);
        }
      }
      tma_3d(db, mb, p0, nt * BN, z, bar);
      break;
    }
  }
}

// RAW: operand A arrives as plain fp32 only (its lo half is split in the kernel)
template <int BN, bool H, bool RAW>
__device__ __forceinline__ void issue_chunk(const Params& p, Smem<BN, H>& S, int s, int q, int mt,
                                            int nt, int z) {
  const uint32_t bar = smem_u32(&S.full[s]);
  if constexpr (H) {
    // halo chunk q = (kernel column v, channel group cg): the input rows
    // y0 - 1 .. y0 + 128 / W of the tile's image, shifted by the column tap
    // (forward x + v - 1, input gradient the flipped 1 - v), once; the three
    // taps (u, v) of the weight operand
    const int v = q / p.Cg, cg = q - v * p.Cg;
    const int HW = p.H * p.W;
    const int m0 = mt * kBM, n0 = m0 / HW, y0 = (m0 - n0 * HW) / p.W;
    const int dx = p.mode == kConvFwd ? v - 1 : 1 - v;
    tma_4d(smem_u32(S.a_hi[s]), &p.ta, cg * kBK, dx, y0 - 1, n0, bar);
    if (!RAW) tma_4d(smem_u32(S.a_lo[s]), &p.ta_lo, cg * kBK, dx, y0 - 1, n0, bar);
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int k0 = (3 * u + v) * p.Cg * kBK + cg * kBK;
      tma_2d(smem_u32(S.b[s][u][0]), &p.tb, k0, nt * BN, bar);
      tma_2d(smem_u32(S.b[s][u][1]), &p.tb_lo, k0, nt * BN, bar);
    }
  } else {
    issue_boxes(p, &p.ta, &p.tb, smem_u32(S.a_hi[s]), smem_u32(S.b[s][0][0]), BN, q, mt, nt, z,
                bar);
    issue_boxes(p, &p.ta_lo, &p.tb_lo, smem_u32(S.a_lo[s]), smem_u32(S.b[s][0][1]), BN, q, mt,
                nt, z, bar, !RAW);
  }
}

// K chunks of a tile: dw-sum walks the positions of every example of its split
__device__ __forceinline__ int tile_chunks(const Params& p, int z) {
  if (p.ksplit > 1) return (z + 1) * p.nchunks / p.ksplit - z * p.nchunks / p.ksplit;
  if (p.mode != kConvDwSum) return p.nchunks;
  const int e0 = z * p.ex_per, e1 = min(p.nex, e0 + p.ex_per);
  return max(0, e1 - e0) * p.nchunks;
}
// chunk q of a tile -> (position chunk, example)
__device__ __forceinline__ void chunk_coords(const Params& p, int q, int z, int& qc, int& ze) {
  if (p.ksplit > 1) {
    qc = z * p.nchunks / p.ksplit + q;
    ze = 0;
  } else if (p.mode != kConvDwSum) {
    qc = q;
    ze = z;
  } else {
    const int k = q / p.nchunks;
    qc = q - k * p.nchunks;
    ze = z * p.ex_per + k;
  }
}

// tile index -> (nt, mt, z), N tiles fastest
__device__ __forceinline__ void tile_coords(const Params& p, int t, int& nt, int& mt, int& z) {
  nt = t % p.ntn;
  const int r = t / p.ntn;
  mt = r % p.ntm;
  z = r / p.ntm;
}

// Persistent: one CTA per SM walks the tiles t = blockIdx.x + k * gridDim.x.
// The TMA ring runs across tile boundaries (the next tile's operands stream in
// while this tile's MMAs finish), and with two accumulator buffers the
// epilogue of a tile overlaps the next tile's MMAs.
// RAW: operand A (activations / shifted copies) is loaded as plain fp32 and
// warps 8-11 write its lo half, x - trunc_tf32(x), next to it in shared
// memory (the tensor core reads the fp32 tile itself as the truncated hi):
// one A load per stage instead of two, and the layout kernels write one tensor.
constexpr int kRawThreads = 384;
template <int BN, bool H = false, bool RAW = false>
__global__ void __launch_bounds__(RAW ? kRawThreads : kThreads, 1)
    tma_gemm_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char raw[];
  // the swizzled tiles need 1024-B alignment of the dynamic window
  Smem<BN, H>& S = *reinterpret_cast<Smem<BN, H>*>(
      (reinterpret_cast<uintptr_t>(raw) + 1023) & ~static_cast<uintptr_t>(1023));
  constexpr int NS = Smem<BN, H>::S;
  constexpr int T = Smem<BN, H>::T;
  constexpr uint32_t kCols = 512;
  constexpr bool kFold = folded<BN>();
  constexpr int NB = nbuf<BN>();
  constexpr int NACC = nacc<BN>();
  constexpr uint32_t kAccStride = acc_stride<BN>();
  constexpr uint32_t kBufCols = 512 / NB;
  // halo tiles with BN <= 32: warps 1-3 each issue one kernel row u into its
  // own accumulator (a single thread issues an MMA only every ~50-120 cycles,
  // and a halo chunk is 3 x 4 x 2 MMAs)
  constexpr bool kMI = H && BN <= 32;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int total = p.ntn * p.ntm * p.nz;
  if (warp == 1) tc::tmem_alloc(&S.tmem, kCols);
  if (t == 0) {
    for (int s = 0; s < NS; ++s) {
      tc::mbar_init(&S.full[s], 1);
      tc::mbar_init(&S.empty[s], kMI ? 3 : 1);  // one commit per issuing warp
      tc::mbar_init(&S.split[s], 4);  // RAW: one arrival per splitting warp
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&S.acc_full[b], kMI ? 3 : 1);
      tc::mbar_init(&S.acc_empty[b], 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&p.ta) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&p.tb) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&p.ta_lo) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&p.tb_lo) : "memory");
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = S.tmem;

  if (warp == 0) {
    // ---- TMA producer ----
    if (lane == 0) {
      int g = 0;  // chunks issued by this CTA (ring position)
      for (int tl = blockIdx.x; tl < total; tl += gridDim.x) {
        int nt, mt, z;
        tile_coords(p, tl, nt, mt, z);
        const uint32_t bytes =
            H ? (RAW ? 1u : 2u) * (uint32_t)(kBM / p.W + 2) * p.W * kBK * 4 + 2u * 3u * BN * kBK * 4
              : (RAW ? 1u : 2u) * a_bytes(p, mt) + 2u * BN * kBK * 4;
        const int nq = tile_chunks(p, z);
        for (int q = 0; q < nq; ++q, ++g) {
          const int s = g % NS;
          if (g >= NS) tc::mbar_wait(&S.empty[s], ((g / NS) - 1) & 1);
          expect_tx(&S.full[s], bytes);
          int qc, ze;
          chunk_coords(p, q, z, qc, ze);
          issue_chunk<BN, H, RAW>(p, S, s, qc, mt, nt, ze);
        }
      }
    }
  } else if (warp == 1 || (kMI && warp <= 3)) {
    // ---- MMA issuer(s) ----
    if (lane == 0) {
      const int u0 = kMI ? warp - 1 : 0, u1 = kMI ? warp : T;
      constexpr uint32_t idesc = tc::idesc_tf32(kBM, kFold ? 2 * BN : (BN < 16 ? 16 : BN));
      constexpr uint32_t idesc_lo = tc::idesc_tf32(kBM, BN < 16 ? 16 : BN);
      int g = 0, lt = 0;
      for (int tl = blockIdx.x; tl < total; tl += gridDim.x, ++lt) {
        int nt_, mt_, z_;
        tile_coords(p, tl, nt_, mt_, z_);
        const int nq = tile_chunks(p, z_);
        const int bsel = NB == 2 ? (lt & 1) : 0;
        const int use = NB == 2 ? (lt >> 1) : lt;  // earlier uses of this buffer
        if (use > 0) tc::mbar_wait(&S.acc_empty[bsel], (use - 1) & 1);
        tc::fence_after_sync();
        const uint32_t buf = tmem + (uint32_t)bsel * kBufCols;
        for (int q = 0; q < nq; ++q, ++g) {
          const int s = g % NS;
          tc::mbar_wait(RAW ? &S.split[s] : &S.full[s], (g / NS) & 1);
          tc::fence_after_sync();
#pragma unroll
          for (int u = u0; u < u1; ++u) {
            // halo: kernel row u reads the stage's rows from u (forward) or
            // 2 - u (input gradient, the flipped tap) times W
            const uint32_t ao =
                H ? (uint32_t)((p.mode == kConvFwd ? u : 2 - u) * p.W * kBK * 4) : 0u;
            const uint32_t ah = smem_u32(S.a_hi[s]) + ao, al = smem_u32(S.a_lo[s]) + ao;
            const uint32_t bh = smem_u32(S.b[s][u][0]), bl = smem_u32(S.b[s][u][1]);
            const int qa = q * T + u;  // accumulator chain step
            const uint32_t dmain = buf + (uint32_t)(kMI ? u : qa % NACC) * kAccStride;
            const bool acc0 = kMI ? q > 0 : qa >= NACC;  // the accumulator already holds a chunk
#pragma unroll
            for (int k = 0; k < kBK / 8; ++k) {
              const uint32_t o = 32u * k;
              if constexpr (kFold) {
                // [Bhi; Blo] is one 2 BN-row operand starting at bh
                tc::mma_tf32(dmain, desc_sw128(ah + o), desc_sw128(bh + o), idesc,
                             (acc0 || k) ? 1u : 0u);
                if (p.narrow)
                  tc::mma_tf32(dmain, desc_sw128(al + o), desc_sw128(bh + o), idesc_lo, 1u);
                else
                  tc::mma_tf32(dmain, desc_sw128(al + o), desc_sw128(bh + o), idesc, 1u);
              } else {
                const uint32_t dcorr = buf + (uint32_t)NACC * kAccStride;
                tc::mma_tf32(dmain, desc_sw128(ah + o), desc_sw128(bh + o), idesc,
                             (qa >= NACC || k) ? 1u : 0u);
                tc::mma_tf32(dcorr, desc_sw128(ah + o), desc_sw128(bl + o), idesc,
                             (qa | k) ? 1u : 0u);
                tc::mma_tf32(dcorr, desc_sw128(al + o), desc_sw128(bh + o), idesc, 1u);
              }
            }
          }
          tc::commit(&S.empty[s]);
        }
        tc::commit(&S.acc_full[bsel]);
      }
    }
  } else if (RAW && warp >= 8) {
    // ---- lo half of each stage's A operand, then release the stage to the MMA ----
    const int ct = t - 256;
    constexpr int na4 = Smem<BN, H>::RA * kBK / 4;
    int g = 0;
    for (int tl = blockIdx.x; tl < total; tl += gridDim.x) {
      int nt, mt, z;
      tile_coords(p, tl, nt, mt, z);
      const int nq = tile_chunks(p, z);
      for (int q = 0; q < nq; ++q, ++g) {
        const int s = g % NS;
        tc::mbar_wait(&S.full[s], (g / NS) & 1);
        const float4* ah = reinterpret_cast<const float4*>(S.a_hi[s]);
        float4* al = reinterpret_cast<float4*>(S.a_lo[s]);
#pragma unroll 4
        for (int e = ct; e < na4; e += 128) al[e] = lo_of(ah[e]);
        tc::fence_proxy_async();  // generic-proxy writes -> the tensor core's reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.split[s]);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---- epilogue: TMEM -> registers -> global ----
    const int q4 = warp & 3, r = q4 * 32 + lane;
    int lt = 0;
    for (int tl = blockIdx.x; tl < total; tl += gridDim.x, ++lt) {
      int nt, mt, z;
      tile_coords(p, tl, nt, mt, z);
      const int nq = tile_chunks(p, z) * T;  // accumulator chain steps
      const int used = kMI ? T : nq < NACC ? nq : NACC;
      const int bsel = NB == 2 ? (lt & 1) : 0;
      const int use = NB == 2 ? (lt >> 1) : lt;
      // input gradient: the tile's ReLU-mask row loaded while the MMAs run
      // (the epilogue's dependent DRAM round trips were the bound of the
      // 32x32 layer: 141 us against 70 us for the same-shape forward)
      float mkpre[BN <= 64 ? BN : 1];
      const bool mk_ahead = BN <= 64 && p.mode == kConvDx && p.mask && p.ksplit <= 1;
      if constexpr (BN <= 64) {
        if (mk_ahead) {
          const int HW = p.H * p.W, m = mt * kBM + r;
          const int img = m / HW, pos = m - img * HW;
          const size_t i0 = ((size_t)img * p.C + nt * BN) * HW + pos;
#pragma unroll
          for (int j = 0; j < BN; ++j)
            mkpre[j] = (m < p.M && nt * BN + j < p.N) ? __ldg(p.mask + i0 + (size_t)j * HW) : 1.0f;
        }
      }
      tc::mbar_wait(&S.acc_full[bsel], use & 1);
      tc::fence_after_sync();
      const uint32_t lane_base =
          tmem + (uint32_t)bsel * kBufCols + ((uint32_t)(q4 * 32) << 16);
      double sq = 0.0;
      const int m = mt * kBM + r;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 8) {
        float v[8], w[8];
        if constexpr (kFold) {
          tc::tmem_ld8(lane_base + (uint32_t)c0, v);
          tc::tmem_ld8(lane_base + (uint32_t)(BN + c0), w);
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] += w[j];
#pragma unroll 1
          for (int a = 1; a < used; ++a) {
            tc::tmem_ld8(lane_base + (uint32_t)(a * kAccStride + c0), w);
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] += w[j];
            tc::tmem_ld8(lane_base + (uint32_t)(a * kAccStride + BN + c0), w);
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] += w[j];
          }
        } else {
          tc::tmem_ld8(lane_base + (uint32_t)(NACC * kAccStride + c0), v);  // corrections
#pragma unroll 1
          for (int a = 0; a < used; ++a) {
            tc::tmem_ld8(lane_base + (uint32_t)(a * kAccStride + c0), w);
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] += w[j];
          }
        }
        const int n0 = nt * BN + c0;
        if (p.ksplit > 1) {  // a K split: the raw tile, summed by splitk_epilogue_kernel
          float* w = p.ws + (((size_t)z * p.ntm + mt) * (size_t)(p.ntn * BN) + n0) * kBM + r;
#pragma unroll
          for (int j = 0; j < 8; ++j) w[(size_t)j * kBM] = v[j];
          continue;
        }
        switch (p.mode) {
          case kPlain:
            if (m < p.M)
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (n0 + j < p.N) p.out[(size_t)m * p.ldc + n0 + j] = v[j];
            break;
          // (every load of a column group is issued before its stores: out
          // may alias the inputs as far as the compiler knows, so a load
          // after a store would wait for it -- 8 serial round trips)
          case kConvFwd: {
            const int HW = p.H * p.W, img = m / HW, pos = m - img * HW;
            float bv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) bv[j] = n0 + j < p.N ? __ldg(p.bias + n0 + j) : 0.0f;
            if (m < p.M)
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int d = n0 + j;
                if (d < p.N) {
                  float o = v[j] + bv[j];
                  if (p.relu) o = fmaxf(o, 0.0f);
                  p.out[((size_t)img * p.D + d) * HW + pos] = o;
                }
              }
            break;
          }
          case kConvDx: {
            const int HW = p.H * p.W, img = m / HW, pos = m - img * HW;
            const size_t i0 = ((size_t)img * p.C + n0) * HW + pos;
            float mk[8];
            if (mk_ahead) {
#pragma unroll
              for (int j = 0; j < 8; ++j) mk[j] = mkpre[(c0 + j) & (BN <= 64 ? BN - 1 : 0)];
            } else {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                mk[j] = (p.mask && m < p.M && n0 + j < p.N) ? __ldg(p.mask + i0 + (size_t)j * HW) : 1.0f;
            }
            if (m < p.M)
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int c = n0 + j;
                if (c < p.N) p.out[i0 + (size_t)j * HW] = !(mk[j] > 0.0f) ? 0.0f : v[j];
              }
            break;
          }
          case kConvDwSum: {
            float* w = p.ws + (((size_t)z * p.ntm + mt) * (size_t)(p.ntn * BN) + n0) * kBM + r;
#pragma unroll
            for (int j = 0; j < 8; ++j) w[(size_t)j * kBM] = used > 0 ? v[j] : 0.0f;
            break;
          }
          case kConvDw: {
            int tap, c;
            if (p.big_c) {
              const int cgs = p.C / kBM;
              tap = mt / cgs;
              c = (mt - tap * cgs) * kBM + r;
            } else {
              const int sl = r / p.Cr;
              // (rows past the T slots -- 128 % Cr of them -- hold no tap)
              tap = sl < p.T ? mt * p.T + sl : 9;
              c = r - sl * p.Cr;
            }
            if (tap < 9 && c < p.C) {
              float* st = p.out + (size_t)z * p.D * p.C * 9;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const int d = n0 + j;
                if (d < p.N) {
                  st[((size_t)d * p.C + c) * 9 + tap] = v[j];
                  sq = fma((double)v[j], (double)v[j], sq);
                }
              }
            }
            break;
          }
        }
      }
      // the accumulator buffer is free once every epilogue warp has read it
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.acc_empty[bsel]);
      if (p.mode == kConvDw && p.tile_sq) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) S.sq[q4] = sq;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (t == 128)
          p.tile_sq[(size_t)z * p.tiles + mt * p.ntn + nt] =
              ((S.sq[0] + S.sq[1]) + S.sq[2]) + S.sq[3];
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, kCols);
}

template <int BN, bool H = false>
inline size_t smem_bytes() {
  return sizeof(Smem<BN, H>) + 1024;
}

// ---------------------------------------------------------------------------
// Per-example dW with halo reuse (3x3 / stride 1 / pad 1, W a multiple of 8,
// W <= 32, C <= 128, 32 output channels per tile). The dW of example z is
//   dW[d][c][u][v] = sum_p' xv[c][p'] g[d][p' - (u - 1) W]
// over the flattened positions p', xv the column-shifted copy v of the input
// (shift3_kernel: the +-1 column taps as whole copies, since a SWIZZLE_128B
// box starts on a 16-byte boundary). A stage is one K chunk of 32 positions:
// operand A = the three copies v (M rows = (v, c), Cr rows per copy) at
// [p0, p0 + 32); operand B = the cotangent at [p0 - W, p0 + 32 + W) (1 + W/16
// boxes of 32, zeros outside the image). The kernel row u reads B at a K
// offset of (2 - u) W positions -- a multiple of the 8-position MMA K step, so
// each step's descriptor starts inside one box -- into its own accumulator.
// Each input and cotangent element thus crosses L2 -> SMEM once per chunk
// (the cotangent once per box overlap) instead of once per tap: the tap-slot
// tiling of tma_gemm_kernel<kConvDw> re-reads both for every tap.
// Epilogue: the reference's stack layout (B, D, C, 3, 3) (strategies.cpp:156-170)
// and the tile's squared sum (fp64) for the per-example norm.
// ---------------------------------------------------------------------------
constexpr int kDwhBN = 32, kDwhStages = 3, kDwhBoxes = 3;

// 32 consecutive TMEM columns of the warp's 32 lanes (no wait: the caller
// issues tcgen05.wait::ld once for a batch of loads)
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
struct DwhSmem {
  float a_hi[kDwhStages][kBM * kBK];
  float a_lo[kDwhStages][kBM * kBK];
  float b[kDwhStages][kDwhBoxes][2][kDwhBN * kBK];  // per box: hi rows, then lo rows
  uint64_t full[kDwhStages], empty[kDwhStages], split[kDwhStages];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem;
  double sq[4];
  alignas(16) float stage[kDwhBN * 32 * 9];  // the tile's output rows (d, c, u, v), copied out coalesced
};

// RAW: the operands arrive as plain fp32 (one TMA load each) and warps 8-11
// write each stage's lo halves, x - trunc_tf32(x), next to them (the tensor
// core reads the fp32 tile itself as the truncated hi); else the hi and lo
// tensors are both loaded (split by the layout kernels).
constexpr int kDwhRawThreads = 384;

template <bool RAW>
__global__ void __launch_bounds__(RAW ? kDwhRawThreads : kThreads, 1)
    tma_dw_halo_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char raw[];
  DwhSmem& S = *reinterpret_cast<DwhSmem*>(
      (reinterpret_cast<uintptr_t>(raw) + 1023) & ~static_cast<uintptr_t>(1023));
  constexpr int NS = kDwhStages, BN = kDwhBN;
  constexpr uint32_t kCols = 512, kAcc = 2 * BN;  // folded accumulator: hi cols, then lo cols
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int total = p.ntn * p.ntm * p.nz;
  const int rot = p.rot, NB = rot == 1 ? 2 : 1;
  const uint32_t buf_cols = kCols / NB;
  const int nbox = 1 + (2 * p.W + kBK - 1) / kBK;  // cotangent halo boxes (W = 8, 16: 2; 32: 3)
  if (warp == 1) tc::tmem_alloc(&S.tmem, kCols);
  if (t == 0) {
    for (int s = 0; s < NS; ++s) {
      tc::mbar_init(&S.full[s], 1);
      tc::mbar_init(&S.empty[s], 3);  // one commit per issuing warp
      tc::mbar_init(&S.split[s], 4);  // one arrival per splitting warp
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&S.acc_full[b], 3);
      tc::mbar_init(&S.acc_empty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&p.ta) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&p.tb) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&p.ta_lo) : "memory");
    asm volatile("prefetch.tensormap [%0];" :: "l"(&p.tb_lo) : "memory");
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = S.tmem;

  if (warp == 0) {
    // ---- TMA producer ----
    if (lane == 0) {
      int g = 0;
      for (int tl = blockIdx.x; tl < total; tl += gridDim.x) {
        int nt, mt, z;
        tile_coords(p, tl, nt, mt, z);
        const uint32_t bytes =
            (RAW ? 1u : 2u) * ((uint32_t)(3 * p.Cr) * kBK * 4 + (uint32_t)(nbox * BN) * kBK * 4);
        for (int q = 0; q < p.nchunks; ++q, ++g) {
          const int s = g % NS;
          if (g >= NS) tc::mbar_wait(&S.empty[s], ((g / NS) - 1) & 1);
          const uint32_t bar = smem_u32(&S.full[s]);
          expect_tx(&S.full[s], bytes);
          const int p0 = q * kBK;
          for (int v = 0; v < 3; ++v) {  // rows (v, channel mt * Cr + c)
            const uint32_t o = (uint32_t)(v * p.Cr) * kBK * 4;
            tma_4d(smem_u32(S.a_hi[s]) + o, &p.ta, p0, mt * p.Cr, z, v, bar);
            if (!RAW) tma_4d(smem_u32(S.a_lo[s]) + o, &p.ta_lo, p0, mt * p.Cr, z, v, bar);
          }
          for (int i = 0; i < nbox; ++i) {
            const int pb = p0 - p.W + i * kBK;
            tma_3d(smem_u32(S.b[s][i][0]), &p.tb, pb, nt * BN, z, bar);
            if (!RAW) tma_3d(smem_u32(S.b[s][i][1]), &p.tb_lo, pb, nt * BN, z, bar);
          }
        }
      }
    }
  } else if (warp <= 3) {
    // ---- MMA issuers: warp 1 + u issues kernel row u into its own
    // accumulator (one thread issues an MMA only every ~50-120 cycles; three
    // issuers keep the tensor core fed, scripts/umma_rate.py) ----
    if (lane == 0) {
      const int u = warp - 1;
      const bool lo_narrow = p.narrow;
      constexpr uint32_t idesc = tc::idesc_tf32(kBM, 2 * BN);
      constexpr uint32_t idesc_lo = tc::idesc_tf32(kBM, BN);
      int g = 0, lt = 0;
      for (int tl = blockIdx.x; tl < total; tl += gridDim.x, ++lt) {
        const int bsel = NB == 2 ? (lt & 1) : 0;
        const int use = NB == 2 ? (lt >> 1) : lt;
        if (use > 0) tc::mbar_wait(&S.acc_empty[bsel], (use - 1) & 1);
        tc::fence_after_sync();
        const uint32_t buf = tmem + (uint32_t)bsel * buf_cols;
        for (int q = 0; q < p.nchunks; ++q, ++g) {
          const int s = g % NS;
          tc::mbar_wait(RAW ? &S.split[s] : &S.full[s], (g / NS) & 1);
          tc::fence_after_sync();
          const uint32_t ah = smem_u32(S.a_hi[s]), al = smem_u32(S.a_lo[s]);
          const int r = rot == 1 ? 0 : (q & 1);
          const bool first = q < rot;
          const uint32_t d = buf + (uint32_t)(u * rot + r) * kAcc;
#pragma unroll
          for (int k = 0; k < kBK / 8; ++k) {
            const int o = 8 * k + (2 - u) * p.W;  // cotangent position offset in the halo
            const uint32_t bh = smem_u32(S.b[s][o >> 5][0]) + 32u * ((o >> 3) & 3);
            tc::mma_tf32(d, desc_sw128(ah + 32u * k), desc_sw128(bh), idesc,
                         (!first || k) ? 1u : 0u);
            // Alo.Bhi only (N = BN): the lo.lo product is below the split's error
            if (lo_narrow)
              tc::mma_tf32(d, desc_sw128(al + 32u * k), desc_sw128(bh), idesc_lo, 1u);
            else
              tc::mma_tf32(d, desc_sw128(al + 32u * k), desc_sw128(bh), idesc, 1u);
          }
          tc::commit(&S.empty[s]);
        }
        tc::commit(&S.acc_full[bsel]);
      }
    }
  } else if (RAW && warp >= 8) {
    // ---- lo halves of each stage (both operands), then release it to the MMAs ----
    const int ct = t - 256;
    const int na4 = 3 * p.Cr * kBK / 4, nb4 = BN * kBK / 4;
    int g = 0;
    for (int tl = blockIdx.x; tl < total; tl += gridDim.x)
      for (int q = 0; q < p.nchunks; ++q, ++g) {
        const int s = g % NS;
        tc::mbar_wait(&S.full[s], (g / NS) & 1);
        const float4* ah = reinterpret_cast<const float4*>(S.a_hi[s]);
        float4* al = reinterpret_cast<float4*>(S.a_lo[s]);
        for (int e = ct; e < na4; e += 128) al[e] = lo_of(ah[e]);
        for (int i = 0; i < nbox; ++i) {
          const float4* bh = reinterpret_cast<const float4*>(S.b[s][i][0]);
          float4* bl = reinterpret_cast<float4*>(S.b[s][i][1]);
          for (int e = ct; e < nb4; e += 128) bl[e] = lo_of(bh[e]);
        }
        tc::fence_proxy_async();  // generic-proxy writes -> the tensor core's reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.split[s]);
      }
  } else if (warp >= 4 && warp < 8) {
    // ---- epilogue: TMEM -> registers -> the stack ----
    const int q4 = warp & 3, r = q4 * 32 + lane;
    const int v = r / p.Cr, cl = r - v * p.Cr;
    const int used = min(rot, p.nchunks);
    int lt = 0;
    for (int tl = blockIdx.x; tl < total; tl += gridDim.x, ++lt) {
      int nt, mt, z;
      tile_coords(p, tl, nt, mt, z);
      const int bsel = NB == 2 ? (lt & 1) : 0;
      const int use = NB == 2 ? (lt >> 1) : lt;
      tc::mbar_wait(&S.acc_full[bsel], use & 1);
      tc::fence_after_sync();
      const uint32_t lane_base = tmem + (uint32_t)bsel * buf_cols + ((uint32_t)(q4 * 32) << 16);
      const int c0t = mt * p.Cr, cval = min(p.Cr, p.C - c0t);  // the tile's channels
      const bool ok = v < 3 && cl < cval;
      float* sg = S.stage + cl * 9 + v;
      double sqj[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // independent fp64 chains
      const int nd = min(BN, p.N - nt * BN);
#pragma unroll 1
      for (int u = 0; u < 3; ++u) {
        uint32_t h[BN], l[BN];
        const uint32_t base = lane_base + (uint32_t)(u * rot) * kAcc;
        tmem_ld32_nowait(base, h);       // hi.hi + lo.hi
        tmem_ld32_nowait(base + BN, l);  // hi.lo + lo.lo
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float a[BN];
#pragma unroll
        for (int j = 0; j < BN; ++j) a[j] = __uint_as_float(h[j]) + __uint_as_float(l[j]);
        for (int e = 1; e < used; ++e) {
          tmem_ld32_nowait(base + (uint32_t)e * kAcc, h);
          tmem_ld32_nowait(base + (uint32_t)e * kAcc + BN, l);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < BN; ++j) a[j] += __uint_as_float(h[j]) + __uint_as_float(l[j]);
        }
        if (ok) {
          // stage[d][c][u][v]: lanes are consecutive c, a stride of 9 words (conflict-free)
#pragma unroll
          for (int j = 0; j < BN; ++j)
            if (j < nd) {
              sg[j * cval * 9 + 3 * u] = a[j];
              sqj[j & 7] = fma((double)a[j], (double)a[j], sqj[j & 7]);
            }
        }
      }
      double sq = ((sqj[0] + sqj[1]) + (sqj[2] + sqj[3])) + ((sqj[4] + sqj[5]) + (sqj[6] + sqj[7]));
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.acc_empty[bsel]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
      if (lane == 0) S.sq[q4] = sq;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (t == 128 && p.tile_sq)
        p.tile_sq[(size_t)z * p.tiles + mt * p.ntn + nt] = ((S.sq[0] + S.sq[1]) + S.sq[2]) + S.sq[3];
      // the staged rows: per output channel d, cval * 9 contiguous floats of
      // the reference's stack (B, D, C, 3, 3) (strategies.cpp:156-170)
      {
        const int row = cval * 9;
        float* dst = p.out + ((size_t)z * p.D + nt * BN) * p.C * 9 + (size_t)c0t * 9;
        const size_t ld = (size_t)p.C * 9;
        if (row % 4 == 0 && ld % 4 == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
          const int r4 = row / 4;
          for (int e = t - 128; e < nd * r4; e += 128) {
            const int d = e / r4, k = e - d * r4;
            *reinterpret_cast<float4*>(dst + d * ld + 4 * k) =
                *reinterpret_cast<const float4*>(S.stage + d * row + 4 * k);
          }
        } else {
          for (int e = t - 128; e < nd * row; e += 128) {
            const int d = e / row, k = e - d * row;
            dst[d * ld + k] = S.stage[e];
          }
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, kCols);
}

}  // namespace tg
}  // namespace pgb

// ---------------------------------------------------------------------------
// Layout kernels feeding the TMA operands, and the host side.
// ---------------------------------------------------------------------------
namespace pgb {
namespace tg {

// NCHW (B, C, HW) -> NHWC (B, HW, Cp) as the 3xTF32 pair (hi, lo), channels
// zero-padded to Cp (32 x 32 tiles through shared memory: coalesced on both
// sides)
__global__ void nchw_to_nhwc_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                    float* __restrict__ dst_lo, int C, int HW, int Cp) {
  __shared__ float tile[32][33];
  const int n = blockIdx.z, p0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int c = c0 + j, p = p0 + threadIdx.x;
    tile[j][threadIdx.x] = (c < C && p < HW) ? src[((size_t)n * C + c) * HW + p] : 0.0f;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int p = p0 + j, c = c0 + threadIdx.x;
    if (p < HW) {
      if (!dst_lo) {  // plain fp32 (the GEMM splits the lo half itself)
        dst[((size_t)n * HW + p) * Cp + c] = tile[threadIdx.x][j];
        continue;
      }
      float hi, lo;
      split2(tile[threadIdx.x][j], hi, lo);
      dst[((size_t)n * HW + p) * Cp + c] = hi;
      dst_lo[((size_t)n * HW + p) * Cp + c] = lo;
    }
  }
}

// nchw_to_nhwc_kernel over CB channels x 32 NQ positions per block (4096
// elements: (32, 128), (64, 64) or (128, 32)): each thread has its 16 loads in
// flight before the first store (the 32 x 32 version keeps ~4 KB per block in
// flight and ran at ~40% of HBM on the 32 x 32 CIFAR maps). Same values, same
// layout; the tile rows padded by one float keep both passes conflict-free.
template <int NQ, int CB>
__global__ void __launch_bounds__(256) nchw_to_nhwc_wide_kernel(const float* __restrict__ src,
                                                                float* __restrict__ dst,
                                                                float* __restrict__ dst_lo, int C,
                                                                int HW, int Cp) {
  static_assert(NQ * CB == 128, "16 elements per thread");
  constexpr int PB = 32 * NQ;
  __shared__ float tile[CB][PB + 1];  // [c][p]
  const int n = blockIdx.z, p0 = blockIdx.x * PB, c0 = blockIdx.y * CB;
  const int tx = threadIdx.x, ty = threadIdx.y;
  float v[CB / 8][NQ];
#pragma unroll
  for (int j = 0; j < CB / 8; ++j) {
    const int c = c0 + ty + 8 * j;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int p = p0 + 32 * q + tx;
      v[j][q] = (c < C && p < HW) ? __ldg(src + ((size_t)n * C + c) * HW + p) : 0.0f;
    }
  }
#pragma unroll
  for (int j = 0; j < CB / 8; ++j)
#pragma unroll
    for (int q = 0; q < NQ; ++q) tile[ty + 8 * j][32 * q + tx] = v[j][q];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < PB / 8; ++j) {
    const int pp = ty + 8 * j, p = p0 + pp;
    if (p < HW) {
#pragma unroll
      for (int k = 0; k < CB / 32; ++k) {
        const int c = c0 + tx + 32 * k;
        const float x = tile[tx + 32 * k][pp];
        if (!dst_lo) {
          dst[((size_t)n * HW + p) * Cp + c] = x;
        } else {
          float hi, lo;
          split2(x, hi, lo);
          dst[((size_t)n * HW + p) * Cp + c] = hi;
          dst_lo[((size_t)n * HW + p) * Cp + c] = lo;
        }
      }
    }
  }
}

// NCHW -> NHWC (channels padded to Cp) of Bi examples: 4096-element tiles
// shaped to the map (positions x channels), else the 32 x 32 kernel
inline void nchw_to_nhwc(const float* src, float* dst, float* dst_lo, int C, int HW, int Cp,
                         int Bi, cudaStream_t s) {
  const dim3 blk(32, 8);
  if (HW >= 128)
    nchw_to_nhwc_wide_kernel<4, 32><<<dim3((HW + 127) / 128, Cp / 32, Bi), blk, 0, s>>>(
        src, dst, dst_lo, C, HW, Cp);
  else if (HW > 32 && Cp % 64 == 0)
    nchw_to_nhwc_wide_kernel<2, 64><<<dim3((HW + 63) / 64, Cp / 64, Bi), blk, 0, s>>>(
        src, dst, dst_lo, C, HW, Cp);
  else if (Cp % 128 == 0)
    nchw_to_nhwc_wide_kernel<1, 128><<<dim3((HW + 31) / 32, Cp / 128, Bi), blk, 0, s>>>(
        src, dst, dst_lo, C, HW, Cp);
  else
    nchw_to_nhwc_kernel<<<dim3((HW + 31) / 32, Cp / 32, Bi), blk, 0, s>>>(src, dst, dst_lo, C, HW,
                                                                         Cp);
}

// the 3xTF32 pair of a tensor, element-wise
__global__ void split_kernel(const float* __restrict__ src, float* __restrict__ hi,
                             float* __restrict__ lo, long long n) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    split2(src[e], hi[e], lo[e]);
}

// dst[v][i] = src[i + v - 1] within the row (x + v - 1 in [0, W)), else 0:
// the three column-shifted copies the per-example dW boxes read
__global__ void shift3_kernel(const float* __restrict__ src, float* __restrict__ dst,
                              float* __restrict__ dst_lo, long long total, int W) {
  // one thread per source element writes its three copies (the row's
  // neighbours read once); 32-bit index math when the tensor allows it (the
  // 64-bit division per element was this kernel's bound)
  if (total < (1ll << 31)) {
    const unsigned T = (unsigned)total;
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < T; i += gridDim.x * blockDim.x) {
      const unsigned x = i % (unsigned)W;
      const float c = src[i];
      const float l = x > 0 ? src[i - 1] : 0.0f;
      const float r = x + 1 < (unsigned)W ? src[i + 1] : 0.0f;
      if (!dst_lo) {  // plain fp32 copies (the consumer splits them)
        dst[i] = l;
        dst[T + i] = c;
        dst[2ull * T + i] = r;
        continue;
      }
      split2(l, dst[i], dst_lo[i]);
      split2(c, dst[T + i], dst_lo[T + i]);
      split2(r, dst[2ull * T + i], dst_lo[2ull * T + i]);
    }
    return;
  }
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < 3 * total;
       e += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(e / total);
    const long long i = e - v * total;
    const int x = (int)(i % W), xs = x + v - 1;
    const float val = (xs >= 0 && xs < W) ? src[i + v - 1] : 0.0f;
    if (dst_lo)
      split2(val, dst[e], dst_lo[e]);
    else
      dst[e] = val;
  }
}

// The K splits of a forward / input-gradient GEMM added in split order, then
// that mode's epilogue (bias + relu into NCHW; relu mask into NCHW).
__global__ void splitk_epilogue_kernel(const Params p) {
  // four consecutive tile rows (positions) per thread: 16-byte loads of every
  // split issued before the ordered sum (the splits' loads were serialised
  // behind the running sum before), 16-byte mask loads and output stores;
  // 32-bit index math (a split is < 2^31 elements)
  const unsigned npad = (unsigned)p.ntn * (p.N <= 16 ? 16 : p.N <= 32 ? 32 : p.N <= 64 ? 64 : 128);
  const unsigned per_split = (unsigned)p.ntm * npad * kBM;
  const unsigned HW = p.mode == kPlain ? 1u : (unsigned)(p.H * p.W);
  const unsigned N = (unsigned)p.N, M = (unsigned)p.M;
  const bool vec = p.mode != kPlain && HW % 4 == 0;
  const int S = p.ksplit;
  for (unsigned q = blockIdx.x * blockDim.x + threadIdx.x; q < per_split / 4;
       q += gridDim.x * blockDim.x) {
    const unsigned e = 4 * q, r = e & (kBM - 1), t = e >> 7;
    const unsigned mt = t / npad, n = t - mt * npad;
    const unsigned m = mt * kBM + r;
    if (m >= M || n >= N) continue;
    float4 acc = *reinterpret_cast<const float4*>(p.ws + e);
    for (int z0 = 1; z0 < S; z0 += 8) {
      float4 u[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (z0 + k < S) u[k] = __ldcg(reinterpret_cast<const float4*>(p.ws + (size_t)(z0 + k) * per_split + e));
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (z0 + k < S) {
          acc.x += u[k].x;
          acc.y += u[k].y;
          acc.z += u[k].z;
          acc.w += u[k].w;
        }
    }
    float a[4] = {acc.x, acc.y, acc.z, acc.w};
    if (p.mode == kPlain) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (m + j < M) p.out[(size_t)(m + j) * p.ldc + n] = a[j];
      continue;
    }
    const unsigned img = m / HW, pos = m - img * HW;
    if (p.mode == kConvFwd) {
      const float b = p.bias[n];
      const size_t o = ((size_t)img * p.D + n) * HW + pos;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        a[j] += b;
        if (p.relu) a[j] = fmaxf(a[j], 0.0f);
      }
      if (vec) {
        *reinterpret_cast<float4*>(p.out + o) = make_float4(a[0], a[1], a[2], a[3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) p.out[o + j] = a[j];
      }
    } else {
      const size_t i = ((size_t)img * p.C + n) * HW + pos;
      float mk[4] = {1.0f, 1.0f, 1.0f, 1.0f};
      if (p.mask) {
        if (vec) {
          const float4 mv = *reinterpret_cast<const float4*>(p.mask + i);
          mk[0] = mv.x; mk[1] = mv.y; mk[2] = mv.z; mk[3] = mv.w;
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) mk[j] = p.mask[i + j];
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) a[j] = !(mk[j] > 0.0f) ? 0.0f : a[j];
      if (vec) {
        *reinterpret_cast<float4*>(p.out + i) = make_float4(a[0], a[1], a[2], a[3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) p.out[i + j] = a[j];
      }
    }
  }
}

// the clip-scaled cotangent of the summed weight gradient, as the 3xTF32 pair:
// fl(g * s_i) split into hi / lo (per element the reference's fl(g_ij * s_i)
// rounding moves from the weight gradient to the cotangent it is built from)
__global__ void scale_split_kernel(const float* __restrict__ g, const float* __restrict__ scale,
                                   long long per_ex, long long total, float* __restrict__ hi,
                                   float* __restrict__ lo) {
  if (total < (1ll << 31)) {  // 32-bit index math
    const unsigned T = (unsigned)total, pe = (unsigned)per_ex;
    for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < T; e += gridDim.x * blockDim.x)
      split2(__fmul_rn(g[e], scale[e / pe]), hi[e], lo[e]);
    return;
  }
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x)
    split2(__fmul_rn(g[e], scale[e / per_ex]), hi[e], lo[e]);
}

// Sum the example splits of the kConvDwSum workspace in split order (fixed:
// run-to-run deterministic) and scatter the tile rows (tap slot, channel) to
// the (D, C, 3, 3) parameter layout of the clipped-sum vector.
__global__ void dw_sum_reduce_kernel(const float* __restrict__ ws, int splits, int ntm, int npad,
                                     int C, int D, int Cr, int T, int big,
                                     float* __restrict__ out) {
  // 32-bit index math (a split of the workspace is < 2^31 elements)
  const unsigned per_split = (unsigned)ntm * npad * kBM;
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < per_split;
       e += gridDim.x * blockDim.x) {
    const int r = (int)(e & (kBM - 1));
    const unsigned t = e >> 7;
    const int mt = (int)(t / (unsigned)npad), n = (int)(t - (unsigned)mt * npad);
    int tap, c;
    if (big) {
      const int cgs = C / kBM;
      tap = mt / cgs;
      c = (mt - tap * cgs) * kBM + r;
    } else {
      const int sl = r / Cr;
      tap = mt * T + sl;
      c = r - sl * Cr;
    }
    if (tap >= 9 || c >= C || n >= D) continue;
    float acc = ws[e];
    for (int z = 1; z < splits; ++z) acc = __fadd_rn(acc, ws[(size_t)z * per_split + e]);
    out[((size_t)n * C + c) * 9 + tap] = acc;
  }
}

// Every TMA conv layer's forward and input-gradient weight operands in one
// launch per step (they change only at the update): segment k writes the
// conv_wt_fwd_kernel (kind 0) or conv_wt_dx_kernel (kind 1) layout of W.
constexpr int kMaxWtSegs = 32;
struct WtAll {
  int n;
  const float* W[kMaxWtSegs];
  int D[kMaxWtSegs], C[kMaxWtSegs], P[kMaxWtSegs], kind[kMaxWtSegs];  // P: Cp or Dp
  long long off[kMaxWtSegs + 1];  // element offsets into the output (prefix sums)
  float* hi;
  float* lo;
};

__global__ void conv_wt_all_kernel(const WtAll A) {
  const long long total = A.off[A.n];
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int k = 0;
    while (k + 1 < A.n && A.off[k + 1] <= e) ++k;
    const int r0 = (int)(e - A.off[k]);
    const int D = A.D[k], C = A.C[k], Pp = A.P[k];
    float v;
    if (A.kind[k] == 0) {  // Wt[d][tap * Cp + c]
      const int d = r0 / (9 * Pp), r = r0 - d * 9 * Pp, tap = r / Pp, c = r - tap * Pp;
      v = c < C ? A.W[k][((size_t)d * C + c) * 9 + tap] : 0.0f;
    } else {  // Wt2[c][tap * Dp + d]
      const int c = r0 / (9 * Pp), r = r0 - c * 9 * Pp, tap = r / Pp, d = r - tap * Pp;
      v = d < D ? A.W[k][((size_t)d * C + c) * 9 + tap] : 0.0f;
    }
    split2(v, A.hi[e], A.lo[e]);
  }
}

// Probe (self-test): one TMA box {32, 4} of a SWIZZLE_128B map at an arbitrary
// (possibly misaligned or negative) innermost coordinate x0, unswizzled into out
// (4 rows x 32): does a box start need 16-byte alignment in the innermost dim?
__global__ void tma_box_probe_kernel(const __grid_constant__ CUtensorMap m, int x0, int y0,
                                     float* out) {
  __shared__ __align__(1024) float tile[4 * 32];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    expect_tx(&bar, 4 * 32 * 4);
    tma_2d(smem_u32(tile), &m, x0, y0, smem_u32(&bar));
  }
  __syncthreads();
  tc::mbar_wait(&bar, 0);
  for (int e = threadIdx.x; e < 128; e += blockDim.x) {
    const int r = e / 32, c = e % 32;          // logical row, element
    const int chunk = (c / 4) ^ (r % 8);       // 16-byte chunk after the 128-B swizzle
    out[e] = tile[r * 32 + chunk * 4 + (c % 4)];
  }
}

// conv weights (D, C, 3, 3) -> the forward B operand Wt[d][tap * Cp + c]
__global__ void conv_wt_fwd_kernel(const float* __restrict__ W, float* __restrict__ wt,
                                   float* __restrict__ wt_lo, int D, int C, int Cp) {
  const int n = D * 9 * Cp;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int d = e / (9 * Cp), r = e - d * 9 * Cp, tap = r / Cp, c = r - tap * Cp;
    split2(c < C ? W[((size_t)d * C + c) * 9 + tap] : 0.0f, wt[e], wt_lo[e]);
  }
}

// conv weights (D, C, 3, 3) -> the input-gradient B operand Wt2[c][tap * Dp + d]
__global__ void conv_wt_dx_kernel(const float* __restrict__ W, float* __restrict__ wt,
                                  float* __restrict__ wt_lo, int D, int C, int Dp) {
  const int n = C * 9 * Dp;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const int c = e / (9 * Dp), r = e - c * 9 * Dp, tap = r / Dp, d = r - tap * Dp;
    split2(d < D ? W[((size_t)d * C + c) * 9 + tap] : 0.0f, wt[e], wt_lo[e]);
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link
// dependency on libcuda)
inline EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        !f || q != cudaDriverEntryPointSuccess)
      raise(PGB_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable");
    fn = reinterpret_cast<EncodeFn>(f);
  }
  return fn;
}

// fp32 tensor map, 128-B swizzle, zero out-of-bounds fill. dims/box innermost
// first; strides (bytes) of dims 1..rank-1.
inline void make_map(CUtensorMap* m, const float* base, int rank, const uint64_t* dims,
                     const uint64_t* strides, const uint32_t* box) {
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = 1;
    if (i + 1 < rank) st[i] = strides[i];
  }
  const CUresult r = encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank,
                               const_cast<float*>(base), d, st, b, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    raise(PGB_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

inline int pick_bn(int n) { return n <= 16 ? 16 : n <= 32 ? 32 : n <= 64 ? 64 : 128; }

inline int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, bool H, bool RAW>
inline void launch_kernel(const Params& p, int ctas, cudaStream_t s) {
  tma_gemm_kernel<BN, H, RAW><<<ctas, RAW ? kRawThreads : kThreads, smem_bytes<BN, H>(), s>>>(p);
}

template <int BN, bool H>
inline void set_attrs() {
  cudaFuncSetAttribute(tma_gemm_kernel<BN, H, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem_bytes<BN, H>());
  cudaFuncSetAttribute(tma_gemm_kernel<BN, H, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem_bytes<BN, H>());
}

template <int BN>
inline void launch_bn(const Params& p, int ctas, cudaStream_t s) {
  static int attr_dev = -1;  // the attribute is set once per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    set_attrs<BN, false>();
    if constexpr (BN <= 64) set_attrs<BN, true>();
    attr_dev = dev;
  }
  if constexpr (BN <= 64) {
    if (p.halo) {
      if (p.raw)
        launch_kernel<BN, true, true>(p, ctas, s);
      else
        launch_kernel<BN, true, false>(p, ctas, s);
      return;
    }
  }
  if (p.raw)
    launch_kernel<BN, false, true>(p, ctas, s);
  else
    launch_kernel<BN, false, false>(p, ctas, s);
}

inline size_t dwh_smem_bytes() { return sizeof(DwhSmem) + 1024; }

// folded tiles issue lo.hi at N = BN, dropping the lo.lo product (PGB_LOLO=1:
// the 2 BN-wide lo MMA, lo.lo included; read once per process)
inline bool narrow_lo() {
  static const bool v = std::getenv("PGB_LOLO") == nullptr;
  return v;
}

// tiles: (N tiles, M tiles, examples)
inline void launch_dwh(const Params& p0, dim3 tiles, cudaStream_t s) {
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(tma_dw_halo_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)dwh_smem_bytes());
    cudaFuncSetAttribute(tma_dw_halo_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)dwh_smem_bytes());
    attr_dev = dev;
  }
  Params p = p0;
  p.ntn = (int)tiles.x;
  p.ntm = (int)tiles.y;
  p.nz = (int)tiles.z;
  p.narrow = narrow_lo() ? 1 : 0;
  const long long total = (long long)p.ntn * p.ntm * p.nz;
  const int ctas = (int)std::min<long long>(total, num_sms());
  if (p.raw)
    tma_dw_halo_kernel<true><<<ctas, kDwhRawThreads, dwh_smem_bytes(), s>>>(p);
  else
    tma_dw_halo_kernel<false><<<ctas, kThreads, dwh_smem_bytes(), s>>>(p);
}

// tiles: (N tiles, M tiles, GEMMs); one persistent CTA per SM walks them
inline void launch(const Params& p0, int bn, dim3 tiles, cudaStream_t s) {
  Params p = p0;
  p.ntn = (int)tiles.x;
  p.ntm = (int)tiles.y;
  p.nz = (int)tiles.z;
  p.narrow = narrow_lo() ? 1 : 0;
  const long long total = (long long)p.ntn * p.ntm * p.nz;
  const int ctas = (int)std::min<long long>(total, num_sms());
  switch (bn) {
    case 16: launch_bn<16>(p, ctas, s); break;
    case 32: launch_bn<32>(p, ctas, s); break;
    case 64: launch_bn<64>(p, ctas, s); break;
    default: launch_bn<128>(p, ctas, s); break;
  }
}

// The TMA engine takes 3x3 / stride 1 / pad 1 convolutions whose rows tile a
// 128-position block: W in {4, 8, 16, 32}, and either 128 | H*W or H*W | 128.
inline bool conv_ok(const ConvGeom& g) {
  if (g.k != 3 || g.stride != 1 || g.pad != 1 || g.Ho != g.H || g.Wo != g.W) return false;
  if (!(g.W == 4 || g.W == 8 || g.W == 16 || g.W == 32)) return false;
  const int hw = g.H * g.W;
  return hw >= 128 ? hw % 128 == 0 : 128 % hw == 0;
}

// the halo per-example dW fits: 3x3 / stride 1 / pad 1, W a multiple of 8
// up to 32, C <= 128
inline bool dwh_ok(const ConvGeom& g) {
  return conv_ok(g) && g.W % 8 == 0 && g.W <= 32 && g.C <= 128;
}

// halo per-example dW M tiling: M rows (v, c) for Cr channels per tile
inline void dwh_tiling(int C, int& Cr, int& T, int& mtiles) {
  Cr = std::min(32, (C + 7) / 8 * 8);  // channels per tile (rows per copy v)
  T = 3;
  mtiles = (C + Cr - 1) / Cr;
}

inline int round32(int c) { return (c + 31) / 32 * 32; }

// A-operand box of the forward / input-gradient GEMMs: 32 channels x W x by rows x bn images
inline void fwd_box(const ConvGeom& g, int& by, int& bn) {
  const int rows = 128 / g.W;
  by = rows < g.H ? rows : g.H;
  bn = 128 / (g.W * by);
}

// per-example dW M tiling: rows per tap slot Cr, slots per tile T, tiles
inline void dw_tiling(int C, int& Cr, int& T, int& big, int& mtiles) {
  big = C >= 128 && C % 128 == 0;
  if (big) {
    Cr = 128;
    T = 1;
    mtiles = 9 * C / 128;
  } else {
    Cr = (C + 7) / 8 * 8;
    T = 128 / Cr;
    if (T < 1) T = 1;
    mtiles = (9 + T - 1) / T;
  }
}

}  // namespace tg
}  // namespace pgb
