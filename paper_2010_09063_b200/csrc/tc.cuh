// tcgen05 (5th-generation tensor core) building blocks for sm_100a:
// TMEM allocation, UMMA shared-memory descriptors (K-major, no swizzle),
// kind::tf32 MMA issue, commit-to-mbarrier, TMEM -> register loads.
//
// fp32 accuracy comes from the 3xTF32 split: x = hi + lo with
// hi = rna_tf32(x), lo = x - hi; D += Ahi.Bhi + Ahi.Blo + Alo.Bhi gives
// ~1e-7 normwise error (1xTF32 gives ~3e-4 and fails the 1e-5 parity bar,
// SURVEY 8(d)).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace pgb {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA shared-memory matrix descriptor, SWIZZLE_NONE, K-major canonical
// layout ((8,m),(4,2)) : ((16B, SBO), (4B, LBO)) -- core matrices of
// 8 rows x 16 bytes, LBO between the two K-adjacent core matrices of one MMA,
// SBO between 8-row groups.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

// Instruction descriptor: kind::tf32, fp32 accumulate, both operands K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4)                       // D format f32
         | (2u << 7)                     // A format tf32
         | (2u << 10)                    // B format tf32
         | ((uint32_t)(N >> 3) << 17)    // N / 8
         | ((uint32_t)(M >> 4) << 24);   // M / 16
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
      :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// Arrive on `bar` once every previously issued tcgen05.mma of this thread
// has completed (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
      :: "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// One full warp: allocate `ncols` TMEM columns (power of 2 >= 32); the base
// address lands in *slot.
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               :: "r"(smem_u32(slot)), "r"(ncols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;"
               :: "r"(taddr), "r"(ncols) : "memory");
}

// Warp w reads TMEM lanes 32w..32w+31 (one accumulator row per thread),
// 8 consecutive 32-bit columns starting at `taddr`'s column.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
}

// 3xTF32 split.
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  lo = x - hi;
}

// Float offset of element (r, k) inside one K-major canonical tile whose K
// extent is BK: 8x4 core matrices, K-adjacent cores 32 floats apart (LBO =
// 128 B), 8-row groups BK*8 floats apart (SBO = BK*32 B).
template <int BK>
__device__ __forceinline__ int canon_off(int r, int k) {
  return (r & 7) * 4 + (k & 3) + (r >> 3) * (BK * 8) + (k >> 2) * 32;
}

// ---------------------------------------------------------------------------
// Generic tcgen05 GEMM with gathered operands:
//   C[z][m][n] = sum_k A(z,m,k) * B(z,n,k)       (then op.store)
// BM = 128 rows per CTA (UMMA_M = 128, one accumulator row per TMEM lane),
// BN columns (multiple of 16, <= 128), BK = 32 per pipeline stage, 2 stages.
// NT threads all gather (fp32 -> hi/lo tf32 in the canonical layout); thread
// 0 issues 4 k-steps x 3 MMAs per stage and commits to the stage's mbarrier,
// so the gather of the next stage overlaps the tensor core. Three TMEM
// accumulators (hi.hi even/odd chunks + the hi.lo/lo.hi correction) keep the
// fp32 accumulation chains short. Epilogue: tcgen05.ld TMEM -> registers.
//
// Ops with kTableA gather A as an implicit im2col window:
//   A(m,k) = src[row.base + k.base + (row.iy + k.dy) * W + (row.ix + k.dx)]
// (zero outside [0,H) x [0,W)), with per-row info computed once per CTA and
// per-k info once per K chunk -- a few integer ops per element.
// ---------------------------------------------------------------------------
constexpr int kBM = 128, kBK = 32;

template <int BN>
struct TcSmem {
  float ahi[2][kBM * kBK], alo[2][kBM * kBK];
  float bhi[2][BN * kBK], blo[2][BN * kBK];
  int4 rowinfo[kBM];
  int4 kinfo[2][kBK];
  uint64_t bar[2];
  uint32_t tmem;
};

struct NoTable {
  static constexpr bool kTableA = false;
};

// Ops with a `double* tile_sq` member also get each tile's sum of squared
// outputs (fp64), written to tile_sq[z * tiles + tile]: the per-example norm
// of a materialised gradient block without a second pass over it.
// Ops with a4 / b4 gather four consecutive k at once (one index computation,
// 16-byte shared-memory stores; the per-example conv dW, where k runs along an
// output row) when op.vec_ok()
template <class T, class = void>
struct HasA4 : std::false_type {};
template <class T>
struct HasA4<T, std::void_t<decltype(&T::a4)>> : std::true_type {};

template <class T, class = void>
struct HasPre : std::false_type {};
template <class T>
struct HasPre<T, std::void_t<decltype(&T::pre)>> : std::true_type {};

template <class T, class = void>
struct HasTileSq : std::false_type {};
template <class T>
struct HasTileSq<T, std::void_t<decltype(&T::tile_sq)>> : std::true_type {};

template <class Op, int BN, int NT>
__global__ void __launch_bounds__(NT) tc_gemm_kernel(Op op) {
  extern __shared__ __align__(1024) unsigned char raw[];
  TcSmem<BN>& S = *reinterpret_cast<TcSmem<BN>*>(raw);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int z = blockIdx.z;
  const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * BN;
  const int M = op.M, N = op.N, K = op.K;
  // four accumulators: hi.hi alternating between two (even / odd K chunks),
  // hi.lo and lo.hi each their own, so the three MMAs of a K step come from
  // three issuing warps (one thread issues a tcgen05.mma only every ~120
  // cycles; scripts/umma_rate.py)
  constexpr uint32_t kCols = 4 * BN <= 32 ? 32 : 4 * BN <= 64 ? 64 : 4 * BN <= 128 ? 128
                             : 4 * BN <= 256 ? 256 : 512;
  static_assert(4 * BN <= 512, "BN too large for four TMEM accumulators");
  static_assert(NT >= 96, "three issuing warps");
  if (warp == 0) tmem_alloc(&S.tmem, kCols);
  if (t == 0) {
    mbar_init(&S.bar[0], 3);
    mbar_init(&S.bar[1], 3);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (Op::kTableA) {
    for (int r = t; r < kBM; r += NT) S.rowinfo[r] = op.row_info(z, m0 + r);
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = S.tmem;
  constexpr uint32_t idesc = idesc_tf32(kBM, BN);
  const int nk = (K + kBK - 1) / kBK;
  int H = 0, Wd = 0;
  const float* src = nullptr;
  if constexpr (Op::kTableA) {
    H = op.img_h();
    Wd = op.img_w();
    src = op.img(z);
  }
  // Operands are gathered one K chunk ahead into registers (kA + kB values
  // per thread), so the global-load latency of chunk kc+1 overlaps the split,
  // the shared stores and the MMAs of chunk kc.
  constexpr int kA = kBM * kBK / NT, kB = (BN * kBK + NT - 1) / NT;
  float ra[kA], rb[kB];
  // per-k gather info of a chunk, computed once per CTA into kinfo[kc & 1]
  auto kinfo_fill = [&](int kc) {
    if constexpr (Op::kTableA) {
      if (t < kBK) S.kinfo[kc & 1][t] = op.k_info(z, kc * kBK + t);
    }
  };
  auto fetch = [&](int kc) {
    const int k0 = kc * kBK;
#pragma unroll
    for (int i = 0; i < kA; ++i) {
      const int e = t + i * NT;
      const int core = e >> 5, in = e & 31;
      const int r = (core % (kBM / 8)) * 8 + (in >> 2);
      const int k = (core / (kBM / 8)) * 4 + (in & 3);
      float v;
      if constexpr (Op::kTableA) {
        const int4 ri = S.rowinfo[r];
        const int4 ki = S.kinfo[kc & 1][k];
        const int iy = ri.y + ki.y, ix = ri.z + ki.z;
        const bool ok = (ri.w & ki.w) && (unsigned)iy < (unsigned)H && (unsigned)ix < (unsigned)Wd;
        v = ok ? __ldg(src + ri.x + ki.x + iy * Wd + ix) : 0.0f;
      } else {
        const int m = m0 + r, kk = k0 + k;
        v = (m < M && kk < K) ? op.a(z, m, kk) : 0.0f;
      }
      ra[i] = v;
    }
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      const int e = t + i * NT;
      float v = 0.0f;
      if (e < BN * kBK) {
        const int core = e >> 5, in = e & 31;
        const int r = (core % (BN / 8)) * 8 + (in >> 2);
        const int k = (core / (BN / 8)) * 4 + (in & 3);
        const int n = n0 + r, kk = k0 + k;
        v = (n < N && kk < K) ? op.b(z, n, kk) : 0.0f;
      }
      rb[i] = v;
    }
  };
  // four consecutive k per thread (HasA4 ops). A warp covers 8 rows x 4 quads:
  // lane = 8 * (k4 % 4) + row % 8, so each 8-lane phase of a 16-byte store
  // hits 8 distinct 16-B slots of the core-matrix rows (conflict-free) and
  // each load instruction touches 8 rows x 64 contiguous bytes
  constexpr int kA4 = kBM * kBK / 4 / NT, kB4 = (BN * kBK / 4 + NT - 1) / NT;
  auto quad = [](int eq, int rows, int& r, int& k4) {
    const int l = eq & 31, gi = eq >> 5, rg = rows / 8;
    r = (gi % rg) * 8 + (l & 7);
    k4 = (gi / rg) * 4 + (l >> 3);
  };
  bool vec = false;
  if constexpr (HasA4<Op>::value) vec = op.vec_ok();
  float4 ra4[HasA4<Op>::value ? kA4 : 1], rb4[HasA4<Op>::value ? kB4 : 1];
  auto fetch4 = [&](int kc) {
    if constexpr (HasA4<Op>::value) {
      const int k0 = kc * kBK;
#pragma unroll
      for (int i = 0; i < kA4; ++i) {
        int r, k4;
        quad(t + i * NT, kBM, r, k4);
        ra4[i] = op.a4(z, S.rowinfo[r], k0 + 4 * k4);
      }
#pragma unroll
      for (int i = 0; i < kB4; ++i) {
        const int eq = t + i * NT;
        int n, k4;
        quad(eq, BN, n, k4);
        rb4[i] = eq < BN * kBK / 4 ? op.b4(z, n0 + n, k0 + 4 * k4) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  };
  auto store4 = [&](int s) {
    if constexpr (HasA4<Op>::value) {
      auto put = [&](float* hi_base, float* lo_base, int r, int k4, const float4& v) {
        float4 h, l;
        split_tf32(v.x, h.x, l.x);
        split_tf32(v.y, h.y, l.y);
        split_tf32(v.z, h.z, l.z);
        split_tf32(v.w, h.w, l.w);
        const int o = canon_off<kBK>(r, 4 * k4);
        *reinterpret_cast<float4*>(hi_base + o) = h;
        *reinterpret_cast<float4*>(lo_base + o) = l;
      };
#pragma unroll
      for (int i = 0; i < kA4; ++i) {
        int r, k4;
        quad(t + i * NT, kBM, r, k4);
        put(S.ahi[s], S.alo[s], r, k4, ra4[i]);
      }
#pragma unroll
      for (int i = 0; i < kB4; ++i) {
        const int eq = t + i * NT;
        int n, k4;
        quad(eq, BN, n, k4);
        if (eq < BN * kBK / 4) put(S.bhi[s], S.blo[s], n, k4, rb4[i]);
      }
    }
  };
  kinfo_fill(0);
  __syncthreads();
  if (vec) fetch4(0);
  else fetch(0);
  for (int kc = 0; kc < nk; ++kc) {
    const int s = kc & 1;
    // chunk kc+1's gather info (slot s^1 was last read by fetch(kc-1), two
    // barriers ago); made visible by this iteration's barrier
    if (kc + 1 < nk) kinfo_fill(kc + 1);
    if (kc >= 2) mbar_wait(&S.bar[s], ((kc - 2) >> 1) & 1);
    // split + store this chunk (lanes cover one 8x4 core matrix: conflict-free)
    if (vec) {
      store4(s);
    } else {
#pragma unroll
    for (int i = 0; i < kA; ++i) {
      const int e = t + i * NT;
      const int core = e >> 5, in = e & 31;
      const int r = (core % (kBM / 8)) * 8 + (in >> 2);
      const int k = (core / (kBM / 8)) * 4 + (in & 3);
      float hi, lo;
      split_tf32(ra[i], hi, lo);
      const int o = canon_off<kBK>(r, k);
      S.ahi[s][o] = hi;
      S.alo[s][o] = lo;
    }
#pragma unroll
    for (int i = 0; i < kB; ++i) {
      const int e = t + i * NT;
      if (e < BN * kBK) {
        const int core = e >> 5, in = e & 31;
        const int r = (core % (BN / 8)) * 8 + (in >> 2);
        const int k = (core / (BN / 8)) * 4 + (in & 3);
        float hi, lo;
        split_tf32(rb[i], hi, lo);
        const int o = canon_off<kBK>(r, k);
        S.bhi[s][o] = hi;
        S.blo[s][o] = lo;
      }
    }
    }  // scalar store
    fence_proxy_async();
    __syncthreads();
    if (lane == 0 && warp < 3) {
      // warp 0: hi.hi, warp 1: hi.lo, warp 2: lo.hi
      fence_after_sync();
      const uint32_t a = smem_u32(warp == 2 ? S.alo[s] : S.ahi[s]);
      const uint32_t b = smem_u32(warp == 1 ? S.blo[s] : S.bhi[s]);
      const uint32_t d = warp == 0 ? tmem + (uint32_t)((kc & 1) * BN) : tmem + (uint32_t)((1 + warp) * BN);
      const bool first = warp == 0 ? kc <= 1 : kc == 0;
#pragma unroll
      for (int ks = 0; ks < kBK / 8; ++ks) {
        const uint32_t off = ks * 256;  // two 128-B core matrices per k-step
        mma_tf32(d, make_desc(a + off, 128, kBK * 32), make_desc(b + off, 128, kBK * 32), idesc,
                 (first && ks == 0) ? 0u : 1u);
      }
      commit(&S.bar[s]);
    }
    // next chunk's operands into registers while the tensor core runs
    if (kc + 1 < nk) {
      if (vec) fetch4(kc + 1);
      else fetch(kc + 1);
    }
  }
  // all MMAs done once the last commit lands (they complete in issue order)
  mbar_wait(&S.bar[(nk - 1) & 1], ((nk - 1) >> 1) & 1);
  fence_after_sync();
  // warp w reads TMEM lanes 32(w%4).. ; warps >= 4 take the upper column half
  constexpr int kGroups = NT / 128;
  const int row = m0 + (warp & 3) * 32 + lane;
  const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const int cbeg = (warp >> 2) * (BN / kGroups), cend = cbeg + BN / kGroups;
  double sq = 0.0;
#pragma unroll 1
  for (int c0 = cbeg; c0 < cend; c0 += 8) {
    float v[8], v1[8], vc[8], vd[8];
    tmem_ld8(lane_base + (uint32_t)c0, v);
    tmem_ld8(lane_base + (uint32_t)(2 * BN + c0), vc);
    tmem_ld8(lane_base + (uint32_t)(3 * BN + c0), vd);
    if (nk > 1) {
      tmem_ld8(lane_base + (uint32_t)(BN + c0), v1);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] += v1[j];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] += vc[j] + vd[j];
    if (row < M) {
      if constexpr (HasPre<Op>::value) {
        // every load of the group before its stores (a load after a
        // possibly-aliasing store waits for it)
        float pv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) pv[j] = n0 + c0 + j < N ? op.pre(z, row, n0 + c0 + j) : 0.0f;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (n0 + c0 + j < N) op.store_pre(z, row, n0 + c0 + j, v[j], pv[j]);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (n0 + c0 + j < N) {
            op.store(z, row, n0 + c0 + j, v[j]);
            if constexpr (HasTileSq<Op>::value) sq = fma((double)v[j], (double)v[j], sq);
          }
      }
    }
  }
  if constexpr (HasTileSq<Op>::value) {
    __shared__ double sq_red[NT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if (lane == 0) sq_red[warp] = sq;
    fence_before_sync();
    __syncthreads();
    if (t == 0) {
      double tot = 0.0;
#pragma unroll
      for (int w = 0; w < NT / 32; ++w) tot += sq_red[w];
      const int tiles = gridDim.x * gridDim.y;
      op.tile_sq[(size_t)z * tiles + blockIdx.y * gridDim.x + blockIdx.x] = tot;
    }
  } else {
    fence_before_sync();
    __syncthreads();
  }
  if (warp == 0) tmem_dealloc(tmem, kCols);
}

template <class Op, int BN>
inline size_t tc_smem_bytes() {
  return sizeof(TcSmem<BN>);
}

// ---------------------------------------------------------------------------
// Operand layouts without swizzle (byte offsets inside one operand tile).
// K-major: core matrices of 8 rows x 16 B (4 tf32 along K); rows 16 B apart,
//   8-row groups SBO apart, the two K-adjacent cores of one K=8 step LBO apart.
// MN-major: core matrices of 8 K-rows x 16 B (4 tf32 along M/N); 4-element
//   M/N groups SBO apart, K rows 16 B apart (one core spans a K=8 step).
// In both, the block [8 rows][4 floats] with the 4 floats contiguous is the
// same 128-byte core, which lets one shared-memory buffer serve as a K-major
// operand of one GEMM and an MN-major operand of another.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr uint32_t idesc_tf32_mj(int M, int N, int a_mn, int b_mn) {
  return idesc_tf32(M, N) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16);
}

__device__ __forceinline__ uint32_t kmaj_off(int r, int k, uint32_t sbo, uint32_t lbo) {
  return (uint32_t)((r & 7) * 16 + (k & 3) * 4) + (uint32_t)(r >> 3) * sbo + (uint32_t)(k >> 2) * lbo;
}
__device__ __forceinline__ uint32_t mnmaj_off(int r, int k, uint32_t sbo, uint32_t lbo) {
  return (uint32_t)((r & 3) * 4 + (k & 7) * 16) + (uint32_t)(r >> 2) * sbo + (uint32_t)(k >> 3) * lbo;
}

// Layout probe (self-test): D (M x N) = A (M x K) . B (N x K)^T with A and
// B staged in the K-major or MN-major layouts above, cores packed along M/N
// (SBO = 128 B) then along K. One CTA of 128 threads; the raw TMEM contents
// (128 lanes x N columns) are dumped so the host checks the accumulator row
// -> lane map too (M = 128: lane m; M = 64: lane m % 16 + 32 (m / 16)).
__global__ void __launch_bounds__(128) umma_probe_kernel(const float* __restrict__ A,
                                                         const float* __restrict__ B,
                                                         float* __restrict__ Draw, int M, int N,
                                                         int K, int a_mn, int b_mn) {
  extern __shared__ __align__(1024) unsigned char raw[];
  float* sa = reinterpret_cast<float*>(raw);
  float* sb = sa + 128 * 32;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const uint32_t a_lbo = a_mn ? (uint32_t)(M / 4) * 128 : (uint32_t)(M / 8) * 128;
  const uint32_t b_lbo = b_mn ? (uint32_t)(N / 4) * 128 : (uint32_t)(N / 8) * 128;
  for (int e = t; e < 128 * 32 + 256 * 32; e += 128) sa[e] = 0.0f;
  __syncthreads();
  for (int e = t; e < M * K; e += 128) {
    const int r = e / K, k = e % K;
    const uint32_t o = a_mn ? mnmaj_off(r, k, 128, a_lbo) : kmaj_off(r, k, 128, a_lbo);
    sa[o / 4] = A[e];
  }
  for (int e = t; e < N * K; e += 128) {
    const int r = e / K, k = e % K;
    const uint32_t o = b_mn ? mnmaj_off(r, k, 128, b_lbo) : kmaj_off(r, k, 128, b_lbo);
    sb[o / 4] = B[e];
  }
  if (warp == 0) tmem_alloc(&tslot, 256);
  if (t == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tslot;
  if (t == 0) {
    const uint32_t idesc = idesc_tf32_mj(M, N, a_mn, b_mn);
    for (int s = 0; s < K / 8; ++s) {
      const uint32_t ao = a_mn ? (uint32_t)s * a_lbo : (uint32_t)s * 2 * a_lbo;
      const uint32_t bo = b_mn ? (uint32_t)s * b_lbo : (uint32_t)s * 2 * b_lbo;
      // MN-major: SBO = M/N-group stride, LBO = K-group stride
      const uint64_t da = make_desc(smem_u32(sa) + ao, a_lbo, 128);
      const uint64_t db = make_desc(smem_u32(sb) + bo, b_lbo, 128);
      mma_tf32(tmem, da, db, idesc, s > 0 ? 1u : 0u);
    }
    commit(&bar);
  }
  mbar_wait(&bar, 0);
  fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 8) {
    float v[8];
    tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
    for (int j = 0; j < 8 && c0 + j < N; ++j) Draw[(warp * 32 + lane) * N + c0 + j] = v[j];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

// Issue-rate microbenchmark: `reps` back-to-back kind::tf32 MMAs of shape
// M x N x 8 from one thread, cycles from the first issue to the commit's
// completion. mode bit 0: alternate two accumulators; bit 1: stream the
// operand addresses (A +4 KB, B +2 KB per MMA, wrapping in 64 KB / 32 KB);
// bit 2: every other thread polls the completion mbarrier meanwhile.
__global__ void __launch_bounds__(1024) umma_rate_kernel(int M, int N, int reps, uint32_t a_lbo,
                                                         uint32_t a_sbo, uint32_t b_lbo,
                                                         uint32_t b_sbo, int mode,
                                                         long long* cycles) {
  extern __shared__ __align__(1024) unsigned char raw[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  float* sm = reinterpret_cast<float*>(raw);
  for (int e = threadIdx.x; e < 48 * 1024; e += blockDim.x) sm[e] = 0.0f;
  if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, (mode & 16) ? 4 : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const int issuers = (mode & 16) ? 4 : 1;
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && w < issuers) {
    const uint32_t idesc = idesc_tf32(M, N);
    const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 32 * 1024);
    const uint64_t da0 = make_desc(a0, a_lbo, a_sbo), db0 = make_desc(b0, b_lbo, b_sbo);
    const long long t0 = clock64();
    for (int r = w; r < reps; r += issuers) {
      const uint32_t ao = (mode & 2) ? (uint32_t)((r * 4096) & 65535) : 0u;
      const uint32_t bo = (mode & 2) ? (uint32_t)((r * 2048) & 32767) : 0u;
      const uint32_t d = tslot + (N <= 128 ? (uint32_t)w * 128u : (uint32_t)(w & 1) * 256u);
      if (mode & 32)
        mma_tf32(d, da0 + (ao >> 4), db0 + (bo >> 4), idesc, r >= issuers ? 1u : 0u);
      else
        mma_tf32(d, make_desc(a0 + ao, a_lbo, a_sbo), make_desc(b0 + bo, b_lbo, b_sbo), idesc,
                 r >= issuers ? 1u : 0u);
    }
    commit(&bar);
    mbar_wait(&bar, 0);
    if (w == 0) cycles[blockIdx.x] = clock64() - t0;
  } else if (mode & 4) {
    mbar_wait(&bar, 0);
  }
  fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tslot, 512);
}

// Plain row-major test GEMM: C (M x N) = A (M x K) . B (N x K)^T.
struct PlainOp {
  static constexpr bool kTableA = false;
  int M, N, K;
  const float* A;
  const float* Bm;
  float* C;
  __device__ float a(int, int m, int k) const { return A[(size_t)m * K + k]; }
  __device__ float b(int, int n, int k) const { return Bm[(size_t)n * K + k]; }
  __device__ void store(int, int m, int n, float v) const { C[(size_t)m * N + n] = v; }
};

}  // namespace tc
}  // namespace pgb
