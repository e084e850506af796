// gemm_tc.cu -- tcgen05 / TMEM / TMA tensor-core GEMM for sm_100a.
//
//   C[m x n] (f32, column-major, ldc) = alpha * op(A)[m x k] . op(B)[k x n]
//
// with bf16 operands in column-major storage.  This is the B200 replacement
// for the reference's matmul step (cjit.py:33-51 / backend.py:338-346), and
// the planner hands it the whole `s * X @ Y.t()` product (plan.py gemm_operand):
//   * the scalar is applied in the epilogue (TMEM -> registers -> *alpha),
//   * a transpose only flips the operand's shared-memory major-ness: a
//     column-major X (m x k) is M-contiguous ("MN-major"); Y.t() read from a
//     column-major Y (n x k) is N-contiguous (MN-major too).  TMA loads either
//     layout straight from the user's buffer and the UMMA descriptors say
//     which one it is -- no transposed copy is ever materialised.
//
// Structure (one CTA per SM, persistent, warp-specialised):
//   warp 0      TMA producer: 4-stage ring of (A 128 x 64, B 256 x 64) bf16
//               tiles, 128-byte swizzled, completion on an mbarrier;
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (M=128, N=256, K=16 per instruction, f32 accumulators);
//   warps 2..5  epilogue: tcgen05.ld 32 lanes x 32 columns at a time,
//               scale, coalesced column-major stores.
// Two 256-column accumulators (all 512 TMEM columns) let the epilogue of
// tile i overlap the MMAs of tile i+1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "ops.cuh"

namespace fm {
namespace tc {

constexpr int BM = 128, BN = 256, BK = 64;          // CTA tile; BK = one 128-byte swizzle row of bf16
constexpr int UMMA_K = 16;                          // K per tcgen05.mma (kind::f16)
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;                // 16 KiB
constexpr int B_BYTES = BN * BK * 2;                // 32 KiB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 2 * BN;                   // double-buffered accumulator
// 2 per TMEM lane quarter, 128 columns each.  10 warps put 3 on some SM
// sub-partition (16K registers each), so ptxas caps the kernel at 168
// registers: the 128 f32 running sums fit, with a few bytes of spill.
constexpr int kEpiWarps = 8;
constexpr int kThreadsTc = (2 + kEpiWarps) * 32;
// k-blocks per TMEM drain.  The tensor core truncates its f32 accumulator at
// every K=16 step; draining every KC*BK = 1024 of K into round-to-nearest f32
// register sums bounds that error by 64 * 2^-23 = 7.6e-6 relative for any K
// (a single 8192-deep accumulation measured 3.1e-5, bound 6.1e-5).  Measured
// at C5 (8192^3 bf16): KC=8 1340 TF/s, 16 1436, 32 1452, unchunked 1465.
constexpr int KC = 16;
// fp16-plane scheme: drain every 8 virtual k-blocks (C5 f32: max rel err
// 6.0e-6 at 16, 2.9e-6 at 8, 1.5e-6 at 4 from the accumulator's per-step
// truncation; 360 / 352 / 335 TF/s)
constexpr int KC_F16 = 8;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int GROUP_M = 8;                          // tile rasterisation: 8 M-blocks share B in L2

// ---- PTX wrappers --------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 TMEM lanes x 32 consecutive f32 columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor, 128-byte swizzle (layout type 2), sm_100 version bits.
//   K-major  : rows of 128 B (64 bf16 along K), 8-row atoms 1024 B apart (SBO); LBO unused.
//   MN-major : 64 MN-elements (128 B) per k-row, 8 k-rows per 1024 B atom; SBO = k-group
//              stride (1024 B), LBO = stride between 64-element MN blocks.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;   // SWIZZLE_128B
  return d;
}

// instruction descriptor, kind::f16: bf16 x bf16 (or fp16 x fp16) -> f32, M = BM, N = BN
__host__ __device__ constexpr uint32_t make_idesc(bool a_mn, bool b_mn, bool f16 = false) {
  return (1u << 4)                                      // D format f32
         | (f16 ? 0u : ((1u << 7) | (1u << 10)))        // A, B format: bf16 = 1, fp16 = 0
         | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16)
         | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

struct Params {
  float *c;
  int64_t ldc;
  int m, n, k;
  float alpha;
  int a_mn, b_mn;   // operand major-ness (1 = MN-contiguous)
  int nkb;          // k-blocks per product
  int nprod;        // 1 (bf16 operands), 3 (f32: 2 fp16 planes) or 6 (f32: 3 bf16 planes)
  int kplane;       // K offset between stacked planes (elements, multiple of BK)
  uint32_t pa, pb;  // plane of A / B used by product p: bits [3p, 3p+3)
  int kc;           // virtual k-blocks per TMEM drain (KC unless overridden)
  const float *cin; // epilogue addend (nullptr: none)
  int64_t ldcin;
  float alpha2, beta;
  int group_m;      // M-blocks per rasterisation group (L2 reuse of B)
  int f16;          // operands are fp16 planes (f32 inputs, two scaled planes)
  const unsigned *amax;  // [2] max |A|, max |B| bits (fp16 planes: power-of-two scales), or nullptr
};

// epilogue scale: alpha * 2^-(ea + eb), exact (a power of two)
__device__ __forceinline__ float epilogue_alpha(const Params &p) {
  if (!p.amax) return p.alpha;
  const int e = f16_scale_exp(p.amax[0]) + f16_scale_exp(p.amax[1]);
  return p.alpha * ldexpf(1.0f, -e);
}

__device__ __forceinline__ void tile_coords(int t, int ntm, int ntn, int &mb, int &nb, int group_m = GROUP_M) {
  const int per_group = group_m * ntn;
  const int g = t / per_group;
  const int first = g * group_m;
  const int gsize = min(group_m, ntm - first);
  const int r = t - g * per_group;
  mb = first + r % gsize;
  nb = r / gsize;
}

__global__ void __launch_bounds__(kThreadsTc, 1)
    k_gemm_bf16(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(smem + STAGES * STAGE_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + STAGES;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_holder = (uint32_t *)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntm = (p.m + BM - 1) / BM, ntn = (p.n + BN - 1) / BN;
  const int ntiles = ntm * ntn;
  const int nv = p.nprod * p.nkb;   // virtual k-blocks per tile (products x k-blocks)

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);   // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ===== TMA producer: virtual k-block v = product * nkb + kb =====
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, ntm, ntn, mb, nb);
        const int m0 = mb * BM, n0 = nb * BN;
        int prod = 0, kb = 0;
        for (int v = 0; v < nv; ++v, ++kb) {
          if (kb == p.nkb) { kb = 0; ++prod; }
          const int ka = (int)((p.pa >> (3 * prod)) & 7u) * p.kplane + kb * BK;
          const int kbb = (int)((p.pb >> (3 * prod)) & 7u) * p.kplane + kb * BK;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t *sa = smem + stage * STAGE_BYTES;
          uint8_t *sb = sa + A_BYTES;
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          if (p.a_mn) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tma_load_2d(sa + j * (64 * BK * 2), &map_a, &full[stage], m0 + 64 * j, ka);
          } else {
            tma_load_2d(sa, &map_a, &full[stage], ka, m0);
          }
          if (p.b_mn) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_load_2d(sb + j * (64 * BK * 2), &map_b, &full[stage], n0 + 64 * j, kbb);
          } else {
            tma_load_2d(sb, &map_b, &full[stage], kbb, n0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer: one TMEM accumulator per chunk of KC virtual k-blocks =====
    const uint32_t idesc = make_idesc(p.a_mn != 0, p.b_mn != 0, p.f16 != 0);
    // per UMMA_K step: K-major advances 32 B inside the swizzled row;
    // MN-major advances two 1024-B k-groups.
    const uint32_t a_step = p.a_mn ? 2048u : 32u, b_step = p.b_mn ? 2048u : 32u;
    const uint32_t a_lbo = p.a_mn ? 64u * BK * 2 : 16u, b_lbo = p.b_mn ? 64u * BK * 2 : 16u;
    int stage = 0;
    uint32_t phase = 0;
    uint32_t gc = 0;   // chunks issued by this CTA (selects the TMEM buffer)
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int v0 = 0; v0 < nv; v0 += p.kc, ++gc) {
        const int acc = (int)(gc & 1u);
        const uint32_t use = gc >> 1;
        mbar_wait(&tempty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        const int vend = min(nv, v0 + p.kc);
        for (int v = v0; v < vend; ++v) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
            const uint32_t sb = sa + A_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / UMMA_K; ++kk) {
              const uint64_t ad = make_desc(sa + kk * a_step, a_lbo, 1024u);
              const uint64_t bd = make_desc(sb + kk * b_step, b_lbo, 1024u);
              umma_bf16(d_tmem, ad, bd, idesc, (v != v0 || kk != 0) ? 1u : 0u);
            }
            umma_commit(&empty[stage]);                    // frees the smem slot when these MMAs finish
            if (v == vend - 1) umma_commit(&tfull[acc]);   // chunk accumulated: hand it to the epilogue
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ===== epilogue: drain each chunk into f32 register sums, then alpha * sum -> column-major stores =====
    const float ealpha = epilogue_alpha(p);
    const int q = warp & 3;                    // TMEM lane quarter this warp may access
    const int h = (warp - 2) >> 2;             // column half (128 columns)
    uint32_t gc = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      int mb, nb;
      tile_coords(t, ntm, ntn, mb, nb);
      float sum[BN / 2];
#pragma unroll
      for (int j = 0; j < BN / 2; ++j) sum[j] = 0.0f;
      for (int v0 = 0; v0 < nv; v0 += p.kc, ++gc) {
        const int acc = (int)(gc & 1u);
        const uint32_t use = gc >> 1;
        mbar_wait(&tfull[acc], use & 1);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + h * (BN / 2));
#pragma unroll
        for (int c4 = 0; c4 < BN / 64; ++c4) {
          uint32_t v[32];
          tmem_ld32_nowait(taddr + c4 * 32, v);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) sum[c4 * 32 + j] = __fadd_rn(sum[c4 * 32 + j], __uint_as_float(v[j]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);   // buffer drained: the MMA warp may reuse it
      }
      const int row = mb * BM + q * 32 + lane;
      if (row < p.m) {
        float *cp = p.c + row;
        const int col0 = nb * BN + h * (BN / 2);
        if (p.cin) {
          const float *ci = p.cin + row;
#pragma unroll
          for (int j = 0; j < BN / 2; ++j)
            if (col0 + j < p.n) {
              const float t = __fmul_rn(ealpha, sum[j]);
              cp[(int64_t)(col0 + j) * p.ldc] =
                  __fadd_rn(__fmul_rn(p.alpha2, t), __fmul_rn(p.beta, ci[(int64_t)(col0 + j) * p.ldcin]));
            }
        } else {
#pragma unroll
          for (int j = 0; j < BN / 2; ++j)
            if (col0 + j < p.n) cp[(int64_t)(col0 + j) * p.ldc] = __fmul_rn(ealpha, sum[j]);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// ---- CTA-pair (cta_group::2) variant ---------------------------------------------------
// A cluster of two CTAs on one TPC computes a 256 x 256 tile: each CTA TMA-
// loads its own 128-row half of A and 128-column half of B (32 KiB per stage
// instead of 48, so 6 stages fit), the leader (rank 0) issues
// tcgen05.mma.cta_group::2 (M=256, N=256) that reads both CTAs' shared
// memory, and each CTA's TMEM holds the accumulator rows of its half.  Both
// CTAs' TMA completions count on the leader's full barrier; MMA commits are
// multicast to both CTAs' empty / tfull barriers; both epilogues report a
// drained accumulator to the leader's tempty barrier.
namespace pair {
constexpr int BM2 = 256, BNH = 128;                  // pair tile 256 x 256, per-CTA B half 128
constexpr int A_BYTES2 = 128 * BK * 2;               // 16 KiB (this CTA's rows)
constexpr int B_BYTES2 = BNH * BK * 2;               // 16 KiB (this CTA's columns)
constexpr int STAGE_BYTES2 = A_BYTES2 + B_BYTES2;
constexpr int STAGES2 = 7;
constexpr int SMEM_BYTES2 = STAGES2 * STAGE_BYTES2 + 1024 + 256;
constexpr int BN2 = 256;                             // accumulator columns per CTA

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p` (a shared::cta address in this CTA) in CTA `rank`
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void *dst, const CUtensorMap *map, uint32_t leader_bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(leader_bar)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_pair(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__host__ __device__ constexpr uint32_t make_idesc_pair(bool a_mn, bool b_mn, bool f16 = false) {
  return (1u << 4) | (f16 ? 0u : ((1u << 7) | (1u << 10))) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(BM2 >> 4) << 24);
}
}  // namespace pair

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsTc, 1)
    k_gemm_bf16_pair(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const Params p) {
  using namespace pair;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(smem + STAGES2 * STAGE_BYTES2);
  uint64_t *empty = full + STAGES2;
  uint64_t *tfull = empty + STAGES2;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_holder = (uint32_t *)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int ntm = (p.m + BM2 - 1) / BM2, ntn = (p.n + BN2 - 1) / BN2;
  const int ntiles = ntm * ntn;
  const int nv = p.nprod * p.nkb;
  const int pair_id = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiWarps);   // both CTAs' epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const uint32_t leader_full0 = mapa(smem_u32(&full[0]), 0);
  const uint32_t leader_tempty0 = mapa(smem_u32(&tempty[0]), 0);

  if (warp == 0) {
    // ===== TMA producer (both CTAs): this CTA's A rows and B columns; bytes count on the leader's barrier
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair_id; t < ntiles; t += npairs) {
        int mb, nb;
        tile_coords(t, ntm, ntn, mb, nb, p.group_m);
        const int m0 = mb * BM2 + 128 * (int)rank, n0 = nb * BN2 + BNH * (int)rank;
        int prod = 0, kb = 0;
        for (int v = 0; v < nv; ++v, ++kb) {
          if (kb == p.nkb) { kb = 0; ++prod; }
          const int ka = (int)((p.pa >> (3 * prod)) & 7u) * p.kplane + kb * BK;
          const int kbb = (int)((p.pb >> (3 * prod)) & 7u) * p.kplane + kb * BK;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t *sa = smem + stage * STAGE_BYTES2;
          uint8_t *sb = sa + A_BYTES2;
          const uint32_t lbar = leader_full0 + (uint32_t)(stage * 8);
          if (leader) mbar_expect_tx(&full[stage], 2 * STAGE_BYTES2);
          if (p.a_mn) {
#pragma unroll
            for (int j = 0; j < 2; ++j) tma_load_2d_pair(sa + j * (64 * BK * 2), &map_a, lbar, m0 + 64 * j, ka);
          } else {
            tma_load_2d_pair(sa, &map_a, lbar, ka, m0);
          }
          if (p.b_mn) {
#pragma unroll
            for (int j = 0; j < BNH / 64; ++j) tma_load_2d_pair(sb + j * (64 * BK * 2), &map_b, lbar, n0 + 64 * j, kbb);
          } else {
            tma_load_2d_pair(sb, &map_b, lbar, kbb, n0);
          }
          if (++stage == STAGES2) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer: leader only
    if (leader) {
      const uint32_t idesc = make_idesc_pair(p.a_mn != 0, p.b_mn != 0, p.f16 != 0);
      const uint32_t a_step = p.a_mn ? 2048u : 32u, b_step = p.b_mn ? 2048u : 32u;
      const uint32_t a_lbo = p.a_mn ? 64u * BK * 2 : 16u, b_lbo = p.b_mn ? 64u * BK * 2 : 16u;
      int stage = 0;
      uint32_t phase = 0;
      uint32_t gc = 0;
      for (int t = pair_id; t < ntiles; t += npairs) {
        for (int v0 = 0; v0 < nv; v0 += p.kc, ++gc) {
          const int acc = (int)(gc & 1u);
          const uint32_t use = gc >> 1;
          mbar_wait(&tempty[acc], (use & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN2);
          const int vend = min(nv, v0 + p.kc);
          for (int v = v0; v < vend; ++v) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            if (lane == 0) {
              const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES2);
              const uint32_t sb = sa + A_BYTES2;
#pragma unroll
              for (int kk = 0; kk < BK / UMMA_K; ++kk) {
                const uint64_t ad = make_desc(sa + kk * a_step, a_lbo, 1024u);
                const uint64_t bd = make_desc(sb + kk * b_step, b_lbo, 1024u);
                umma_bf16_pair(d_tmem, ad, bd, idesc, (v != v0 || kk != 0) ? 1u : 0u);
              }
              umma_commit_pair(&empty[stage]);                   // frees the slot in BOTH CTAs
              if (v == vend - 1) umma_commit_pair(&tfull[acc]);  // accumulator halves ready in both CTAs
            }
            __syncwarp();
            if (++stage == STAGES2) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else {
    // ===== epilogue (both CTAs): this CTA's 128 accumulator rows
    const float ealpha = epilogue_alpha(p);
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;
    uint32_t gc = 0;
    for (int t = pair_id; t < ntiles; t += npairs) {
      int mb, nb;
      tile_coords(t, ntm, ntn, mb, nb, p.group_m);
      float sum[BN2 / 2];
#pragma unroll
      for (int j = 0; j < BN2 / 2; ++j) sum[j] = 0.0f;
      for (int v0 = 0; v0 < nv; v0 += p.kc, ++gc) {
        const int acc = (int)(gc & 1u);
        const uint32_t use = gc >> 1;
        mbar_wait(&tfull[acc], use & 1);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN2 + h * (BN2 / 2));
#pragma unroll
        for (int c4 = 0; c4 < BN2 / 64; ++c4) {
          uint32_t vv[32];
          tmem_ld32_nowait(taddr + c4 * 32, vv);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) sum[c4 * 32 + j] = __fadd_rn(sum[c4 * 32 + j], __uint_as_float(vv[j]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_tempty0 + (uint32_t)(acc * 8));
      }
      const int row = mb * BM2 + 128 * (int)rank + q * 32 + lane;
      if (row < p.m) {
        float *cp = p.c + row;
        const int col0 = nb * BN2 + h * (BN2 / 2);
        if (p.cin) {
          const float *ci = p.cin + row;
#pragma unroll
          for (int j = 0; j < BN2 / 2; ++j)
            if (col0 + j < p.n) {
              const float tt = __fmul_rn(ealpha, sum[j]);
              cp[(int64_t)(col0 + j) * p.ldc] =
                  __fadd_rn(__fmul_rn(p.alpha2, tt), __fmul_rn(p.beta, ci[(int64_t)(col0 + j) * p.ldcin]));
            }
        } else {
#pragma unroll
          for (int j = 0; j < BN2 / 2; ++j)
            if (col0 + j < p.n) cp[(int64_t)(col0 + j) * p.ldc] = __fmul_rn(ealpha, sum[j]);
        }
      }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// split3 (ops.cuh): f32 -> three bf16 planes

// Grid: x over row runs of 4 elements, y over columns (no per-element
// division); 16-byte loads and 8-byte stores per plane when the column runs
// are aligned, scalar otherwise.
__global__ void k_split3(const float *__restrict__ in, int64_t rows, int64_t cols, int64_t ld_in,
                         uint16_t *__restrict__ out, int64_t ld_out, int64_t plane_off) {
  const bool vec = ((ld_in & 3) == 0) && ((ld_out & 3) == 0) && ((plane_off & 3) == 0) &&
                   ((((uintptr_t)in) & 15) == 0) && ((((uintptr_t)out) & 7) == 0);
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y) {
    const float *src = in + j * ld_in;
    uint16_t *dst = out + j * ld_out;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < rows;
         i += (int64_t)gridDim.x * blockDim.x * 4) {
      if (vec && i + 4 <= rows) {
        const float4 x = *(const float4 *)(src + i);
        ushort4 h, m, l;
        split3(x.x, h.x, m.x, l.x);
        split3(x.y, h.y, m.y, l.y);
        split3(x.z, h.z, m.z, l.z);
        split3(x.w, h.w, m.w, l.w);
        *(ushort4 *)(dst + i) = h;
        *(ushort4 *)(dst + i + plane_off) = m;
        *(ushort4 *)(dst + i + 2 * plane_off) = l;
      } else {
        for (int64_t ii = i; ii < i + 4 && ii < rows; ++ii) {
          uint16_t h, m, l;
          split3(src[ii], h, m, l);
          dst[ii] = h;
          dst[ii + plane_off] = m;
          dst[ii + 2 * plane_off] = l;
        }
      }
    }
  }
}

// max |x| of a column-major operand as f32 bits (non-negative floats order
// like their bit patterns; NaN bits sort above +inf) -> atomicMax into *out.
__global__ void k_amax(const float *__restrict__ in, int64_t rows, int64_t cols, int64_t ld, unsigned *out) {
  unsigned m = 0;
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y) {
    const float *src = in + j * ld;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x)
      m = max(m, __float_as_uint(src[i]) & 0x7fffffffu);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_split2h(const float *__restrict__ in, int64_t rows, int64_t cols, int64_t ld_in,
                          uint16_t *__restrict__ out, int64_t ld_out, int64_t plane_off, const unsigned *amax) {
  const float sc = ldexpf(1.0f, f16_scale_exp(*amax));
  const bool vec = ((ld_in & 3) == 0) && ((ld_out & 3) == 0) && ((plane_off & 3) == 0) &&
                   ((((uintptr_t)in) & 15) == 0) && ((((uintptr_t)out) & 7) == 0);
  for (int64_t j = blockIdx.y; j < cols; j += gridDim.y) {
    const float *src = in + j * ld_in;
    uint16_t *dst = out + j * ld_out;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < rows;
         i += (int64_t)gridDim.x * blockDim.x * 4) {
      if (vec && i + 4 <= rows) {
        const float4 x = *(const float4 *)(src + i);
        ushort4 h, l;
        split2h(x.x, sc, h.x, l.x);
        split2h(x.y, sc, h.y, l.y);
        split2h(x.z, sc, h.z, l.z);
        split2h(x.w, sc, h.w, l.w);
        *(ushort4 *)(dst + i) = h;
        *(ushort4 *)(dst + i + plane_off) = l;
      } else {
        for (int64_t ii = i; ii < i + 4 && ii < rows; ++ii) {
          uint16_t h, l;
          split2h(src[ii], sc, h, l);
          dst[ii] = h;
          dst[ii + plane_off] = l;
        }
      }
    }
  }
}

// ---- host side -----------------------------------------------------------------------
// cuTensorMapEncodeTiled comes from the driver through the runtime's entry-point
// query, so libfmb200.so has no link-time dependency on libcuda (it still loads
// on a machine without a driver; the CPU test suite checks its exports).
using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

// 2-D bf16 tensor map over a column-major operand: dim0 = the contiguous
// extent, dim1 = the strided one, box = {64 (128 B, swizzled), rows}.
static int encode_map(CUtensorMap *map, const void *ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                      uint32_t box_inner, uint32_t box_outer) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail_msg("gemm: cuTensorMapEncodeTiled unavailable from the driver");
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld_elems * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail_msg("gemm: cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r));
  return 0;
}

}  // namespace tc

// Tensor-core path: bf16 operands directly; f32 operands scaled by a power
// of two from their max |x| (k_amax) and split into two fp16 planes each
// (k_split2h / the prologue's fused split), multiplied as the three
// significant plane products lo*hi, hi*lo, hi*hi in one kernel launch
// (dropped lo*lo and plane rounding: O(2^-21) relative).  The older
// three-bf16-plane, six-product scheme (k_split3) remains for a prologue
// program with no room for its max pass.  Shapes TMA cannot describe report
// handled = false and run on the exact kernel.
bool gemm_tensor_supported(const fm_gemm_args &g) {
  if (g.out_etype != FM_F32) return false;
  if (g.m > INT32_MAX / 4 || g.n > INT32_MAX / 4 || g.k > INT32_MAX / 8) return false;
  if (g.in_etype == FM_F32) return true;                                   // re-laid out by the split
  if (g.in_etype != FM_BF16) return false;
  if ((((uintptr_t)g.a) & 15) || (((uintptr_t)g.b) & 15)) return false;   // TMA: 16-byte aligned base
  if ((g.lda * 2) % 16 || (g.ldb * 2) % 16) return false;                  // TMA: 16-byte multiple strides
  return true;
}

namespace {
int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// split one f32 operand into stacked bf16 planes; returns the tensor-map
// geometry of the stacked operand (inner extent, outer extent, ld)
struct Planes {
  uint16_t *buf = nullptr;
  uint64_t inner = 0, outer = 0, ld = 0;
};
// nplanes = 3: bf16 hi/mid/lo; nplanes = 2: scaled fp16 hi/lo (amax = max |src| bits on the device)
int split_operand(const float *src, int64_t rows, int64_t cols, int64_t ld_in, bool k_is_cols, int64_t kplane,
                  Planes *pl, cudaStream_t s, const fm_program *prog, int nplanes = 3,
                  const unsigned *amax = nullptr) {
  int64_t ld_out, plane_off, bytes;
  if (k_is_cols) {   // MN-major operand: planes appended along the column (K) dimension
    ld_out = round_up(rows, 8);
    plane_off = kplane * ld_out;
    bytes = nplanes * plane_off * 2;
    pl->inner = (uint64_t)rows; pl->outer = (uint64_t)(nplanes * kplane);
  } else {           // K-major operand: planes stacked along the row (K) dimension
    ld_out = nplanes * kplane;
    plane_off = kplane;
    bytes = ld_out * cols * 2;
    pl->inner = (uint64_t)(nplanes * kplane); pl->outer = (uint64_t)cols;
  }
  pl->ld = (uint64_t)ld_out;
  FM_CHECK(cudaMallocAsync((void **)&pl->buf, (size_t)bytes, s));
  const int64_t kdim = k_is_cols ? cols : rows;
  if (kdim != kplane) FM_CHECK(cudaMemsetAsync(pl->buf, 0, (size_t)bytes, s));   // zero K padding
  if (prog)   // operand prologue: the operand's expression evaluated into the planes (split.cuh)
    return launch_split_program(*prog, pl->buf, rows, cols, ld_out, plane_off, nplanes == 2 ? amax : nullptr, s);
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((rows + 1023) / 1024, 64));
  const unsigned gy = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cols, 65535));
  if (nplanes == 2) {
    tc::k_split2h<<<dim3(gx, gy), 256, 0, s>>>(src, rows, cols, ld_in, pl->buf, ld_out, plane_off, amax);
    FM_CHECK_LAUNCH("f32 -> scaled fp16 plane split kernel");
    return 0;
  }
  tc::k_split3<<<dim3(gx, gy), 256, 0, s>>>(src, rows, cols, ld_in, pl->buf, ld_out, plane_off);
  FM_CHECK_LAUNCH("f32 -> bf16 plane split kernel");
  return 0;
}
}  // namespace

int gemm_tensor(const fm_gemm_args &g, cudaStream_t s, bool *handled, const fm_program *a_prog,
                const fm_program *b_prog) {
  using namespace tc;
  *handled = false;
  if (!gemm_tensor_supported(g)) return 0;
  if ((a_prog || b_prog) && g.in_etype != FM_F32) return 0;   // prologues ride on the f32 operand split
  Params p;
  p.c = (float *)g.c;
  p.ldc = g.ldc;
  p.m = (int)g.m; p.n = (int)g.n; p.k = (int)g.k;
  p.alpha = (float)g.alpha;   // the scalar node is f32 in the tree (expr.py:225), applied in the epilogue
  p.cin = (const float *)g.c_in;
  p.ldcin = g.ld_c_in;
  p.alpha2 = (float)g.alpha2;
  p.beta = (float)g.beta;
  p.a_mn = g.trans_a ? 0 : 1;   // op(A) = A (m x k, M-contiguous) or A^T of a k x m buffer (K-contiguous)
  p.b_mn = g.trans_b ? 1 : 0;   // op(B) = B (k x n, K-contiguous) or B^T of an n x k buffer (N-contiguous)
  p.nkb = (int)((g.k + BK - 1) / BK);
  // CTA-pair kernel (cta_group::2, 256 x 256 pair tiles) by default: C5 1441
  // vs 1405 TF/s on the single-CTA kernel.  FMB200_GEMM_PAIR=0 selects the
  // single-CTA kernel (A/B measurements).
  static int pair_env = [] {
    const char *e = getenv("FMB200_GEMM_PAIR");
    return (e && *e) ? atoi(e) : 1;
  }();
  const bool use_pair = pair_env == 1 && sm_count() >= 2;
  const int b_box_rows = use_pair ? pair::BNH : BN;   // K-major B box: this CTA's columns
  static int kc_env = [] {
    const char *e = getenv("FMB200_GEMM_KC");
    return (e && *e) ? std::max(1, atoi(e)) : KC;
  }();
  p.kc = kc_env;
  static int group_env = [] {
    const char *e = getenv("FMB200_GEMM_GROUP_M");
    return (e && *e) ? std::max(1, atoi(e)) : GROUP_M;
  }();
  p.group_m = group_env;
  CUtensorMap ma, mb;
  int st;
  Planes pa, pb;
  p.f16 = 0;
  p.amax = nullptr;
  unsigned *amax = nullptr;
  if (g.in_etype == FM_F32) {
    const int64_t kplane = round_up(g.k, BK);
    p.kplane = (int)kplane;
    // f32 operands: two fp16 planes each, scaled by a power of two from the
    // operand's max |x| (one short device pass: a max-abs kernel, or for an
    // operand prologue a MAX reduction of |expression|), and the three
    // significant products hi*lo, lo*hi, hi*hi -- half the tensor work of
    // the six-product bf16 scheme at ~2^-21 relative per term.  The bf16
    // scheme remains for a prologue program with no room for the max pass.
    const int64_t ar = p.a_mn ? g.m : g.k, ac = p.a_mn ? g.k : g.m;
    const int64_t br = p.b_mn ? g.n : g.k, bc = p.b_mn ? g.k : g.n;
    bool f16 = true;
    for (const fm_program *P : {a_prog, b_prog})
      if (P && P->n_instr >= FM_MAX_INSTR) f16 = false;
    int nplanes = 3;
    if (f16) {
      nplanes = 2;
      p.f16 = 1;
      p.nprod = 3;
      p.kc = std::min(p.kc, KC_F16);
      const uint32_t A[3] = {0, 1, 0}, B[3] = {1, 0, 0};
      p.pa = p.pb = 0;
      for (int i = 0; i < 3; ++i) { p.pa |= A[i] << (3 * i); p.pb |= B[i] << (3 * i); }
      FM_CHECK(cudaMallocAsync((void **)&amax, 2 * sizeof(unsigned), s));
      FM_CHECK(cudaMemsetAsync(amax, 0, 2 * sizeof(unsigned), s));
      const fm_program *progs[2] = {a_prog, b_prog};
      const void *bufs[2] = {g.a, g.b};
      const int64_t rows[2] = {ar, br}, cols[2] = {ac, bc}, lds[2] = {g.lda, g.ldb};
      for (int o = 0; o < 2; ++o) {
        if (progs[o]) {
          bool ok = false;
          if (int e = launch_amax_program(*progs[o], rows[o], cols[o], amax + o, s, &ok)) { cudaFreeAsync(amax, s); return e; }
        } else {
          tc::k_amax<<<dim3((unsigned)std::min<int64_t>((rows[o] + 255) / 256, 16),
                            (unsigned)std::min<int64_t>(cols[o], 2048)), 256, 0, s>>>((const float *)bufs[o], rows[o],
                                                                                     cols[o], lds[o], amax + o);
          FM_CHECK_LAUNCH("operand max |x| kernel");
        }
      }
      p.amax = amax;
    } else {
      p.nprod = 6;
      // products, smallest first: (0,2) (1,1) (2,0) (0,1) (1,0) (0,0)
      const uint32_t A[6] = {0, 1, 2, 0, 1, 0}, B[6] = {2, 1, 0, 1, 0, 0};
      p.pa = p.pb = 0;
      for (int i = 0; i < 6; ++i) { p.pa |= A[i] << (3 * i); p.pb |= B[i] << (3 * i); }
    }
    st = p.a_mn ? split_operand((const float *)g.a, g.m, g.k, g.lda, true, kplane, &pa, s, a_prog, nplanes, amax)
                : split_operand((const float *)g.a, g.k, g.m, g.lda, false, kplane, &pa, s, a_prog, nplanes, amax);
    if (st) { if (amax) cudaFreeAsync(amax, s); return st; }
    st = p.b_mn ? split_operand((const float *)g.b, g.n, g.k, g.ldb, true, kplane, &pb, s, b_prog, nplanes,
                                amax ? amax + 1 : nullptr)
                : split_operand((const float *)g.b, g.k, g.n, g.ldb, false, kplane, &pb, s, b_prog, nplanes,
                                amax ? amax + 1 : nullptr);
    if (st) { cudaFreeAsync(pa.buf, s); if (amax) cudaFreeAsync(amax, s); return st; }
    st = encode_map(&ma, pa.buf, pa.inner, pa.outer, pa.ld, p.a_mn ? 64 : BK, p.a_mn ? BK : BM);
    if (!st) st = encode_map(&mb, pb.buf, pb.inner, pb.outer, pb.ld, p.b_mn ? 64 : BK, p.b_mn ? BK : b_box_rows);
  } else {
    p.nprod = 1;
    p.kplane = 0;
    p.pa = p.pb = 0;
    if (p.a_mn) st = encode_map(&ma, g.a, (uint64_t)g.m, (uint64_t)g.k, (uint64_t)g.lda, 64, BK);
    else st = encode_map(&ma, g.a, (uint64_t)g.k, (uint64_t)g.m, (uint64_t)g.lda, BK, BM);
    if (!st) {
      if (p.b_mn) st = encode_map(&mb, g.b, (uint64_t)g.n, (uint64_t)g.k, (uint64_t)g.ldb, 64, BK);
      else st = encode_map(&mb, g.b, (uint64_t)g.k, (uint64_t)g.n, (uint64_t)g.ldb, BK, b_box_rows);
    }
  }
  if (!st && use_pair) {
    static bool attr2 = false;
    if (!attr2) {
      cudaError_t e = cudaFuncSetAttribute(k_gemm_bf16_pair, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           pair::SMEM_BYTES2);
      if (e != cudaSuccess) st = fail("cudaFuncSetAttribute(k_gemm_bf16_pair)", e);
      else attr2 = true;
    }
    if (!st) {
      const int ntiles = (int)(((g.m + pair::BM2 - 1) / pair::BM2) * ((g.n + pair::BN2 - 1) / pair::BN2));
      const int grid = std::min(2 * ntiles, sm_count() & ~1);
      k_gemm_bf16_pair<<<grid, kThreadsTc, pair::SMEM_BYTES2, s>>>(ma, mb, p);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) st = fail("tcgen05 gemm kernel (CTA pair)", e);
      else count_launch();
    }
    if (pa.buf) cudaFreeAsync(pa.buf, s);
    if (pb.buf) cudaFreeAsync(pb.buf, s);
    if (amax) cudaFreeAsync(amax, s);
    if (!st) *handled = true;
    return st;
  }
  if (!st) {
    static bool attr_set = false;
    if (!attr_set) {
      cudaError_t e = cudaFuncSetAttribute(k_gemm_bf16, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
      if (e != cudaSuccess) st = fail("cudaFuncSetAttribute(k_gemm_bf16)", e);
      else attr_set = true;
    }
  }
  if (!st) {
    const int ntiles = (int)(((g.m + BM - 1) / BM) * ((g.n + BN - 1) / BN));
    const int grid = std::min(ntiles, sm_count());
    k_gemm_bf16<<<grid, kThreadsTc, SMEM_BYTES, s>>>(ma, mb, p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) st = fail("tcgen05 gemm kernel", e);
    else count_launch();
  }
  if (pa.buf) cudaFreeAsync(pa.buf, s);   // stream-ordered: released after the GEMM reads it
  if (pb.buf) cudaFreeAsync(pb.buf, s);
  if (amax) cudaFreeAsync(amax, s);
  if (!st) *handled = true;
  return st;
}

}  // namespace fm
