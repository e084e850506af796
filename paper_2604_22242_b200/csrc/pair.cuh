// pair.cuh -- tile-pair copy skeleton for square programs with transposed
// leaves (the paper's expr1 `2*(X.t() + Y) + 2*(X + Y.t())`, expr2's
// `(b + c).t()`).
//
// The per-slot staged skeleton (tiled.cuh) copies one tile per SLOT: a
// matrix read both as X and as X.t() is fetched twice, once as block (I,J)
// and once as block (J,I) (r01: expr1 moved 1.85x its algorithmic bytes and
// spent ~113 instructions per element on cp.async address math).  Here one
// CTA owns the output tile PAIR (I,J) + (J,I) of an n x n domain and stages,
// per DISTINCT buffer M, the two blocks M[I,J] and M[J,I] -- exactly the
// blocks both output tiles need, whatever mix of M and M.t() the program
// reads -- so every input byte leaves HBM once.  Staging is 2-D TMA
// (cp.async.bulk.tensor, 128-byte swizzle, one elected thread, completion on
// an mbarrier), so the copy costs no per-element instructions; S stages per
// CTA keep the next pairs' blocks in flight while the current pair is
// evaluated out of shared memory (vm.cuh load_pair).
//
// Thread map: lane = tile column, warp = a V-row chunk of that column
// (32 / V warps).  Untransposed leaves are 16-byte vector reads along the
// column, transposed ones scalar reads along a row of the other block; the
// swizzle makes both conflict-free.
#pragma once
#include <cuda.h>

#include <algorithm>

#include "skeletons.cuh"

namespace fm {
namespace pair {

constexpr int kTile = 32;          // square tile edge (elements)
constexpr int kMaxBuf = 8;         // distinct buffers per program
constexpr int kHalf = 4096;        // one 128-byte x 32-column TMA box
constexpr int kStrip = 8;          // tile columns per strip of the pair order

struct Maps {
  CUtensorMap map[kMaxBuf];        // 2-D, {ld rows, n cols}, box {128 B, 32 cols}, SWIZZLE_128B
  int32_t width[kMaxBuf];          // element bytes (4 or 8)
  int32_t n_buf;
  int32_t tile_bytes;              // bytes per staged tile (32 x 32 x widest element)
  CUtensorMap out_map;             // the output, same box geometry (TMA store epilogue)
  int32_t out_w;                   // output element bytes (4 or 8)
};

FM_DEV uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
FM_DEV void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
FM_DEV void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
FM_DEV void mbar_wait(uint64_t *bar, uint32_t parity) {
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
FM_DEV void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int x, int y, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// One thread: stage tile pair (I, J) into `st` (both blocks of every buffer;
// one block on the diagonal).
FM_DEV void issue(const Maps &M, unsigned char *st, uint64_t *bar, int I, int J, uint64_t policy) {
  const bool diag = I == J;
  uint32_t bytes = 0;
  for (int b = 0; b < M.n_buf; ++b) bytes += (diag ? 1u : 2u) * (uint32_t)(M.width[b] / 4) * kHalf;
  mbar_expect_tx(bar, bytes);
  for (int b = 0; b < M.n_buf; ++b) {
    unsigned char *ta = st + (size_t)(2 * b) * M.tile_bytes;
    const int halves = M.width[b] / 4, rows_per = kTile / halves;
    for (int h = 0; h < halves; ++h) {
      tma_load_2d(ta + h * kHalf, &M.map[b], bar, I * kTile + h * rows_per, J * kTile, policy);
      if (!diag) tma_load_2d(ta + M.tile_bytes + h * kHalf, &M.map[b], bar, J * kTile + h * rows_per, I * kTile, policy);
    }
  }
}

// Does the template evaluator take the direct path (its NIN x V loaded values
// fit in registers)?  The register VM and very wide templates use E::eval.
template <class E, bool VM = E::kIsVm>
struct Direct { static constexpr bool v = false; };
template <class E>
struct Direct<E, false> { static constexpr bool v = E::kNin * E::kV <= 64; };
// element bytes of the direct path's per-thread offsets (the VM computes its own)
template <class E, bool VM = E::kIsVm>
struct ElemBytes { static constexpr int v = 4; };
template <class E>
struct ElemBytes<E, false> { static constexpr int v = (int)sizeof(typename E::Elem); };

// Template evaluator, one chunk: every slot's V values straight from the
// staged tiles at per-thread offsets fixed for the whole launch (tv: the V
// transposed elements of this thread's row, uq: its 16-byte column vectors),
// then the expression per element.
FM_DEV uint4 lds128(uint32_t a) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}
FM_DEV uint32_t lds32(uint32_t a) {
  uint32_t r;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
  return r;
}
FM_DEV uint2 lds64(uint32_t a) {
  uint2 r;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(a));
  return r;
}

// Thread geometry: 32 lanes = the 32 tile columns; 32 / V consumer warps
// cover the rows of one output tile.  Direct-path programs split the pair's
// two output tiles over two warp groups, so a stage feeds twice the warps
// (heavy chains: the FP64 transcendental latency; light ones too since the
// kernel runs at 8 consumer warps per SM otherwise -- expr1 +2-3 % at
// 10000^2 / 8192^2); VM programs evaluate both tiles per thread.  One more
// warp is the producer: it waits for a stage to be released, then stages
// the next pair into it (warp-specialised ring, no block-wide barrier in the
// loop).
template <class E>
struct Geo {
  static constexpr int V = E::kV;
  static constexpr int kWarpsPerTile = kTile / V;
  static constexpr int kGroups = Direct<E>::v ? 2 : 1;
  static constexpr int kConsumerWarps = kWarpsPerTile * kGroups;
  static constexpr int kThreads = 32 * (kConsumerWarps + 1);
};

template <class E>
FM_DEV void eval_direct(const fm_program &P, const unsigned char *stage, uint32_t tile_bytes, int mode,
                        const uint32_t (&tv)[E::kV], const uint32_t (&uq)[E::kV * ElemBytes<E>::v / 16],
                        uint32_t (&lo)[E::kV], uint32_t (&hi)[E::kV]) {
  using T = typename E::Elem;
  constexpr int V = E::kV, NIN = E::kNin, W = 16 / (int)sizeof(T), NQ = V / W;
  T x[NIN][V];
#pragma unroll
  for (int j = 0; j < NIN; ++j) {
    const fm_slot &s = P.slots[j];
    const uint32_t trn = s.transposed != 0;
    const uint32_t sel = mode == 3 ? 0u : (trn ^ (uint32_t)(mode == 2));
    const unsigned char *t = stage + ((uint32_t)s.reserved * 2u + sel) * tile_bytes;
    if (trn) {
#pragma unroll
      for (int v = 0; v < V; ++v) x[j][v] = *(const T *)(t + tv[v]);
    } else {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const uint4 w = *(const uint4 *)(t + uq[q]);
        if constexpr (sizeof(T) == 8) {
          x[j][2 * q] = u2d(w.x, w.y);
          x[j][2 * q + 1] = u2d(w.z, w.w);
        } else {
          x[j][4 * q] = u2f(w.x); x[j][4 * q + 1] = u2f(w.y);
          x[j][4 * q + 2] = u2f(w.z); x[j][4 * q + 3] = u2f(w.w);
        }
      }
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    T xv[NIN];
#pragma unroll
    for (int j = 0; j < NIN; ++j) xv[j] = x[j][v];
    const T r = E::ev_elem(P, xv);
    if constexpr (sizeof(T) == 8) d2u(r, lo[v], hi[v]);
    else { lo[v] = f2u(r); hi[v] = 0u; }
  }
}

FM_DEV void tma_store_2d(const CUtensorMap *map, const void *src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(x),
               "r"(y), "r"(smem_u32(src))
               : "memory");
}
FM_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
FM_DEV void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
FM_DEV void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
FM_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// named barrier over the consumer warps only (the producer never joins)
FM_DEV void consumers_sync(int nthreads) { asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory"); }

// Write this thread's V results (rows tr.., column lane) into an output tile
// laid out like the staged inputs, for the TMA store.
template <int V>
FM_DEV void put_out(unsigned char *t, int w, int tr, int lane, const uint32_t (&lo)[V], const uint32_t (&hi)[V]) {
  if (w == 4) {
#pragma unroll
    for (int q = 0; q < V / 4; ++q)
      *(uint4 *)(t + pair_off(tr + 4 * q, lane, 4)) = make_uint4(lo[4 * q], lo[4 * q + 1], lo[4 * q + 2], lo[4 * q + 3]);
  } else {
#pragma unroll
    for (int q = 0; q < V / 2; ++q)
      *(uint4 *)(t + pair_off(tr + 2 * q, lane, 8)) = make_uint4(lo[2 * q], hi[2 * q], lo[2 * q + 1], hi[2 * q + 1]);
  }
}

FM_DEV void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <class E>
__global__ void __launch_bounds__(Geo<E>::kThreads) k_copy_pair(const __grid_constant__ fm_program P,
                                                                 const __grid_constant__ Maps M, void *out,
                                                                 int64_t n, const uint32_t *__restrict__ order,
                                                                 int stages) {
  using G = Geo<E>;
  constexpr int V = E::kV;
  extern __shared__ unsigned char sm_raw[];
  // 1024-byte aligned (the 128-byte swizzle pattern repeats every 1 KiB); the
  // pointer stays derived from the __shared__ array, so loads are ld.shared
  unsigned char *sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  const size_t stage_bytes = (size_t)M.n_buf * 2 * M.tile_bytes;
  const int out_tile = kTile * kTile * M.out_w;
  unsigned char *obuf = sm + stages * stage_bytes;     // the pair's 2 result tiles
  uint64_t *full = (uint64_t *)(obuf + 2 * out_tile);
  uint64_t *empty = full + stages;
  uint32_t *coord = (uint32_t *)(empty + stages);     // (I | J << 16) of each stage's pair
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nt = (n + kTile - 1) / kTile;
  const int64_t np = nt * (nt + 1) / 2;
  const int step = (int)gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], G::kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == G::kConsumerWarps) {
    // producer: one lane; the pair order is read one pair ahead
    if (lane == 0) {
      uint64_t policy;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      int s = 0;
      uint32_t use = 0;            // completed passes over the ring
      int64_t p = blockIdx.x;
      uint32_t c = p < np ? order[p] : 0u;
      for (; p < np; p += step) {
        const uint32_t cur = c;
        if (p + step < np) c = order[p + step];
        if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
        coord[s] = cur;
        issue(M, sm + s * stage_bytes, &full[s], (int)(cur & 0xffffu), (int)(cur >> 16), policy);
        if (++s == stages) { s = 0; ++use; }
      }
    }
    return;
  }

  // consumers: per-thread tile offsets (direct template path)
  const int group = warp / G::kWarpsPerTile;
  const int tr = (warp % G::kWarpsPerTile) * V;
  constexpr int kW = ElemBytes<E>::v;
  constexpr int NQ = V * kW / 16 > 0 ? V * kW / 16 : 1;
  uint32_t tv[V], uq[NQ];
#pragma unroll
  for (int v = 0; v < V; ++v) tv[v] = pair_off(lane, tr + v, kW);
#pragma unroll
  for (int q = 0; q < NQ; ++q) uq[q] = pair_off(tr + q * (16 / kW), lane, kW);
  int s = 0;
  uint32_t phase = 0;
  for (int64_t p = blockIdx.x; p < np; p += step) {
    mbar_wait(&full[s], phase);
    const uint32_t c = coord[s];
    const int I = (int)(c & 0xffffu), J = (int)(c >> 16);
    const unsigned char *stage = sm + s * stage_bytes;
    const int nout = I == J ? 1 : 2;
    // output tiles of this thread: both (one group), or tile `group` (two)
    constexpr int NO = G::kGroups == 1 ? 2 : 1;
    uint32_t lo[NO][V], hi[NO][V];
#pragma unroll
    for (int k = 0; k < NO; ++k) {
      const int o = G::kGroups == 1 ? k : group;
      if (o >= nout) break;
      const int mode = I == J ? 3 : o + 1;
      if constexpr (Direct<E>::v) {
        eval_direct<E>(P, stage, (uint32_t)M.tile_bytes, mode, tv, uq, lo[k], hi[k]);
      } else {
        const int64_t row0 = (int64_t)(o == 0 ? I : J) * kTile + tr, col = (int64_t)(o == 0 ? J : I) * kTile + lane;
        Chunk ch;
        ch.flat = false;
        ch.stage = stage;
        ch.tile_bytes = M.tile_bytes;
        ch.tr = tr;
        ch.tc = lane;
        ch.pair = mode;
        ch.row0 = row0;
        ch.col = col;
        ch.cnt = (int)max((int64_t)0, min((int64_t)V, n - row0));
        ch.base = row0 + col * n;
        E::eval(P, ch, lo[k], hi[k]);
      }
    }
    // the stage is read: release it to the producer before the stores
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    // epilogue: results into the output tiles (once the previous pair's TMA
    // store has read them -- long done by now), then one thread stores the
    // tiles with 2-D TMA: full 128-byte lines, edges clipped by the map
    // (lane = column stores would write 32 B to each of 32 lines)
    constexpr int kCons = 32 * G::kConsumerWarps;
    if (threadIdx.x == 0) bulk_wait_read_all();   // the previous pair's store has read the buffer
    consumers_sync(kCons);
    unsigned char *ob = obuf;
#pragma unroll
    for (int k = 0; k < NO; ++k) {
      const int o = G::kGroups == 1 ? k : group;
      if (o >= nout) break;
      put_out<V>(ob + o * out_tile, M.out_w, tr, lane, lo[k], hi[k]);
    }
    fence_async_smem();
    consumers_sync(kCons);
    if (threadIdx.x == 0) {
      const int halves = M.out_w / 4, rows_per = kTile / halves;
      for (int h = 0; h < halves; ++h) {
        tma_store_2d(&M.out_map, ob + h * kHalf, I * kTile + h * rows_per, J * kTile);
        if (nout == 2) tma_store_2d(&M.out_map, ob + out_tile + h * kHalf, J * kTile + h * rows_per, I * kTile);
      }
      bulk_commit();
    }
    if (++s == stages) { s = 0; phase ^= 1u; }
  }
  if (threadIdx.x == 0) bulk_wait_all();   // global writes complete before the grid ends
}

}  // namespace pair

// ---- host side ----------------------------------------------------------------------------
// Is the copy program a tile-pair candidate: an n x n domain whose every
// slot is a whole n x n matrix (dense, or a subview at offset 0 with ld = n),
// plain or transposed, 4- or 8-byte elements TMA can address?
inline bool pair_eligible(const fm_program &P, int64_t n_rows, int64_t n_cols) {
  if (n_rows != n_cols || n_rows < pair::kTile || n_rows >= 65536ll * pair::kTile) return false;
  bool transposed = false;
  for (int j = 0; j < P.n_slots; ++j) {
    const fm_slot &s = P.slots[j];
    const int w = s.etype == FM_F64 ? 8 : (s.etype == FM_BF16 ? 2 : 4);
    if (s.map == FM_MAP_DIAG || s.row_off != 0 || s.col_off != 0 || s.ld != n_rows || w == 2) return false;
    if ((((uintptr_t)s.ptr) & 15) || ((n_rows * w) & 15)) return false;
    transposed |= s.transposed != 0;
  }
  return transposed;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
void *tensor_map_encoder();   // runtime.cu: cuTensorMapEncodeTiled via the runtime's entry-point query

// Group the slots by buffer (slot.reserved = buffer index) and encode one
// tensor map per buffer.  Returns false when the program has more distinct
// buffers than the kernel stages.
// one 2-D tensor map over an n x n column-major matrix of w-byte elements,
// box {128 bytes of a column, 32 columns}, 128-byte swizzle; 64-byte L2
// promotion (r02, scripts/gpu_promo.sh: neutral on aligned n, +6 % at
// n = 10000 f32 where odd columns start mid-line; 256 B costs up to 10 %)
inline int pair_encode(CUtensorMap *map, const void *ptr, int64_t n, int w) {
  EncodeTiledFn enc = (EncodeTiledFn)tensor_map_encoder();
  if (!enc) return fail_msg("pair: cuTensorMapEncodeTiled unavailable from the driver");
  const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)n * w};
  const cuuint32_t box[2] = {(cuuint32_t)(128 / w), (cuuint32_t)pair::kTile};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, w == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 2,
                   const_cast<void *>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_64B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail_msg("pair: cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r));
  return 0;
}

// Group the slots by buffer (slot.reserved = buffer index) and encode one
// tensor map per buffer and one for the output.  ok = false when the program
// has more distinct buffers than the kernel stages or a 2-byte result.
inline int pair_prepare(fm_program &P, pair::Maps &M, void *out, int64_t n, bool &ok) {
  ok = false;
  M.n_buf = 0;
  const int ow = P.result_etype == FM_F64 ? 8 : (P.result_etype == FM_BF16 ? 2 : 4);
  if (ow == 2 || (((uintptr_t)out) & 15)) return 0;
  int wmax = 4;
  for (int j = 0; j < P.n_slots; ++j) {
    fm_slot &s = P.slots[j];
    const int w = s.etype == FM_F64 ? 8 : 4;
    int b = -1;
    for (int i = 0; i < j; ++i)
      if (P.slots[i].ptr == s.ptr && (P.slots[i].etype == FM_F64 ? 8 : 4) == w) { b = P.slots[i].reserved; break; }
    if (b < 0) {
      if (M.n_buf == pair::kMaxBuf) return 0;
      b = M.n_buf++;
      M.width[b] = w;
      if (int st = pair_encode(&M.map[b], s.ptr, n, w)) return st;
    }
    s.reserved = b;
    wmax = std::max(wmax, w);
  }
  M.tile_bytes = pair::kTile * pair::kTile * wmax;
  M.out_w = ow;
  if (int st = pair_encode(&M.out_map, out, n, ow)) return st;
  ok = true;
  return 0;
}

// Device table of the pair order for an n x n domain (runtime.cu, cached per
// device and tile count): strips of kStrip tile columns, and in each strip
// row blocks I = 0, 1, ... with the strip's J >= I -- so the CTAs running at
// one time read a few hundred consecutive rows of kStrip x 32 columns
// (blocks (I,J)) and kStrip x 32 consecutive rows of many columns (blocks
// (J,I)): long runs per column instead of one 128-byte segment per column.
int pair_order(int64_t n, const uint32_t **table);

template <class E>
int run_copy_pair(const fm_program &P0, void *out, int64_t n, cudaStream_t s, bool &handled) {
  handled = false;
  fm_program P = P0;
  pair::Maps M;
  bool ok = false;
  if (int st = pair_prepare(P, M, out, n, ok)) return st;
  if (!ok) return 0;
  constexpr int kThreadsPair = pair::Geo<E>::kThreads;
  constexpr int kMaxSmem = 200 * 1024;
  static bool attr = false;
  if (!attr) {
    FM_CHECK(cudaFuncSetAttribute(pair::k_copy_pair<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    attr = true;
  }
  // the deepest ring (<= 6 stages) that still leaves >= 16 resident
  // consumer warps per SM; 2 stages when nothing does
  const size_t stage_bytes = (size_t)M.n_buf * 2 * M.tile_bytes;
  const size_t fixed = 2 * (size_t)pair::kTile * pair::kTile * M.out_w + 1024 + 256;   // out tiles, align, barriers
  // the ring depth (2..6 stages) that keeps the most bytes in flight per SM
  // -- (stages - 1) x stage x resident CTAs, one stage being evaluated --
  // with at least 8 consumer warps per SM when any depth allows it
  int stages = 0, occ = 0;
  int64_t best = -1;
  for (int st = 2; st <= 6; ++st) {
    const size_t sm_b = st * stage_bytes + fixed;
    if (sm_b > (size_t)kMaxSmem) break;
    int o = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, pair::k_copy_pair<E>, kThreadsPair, sm_b) != cudaSuccess)
      o = 0;
    if (o < 1) continue;
    const bool warps_ok = o * pair::Geo<E>::kConsumerWarps >= 8;
    const int64_t score = (int64_t)o * (st - 1) * (int64_t)stage_bytes + (warps_ok ? (1ll << 40) : 0);
    if (score > best) { best = score; stages = st; occ = o; }
  }
  if (stages == 0) return 0;
  const size_t smem = stages * stage_bytes + fixed;
  const uint32_t *order = nullptr;
  if (int st = pair_order(n, &order)) return st;
  const int64_t nt = (n + pair::kTile - 1) / pair::kTile;
  const int64_t np = nt * (nt + 1) / 2;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(np, (int64_t)sm_count() * occ));
  pair::k_copy_pair<E><<<(unsigned)grid, kThreadsPair, smem, s>>>(P, M, out, n, order, stages);
  FM_CHECK_LAUNCH("fused copy kernel (tile pairs)");
  handled = true;
  return 0;
}

}  // namespace fm
