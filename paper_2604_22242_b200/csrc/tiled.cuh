// tiled.cuh -- 2-D tiled, shared-memory staged copy skeleton for the
// register VM.
//
// The chunk path of the VM reads a transposed leaf (`X.t()`) with the
// parent's leading dimension as stride -- every lane touches its own cache
// line -- and reads views / mixed-width leaves one scalar at a time; the
// paper's suite members with such leaves ran at 0.75-2 TB/s
// (bench.py --config suite, r01).  Here a CTA owns a TR x TC output tile:
// every non-diagonal slot's source tile is copied into shared memory with
// `cp.async` along the slot's OWN contiguous dimension (columns of an
// untransposed leaf, rows of a transposed one), double-buffered so the next
// tile's copies are in flight while the VM evaluates the current one from
// shared memory.  Diagonal slots (stride ld+1, no reuse) still read global
// memory.  Also used for flat programs with more leaves than the VM
// prefetches (add-N), where it keeps every leaf's bytes in flight at once.
#pragma once
#include "skeletons.cuh"

namespace fm {
namespace tiled {

FM_DEV void cp_async4(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
FM_DEV void cp_async8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
FM_DEV void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
FM_DEV void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
FM_DEV void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

FM_DEV int etype_width(int e) { return e == FM_F64 ? 8 : (e == FM_BF16 ? 2 : 4); }

// one element of width w, asynchronously where the size allows
FM_DEV void copy_elem(unsigned char *dst, const unsigned char *src, int w) {
  if (w == 4) cp_async4(dst, src);
  else if (w == 8) cp_async8(dst, src);
  else *(uint16_t *)dst = __ldg((const unsigned short *)src);
}

template <int V, int TC, int WMAX>
struct Geo {
  static constexpr int TR = 8 * V;               // 8 row-chunks of V elements per column
  static constexpr int NT = 8 * TC;              // one thread per (row-chunk, column)
  static constexpr int TRP = TR + 8;             // column-major pitch: 16-byte column starts for w = 2, 4, 8
  static constexpr int TCP = TC;                 // row-major pitch (16-byte chunks swizzled, see stage_tile)
  static constexpr int LTR = V == 8 ? 6 : (V == 4 ? 5 : 4);   // log2(TR)
  static constexpr int LTC = TC == 64 ? 6 : (TC == 32 ? 5 : (TC == 16 ? 4 : 3));
  static constexpr int SB0 = (TC * TRP > TR * TCP ? TC * TRP : TR * TCP) * WMAX;
  static constexpr int SLOT_BYTES = (SB0 + 15) / 16 * 16;
};

// Issue the copies of tile (r0, c0) for every staged slot into `buf`.
// Full tiles with 16-byte aligned source runs move 16-byte vectors (index
// math by shifts: TR, TC and the widths are powers of two); edge tiles and
// unaligned views copy element by element.
template <int V, int TC, int WMAX>
FM_DEV void stage_tile(const fm_program &P, unsigned char *buf, int64_t r0, int64_t c0, int rv, int cv) {
  using G = Geo<V, TC, WMAX>;
  const int tid = threadIdx.x;
  const bool full = rv == G::TR && cv == TC;
  for (int j = 0; j < P.n_slots; ++j) {
    const fm_slot &s = P.slots[j];
    if (s.map == FM_MAP_DIAG) continue;
    const int w = etype_width(s.etype);
    const int lw = w == 8 ? 3 : (w == 4 ? 2 : 1);
    unsigned char *dst = buf + (size_t)j * G::SLOT_BYTES;
    const unsigned char *base = (const unsigned char *)s.ptr;
    const bool aligned = ((s.ld * w) & 15) == 0 && (((uintptr_t)base) & 15) == 0;
    if (!s.transposed) {
      // element (r, c) of the tile = parent (r0 + r + row_off, c0 + c + col_off); columns contiguous
      const int64_t prow = r0 + s.row_off, pcol = c0 + s.col_off;
      const unsigned char *src0 = base + (prow + pcol * s.ld) * w;
      if (full && aligned && ((prow * w) & 15) == 0) {
        const int lpc = (G::LTR + lw) - 4;                 // log2(16-byte vectors per column)
        for (int i = tid; i < (TC << lpc); i += G::NT) {
          const int c = i >> lpc, q = i & ((1 << lpc) - 1);
          cp_async16(dst + ((size_t)c * G::TRP << lw) + 16 * q, src0 + (int64_t)c * s.ld * w + 16 * q);
        }
      } else {
        for (int i = tid; i < rv * cv; i += G::NT) {
          const int c = i / rv, r = i - c * rv;
          copy_elem(dst + (size_t)(c * G::TRP + r) * w, src0 + (r + (int64_t)c * s.ld) * w, w);
        }
      }
    } else {
      // transposed: element (r, c) = parent (c0 + c + row_off, r0 + r + col_off); parent columns run
      // along the tile's rows, so tile row r is a contiguous run of the parent.  Row-major tile,
      // pitch TC, 16-byte chunks XOR-swizzled by (r / 8) so a warp's column reads spread over banks.
      const int64_t prow = c0 + s.row_off, pcol = r0 + s.col_off;
      const unsigned char *src0 = base + (prow + pcol * s.ld) * w;
      if (full && aligned && ((prow * w) & 15) == 0) {
        const int lpr = (G::LTC + lw) - 4;                 // log2(16-byte vectors per row)
        const int qmask = (1 << lpr) - 1;
        for (int i = tid; i < (G::TR << lpr); i += G::NT) {
          const int r = i >> lpr, q = i & qmask;
          const int qs = q ^ ((r >> 3) & qmask);
          cp_async16(dst + ((size_t)r * TC << lw) + 16 * qs, src0 + (int64_t)r * s.ld * w + 16 * q);
        }
      } else {
        for (int i = tid; i < rv * cv; i += G::NT) {
          const int r = i / cv, c = i - r * cv;
          const int qmask = (TC * w / 16) - 1;
          const int byte = c * w, qs = (byte >> 4) ^ ((r >> 3) & qmask);
          copy_elem(dst + (size_t)r * TC * w + qs * 16 + (byte & 15), src0 + (c + (int64_t)r * s.ld) * w, w);
        }
      }
    }
  }
}

// Tile t -> (row block, column block), column-major tile order (neighbouring
// CTAs on neighbouring HBM pages).
FM_DEV void tile_of(int64_t t, int64_t ntr, int64_t &bi, int64_t &bj) {
  bi = t % ntr;
  bj = t / ntr;
}

template <class E, int TC>
__global__ void __launch_bounds__(8 * TC) k_copy_tiled(const __grid_constant__ fm_program P, void *out,
                                                        int64_t n_rows, int64_t n_cols) {
  constexpr int V = E::kV, WMAX = E::kWide ? 8 : 4;
  using G = Geo<V, TC, WMAX>;
  extern __shared__ __align__(16) unsigned char sm[];
  const size_t buf_bytes = (size_t)P.n_slots * G::SLOT_BYTES;
  const int64_t ntr = (n_rows + G::TR - 1) / G::TR, ntc = (n_cols + TC - 1) / TC;
  const int64_t ntiles = ntr * ntc;
  const int k = threadIdx.x & 7, cc = threadIdx.x >> 3;
  int64_t t = blockIdx.x;
  if (t < ntiles) {
    int64_t bi, bj;
    tile_of(t, ntr, bi, bj);
    const int64_t r0 = bi * G::TR, c0 = bj * TC;
    stage_tile<V, TC, WMAX>(P, sm, r0, c0, (int)min((int64_t)G::TR, n_rows - r0), (int)min((int64_t)TC, n_cols - c0));
  }
  cp_commit();
  for (int b = 0; t < ntiles; t += gridDim.x, b ^= 1) {
    const int64_t tn = t + gridDim.x;
    if (tn < ntiles) {
      int64_t bi, bj;
      tile_of(tn, ntr, bi, bj);
      const int64_t r0 = bi * G::TR, c0 = bj * TC;
      stage_tile<V, TC, WMAX>(P, sm + (b ^ 1) * buf_bytes, r0, c0, (int)min((int64_t)G::TR, n_rows - r0),
                        (int)min((int64_t)TC, n_cols - c0));
    }
    cp_commit();
    cp_wait<1>();        // this tile's copies (all but the newest group) have landed
    __syncthreads();
    int64_t bi, bj;
    tile_of(t, ntr, bi, bj);
    const int64_t r0 = bi * G::TR, c0 = bj * TC;
    const int rv = (int)min((int64_t)G::TR, n_rows - r0), cv = (int)min((int64_t)TC, n_cols - c0);
    if (cc < cv && k * V < rv) {
      Chunk ch;
      ch.row0 = r0 + k * V;
      ch.col = c0 + cc;
      ch.cnt = min(V, rv - k * V);
      ch.base = ch.row0 + ch.col * n_rows;
      ch.flat = false;
      ch.stage = sm + b * buf_bytes;
      ch.tr = k * V;
      ch.tc = cc;
      ch.trp = G::TRP;
      ch.tcp = G::TCP;
      ch.slot_bytes = G::SLOT_BYTES;
      uint32_t lo[V], hi[V];
      E::eval(P, ch, lo, hi);
      store_chunk<V>(out, P.result_etype, ch.base, ch.cnt, lo, hi);
    }
    __syncthreads();     // every read of buffer b is done before it is refilled
  }
}

}  // namespace tiled
}  // namespace fm

namespace fm {
namespace tiled {

// bytes of dynamic shared memory for a program with n_slots leaves
template <class E, int TC>
constexpr int64_t smem_bytes(int n_slots) {
  return 2ll * n_slots * Geo<E::kV, TC, E::kWide ? 8 : 4>::SLOT_BYTES;
}

}  // namespace tiled
}  // namespace fm
