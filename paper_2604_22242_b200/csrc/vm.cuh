// vm.cuh -- generic fused kernel: a register-stack VM for fm_program.
//
// The program (include/fmb200.h) lives in kernel parameter space, so every
// instruction fetch is a uniform constant-bank read.  Each thread evaluates V
// consecutive elements at once; every instruction is specialised on the stack
// slot it writes ((opcode << 3) | depth), so the stack stays in registers and
// the dispatch cost (one BRX per instruction) is paid once per V elements.
// Leaf slots < NPF are loaded up front (vectorised, all in flight together)
// before the program runs; further slots load at their PUSH.
#pragma once
#include "fmb200.h"
#include "ops.cuh"

namespace fm {

#define FM_DEV __device__ __forceinline__

FM_DEV uint4 ldg_v4(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
FM_DEV uint2 ldg_v2(const void *p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
               : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
FM_DEV uint32_t ldg_u32(const void *p) { return __ldg((const unsigned int *)p); }
FM_DEV uint16_t ldg_u16(const void *p) { return __ldg((const unsigned short *)p); }
FM_DEV unsigned long long ldg_u64(const void *p) { return __ldg((const unsigned long long *)p); }

// Element index of slot `s` for output element (r, c).
FM_DEV int64_t slot_index(const fm_slot &s, int64_t r, int64_t c) {
  if (s.transposed) { int64_t t = r; r = c; c = t; }
  if (s.map == FM_MAP_SUBVIEW) return (r + s.row_off) + (c + s.col_off) * s.ld;
  if (s.map == FM_MAP_DIAG) return (r + s.row_off) + (r + s.col_off) * s.ld;
  return r + c * s.ld;
}

// Load one element of slot `s` at element index `i` into (lo, hi) bits.
FM_DEV void load_one(const fm_slot &s, int64_t i, uint32_t &lo, uint32_t &hi) {
  switch (s.etype) {
    case FM_F64: {
      unsigned long long w = ldg_u64((const unsigned long long *)s.ptr + i);
      lo = (uint32_t)w; hi = (uint32_t)(w >> 32);
      break;
    }
    case FM_BF16: lo = ((uint32_t)ldg_u16((const uint16_t *)s.ptr + i)) << 16; break;
    default: lo = ldg_u32((const uint32_t *)s.ptr + i); break;
  }
}

// A chunk is V consecutive elements.  Flat chunks index every slot by the
// flat index base+v; column chunks are rows row0..row0+V-1 of column `col`.
struct Chunk {
  int64_t base;   // flat index of the first element (output index)
  int64_t row0;
  int64_t col;
  int cnt;        // valid elements (<= V)
  bool flat;
  // shared-memory staged tile (tiled.cuh), or nullptr: read global memory
  const unsigned char *stage = nullptr;
  int tr = 0, tc = 0;        // chunk position inside the tile (first row, column)
  int trp = 0, tcp = 0;      // element pitches of the column-major / transposed layouts
  int slot_bytes = 0;        // bytes per staged slot
  // tile-pair layout (pair.cuh): 0 = the per-slot layouts above; else which
  // output tile of the pair this chunk belongs to (1: (I,J), 2: (J,I),
  // 3: a diagonal tile), and the bytes of one staged 32 x 32 tile
  int pair = 0;
  int tile_bytes = 0;
  // bulk-staged flat chunk (bulk.cuh k_copy_bulk_vm): slot j's elements of
  // the staged chunk start at bstage + slot.reserved; this chunk's first
  // element is element `boff` of it
  const unsigned char *bstage = nullptr;
  int boff = 0;
};

// Load V elements of slot s for a flat chunk (every slot dense, same shape).
template <int V>
FM_DEV void load_slot_flat(const fm_slot &s, const Chunk &ch, uint32_t (&lo)[V], uint32_t (&hi)[V]);

template <int V>
FM_DEV void load_slot_flat(const fm_slot &s, const Chunk &ch, uint32_t (&lo)[V], uint32_t (&hi)[V]) {
  const int64_t b = ch.base;
  if (s.etype == FM_F64) {
    const unsigned long long *p = (const unsigned long long *)s.ptr + b;
    if (ch.cnt == V && (((uintptr_t)p) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < V / 2; ++q) {
        uint4 w = ldg_v4(p + 2 * q);
        lo[2 * q] = w.x; hi[2 * q] = w.y; lo[2 * q + 1] = w.z; hi[2 * q + 1] = w.w;
      }
      return;
    }
  } else if (s.etype == FM_BF16) {
    const uint16_t *p = (const uint16_t *)s.ptr + b;
    if (ch.cnt == V && (((uintptr_t)p) & (2 * V - 1)) == 0 && (V == 4 || V == 8)) {
      if (V == 8) {
        uint4 w = ldg_v4(p);
        uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4 && 2 * q + 1 < V; ++q) {
          lo[2 * q] = ws[q] << 16; lo[2 * q + 1] = ws[q] & 0xffff0000u;
        }
      } else {
        uint2 w = ldg_v2(p);
        lo[0] = w.x << 16; lo[1] = w.x & 0xffff0000u;
        lo[2 % V] = w.y << 16; lo[3 % V] = w.y & 0xffff0000u;
      }
      return;
    }
  } else {
    const uint32_t *p = (const uint32_t *)s.ptr + b;
    if (ch.cnt == V && (((uintptr_t)p) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < V / 4; ++q) {
        uint4 w = ldg_v4(p + 4 * q);
        lo[4 * q] = w.x; lo[4 * q + 1] = w.y; lo[4 * q + 2] = w.z; lo[4 * q + 3] = w.w;
      }
      return;
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    lo[v] = 0; hi[v] = 0;
    if (v < ch.cnt) load_one(s, b + v, lo[v], hi[v]);
  }
  return;
}

// Load V elements of slot s for the chunk.
template <int V>
FM_DEV void load_slot(const fm_slot &s, const Chunk &ch, uint32_t (&lo)[V], uint32_t (&hi)[V]) {
  if (ch.flat) {
    load_slot_flat<V>(s, ch, lo, hi);
    return;
  }
  // untransposed dense / subview leaf: the chunk's V rows are consecutive in
  // one parent column -- vector loads when the run is whole and aligned
  if (!s.transposed && s.map != FM_MAP_DIAG && ch.cnt == V) {
    const int64_t i0 = slot_index(s, ch.row0, ch.col);
    if (s.etype == FM_F64 && V % 2 == 0) {
      const unsigned long long *p = (const unsigned long long *)s.ptr + i0;
      if ((((uintptr_t)p) & 15) == 0) {
#pragma unroll
        for (int q = 0; q < V / 2; ++q) {
          uint4 w = ldg_v4(p + 2 * q);
          lo[2 * q] = w.x; hi[2 * q] = w.y; lo[2 * q + 1] = w.z; hi[2 * q + 1] = w.w;
        }
        return;
      }
    } else if (s.etype != FM_F64 && s.etype != FM_BF16 && V % 4 == 0) {
      const uint32_t *p = (const uint32_t *)s.ptr + i0;
      if ((((uintptr_t)p) & 15) == 0) {
#pragma unroll
        for (int q = 0; q < V / 4; ++q) {
          uint4 w = ldg_v4(p + 4 * q);
          lo[4 * q] = w.x; lo[4 * q + 1] = w.y; lo[4 * q + 2] = w.z; lo[4 * q + 3] = w.w;
        }
        return;
      }
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    lo[v] = 0; hi[v] = 0;
    if (v < ch.cnt) load_one(s, slot_index(s, ch.row0 + v, ch.col), lo[v], hi[v]);
  }
}

// Load V elements of slot `s` from its staged tile.  Untransposed slots are
// staged column-major (element (r, c) at c*trp + r), transposed ones
// row-major (at r*tcp + c), so both are read along the layout they were
// copied in with (coalesced global reads, tiled.cuh).
template <int V>
FM_DEV void load_staged(const fm_slot &s, const unsigned char *buf, const Chunk &ch, uint32_t (&lo)[V],
                        uint32_t (&hi)[V]) {
  const int w = s.etype == FM_F64 ? 8 : (s.etype == FM_BF16 ? 2 : 4);
  if (!s.transposed) {
    const unsigned char *p = buf + (size_t)(ch.tc * ch.trp + ch.tr) * w;
    if (w == 4 && V % 4 == 0) {
#pragma unroll
      for (int q = 0; q < V / 4; ++q) {
        const uint4 x = *(const uint4 *)(p + 16 * q);
        lo[4 * q] = x.x; lo[4 * q + 1] = x.y; lo[4 * q + 2] = x.z; lo[4 * q + 3] = x.w;
      }
      return;
    }
    if (w == 8 && V % 2 == 0) {
#pragma unroll
      for (int q = 0; q < V / 2; ++q) {
        const uint4 x = *(const uint4 *)(p + 16 * q);
        lo[2 * q] = x.x; hi[2 * q] = x.y; lo[2 * q + 1] = x.z; hi[2 * q + 1] = x.w;
      }
      return;
    }
#pragma unroll
    for (int v = 0; v < V; ++v) lo[v] = ((uint32_t)((const uint16_t *)p)[v]) << 16;
    return;
  }
  // row-major tile, pitch tcp elements, 16-byte chunks XOR-swizzled by row/8
  const int qmask = (ch.tcp * w / 16) - 1;
  const int byte = ch.tc * w;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int r = ch.tr + v;
    const unsigned char *p = buf + (size_t)r * ch.tcp * w + ((((byte >> 4) ^ (r >> 3)) & qmask) << 4) + (byte & 15);
    if (w == 8) {
      const uint2 x = *(const uint2 *)p;
      lo[v] = x.x; hi[v] = x.y;
    } else if (w == 4) {
      lo[v] = *(const uint32_t *)p;
    } else {
      lo[v] = ((uint32_t)*(const uint16_t *)p) << 16;
    }
  }
}

// Load V elements of slot `s` from the tile-pair stage (pair.cuh).  Every
// distinct buffer b (slot.reserved) has two 32 x 32 tiles staged by 2-D TMA
// with the 128-byte swizzle: A = M[I-block, J-block] and B = M[J-block,
// I-block], column-major, 128-byte rows (= tile columns, 16 B chunk q of
// column c at q ^ (c & 7)); 8-byte elements take two 16-row half tiles of
// 4 KiB.  Untransposed slots read V rows of one column (16-byte vectors);
// transposed slots read one row across V columns of the other tile.  With
// lane = column both patterns are bank-conflict free.
FM_DEV int pair_off(int r, int c, int w) {
  const int rb = r * w;
  return ((rb >> 7) << 12) + (c << 7) + ((((rb >> 4) ^ c) & 7) << 4) + (rb & 15);
}
FM_DEV const unsigned char *pair_addr(const unsigned char *t, int r, int c, int w) { return t + pair_off(r, c, w); }
template <int V>
FM_DEV void load_pair(const fm_slot &s, const Chunk &ch, uint32_t (&lo)[V], uint32_t (&hi)[V]) {
  const int w = s.etype == FM_F64 ? 8 : 4;
  const int tr = s.transposed != 0;
  const int sel = ch.pair == 3 ? 0 : (tr ^ (ch.pair == 2));
  const unsigned char *t = ch.stage + (size_t)(s.reserved * 2 + sel) * ch.tile_bytes;
  if (!tr) {
    if (w == 4) {
#pragma unroll
      for (int q = 0; q < V / 4; ++q) {
        const uint4 x = *(const uint4 *)pair_addr(t, ch.tr + 4 * q, ch.tc, 4);
        lo[4 * q] = x.x; lo[4 * q + 1] = x.y; lo[4 * q + 2] = x.z; lo[4 * q + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < V / 2; ++q) {
        const uint4 x = *(const uint4 *)pair_addr(t, ch.tr + 2 * q, ch.tc, 8);
        lo[2 * q] = x.x; hi[2 * q] = x.y; lo[2 * q + 1] = x.z; hi[2 * q + 1] = x.w;
      }
    }
    return;
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const unsigned char *p = pair_addr(t, ch.tc, ch.tr + v, w);
    if (w == 8) {
      const uint2 x = *(const uint2 *)p;
      lo[v] = x.x; hi[v] = x.y;
    } else {
      lo[v] = *(const uint32_t *)p;
    }
  }
}

// V elements of slot s from a bulk-staged chunk (vector shared-memory loads)
template <int V>
FM_DEV void load_bulk(const fm_slot &s, const Chunk &ch, uint32_t (&lo)[V], uint32_t (&hi)[V]) {
  const unsigned char *p = ch.bstage + s.reserved;
  if (s.etype == FM_F64) {
    p += (size_t)ch.boff * 8;
#pragma unroll
    for (int q = 0; q < V / 2; ++q) {
      const uint4 x = *(const uint4 *)(p + 16 * q);
      lo[2 * q] = x.x; hi[2 * q] = x.y; lo[2 * q + 1] = x.z; hi[2 * q + 1] = x.w;
    }
  } else if (s.etype == FM_BF16) {
    p += (size_t)ch.boff * 2;
    if constexpr (V == 8) {
      const uint4 x = *(const uint4 *)p;
      const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) { lo[2 * q] = w[q] << 16; lo[2 * q + 1] = w[q] & 0xffff0000u; }
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) lo[v] = ((uint32_t)((const uint16_t *)p)[v]) << 16;
    }
  } else {
    p += (size_t)ch.boff * 4;
#pragma unroll
    for (int q = 0; q < V / 4; ++q) {
      const uint4 x = *(const uint4 *)(p + 16 * q);
      lo[4 * q] = x.x; lo[4 * q + 1] = x.y; lo[4 * q + 2] = x.z; lo[4 * q + 3] = x.w;
    }
  }
}

// Slot j of the program for the chunk: staged tile when the kernel staged it
// (every slot but diagonals), global memory otherwise.
template <int V, bool FLAT_ONLY = false>
FM_DEV void fetch_slot(const fm_program &P, int j, const Chunk &ch, uint32_t (&lo)[V], uint32_t (&hi)[V]) {
  const fm_slot &s = P.slots[j];
  if constexpr (FLAT_ONLY) {
    // evaluators whose programs are always flat (flat-signature templates)
    // carry no view / staging code: fewer live registers
    load_slot_flat<V>(s, ch, lo, hi);
  } else {
    if (ch.bstage) load_bulk<V>(s, ch, lo, hi);
    else if (ch.pair) load_pair<V>(s, ch, lo, hi);
    else if (ch.stage && s.map != FM_MAP_DIAG) load_staged<V>(s, ch.stage + (size_t)j * ch.slot_bytes, ch, lo, hi);
    else load_slot<V>(s, ch, lo, hi);
  }
}

// -----------------------------------------------------------------------------
// The interpreter.  WIDE: registers carry 64-bit values (any f64 in the
// program).  MAXD: stack depth.  V: elements per thread.  NPF: prefetched slots.
template <bool WIDE, int MAXD, int V, int NPF>
struct Vm {
  static constexpr int kV = V;
  static constexpr bool kWide = WIDE;
  static constexpr bool kIsVm = true;
  static constexpr int kMinBlocks = 1;
  static constexpr bool kTiled = true;
  static constexpr bool kFast = false;
  FM_DEV static bool fast_ok(const fm_program &, const void *) { return false; }
  static constexpr int HD = WIDE ? MAXD : 1;
  static constexpr int HP = WIDE && NPF > 0 ? NPF : 1;

  // Evaluate the chunk; result bits land in (lo0, hi0).
  FM_DEV static void eval(const fm_program &P, const Chunk &ch, uint32_t (&lo0)[V], uint32_t (&hi0)[V]) {
    uint32_t lo[MAXD][V];
    uint32_t hi[HD][V];
    uint32_t plo[NPF > 0 ? NPF : 1][V];
    uint32_t phi[HP > 0 ? HP : 1][V];

    // Prefetch: all loads issued back to back.
#pragma unroll
    for (int j = 0; j < NPF; ++j) {
      if (j < P.n_slots) {
        uint32_t th[V];
        fetch_slot<V>(P, j, ch, plo[j], th);
        if constexpr (WIDE) {
#pragma unroll
          for (int v = 0; v < V; ++v) phi[j < HP ? j : 0][v] = th[v];
        }
      }
    }

#define LO(d) lo[((d) < MAXD) ? (d) : 0]
#define HI(d) hi[(WIDE && (d) < MAXD) ? (d) : 0]
#define VLOOP _Pragma("unroll") for (int v = 0; v < V; ++v)
#define CASE(OP, D) case ((FM_OP_##OP << 3) | (D)):
#define OKD(D) ((D) < MAXD)
#define OKB(D) ((D) + 1 < MAXD)

#define PUSH32(D)                                                               \
  CASE(PUSH32, D) if constexpr (OKD(D)) {                                       \
    switch (a) {                                                                \
      case 0: if constexpr (NPF > 0) { VLOOP LO(D)[v] = plo[0][v]; break; }     \
      case 1: if constexpr (NPF > 1) { VLOOP LO(D)[v] = plo[1 % NPF][v]; break; } \
      case 2: if constexpr (NPF > 2) { VLOOP LO(D)[v] = plo[2 % NPF][v]; break; } \
      case 3: if constexpr (NPF > 3) { VLOOP LO(D)[v] = plo[3 % NPF][v]; break; } \
      default: { uint32_t th[V]; fetch_slot<V>(P, a, ch, LO(D), th); }         \
    }                                                                           \
  } break;

#define PUSH64(D)                                                               \
  CASE(PUSH64, D) if constexpr (WIDE && OKD(D)) {                               \
    if (a < NPF) {                                                              \
      switch (a) {                                                              \
        case 0: VLOOP { LO(D)[v] = plo[0][v]; HI(D)[v] = phi[0][v]; } break;     \
        case 1: VLOOP { LO(D)[v] = plo[1 % NPF][v]; HI(D)[v] = phi[1 % HP][v]; } break; \
        case 2: VLOOP { LO(D)[v] = plo[2 % NPF][v]; HI(D)[v] = phi[2 % HP][v]; } break; \
        default: VLOOP { LO(D)[v] = plo[3 % NPF][v]; HI(D)[v] = phi[3 % HP][v]; } break; \
      }                                                                         \
    } else {                                                                    \
      fetch_slot<V>(P, a, ch, LO(D), HI(D));                                    \
    }                                                                           \
  } break;

#define BIN_F(OP, EXPR, D)                                                      \
  CASE(OP, D) if constexpr (OKB(D)) {                                           \
    VLOOP { float x = u2f(LO(D)[v]), y = u2f(LO((D) + 1)[v]); LO(D)[v] = f2u(EXPR); } \
  } break;
#define BIN_D(OP, EXPR, D)                                                      \
  CASE(OP, D) if constexpr (WIDE && OKB(D)) {                                   \
    VLOOP { double x = u2d(LO(D)[v], HI(D)[v]), y = u2d(LO((D) + 1)[v], HI((D) + 1)[v]); \
            d2u(EXPR, LO(D)[v], HI(D)[v]); }                                    \
  } break;
#define BIN_I(OP, EXPR, D)                                                      \
  CASE(OP, D) if constexpr (OKB(D)) {                                           \
    VLOOP { uint32_t x = LO(D)[v], y = LO((D) + 1)[v]; LO(D)[v] = (EXPR); }     \
  } break;
// fused binary ops: the slot operand (yl, yh) is loaded once per
// instruction before the dispatch (one fetch_slot call site for all of them)
#define BINS_F(OP, EXPR, D)                                                     \
  CASE(OP, D) if constexpr (OKD(D)) {                                           \
    VLOOP { float x = u2f(LO(D)[v]), y = u2f(yl[v]); LO(D)[v] = f2u(EXPR); }    \
  } break;
#define BINS_D(OP, EXPR, D)                                                     \
  CASE(OP, D) if constexpr (WIDE && OKD(D)) {                                   \
    VLOOP { double x = u2d(LO(D)[v], HI(D)[v]), y = u2d(yl[v], yh[v]);          \
            d2u(EXPR, LO(D)[v], HI(D)[v]); }                                    \
  } break;
#define BINS_I(OP, EXPR, D)                                                     \
  CASE(OP, D) if constexpr (OKD(D)) {                                           \
    VLOOP { uint32_t x = LO(D)[v], y = yl[v]; LO(D)[v] = (EXPR); }              \
  } break;
#define UN_F(OP, EXPR, D)                                                       \
  CASE(OP, D) if constexpr (OKD(D)) {                                           \
    const float s = u2f((uint32_t)sb); (void)s;                                 \
    VLOOP { float x = u2f(LO(D)[v]); LO(D)[v] = f2u(EXPR); }                    \
  } break;
#define UN_D(OP, EXPR, D)                                                       \
  CASE(OP, D) if constexpr (WIDE && OKD(D)) {                                   \
    const double s = __longlong_as_double((long long)sb); (void)s;              \
    VLOOP { double x = u2d(LO(D)[v], HI(D)[v]); d2u(EXPR, LO(D)[v], HI(D)[v]); } \
  } break;
#define UN_I(OP, EXPR, D)                                                       \
  CASE(OP, D) if constexpr (OKD(D)) {                                           \
    const uint32_t s = (uint32_t)sb; (void)s;                                   \
    VLOOP { uint32_t x = LO(D)[v]; LO(D)[v] = (EXPR); }                         \
  } break;
// widening / narrowing conversions
#define CV_TO_D(OP, EXPR, D)                                                    \
  CASE(OP, D) if constexpr (WIDE && OKD(D)) {                                   \
    VLOOP { uint32_t xb = LO(D)[v]; (void)xb; float xf = u2f(xb); (void)xf;     \
            d2u(EXPR, LO(D)[v], HI(D)[v]); }                                    \
  } break;
#define CV_FROM_D(OP, EXPR, D)                                                  \
  CASE(OP, D) if constexpr (WIDE && OKD(D)) {                                   \
    VLOOP { double x = u2d(LO(D)[v], HI(D)[v]); LO(D)[v] = (EXPR); }            \
  } break;

#define ALLD(M, ...) M(__VA_ARGS__, 0) M(__VA_ARGS__, 1) M(__VA_ARGS__, 2) M(__VA_ARGS__, 3) \
                     M(__VA_ARGS__, 4) M(__VA_ARGS__, 5) M(__VA_ARGS__, 6) M(__VA_ARGS__, 7)

    const int n = P.n_instr;
    for (int pc = 0; pc < n; ++pc) {
      const fm_instr ins = P.code[pc];
      const int a = ins.arg;
      const uint64_t sb = P.scalars[a & (FM_MAX_SCALARS - 1)];
      (void)sb;
      uint32_t yl[V], yh[V];
      if (ins.key >= (FM_OP_ADD_F_S << 3)) {   // slot operand of a fused binary op
        bool pre = false;
#pragma unroll
        for (int j = 0; j < NPF; ++j)
          if (a == j) {
            VLOOP { yl[v] = plo[j][v]; yh[v] = phi[j < HP ? j : 0][v]; }
            pre = true;
          }
        if (!pre) fetch_slot<V>(P, a, ch, yl, yh);
      }
      switch (ins.key) {
        PUSH32(0) PUSH32(1) PUSH32(2) PUSH32(3) PUSH32(4) PUSH32(5) PUSH32(6) PUSH32(7)
        PUSH64(0) PUSH64(1) PUSH64(2) PUSH64(3) PUSH64(4) PUSH64(5) PUSH64(6) PUSH64(7)
        ALLD(BIN_F, ADD_F, add_f(x, y))
        ALLD(BIN_F, SUB_F, sub_f(x, y))
        ALLD(BIN_F, RSUB_F, sub_f(y, x))
        ALLD(BIN_F, MUL_F, mul_f(x, y))
        ALLD(BIN_F, DIV_F, div_f(x, y))
        ALLD(BIN_F, RDIV_F, div_f(y, x))
        ALLD(BIN_D, ADD_D, add_d(x, y))
        ALLD(BIN_D, SUB_D, sub_d(x, y))
        ALLD(BIN_D, RSUB_D, sub_d(y, x))
        ALLD(BIN_D, MUL_D, mul_d(x, y))
        ALLD(BIN_D, DIV_D, div_d(x, y))
        ALLD(BIN_D, RDIV_D, div_d(y, x))
        ALLD(BIN_I, ADD_I, add_i(x, y))
        ALLD(BIN_I, SUB_I, sub_i(x, y))
        ALLD(BIN_I, RSUB_I, sub_i(y, x))
        ALLD(BIN_I, MUL_I, mul_i(x, y))
        ALLD(BINS_F, ADD_F_S, add_f(x, y))
        ALLD(BINS_F, SUB_F_S, sub_f(x, y))
        ALLD(BINS_F, RSUB_F_S, sub_f(y, x))
        ALLD(BINS_F, MUL_F_S, mul_f(x, y))
        ALLD(BINS_F, DIV_F_S, div_f(x, y))
        ALLD(BINS_F, RDIV_F_S, div_f(y, x))
        ALLD(BINS_D, ADD_D_S, add_d(x, y))
        ALLD(BINS_D, SUB_D_S, sub_d(x, y))
        ALLD(BINS_D, RSUB_D_S, sub_d(y, x))
        ALLD(BINS_D, MUL_D_S, mul_d(x, y))
        ALLD(BINS_D, DIV_D_S, div_d(x, y))
        ALLD(BINS_D, RDIV_D_S, div_d(y, x))
        ALLD(BINS_I, ADD_I_S, add_i(x, y))
        ALLD(BINS_I, SUB_I_S, sub_i(x, y))
        ALLD(BINS_I, RSUB_I_S, sub_i(y, x))
        ALLD(BINS_I, MUL_I_S, mul_i(x, y))
        ALLD(UN_F, SADD_F, add_f(x, s))
        ALLD(UN_F, SMUL_F, mul_f(s, x))
        ALLD(UN_F, SDIV_F, div_f(s, x))
        ALLD(UN_F, GTS_F, gts_f(x, s))
        ALLD(UN_D, SADD_D, add_d(x, s))
        ALLD(UN_D, SMUL_D, mul_d(s, x))
        ALLD(UN_D, SDIV_D, div_d(s, x))
        ALLD(UN_D, GTS_D, gts_d(x, s))
        ALLD(UN_I, SADD_I, add_i(x, s))
        ALLD(UN_I, SMUL_I, mul_i(s, x))
        ALLD(UN_I, GTS_I32, gts_i32(x, s))
        ALLD(UN_I, GTS_U32, gts_u32(x, s))
        ALLD(UN_F, NEG_F, neg_f(x))
        ALLD(UN_D, NEG_D, neg_d(x))
        ALLD(UN_I, NEG_I, neg_i(x))
        ALLD(UN_F, ABS_F, abs_f(x))
        ALLD(UN_D, ABS_D, abs_d(x))
        ALLD(UN_I, ABS_I32, abs_i32(x))
        ALLD(UN_F, EXP_F, exp_f(x))
        ALLD(UN_F, LOG_F, log_f(x))
        ALLD(UN_F, SQRT_F, sqrt_f(x))
        ALLD(UN_F, TANH_F, tanh_f(x))
        ALLD(UN_D, EXP_D, exp_d(x))
        ALLD(UN_D, LOG_D, log_d(x))
        ALLD(UN_D, SQRT_D, sqrt_d(x))
        ALLD(UN_D, TANH_D, tanh_d(x))
        ALLD(UN_F, POW_F, pow_f(x, a))
        ALLD(UN_D, POW_D, pow_d(x, a))
        ALLD(UN_I, POW_I, pow_i(x, a))
        ALLD(UN_F, ONE_F, 1.0f)
        ALLD(UN_D, ONE_D, 1.0)
        ALLD(UN_I, ONE_I, 1u)
        ALLD(CV_TO_D, CVT_F_D, (double)xf)
        ALLD(CV_FROM_D, CVT_D_F, f2u(d_to_f(x)))
        ALLD(UN_F, CVT_F_I, __uint_as_float(f_to_i32bits(x)))
        ALLD(CV_FROM_D, CVT_D_I, d_to_i32bits(x))
        ALLD(UN_I, CVT_I32_F, f2u(i32_to_f(x)))
        ALLD(UN_I, CVT_U32_F, f2u(u32_to_f(x)))
        ALLD(CV_TO_D, CVT_I32_D, i32_to_d(xb))
        ALLD(CV_TO_D, CVT_U32_D, u32_to_d(xb))
        ALLD(UN_F, RND_BF_F, rnd_bf_f(x))
        ALLD(CV_FROM_D, CVT_D_BF, f2u(d_to_bf(x)))
        default: break;
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      lo0[v] = lo[0][v];
      hi0[v] = WIDE ? hi[0][v] : 0u;
    }
#undef LO
#undef HI
#undef VLOOP
#undef CASE
#undef OKD
#undef OKB
#undef PUSH32
#undef PUSH64
#undef BIN_F
#undef BIN_D
#undef BIN_I
#undef BINS_F
#undef BINS_D
#undef BINS_I
#undef UN_F
#undef UN_D
#undef UN_I
#undef CV_TO_D
#undef CV_FROM_D
#undef ALLD
  }
};

// The same VM without prefetched slots: for kernels whose slots come from
// shared memory (bulk.cuh k_copy_bulk_vm) a PUSH is a short LDS, and the
// prefetch registers (NPF x V words) only cost occupancy.
template <class E> struct NoPrefetch { using type = E; };
template <bool W, int D, int V, int N> struct NoPrefetch<Vm<W, D, V, N>> { using type = Vm<W, D, V, 0>; };

}  // namespace fm
