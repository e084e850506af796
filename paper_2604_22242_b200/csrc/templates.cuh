// templates.cuh -- expression templates (the paper's eOp/eGlue types) for the
// ahead-of-time kernels.  A registered signature becomes a C++ type such as
//   Add<SMul<0, Mul<In<0>, In<1>>>, In<0>>        (C1: 2*(X%Y)+X)
// whose ev() inlines the whole element expression, so nvcc schedules the
// loads of all inputs together and the chain runs as straight-line code.
// Numerics come from ops.cuh, identical to the VM's.
#pragma once
#include "launch.cuh"

namespace fm {
namespace tx {

FM_DEV float tadd(float a, float b) { return add_f(a, b); }
FM_DEV double tadd(double a, double b) { return add_d(a, b); }
FM_DEV float tsub(float a, float b) { return sub_f(a, b); }
FM_DEV double tsub(double a, double b) { return sub_d(a, b); }
FM_DEV float tmul(float a, float b) { return mul_f(a, b); }
FM_DEV double tmul(double a, double b) { return mul_d(a, b); }
FM_DEV float tdiv(float a, float b) { return div_f(a, b); }
FM_DEV double tdiv(double a, double b) { return div_d(a, b); }
FM_DEV float tneg(float a) { return neg_f(a); }
FM_DEV double tneg(double a) { return neg_d(a); }
FM_DEV float tabs(float a) { return abs_f(a); }
FM_DEV double tabs(double a) { return abs_d(a); }
FM_DEV float tgt(float a, float s) { return gts_f(a, s); }
FM_DEV double tgt(double a, double s) { return gts_d(a, s); }
FM_DEV float texp(float a) { return exp_f(a); }
FM_DEV double texp(double a) { return exp_d(a); }
FM_DEV float tlog(float a) { return log_f(a); }
FM_DEV double tlog(double a) { return log_d(a); }
FM_DEV float tsqrt(float a) { return sqrt_f(a); }
FM_DEV double tsqrt(double a) { return sqrt_d(a); }
FM_DEV float ttanh(float a) { return tanh_f(a); }
FM_DEV double ttanh(double a) { return tanh_d(a); }

template <class T> FM_DEV T scal(uint64_t b);
template <> FM_DEV float scal<float>(uint64_t b) { return u2f((uint32_t)b); }
template <> FM_DEV double scal<double>(uint64_t b) { return __longlong_as_double((long long)b); }

#define FM_EV template <class T> FM_DEV static T ev(const T *x, const uint64_t *s)

template <int I> struct In { FM_EV { return x[I]; } };
template <class A, class B> struct Add { FM_EV { return tadd(A::ev(x, s), B::ev(x, s)); } };
template <class A, class B> struct Sub { FM_EV { return tsub(A::ev(x, s), B::ev(x, s)); } };
template <class A, class B> struct Mul { FM_EV { return tmul(A::ev(x, s), B::ev(x, s)); } };
template <class A, class B> struct Div { FM_EV { return tdiv(A::ev(x, s), B::ev(x, s)); } };
template <int S, class A> struct SAdd { FM_EV { return tadd(A::ev(x, s), scal<T>(s[S])); } };
template <int S, class A> struct SMul { FM_EV { return tmul(scal<T>(s[S]), A::ev(x, s)); } };
template <int S, class A> struct SDiv { FM_EV { return tdiv(scal<T>(s[S]), A::ev(x, s)); } };
template <int S, class A> struct Gts { FM_EV { return tgt(A::ev(x, s), scal<T>(s[S])); } };
// conversion of an integer leaf (slot I holds u32 / i32 bits) to T, as the
// reference's C cast (codegen.py:217-218): round to nearest
template <class T> FM_DEV uint32_t leaf_bits(T v);
template <> FM_DEV uint32_t leaf_bits<float>(float v) { return __float_as_uint(v); }
template <> FM_DEV uint32_t leaf_bits<double>(double v) { return (uint32_t)__double2loint(v); }
template <int I> struct CvtU32 { FM_EV { return (T)leaf_bits<T>(x[I]); } };
template <int I> struct CvtI32 { FM_EV { return (T)(int32_t)leaf_bits<T>(x[I]); } };
template <class A> struct Neg { FM_EV { return tneg(A::ev(x, s)); } };
template <class A> struct Abs { FM_EV { return tabs(A::ev(x, s)); } };
template <class A> struct Exp { FM_EV { return texp(A::ev(x, s)); } };
template <class A> struct Log { FM_EV { return tlog(A::ev(x, s)); } };
template <class A> struct Sqrt { FM_EV { return tsqrt(A::ev(x, s)); } };
template <class A> struct Tanh { FM_EV { return ttanh(A::ev(x, s)); } };
template <int K, class A> struct Pow {
  FM_EV {
    const T a = A::ev(x, s);
    if (K == 0) return T(1);
    T acc = a;
#pragma unroll
    for (int i = 1; i < K; ++i) acc = tmul(acc, a);
    return acc;
  }
};
#undef FM_EV

// Heavy<Expr>::v -- the chain contains a transcendental: its per-element math
// is long enough that the copy skeleton should stage inputs through shared
// memory with TMA bulk copies (bulk.cuh) instead of register tiles.
template <class X> struct Heavy { static constexpr bool v = false; };
template <class A> struct Heavy<Exp<A>> { static constexpr bool v = true; };
template <class A> struct Heavy<Log<A>> { static constexpr bool v = true; };
template <class A> struct Heavy<Tanh<A>> { static constexpr bool v = true; };
template <class A> struct Heavy<Neg<A>> { static constexpr bool v = Heavy<A>::v; };
template <class A> struct Heavy<Abs<A>> { static constexpr bool v = Heavy<A>::v; };
template <class A> struct Heavy<Sqrt<A>> { static constexpr bool v = Heavy<A>::v; };
template <int K, class A> struct Heavy<Pow<K, A>> { static constexpr bool v = Heavy<A>::v; };
template <int S, class A> struct Heavy<SAdd<S, A>> { static constexpr bool v = Heavy<A>::v; };
template <int S, class A> struct Heavy<SMul<S, A>> { static constexpr bool v = Heavy<A>::v; };
template <int S, class A> struct Heavy<SDiv<S, A>> { static constexpr bool v = Heavy<A>::v; };
template <int S, class A> struct Heavy<Gts<S, A>> { static constexpr bool v = Heavy<A>::v; };
template <class A, class B> struct Heavy<Add<A, B>> { static constexpr bool v = Heavy<A>::v || Heavy<B>::v; };
template <class A, class B> struct Heavy<Sub<A, B>> { static constexpr bool v = Heavy<A>::v || Heavy<B>::v; };
template <class A, class B> struct Heavy<Mul<A, B>> { static constexpr bool v = Heavy<A>::v || Heavy<B>::v; };
template <class A, class B> struct Heavy<Div<A, B>> { static constexpr bool v = Heavy<A>::v || Heavy<B>::v; };

// RegTiles<Expr>::v -- stream on register tiles even beyond L2: a chain with
// an elementwise division needs the register path's 32-40 resident warps to
// hide it.  Measured at 10000^2 f32 (bench.py --config suite): swish 4.25
// (tiles) vs 4.04 TB/s (bulk, 24 consumer warps for transcendental chains),
// while gelu (tanh) 3.83 vs 4.04, sigmoid (scalar division) and C3 favour
// bulk.  (With 16 bulk consumer warps tanh chains were faster on tiles too.)
template <class X> struct RegTiles { static constexpr bool v = false; };
template <class A> struct RegTiles<Tanh<A>> { static constexpr bool v = RegTiles<A>::v; };
template <class A, class B> struct RegTiles<Div<A, B>> { static constexpr bool v = true; };
template <class A> struct RegTiles<Exp<A>> { static constexpr bool v = RegTiles<A>::v; };
template <class A> struct RegTiles<Log<A>> { static constexpr bool v = RegTiles<A>::v; };
template <class A> struct RegTiles<Neg<A>> { static constexpr bool v = RegTiles<A>::v; };
template <class A> struct RegTiles<Abs<A>> { static constexpr bool v = RegTiles<A>::v; };
template <class A> struct RegTiles<Sqrt<A>> { static constexpr bool v = RegTiles<A>::v; };
template <int K, class A> struct RegTiles<Pow<K, A>> { static constexpr bool v = RegTiles<A>::v; };
template <int S, class A> struct RegTiles<SAdd<S, A>> { static constexpr bool v = RegTiles<A>::v; };
template <int S, class A> struct RegTiles<SMul<S, A>> { static constexpr bool v = RegTiles<A>::v; };
template <int S, class A> struct RegTiles<SDiv<S, A>> { static constexpr bool v = RegTiles<A>::v; };
template <int S, class A> struct RegTiles<Gts<S, A>> { static constexpr bool v = RegTiles<A>::v; };
template <class A, class B> struct RegTiles<Add<A, B>> { static constexpr bool v = RegTiles<A>::v || RegTiles<B>::v; };
template <class A, class B> struct RegTiles<Sub<A, B>> { static constexpr bool v = RegTiles<A>::v || RegTiles<B>::v; };
template <class A, class B> struct RegTiles<Mul<A, B>> { static constexpr bool v = RegTiles<A>::v || RegTiles<B>::v; };

// Evaluator over a chunk: all NIN inputs share type T (f32 or f64), and so
// does the result.  eval() is the general path (any index map, ragged
// chunks); the *_tile members serve the steady state of a flat program whose
// buffers are all 16-byte aligned: typed 128-bit loads and stores with no
// per-element type dispatch or bounds checks.
template <class Expr, class T, int NIN, int V, bool TILED = false>
struct TEval {
  // TILED: the signature has transposed / view leaves, so copies run on the
  // tiled staged skeleton (instantiated only for those templates)
  static constexpr bool kTiled = TILED;
  using Elem = T;
  static constexpr int kV = V;
  static constexpr int kNin = NIN;
  // warp-tile fast path (a second tile of every input in flight) up to 8
  // inputs; wider chains (add-N) load all inputs of a chunk at once instead
  static constexpr bool kFast = NIN <= 8;
  // the wide add-N chains (9..32 inputs) take the copy skeleton's warp tiles
  // too, one tile per warp at a time (NIN x V words per lane already keep
  // 128-512 B per lane in flight); before, they ran the general chunk path at
  // ~200 instructions per element (profiles: add32N issue 24 %, LDL/STL)
  static constexpr bool kWideTile = NIN > 8 && NIN <= 32;
  static constexpr bool kIsVm = false;
  // the widest chains (add-N, N > 16) hold NIN x V loaded words per thread:
  // ask for two resident blocks so they keep 16 warps per SM
  static constexpr int kMinBlocks = 1;
  static constexpr bool kWide = sizeof(T) == 8;
  static constexpr bool kHeavy = Heavy<Expr>::v;
  static constexpr bool kRegTiles = RegTiles<Expr>::v;

  FM_DEV static T ev_elem(const fm_program &P, const T (&x)[NIN]) {
    return Expr::template ev<T>(x, P.scalars);
  }
  static constexpr int kEtype = sizeof(T) == 8 ? FM_F64 : FM_F32;
  static_assert(V * sizeof(T) % 16 == 0, "tiles move whole 16-byte vectors");

  FM_DEV static void eval(const fm_program &P, const Chunk &ch, uint32_t (&lo)[V], uint32_t (&hi)[V]) {
    uint32_t xl[NIN][V], xh[NIN][V];
#pragma unroll
    for (int i = 0; i < NIN; ++i) fetch_slot<V, !TILED>(P, i, ch, xl[i], xh[i]);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      T xv[NIN];
#pragma unroll
      for (int i = 0; i < NIN; ++i) {
        if constexpr (sizeof(T) == 8) xv[i] = u2d(xl[i][v], xh[i][v]);
        else xv[i] = u2f(xl[i][v]);
      }
      const T r = Expr::template ev<T>(xv, P.scalars);
      if constexpr (sizeof(T) == 8) d2u(r, lo[v], hi[v]);
      else { lo[v] = f2u(r); hi[v] = 0u; }
    }
  }

  // uniform per launch: may the tile members run?
  // a slot the tile paths can move as T-sized words: T itself, or (f32
  // templates) the u32 / i32 leaf of a CvtU32 / CvtI32 node
  FM_DEV static constexpr bool slot_ok(int et) {
    return et == kEtype || (sizeof(T) == 4 && (et == FM_U32 || et == FM_I32));
  }
  FM_DEV static bool fast_ok(const fm_program &P, const void *out) {
    if (!P.flat || P.result_etype != kEtype || (((uintptr_t)out) & 15)) return false;
#pragma unroll
    for (int i = 0; i < NIN; ++i)
      if ((((uintptr_t)P.slots[i].ptr) & 15) || !slot_ok(P.slots[i].etype)) return false;
    return true;
  }

  // ---- warp tiles: 32 lanes x V elements, every vector access one fully
  // coalesced 512-byte warp transaction.  Lane l owns, for q < V/W, the W
  // elements at tile_base + q*32*W + l*W.  The skeletons keep one tile in
  // flight (load t+1, then compute t) so HBM requests never wait on math.
  static constexpr int kW = 16 / sizeof(T);   // elements per 128-bit vector
  static constexpr int kTile = 32 * V;
  struct Buf {
    uint4 w[NIN][V / kW];
  };

  FM_DEV static void load_tile(const fm_program &P, int64_t base, int lane, Buf &b) {
#pragma unroll
    for (int i = 0; i < NIN; ++i) {
      const T *p = (const T *)P.slots[i].ptr + base + lane * kW;
#pragma unroll
      for (int q = 0; q < V / kW; ++q) b.w[i][q] = ldg_v4(p + q * 32 * kW);
    }
  }

  FM_DEV static void eval_tile(const fm_program &P, const Buf &b, T (&r)[V]) {
#pragma unroll
    for (int q = 0; q < V / kW; ++q) {
#pragma unroll
      for (int e = 0; e < kW; ++e) {
        T x[NIN];
#pragma unroll
        for (int i = 0; i < NIN; ++i) {
          const uint4 &w = b.w[i][q];
          if constexpr (sizeof(T) == 8) x[i] = e == 0 ? u2d(w.x, w.y) : u2d(w.z, w.w);
          else x[i] = u2f(e == 0 ? w.x : e == 1 ? w.y : e == 2 ? w.z : w.w);
        }
        r[q * kW + e] = Expr::template ev<T>(x, P.scalars);
      }
    }
  }

  FM_DEV static void copy_tile(const fm_program &P, void *out, int64_t base, int lane, const Buf &b) {
    T r[V];
    eval_tile(P, b, r);
    T *o = (T *)out + base + lane * kW;
#pragma unroll
    for (int q = 0; q < V / kW; ++q) {
      if constexpr (sizeof(T) == 8) {
        uint32_t a0, a1, b0, b1;
        d2u(r[q * 2], a0, a1);
        d2u(r[q * 2 + 1], b0, b1);
        st_v4(o + q * 32 * kW, a0, a1, b0, b1);
      } else {
        st_v4(o + q * 32 * kW, f2u(r[q * 4]), f2u(r[q * 4 + 1]), f2u(r[q * 4 + 2]), f2u(r[q * 4 + 3]));
      }
    }
  }

  // add the lane's V results to the f64 accumulator (the reduce_accu
  // accumulator type, codegen.py:47-49)
  FM_DEV static void accu_tile(const fm_program &P, const Buf &b, double &acc) {
    T r[V];
    eval_tile(P, b, r);
#pragma unroll
    for (int v = 0; v < V; ++v) acc = add_d(acc, (double)r[v]);
  }
};

template <class E> int t_copy(const fm_program &P, void *o, int64_t r, int64_t c, cudaStream_t s) {
  return run_copy<E>(P, o, r, c, s);
}
template <class E> int t_accu(const fm_program &P, void *o, int64_t r, int64_t c, int f, cudaStream_t s) {
  return run_accu<E>(P, o, r, c, f, s);
}
template <class E>
int t_dim(const fm_program &P, int d, int64_t r, int64_t c, const ReduceOuts &R, cudaStream_t s) {
  return run_reduce_dim<E>(P, d, r, c, R, s);
}

}  // namespace tx
}  // namespace fm
