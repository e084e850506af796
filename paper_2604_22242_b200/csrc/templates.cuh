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
FM_DEV float texp(float a, const double *tab) { return exp_f(a, tab); }
FM_DEV double texp(double a, const double *) { return exp_d(a); }
FM_DEV float tlog(float a) { return log_f(a); }
FM_DEV double tlog(double a) { return log_d(a); }
FM_DEV float tsqrt(float a) { return sqrt_f(a); }
FM_DEV double tsqrt(double a) { return sqrt_d(a); }
FM_DEV float ttanh(float a) { return tanh_f(a); }
FM_DEV double ttanh(double a) { return tanh_d(a); }

template <class T> FM_DEV T scal(uint64_t b);
template <> FM_DEV float scal<float>(uint64_t b) { return u2f((uint32_t)b); }
template <> FM_DEV double scal<double>(uint64_t b) { return __longlong_as_double((long long)b); }

#define FM_EV template <class T> FM_DEV static T ev(const T *x, const uint64_t *s, const double *tab)

template <int I> struct In { FM_EV { return x[I]; } };
template <class A, class B> struct Add { FM_EV { return tadd(A::ev(x, s, tab), B::ev(x, s, tab)); } };
template <class A, class B> struct Sub { FM_EV { return tsub(A::ev(x, s, tab), B::ev(x, s, tab)); } };
template <class A, class B> struct Mul { FM_EV { return tmul(A::ev(x, s, tab), B::ev(x, s, tab)); } };
template <class A, class B> struct Div { FM_EV { return tdiv(A::ev(x, s, tab), B::ev(x, s, tab)); } };
template <int S, class A> struct SAdd { FM_EV { return tadd(A::ev(x, s, tab), scal<T>(s[S])); } };
template <int S, class A> struct SMul { FM_EV { return tmul(scal<T>(s[S]), A::ev(x, s, tab)); } };
template <int S, class A> struct SDiv { FM_EV { return tdiv(scal<T>(s[S]), A::ev(x, s, tab)); } };
template <int S, class A> struct Gts { FM_EV { return tgt(A::ev(x, s, tab), scal<T>(s[S])); } };
template <class A> struct Neg { FM_EV { return tneg(A::ev(x, s, tab)); } };
template <class A> struct Abs { FM_EV { return tabs(A::ev(x, s, tab)); } };
template <class A> struct Exp { FM_EV { return texp(A::ev(x, s, tab), tab); } };
template <class A> struct Log { FM_EV { return tlog(A::ev(x, s, tab)); } };
template <class A> struct Sqrt { FM_EV { return tsqrt(A::ev(x, s, tab)); } };
template <class A> struct Tanh { FM_EV { return ttanh(A::ev(x, s, tab)); } };
template <int K, class A> struct Pow {
  FM_EV {
    const T a = A::ev(x, s, tab);
    if (K == 0) return T(1);
    T acc = a;
#pragma unroll
    for (int i = 1; i < K; ++i) acc = tmul(acc, a);
    return acc;
  }
};
#undef FM_EV

// Evaluator over a flat chunk: all NIN inputs share type T (f32 or f64).
template <class Expr, class T, int NIN, int V>
struct TEval {
  static constexpr int kV = V;
  FM_DEV static void eval(const fm_program &P, const Chunk &ch, uint32_t (&lo)[V], uint32_t (&hi)[V]) {
    uint32_t xl[NIN][V], xh[NIN][V];
#pragma unroll
    for (int i = 0; i < NIN; ++i) load_slot<V>(P.slots[i], ch, xl[i], xh[i]);
    const double *tab = kExp2Table;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      T xv[NIN];
#pragma unroll
      for (int i = 0; i < NIN; ++i) {
        if constexpr (sizeof(T) == 8) xv[i] = u2d(xl[i][v], xh[i][v]);
        else xv[i] = u2f(xl[i][v]);
      }
      const T r = Expr::template ev<T>(xv, P.scalars, tab);
      if constexpr (sizeof(T) == 8) d2u(r, lo[v], hi[v]);
      else { lo[v] = f2u(r); hi[v] = 0u; }
    }
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
