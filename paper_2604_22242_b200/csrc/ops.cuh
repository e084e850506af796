// ops.cuh -- per-node numerics of the fused path, shared by the register VM
// and the ahead-of-time template kernels so both round identically.
//
// Contract (reference /root/reference/pkg/src/fusemat/codegen.py:149-227 and
// backend.py:115-168):
//   * every node rounds to its element type; explicit _rn intrinsics stop
//     nvcc from contracting a*b+c into an FMA (the reference's cjit build has
//     no -mfma, so it never fuses either);
//   * integer arithmetic wraps mod 2^32 (-fwrapv, cjit.py:102);
//   * float -> integer truncates through int64 with x86 "integer indefinite"
//     (INT64_MIN) for NaN / out-of-range, then keeps the low 32 bits
//     (codegen.py:164-169, oracle.py:89-92);
//   * f32 exp/log/tanh are evaluated in f64 and rounded once, so they are
//     correctly rounded in practice (policy in DESIGN.md: the oracle's own
//     numpy/glibc f32 transcendentals are not).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fm {

__device__ __forceinline__ float u2f(uint32_t u) { return __uint_as_float(u); }
__device__ __forceinline__ uint32_t f2u(float f) { return __float_as_uint(f); }
__device__ __forceinline__ double u2d(uint32_t lo, uint32_t hi) {
  return __hiloint2double((int)hi, (int)lo);
}
__device__ __forceinline__ void d2u(double d, uint32_t &lo, uint32_t &hi) {
  lo = (uint32_t)__double2loint(d);
  hi = (uint32_t)__double2hiint(d);
}

// ---- f32 --------------------------------------------------------------------
__device__ __forceinline__ float add_f(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_f(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul_f(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float div_f(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float neg_f(float a) { return __uint_as_float(__float_as_uint(a) ^ 0x80000000u); }
__device__ __forceinline__ float abs_f(float a) { return __uint_as_float(__float_as_uint(a) & 0x7fffffffu); }
__device__ __forceinline__ float gts_f(float a, float s) { return a > s ? 1.0f : 0.0f; }
__device__ __forceinline__ float sqrt_f(float a) { return __fsqrt_rn(a); }

// ---- f64 --------------------------------------------------------------------
__device__ __forceinline__ double add_d(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_d(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_d(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double div_d(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double neg_d(double a) {
  return __longlong_as_double(__double_as_longlong(a) ^ (long long)0x8000000000000000ull);
}
__device__ __forceinline__ double abs_d(double a) {
  return __longlong_as_double(__double_as_longlong(a) & 0x7fffffffffffffffll);
}
__device__ __forceinline__ double gts_d(double a, double s) { return a > s ? 1.0 : 0.0; }
__device__ __forceinline__ double sqrt_d(double a) { return __dsqrt_rn(a); }

// exp of an f32 argument, correctly rounded in practice: evaluated in f64
// (relative error ~2^-52) and rounded once to f32.  Branch-free and
// table-free so a fused chain stays memory-bound (C3 is one exp per element):
//   k = rint(x / ln2)  (magic-constant rounding inside one DFMA),
//   r = x - k*ln2      (Cody-Waite hi/lo, exact hi product), |r| <= ln2/2,
//   exp(r)             degree-11 Chebyshev fit (approximation error 2^-58),
//   2^k                added to the exponent field (k in [-150, 129]: the
//                      f64 result stays normal; f32 overflow/underflow and
//                      subnormal rounding happen in the final conversion).
// Arguments are clamped to [-104, 89]: exp(-104) < 2^-150 rounds to +0 and
// exp(89) > FLT_MAX rounds to +inf, exactly as the unclamped values would.
__device__ __forceinline__ double exp_poly_d(double r) {
  double p = 0x1.af632a0f7e2cep-26;
  p = fma(p, r, 0x1.28b4101c77212p-22);
  p = fma(p, r, 0x1.71ddf56d8deb5p-19);
  p = fma(p, r, 0x1.a01991a10d9aep-16);
  p = fma(p, r, 0x1.a01a01b1461c5p-13);
  p = fma(p, r, 0x1.6c16c1880029fp-10);
  p = fma(p, r, 0x1.111111110f21ep-7);
  p = fma(p, r, 0x1.555555554f0bap-5);
  p = fma(p, r, 0x1.555555555555ap-3);
  p = fma(p, r, 0x1.0000000000011p-1);
  p = fma(p, r, 1.0);
  return fma(p, r, 1.0);
}

__device__ __forceinline__ float exp_f(float a) {
  const float c = fminf(fmaxf(a, -104.0f), 89.0f);
  const double x = (double)c;
  const double kMagic = 0x1.8p52;
  const double t = fma(x, 0x1.71547652b82fep0, kMagic);   // rint(x/ln2) + 1.5*2^52
  const double k = __dsub_rn(t, kMagic);
  const int ki = __double2loint(t);
  double r = fma(-k, 0x1.62e42fee00000p-1, x);              // ln2 hi (exact k*hi)
  r = fma(-k, 0x1.a39ef35793c76p-33, r);                    // ln2 lo
  const double p = exp_poly_d(r);
  const double y = __hiloint2double(__double2hiint(p) + (int)((unsigned)ki << 20), __double2loint(p));
  const float res = __double2float_rn(y);
  return (a != a) ? a : res;
}
__device__ __forceinline__ float log_f(float a) { return __double2float_rn(log((double)a)); }
__device__ __forceinline__ float tanh_f(float a) { return __double2float_rn(tanh((double)a)); }
__device__ __forceinline__ double exp_d(double a) { return exp(a); }
__device__ __forceinline__ double log_d(double a) { return log(a); }
__device__ __forceinline__ double tanh_d(double a) { return tanh(a); }

// ---- 32-bit integers (u32 and i32 share wrapping bit arithmetic) ------------
__device__ __forceinline__ uint32_t add_i(uint32_t a, uint32_t b) { return a + b; }
__device__ __forceinline__ uint32_t sub_i(uint32_t a, uint32_t b) { return a - b; }
__device__ __forceinline__ uint32_t mul_i(uint32_t a, uint32_t b) { return a * b; }
__device__ __forceinline__ uint32_t neg_i(uint32_t a) { return 0u - a; }
__device__ __forceinline__ uint32_t abs_i32(uint32_t a) {
  return ((int32_t)a < 0) ? 0u - a : a;
}
__device__ __forceinline__ uint32_t gts_i32(uint32_t a, uint32_t s) { return (int32_t)a > (int32_t)s ? 1u : 0u; }
__device__ __forceinline__ uint32_t gts_u32(uint32_t a, uint32_t s) { return a > s ? 1u : 0u; }

// ---- conversions ---------------------------------------------------------------
// x86 cvttsd2si semantics: NaN or |x| >= 2^63 -> INT64_MIN; then wrap to 32 bits.
__device__ __forceinline__ uint32_t d_to_i32bits(double x) {
  long long v;
  if (!(x == x) || x >= 9223372036854775808.0 || x < -9223372036854775808.0)
    v = (long long)0x8000000000000000ull;
  else
    v = __double2ll_rz(x);
  return (uint32_t)(unsigned long long)v;
}
__device__ __forceinline__ uint32_t f_to_i32bits(float x) { return d_to_i32bits((double)x); }
__device__ __forceinline__ float i32_to_f(uint32_t a) { return __int2float_rn((int)a); }
__device__ __forceinline__ float u32_to_f(uint32_t a) { return __uint2float_rn(a); }
__device__ __forceinline__ double i32_to_d(uint32_t a) { return (double)(int)a; }
__device__ __forceinline__ double u32_to_d(uint32_t a) { return (double)a; }
__device__ __forceinline__ float d_to_f(double a) { return __double2float_rn(a); }

// round an f32 to the nearest-even bf16 value (kept in an f32 container)
__device__ __forceinline__ float rnd_bf_f(float a) {
  uint32_t u = __float_as_uint(a);
  if ((u & 0x7fffffffu) > 0x7f800000u) return __uint_as_float((u | 0x00400000u) & 0xffff0000u);
  u = u + 0x7fffu + ((u >> 16) & 1u);
  return __uint_as_float(u & 0xffff0000u);
}
// f64 -> bf16 with a single rounding (round-to-odd to f32 first keeps it exact)
__device__ __forceinline__ float d_to_bf(double a) {
  if (!(a == a)) return __uint_as_float(0x7fc00000u);
  float lo = __double2float_rz(a);
  uint32_t u = __float_as_uint(lo);
  if ((double)lo != a && (u & 0x7f800000u) != 0x7f800000u) u |= 1u;   // sticky bit (round to odd)
  return rnd_bf_f(__uint_as_float(u));
}
__device__ __forceinline__ float bf16_bits_to_f(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }
__device__ __forceinline__ uint16_t f_to_bf16_bits(float a) { return (uint16_t)(__float_as_uint(rnd_bf_f(a)) >> 16); }

// ---- pow: left-associated repeated product (codegen.py:211-216) ------------------
__device__ __forceinline__ float pow_f(float x, int k) {
  float acc = x;
  for (int i = 1; i < k; ++i) acc = mul_f(acc, x);
  return acc;
}
__device__ __forceinline__ double pow_d(double x, int k) {
  double acc = x;
  for (int i = 1; i < k; ++i) acc = mul_d(acc, x);
  return acc;
}
__device__ __forceinline__ uint32_t pow_i(uint32_t x, int k) {
  uint32_t acc = x;
  for (int i = 1; i < k; ++i) acc = acc * x;
  return acc;
}

}  // namespace fm
