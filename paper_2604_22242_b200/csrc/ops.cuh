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
// (relative error ~2^-52) and rounded once to f32.  Branch-free, so a fused
// chain stays memory-bound (C3 is one exp per element), and short: 10 FP64
// operations per element (the previous table-free degree-11 form took 16 and
// kept C3 issue-bound, profiles/r01/ncu_c3_copy.txt):
//   n = rint(x * 64/ln2)   (magic-constant rounding inside one DFMA),
//   r = x - n*ln2/64       (Cody-Waite hi/lo, exact hi product), |r| <= ln2/128,
//   exp(r) - 1             degree-5 Taylor polynomial (truncation 2^-54.6),
//   2^(j/64)               64-entry table of correctly rounded f64 values
//                          (j = n mod 64; read through L1, 512 bytes),
//   2^(n div 64)           added to the exponent field (in [-150, 129]: the
//                          f64 result stays normal; f32 overflow/underflow and
//                          subnormal rounding happen in the final conversion).
// Arguments are clamped to [-104, 89]: exp(-104) < 2^-150 rounds to +0 and
// exp(89) > FLT_MAX rounds to +inf, exactly as the unclamped values would.
static __device__ const double kExp2Tab64[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0,
};

__device__ __forceinline__ float exp_f(float a) {
  const float c = fminf(fmaxf(a, -104.0f), 89.0f);
  const double x = (double)c;
  const double kMagic = 0x1.8p52;
  const double t = fma(x, 0x1.71547652b82fep+6, kMagic);   // rint(x*64/ln2) + 1.5*2^52
  const double n = __dsub_rn(t, kMagic);
  const int ni = __double2loint(t);
  double r = fma(-n, 0x1.62e42fee00000p-7, x);             // ln2/64 hi (exact n*hi)
  r = fma(-n, 0x1.a39ef35793c76p-39, r);                   // ln2/64 lo
  double q = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  q = fma(q, r, 1.0 / 6.0);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  const double p = __dmul_rn(q, r);                         // exp(r) - 1
  const double tj = __ldg(&kExp2Tab64[ni & 63]);
  const double y0 = fma(tj, p, tj);                         // 2^(j/64) * exp(r)
  const double y = __hiloint2double(__double2hiint(y0) + (int)((unsigned)(ni >> 6) << 20), __double2loint(y0));
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
