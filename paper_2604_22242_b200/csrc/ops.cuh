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
#include <cuda_bf16.h>
#include <cuda_fp16.h>

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
//   n = rint(x * 64/ln2)   (magic-constant rounding inside one DFMA; the
//                          multiplier kept to 20 bits so it is an instruction
//                          immediate -- n may differ by one at a boundary,
//                          |r| stays <= ln2/128 * (1 + 2^-13)),
//   r = x - n*ln2/64       (Cody-Waite: a 21-bit hi, so n*hi and x - n*hi are
//                          exact, and a full f64 lo), |r| <= ln2/128,
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
  const double t = fma(x, 0x1.71547p+6, kMagic);          // rint(x*64/ln2) + 1.5*2^52 (20-bit multiplier)
  const double n = __dsub_rn(t, kMagic);
  const int ni = __double2loint(t);
  double r = fma(-n, 0x1.62e43p-7, x);                     // ln2/64 hi, 21 bits (n*hi and x - n*hi exact)
  r = fma(n, 0x1.05c610ca86c39p-35, r);                    // - ln2/64 lo (hi - ln2/64)
  double q = fma(r, 0x1.11111p-7, 0x1.5555555555555p-5);   // 1/120 (20 bits: error r^5 2^-21 < 2^-60), 1/24
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
// log of an f32 argument, correctly rounded in practice: evaluated in f64
// and rounded once (like exp_f), table-driven so it costs ~12 FP64
// operations instead of libdevice log's ~30 (the paper's expr2 / expr3):
//   x = 2^e * m, m in [1, 2); j = top 7 bits of m; c_j = 1 + (j + 1/2)/128
//   r = m * (1/c_j) - 1          one FMA, |r| <= 2^-8 (1/c_j correctly rounded)
//   log x = e*ln2 + (-log(1/c_j)) + log1p(r)
// with -log(1/c_j) tabulated from the ROUNDED reciprocal, so the identity is
// exact; log1p by its degree-8 series.  Arguments within 2^-7 of 1 take
// log1p(x - 1) directly (x - 1 exact) so results near 0 keep full relative
// accuracy.
static __device__ const double kLogInvC[128] = {
    0x1.fe01fe01fe020p-1, 0x1.fa11caa01fa12p-1, 0x1.f6310aca0dbb5p-1, 0x1.f25f644230ab5p-1,
    0x1.ee9c7f8458e02p-1, 0x1.eae807aba01ebp-1, 0x1.e741aa59750e4p-1, 0x1.e3a9179dc1a73p-1,
    0x1.e01e01e01e01ep-1, 0x1.dca01dca01dcap-1, 0x1.d92f2231e7f8ap-1, 0x1.d5cac807572b2p-1,
    0x1.d272ca3fc5b1ap-1, 0x1.cf26e5c44bfc6p-1, 0x1.cbe6d9601cbe7p-1, 0x1.c8b265afb8a42p-1,
    0x1.c5894d10d4986p-1, 0x1.c26b5392ea01cp-1, 0x1.bf583ee868d8bp-1, 0x1.bc4fd65883e7bp-1,
    0x1.b951e2b18ff23p-1, 0x1.b65e2e3beee05p-1, 0x1.b37484ad806cep-1, 0x1.b094b31d922a4p-1,
    0x1.adbe87f94905ep-1, 0x1.aaf1d2f87ebfdp-1, 0x1.a82e65130e159p-1, 0x1.a574107688a4ap-1,
    0x1.a2c2a87c51ca0p-1, 0x1.a01a01a01a01ap-1, 0x1.9d79f176b682dp-1, 0x1.9ae24ea5510dap-1,
    0x1.9852f0d8ec0ffp-1, 0x1.95cbb0be377aep-1, 0x1.934c67f9b2ce6p-1, 0x1.90d4f120190d5p-1,
    0x1.8e6527af1373fp-1, 0x1.8bfce8062ff3ap-1, 0x1.899c0f601899cp-1, 0x1.87427bcc092b9p-1,
    0x1.84f00c2780614p-1, 0x1.82a4a0182a4a0p-1, 0x1.8060180601806p-1, 0x1.7e225515a4f1dp-1,
    0x1.7beb3922e017cp-1, 0x1.79baa6bb6398bp-1, 0x1.77908119ac60dp-1, 0x1.756cac201756dp-1,
    0x1.734f0c541fe8dp-1, 0x1.713786d9c7c09p-1, 0x1.6f26016f26017p-1, 0x1.6d1a62681c861p-1,
    0x1.6b1490aa31a3dp-1, 0x1.691473a88d0c0p-1, 0x1.6719f3601671ap-1, 0x1.6524f853b4aa3p-1,
    0x1.63356b88ac0dep-1, 0x1.614b36831ae94p-1, 0x1.5f66434292dfcp-1, 0x1.5d867c3ece2a5p-1,
    0x1.5babcc647fa91p-1, 0x1.59d61f123ccaap-1, 0x1.5805601580560p-1, 0x1.56397ba7c52e2p-1,
    0x1.54725e6bb82fep-1, 0x1.52aff56a8054bp-1, 0x1.50f22e111c4c5p-1, 0x1.4f38f62dd4c9bp-1,
    0x1.4d843bedc2c4cp-1, 0x1.4bd3edda68fe1p-1, 0x1.4a27fad76014ap-1, 0x1.4880522014880p-1,
    0x1.46dce34596066p-1, 0x1.453d9e2c776cap-1, 0x1.43a2730abee4dp-1, 0x1.420b5265e5951p-1,
    0x1.40782d10e6566p-1, 0x1.3ee8f42a5af07p-1, 0x1.3d5d991aa75c6p-1, 0x1.3bd60d9232955p-1,
    0x1.3a524387ac822p-1, 0x1.38d22d366088ep-1, 0x1.3755bd1c945eep-1, 0x1.35dce5f9f2af8p-1,
    0x1.34679ace01346p-1, 0x1.32f5ced6a1dfap-1, 0x1.3187758e9ebb6p-1, 0x1.301c82ac40260p-1,
    0x1.2eb4ea1fed14bp-1, 0x1.2d50a012d50a0p-1, 0x1.2bef98e5a3711p-1, 0x1.2a91c92f3c105p-1,
    0x1.293725bb804a5p-1, 0x1.27dfa38a1ce4dp-1, 0x1.268b37cd60127p-1, 0x1.2539d7e9177b2p-1,
    0x1.23eb79717605bp-1, 0x1.22a0122a0122ap-1, 0x1.21579804855e6p-1, 0x1.2012012012012p-1,
    0x1.1ecf43c7fb84cp-1, 0x1.1d8f5672e4abdp-1, 0x1.1c522fc1ce059p-1, 0x1.1b17c67f2bae3p-1,
    0x1.19e0119e0119ep-1, 0x1.18ab083902bdbp-1, 0x1.1778a191bd684p-1, 0x1.1648d50fc3201p-1,
    0x1.151b9a3fdd5c9p-1, 0x1.13f0e8d344724p-1, 0x1.12c8b89edc0acp-1, 0x1.11a3019a74826p-1,
    0x1.107fbbe011080p-1, 0x1.0f5edfab325a2p-1, 0x1.0e40655826011p-1, 0x1.0d24456359e3ap-1,
    0x1.0c0a7868b4171p-1, 0x1.0af2f722eecb5p-1, 0x1.09ddba6af8360p-1, 0x1.08cabb37565e2p-1,
    0x1.07b9f29b8eae2p-1, 0x1.06ab59c7912fbp-1, 0x1.059eea0727586p-1, 0x1.04949cc1664c5p-1,
    0x1.038c6b78247fcp-1, 0x1.02864fc7729e9p-1, 0x1.0182436517a37p-1, 0x1.0080402010080p-1,
};
static __device__ const double kLogC[128] = {
    0x1.ff00aa2b10ba0p-9, 0x1.7dc475f810a69p-7, 0x1.3cea44346a584p-6, 0x1.b9fc027af919ap-6,
    0x1.1b0d98923d97fp-5, 0x1.58a5bafc8e4d3p-5, 0x1.95c830ec8e3f2p-5, 0x1.d276b8adb0b56p-5,
    0x1.075983598e471p-4, 0x1.253f62f0a1417p-4, 0x1.42edcbea646eep-4, 0x1.60658a93750c4p-4,
    0x1.7da766d7b12d0p-4, 0x1.9ab42462033aep-4, 0x1.b78c82bb0eda0p-4, 0x1.d4313d66cb35dp-4,
    0x1.f0a30c01162a4p-4, 0x1.0671512ca596fp-3, 0x1.14785846742acp-3, 0x1.2266f190a5acdp-3,
    0x1.303d718e47fd5p-3, 0x1.3dfc2b0ecc62ap-3, 0x1.4ba36f39a55e5p-3, 0x1.59338d9982085p-3,
    0x1.66acd4272ad51p-3, 0x1.740f8f54037a3p-3, 0x1.815c0a14357e9p-3, 0x1.8e928de886d41p-3,
    0x1.9bb362e7dfb85p-3, 0x1.a8becfc882f19p-3, 0x1.b5b519e8fb5a6p-3, 0x1.c2968558c18c2p-3,
    0x1.cf6354e09c5ddp-3, 0x1.dc1bca0abec7bp-3, 0x1.e8c0252aa5a60p-3, 0x1.f550a564b7b37p-3,
    0x1.00e6c45ad501dp-2, 0x1.071b85fcd590dp-2, 0x1.0d46b579ab74bp-2, 0x1.136870293a8b0p-2,
    0x1.1980d2dd4236fp-2, 0x1.1f8ff9e48a2f3p-2, 0x1.2596010df763ap-2, 0x1.2b9303ab89d25p-2,
    0x1.31871c9544185p-2, 0x1.3772662bfd85cp-2, 0x1.3d54fa5c1f710p-2, 0x1.432ef2a04e813p-2,
    0x1.49006804009d0p-2, 0x1.4ec9732600269p-2, 0x1.548a2c3add263p-2, 0x1.5a42ab0f4cfe2p-2,
    0x1.5ff3070a793d4p-2, 0x1.659b57303e1f2p-2, 0x1.6b3bb2235943dp-2, 0x1.70d42e2789236p-2,
    0x1.7664e1239dbcfp-2, 0x1.7bede0a37afbfp-2, 0x1.816f41da0d495p-2, 0x1.86e919a330ba1p-2,
    0x1.8c5b7c858b48bp-2, 0x1.91c67eb45a83ep-2, 0x1.972a341135159p-2, 0x1.9c86b02dc0862p-2,
    0x1.a1dc064d5b995p-2, 0x1.a72a4966bd9e9p-2, 0x1.ac718c258b0e5p-2, 0x1.b1b1e0ebdfc5ap-2,
    0x1.b6eb59d3cf35cp-2, 0x1.bc1e08b0dad0ap-2, 0x1.c149ff115f027p-2, 0x1.c66f4e3ff6ff9p-2,
    0x1.cb8e0744d7acap-2, 0x1.d0a63ae721e64p-2, 0x1.d5b7f9ae2c684p-2, 0x1.dac353e2c5955p-2,
    0x1.dfc859906d5b5p-2, 0x1.e4c71a8687704p-2, 0x1.e9bfa659861f5p-2, 0x1.eeb20c640ddf3p-2,
    0x1.f39e5bc811e5dp-2, 0x1.f884a36fe9ec1p-2, 0x1.fd64f20f61571p-2, 0x1.011fab125ff8ap-1,
    0x1.0389eefce633cp-1, 0x1.05f14bd26459cp-1, 0x1.0855c884b450ep-1, 0x1.0ab76bece14d2p-1,
    0x1.0d163ccb9d6b8p-1, 0x1.0f7241c9b497dp-1, 0x1.11cb81787ccf8p-1, 0x1.1422025243d45p-1,
    0x1.1675cababa60ep-1, 0x1.18c6e0ff5cf07p-1, 0x1.1b154b57da29ep-1, 0x1.1d610fe677003p-1,
    0x1.1faa34b87094cp-1, 0x1.21f0bfc65beecp-1, 0x1.2434b6f483934p-1, 0x1.26762013430e0p-1,
    0x1.28b500df60783p-1, 0x1.2af15f02640acp-1, 0x1.2d2b4012edc9dp-1, 0x1.2f62a99509546p-1,
    0x1.3197a0fa7fe6ap-1, 0x1.33ca2ba328994p-1, 0x1.35fa4edd36ea0p-1, 0x1.38280fe58797fp-1,
    0x1.3a5373e7ebdf9p-1, 0x1.3c7c7fff73206p-1, 0x1.3ea33936b2f5bp-1, 0x1.40c7a4880dceap-1,
    0x1.42e9c6ddf80bfp-1, 0x1.4509a5133bb0ap-1, 0x1.472743f33aaadp-1, 0x1.4942a83a2fc07p-1,
    0x1.4b5bd6956e273p-1, 0x1.4d72d3a39fd01p-1, 0x1.4f87a3f5026e9p-1, 0x1.519a4c0ba3446p-1,
    0x1.53aad05b99b7cp-1, 0x1.55b9354b40bcep-1, 0x1.57c57f336f191p-1, 0x1.59cfb25fae87fp-1,
    0x1.5bd7d30e71c73p-1, 0x1.5ddde57149923p-1, 0x1.5fe1edad18919p-1, 0x1.61e3efda46467p-1,
};

__device__ __forceinline__ double log1p_series(double r) {
  double q = fma(r, -0.125, 0x1.2492492492492p-3);   // 1/7
  q = fma(q, r, -0x1.5555555555555p-3);               // -1/6
  q = fma(q, r, 0.2);
  q = fma(q, r, -0.25);
  q = fma(q, r, 0x1.5555555555555p-2);                // 1/3
  q = fma(q, r, -0.5);
  return fma(__dmul_rn(q, r), r, r);
}

__device__ __forceinline__ float log_f(float a) {
  const double x = (double)a;
  double y;
  const double d = __dsub_rn(x, 1.0);
  if (fabs(d) < 0x1p-7) {
    y = log1p_series(d);
  } else {
    const int hi = __double2hiint(x);
    const int e = (hi >> 20) - 1023;
    const int j = (hi >> 13) & 127;
    const double m = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, __double2loint(x));
    const double r = fma(m, __ldg(&kLogInvC[j]), -1.0);
    const double de = (double)e;
    y = __dadd_rn(fma(de, 0x1.62e42fee00000p-1, __ldg(&kLogC[j])), fma(de, 0x1.a39ef35793c76p-33, log1p_series(r)));
  }
  float res = __double2float_rn(y);
  if (!(a > 0.0f)) res = (a == 0.0f) ? -__int_as_float(0x7f800000) : __int_as_float(0x7fc00000);
  if (a != a) res = a;
  if (a == __int_as_float(0x7f800000)) res = a;
  return res;
}
// tanh of an f32 argument, correctly rounded in practice (f64 evaluation,
// one rounding): tanh|x| = m / (m + 2) with m = expm1(2|x|) from the same
// 64-entry exp table (2^(j/64) * (1 + p) - 1: absolute error ~2^-53,
// relative <= 2^-41 for 2|x| >= 2^-11; for n = 0, m = p itself, so tiny
// arguments keep full relative accuracy down to subnormals and tanh x
// rounds to x with no special case) and a branch-free quotient: the
// hardware's approximate f64 reciprocal of d = m + 2 in [2, 2^28), one
// Newton step (relative error ~2^-46), the quotient and one residual
// correction (~2^-53) -- 6 FP64 operations where __drcp_rn + a multiply
// took 7 plus a range check and branch.  |x| is clamped to 9.5, where the
// quotient already rounds to 1.0f.  (r01 gelu issue-bound at 66
// instructions per element, profiles/r02/ncu_gelu.)
__device__ __forceinline__ double rcp_approx_f64(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  return r;
}
__device__ __forceinline__ float tanh_f(float a) {
  const float ax = fabsf(a);
  const double y = 2.0 * (double)fminf(ax, 9.5f);
  const double kMagic = 0x1.8p52;
  const double t = fma(y, 0x1.71547p+6, kMagic);          // rint(y*64/ln2) + 1.5*2^52 (20-bit multiplier)
  const double n = __dsub_rn(t, kMagic);
  const int ni = __double2loint(t);
  double r = fma(-n, 0x1.62e43p-7, y);
  r = fma(n, 0x1.05c610ca86c39p-35, r);
  double q = fma(r, 0x1.11111p-7, 0x1.5555555555555p-5);
  q = fma(q, r, 1.0 / 6.0);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  const double p = __dmul_rn(q, r);                         // exp(r) - 1
  const double tj = __ldg(&kExp2Tab64[ni & 63]);
  const double sc = __hiloint2double(__double2hiint(tj) + (int)((unsigned)(ni >> 6) << 20), __double2loint(tj));
  const double m = fma(sc, p, __dsub_rn(sc, 1.0));          // 2^(n/64) (1 + p) - 1 >= 0
  const double d = __dadd_rn(m, 2.0);
  const double r0 = rcp_approx_f64(d);
  const double r1 = fma(r0, fma(-d, r0, 1.0), r0);          // 1/d to ~2^-46
  const double q0 = __dmul_rn(m, r1);
  const double th = fma(r1, fma(-d, q0, m), q0);            // m/d to ~2^-53
  const float res = copysignf(__double2float_rn(th), a);
  return (a != a) ? a : res;
}
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

// f32 -> three bf16 planes with x = hi + mid + lo + O(2^-24 |x|): each
// residual is exact in f32 (Sterbenz), each plane the round-to-nearest bf16
// of the residual (the f32 GEMM's operand planes, gemm_tc.cu).
__device__ __forceinline__ void split3(float x, uint16_t &h, uint16_t &m, uint16_t &l) {
  const __nv_bfloat16 hi = __float2bfloat16_rn(x);
  const float r1 = __fsub_rn(x, __bfloat162float(hi));
  const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
  const float r2 = __fsub_rn(r1, __bfloat162float(mid));
  h = __bfloat16_as_ushort(hi);
  m = __bfloat16_as_ushort(mid);
  l = __bfloat16_as_ushort(__float2bfloat16_rn(r2));
}

// The f32 GEMM's fp16 operand planes (gemm_tc.cu): an operand is scaled by
// 2^e with max|x| * 2^e in [2^14, 2^15) -- fp16 keeps 11 significant bits
// over ~30 binades; the scale keeps the hi plane far from overflow and the lo
// plane mostly normal -- then x * 2^e = hi + lo + O(2^-22 |x * 2^e|) with
// hi = fp16(x * 2^e), lo = fp16(x * 2^e - hi) (the residual is exact in f32).
__host__ __device__ inline int f16_scale_exp(unsigned amax_bits) {
  const int be = (int)((amax_bits >> 23) & 0xff);
  if (be == 0 || be == 0xff) return 0;   // zero / subnormal max, or a non-finite input: unscaled
  return 14 - (be - 127);
}
__device__ __forceinline__ void split2h(float x, float sc, uint16_t &h, uint16_t &l) {
  const float y = __fmul_rn(x, sc);
  const __half hi = __float2half_rn(y);
  h = __half_as_ushort(hi);
  l = __half_as_ushort(__float2half_rn(__fsub_rn(y, __half2float(hi))));
}

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
