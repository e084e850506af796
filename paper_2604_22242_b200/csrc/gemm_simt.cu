// gemm_simt.cu -- exact GEMM: f64 accumulation in the reference's order.
//
// Reference numerics (/root/reference/pkg/src/fusemat/cjit.py:33-51): each
// output c[i + j*m] = (T) sum_{p=0..k-1} (double)a(i,p) * (double)b(p,j),
// summed sequentially in p.  This kernel keeps that per-element order (the
// k loop is sequential per output), so for f32/bf16 inputs -- whose products
// are exact in f64 -- it is bit-identical to the reference cjit GEMM.  It
// also serves f64 GEMMs.  alpha and operand transposes are folded in.
// The tensor-core path (gemm_tc.cu) is the fast path; this one is the
// FM_GEMM_EXACT mode and the f64 path.
#include "common.cuh"
#include "ops.cuh"

namespace fm {

constexpr int TM = 64, TN = 64, TK = 16;

__device__ __forceinline__ double load_elem(const void *p, int etype, int64_t idx) {
  switch (etype) {
    case FM_F64: return ((const double *)p)[idx];
    case FM_BF16: return (double)bf16_bits_to_f(((const uint16_t *)p)[idx]);
    default: return (double)((const float *)p)[idx];
  }
}

__global__ void __launch_bounds__(256) k_gemm_exact(fm_gemm_args g) {
  __shared__ double As[TK][TM + 1];
  __shared__ double Bs[TK][TN + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t i0 = (int64_t)blockIdx.x * TM, j0 = (int64_t)blockIdx.y * TN;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t p0 = 0; p0 < g.k; p0 += TK) {
    for (int t = threadIdx.x; t < TK * TM; t += 256) {
      const int pp = t / TM, ii = t % TM;
      const int64_t i = i0 + ii, p = p0 + pp;
      double v = 0.0;
      if (i < g.m && p < g.k) v = load_elem(g.a, g.in_etype, g.trans_a ? p + i * g.lda : i + p * g.lda);
      As[pp][ii] = v;
    }
    for (int t = threadIdx.x; t < TK * TN; t += 256) {
      const int jj = t / TK, pp = t % TK;
      const int64_t j = j0 + jj, p = p0 + pp;
      double v = 0.0;
      if (j < g.n && p < g.k) v = load_elem(g.b, g.in_etype, g.trans_b ? j + p * g.ldb : p + j * g.ldb);
      Bs[pp][jj] = v;
    }
    __syncthreads();
    const int pmax = (int)min((int64_t)TK, g.k - p0);
    for (int pp = 0; pp < pmax; ++pp) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[pp][tx + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[pp][ty + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(av[a], bv[b]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t i = i0 + tx + 16 * a, j = j0 + ty + 16 * b;
      if (i < g.m && j < g.n) {
        double v = acc[a][b];
        if (g.alpha != 1.0) v = __dmul_rn(g.alpha, v);
        if (g.out_etype == FM_F64) {
          if (g.c_in) v = __dadd_rn(__dmul_rn(g.alpha2, v), __dmul_rn(g.beta, ((const double *)g.c_in)[i + j * g.ld_c_in]));
          ((double *)g.c)[i + j * g.ldc] = v;
        } else {
          float t = __double2float_rn(v);
          if (g.c_in)
            t = __fadd_rn(__fmul_rn((float)g.alpha2, t), __fmul_rn((float)g.beta, ((const float *)g.c_in)[i + j * g.ld_c_in]));
          ((float *)g.c)[i + j * g.ldc] = t;
        }
      }
    }
}

int gemm_exact(const fm_gemm_args &g, cudaStream_t s) {
  dim3 grid((unsigned)((g.m + TM - 1) / TM), (unsigned)((g.n + TN - 1) / TN));
  if (grid.y > 65535) return fail_msg("gemm: n too large for the exact kernel");
  k_gemm_exact<<<grid, 256, 0, s>>>(g);
  FM_CHECK_LAUNCH("exact gemm kernel");
  return 0;
}

// defined in gemm_tc.cu
int gemm_tensor(const fm_gemm_args &g, cudaStream_t s, bool *handled, const fm_program *a_prog = nullptr,
                const fm_program *b_prog = nullptr);
bool gemm_tensor_supported(const fm_gemm_args &g);

}  // namespace fm

using namespace fm;

// FM_GEMM_AUTO: bf16 always on the tensor cores (exact products, ~1e-6);
// f32 on the split-bf16 tensor path only when the product is big enough to
// pay for the operand splits -- small f32 GEMMs keep the reference's exact
// f64-accumulated numerics bit for bit (cjit.py:33-51) at no cost.
static bool use_tensor(const fm_gemm_args &g) {
  if (g.precision == FM_GEMM_EXACT || g.in_etype == FM_F64) return false;
  if (g.m <= 0 || g.n <= 0 || g.k <= 0 || !gemm_tensor_supported(g)) return false;
  if (g.precision == FM_GEMM_AUTO && g.in_etype == FM_F32 && (double)g.m * g.n * g.k < (double)(1ll << 28))
    return false;
  return true;
}

extern "C" int fm_gemm_plan(const fm_gemm_args *args, int *path) {
  if (!args || !path) return fail_msg("gemm_plan: null argument");
  *path = use_tensor(*args) ? FM_GEMM_PATH_TCGEN05 : FM_GEMM_PATH_EXACT;
  return 0;
}

extern "C" int fm_gemm(const fm_gemm_args *args, void *stream) {
  if (!args) return fail_msg("gemm: null args");
  const fm_gemm_args &g = *args;
  if (g.m < 0 || g.n < 0 || g.k < 0) return fail_msg("gemm: negative dimension");
  if (g.in_etype != FM_F32 && g.in_etype != FM_F64 && g.in_etype != FM_BF16)
    return fail_msg("gemm: float operands only");
  if ((g.in_etype == FM_F64) != (g.out_etype == FM_F64)) return fail_msg("gemm: f64 in <-> f64 out");
  if (g.out_etype != FM_F32 && g.out_etype != FM_F64) return fail_msg("gemm: output must be f32 or f64");
  if (g.m == 0 || g.n == 0) return 0;
  if (g.c_in && g.ld_c_in < g.m) return fail_msg("gemm: ld_c_in < m");
  cudaStream_t s = (cudaStream_t)stream;
  if (g.k == 0 && !g.c_in) {
    const size_t w = g.out_etype == FM_F64 ? 8 : 4;
    for (int64_t j = 0; j < g.n; ++j) FM_CHECK(cudaMemsetAsync((char *)g.c + j * g.ldc * w, 0, g.m * w, s));
    return 0;
  }
  if (use_tensor(g)) {
    bool handled = false;
    int st = gemm_tensor(g, s, &handled);
    if (st || handled) return st;
    if (g.precision == FM_GEMM_TENSOR) return fail_msg("gemm: shape not supported by the tensor-core kernel");
  }
  return gemm_exact(g, s);
}

// GEMM with elementwise operand prologues (include/fmb200.h): operand A (B)
// is the value of `a_prog` (`b_prog`) over its stored shape instead of the
// buffer g.a (g.b).  On the f32 tensor path the expression is evaluated into
// the bf16 operand planes the GEMM reads anyway (split.cuh) -- no operand
// temp; elsewhere (exact / f64 / bf16 paths) it is materialised into a
// stream-ordered temp first, exactly the reference's plan (plan.py:125-151).
extern "C" int fm_gemm_prologue(const fm_gemm_args *args, const fm_program *a_prog, const fm_program *b_prog,
                                void *stream) {
  if (!args) return fail_msg("gemm: null args");
  if (!a_prog && !b_prog) return fm_gemm(args, stream);
  fm_gemm_args g = *args;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t ar = g.trans_a ? g.k : g.m, ac = g.trans_a ? g.m : g.k;
  const int64_t br = g.trans_b ? g.n : g.k, bc = g.trans_b ? g.k : g.n;
  for (const fm_program *P : {a_prog, b_prog}) {
    if (!P) continue;
    if (int st = validate_program(P)) return st;
    if (P->result_etype != g.in_etype) return fail_msg("gemm prologue: expression type differs from the operand type");
  }
  if (a_prog) g.lda = ar;
  if (b_prog) g.ldb = br;
  if (g.m == 0 || g.n == 0 || g.k == 0) return fm_gemm(&g, stream);
  if (g.in_etype == FM_F32 && use_tensor(g)) {
    bool handled = false;
    int st = gemm_tensor(g, s, &handled, a_prog, b_prog);
    if (st || handled) return st;
  }
  const size_t w = g.in_etype == FM_F64 ? 8 : (g.in_etype == FM_BF16 ? 2 : 4);
  void *ta = nullptr, *tb = nullptr;
  int st = 0;
  if (a_prog) {
    FM_CHECK(cudaMallocAsync(&ta, (size_t)(ar * ac) * w, s));
    st = launch_copy_program(*a_prog, ta, ar, ac, s);
    g.a = ta;
  }
  if (!st && b_prog) {
    cudaError_t e = cudaMallocAsync(&tb, (size_t)(br * bc) * w, s);
    st = e == cudaSuccess ? launch_copy_program(*b_prog, tb, br, bc, s) : fail("cudaMallocAsync", e);
    g.b = tb;
  }
  if (!st) st = fm_gemm(&g, stream);
  if (ta) cudaFreeAsync(ta, s);
  if (tb) cudaFreeAsync(tb, s);
  return st;
}
