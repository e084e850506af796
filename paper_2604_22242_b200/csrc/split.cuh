// split.cuh -- GEMM operand prologue: an elementwise expression evaluated
// straight into the f32 GEMM's three bf16 operand planes.
//
// The reference materialises every MatMul operand that is not a plain
// matrix into a temp before the product (plan.py:125-151: `(X + Y) @ Z` is a
// fused copy into T, then T @ Z).  The f32 tensor-core GEMM here reads its
// operands as three bf16 planes (gemm_tc.cu) that a split pass writes from
// the f32 operand anyway, so the operand's expression is evaluated in that
// pass instead: the f32 value of each element is exactly the temp's (same
// per-node rounding, ops.cuh), split into hi/mid/lo planes, and the temp's
// write and re-read disappear.
//
// Column chunks of V rows (any program: views, transposes, mixed types),
// grid-stride over one wave; plane p of element (i, j) goes to
// out[p*plane_off + i + j*ld_out].  Planes: two scaled fp16 (the default f32
// scheme; the operand's max |x| comes from a MAX reduction of |expression|
// first, fused.cu launch_amax_program) or three bf16.
#pragma once
#include "skeletons.cuh"

namespace fm {

// amax == nullptr: three bf16 planes (split3); else two fp16 planes scaled
// from *amax = max |operand| bits (split2h, the default f32 scheme)
template <class E>
__global__ void __launch_bounds__(kThreads) k_split_fused(const __grid_constant__ fm_program P, uint16_t *out,
                                                          int64_t n_rows, int64_t n_cols, int64_t ld_out,
                                                          int64_t plane_off, const unsigned *amax) {
  constexpr int V = E::kV;
  const float sc = amax ? ldexpf(1.0f, f16_scale_exp(*amax)) : 1.0f;
  const int64_t nrb = (n_rows + V - 1) / V;
  const int64_t nch = nrb * n_cols;
  const bool vec = V % 4 == 0 && (ld_out & 3) == 0 && (plane_off & 3) == 0 && (((uintptr_t)out) & 7) == 0;
  for (int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x; c < nch; c += (int64_t)gridDim.x * kThreads) {
    Chunk ch;
    ch.col = c / nrb;
    ch.row0 = (c - ch.col * nrb) * V;
    ch.cnt = (int)min((int64_t)V, n_rows - ch.row0);
    ch.base = ch.row0 + ch.col * n_rows;
    ch.flat = false;
    uint32_t lo[V], hi[V];
    E::eval(P, ch, lo, hi);
    uint16_t h[V], m[V], l[V];
    if (amax) {
#pragma unroll
      for (int v = 0; v < V; ++v) split2h(u2f(lo[v]), sc, h[v], m[v]);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) split3(u2f(lo[v]), h[v], m[v], l[v]);
    }
    uint16_t *dst = out + ch.row0 + ch.col * ld_out;
    if (vec && ch.cnt == V) {
#pragma unroll
      for (int q = 0; q < V / 4; ++q) {
        *(ushort4 *)(dst + 4 * q) = make_ushort4(h[4 * q], h[4 * q + 1], h[4 * q + 2], h[4 * q + 3]);
        *(ushort4 *)(dst + plane_off + 4 * q) = make_ushort4(m[4 * q], m[4 * q + 1], m[4 * q + 2], m[4 * q + 3]);
        if (!amax)
          *(ushort4 *)(dst + 2 * plane_off + 4 * q) =
              make_ushort4(l[4 * q], l[4 * q + 1], l[4 * q + 2], l[4 * q + 3]);
      }
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (v < ch.cnt) {
          dst[v] = h[v];
          dst[v + plane_off] = m[v];
          if (!amax) dst[v + 2 * plane_off] = l[v];
        }
    }
  }
}

template <class E>
int run_split(const fm_program &P, uint16_t *out, int64_t n_rows, int64_t n_cols, int64_t ld_out, int64_t plane_off,
              const unsigned *amax, cudaStream_t s) {
  if (n_rows == 0 || n_cols == 0) return 0;
  if (P.result_etype != FM_F32) return fail_msg("gemm prologue: the operand expression must be f32");
  const int64_t nch = ((n_rows + E::kV - 1) / E::kV) * n_cols;
  const int64_t grid = wave_grid<GridTag<E, 7>>(k_split_fused<E>, (nch + kThreads - 1) / kThreads);
  k_split_fused<E><<<(unsigned)grid, kThreads, 0, s>>>(P, out, n_rows, n_cols, ld_out, plane_off, amax);
  FM_CHECK_LAUNCH("gemm operand prologue (fused split kernel)");
  return 0;
}

}  // namespace fm
