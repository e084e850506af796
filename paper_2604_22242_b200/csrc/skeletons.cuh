// skeletons.cuh -- the three launch skeletons, templated on an evaluator.
//
//   copy       : out[r + c*n_rows] = EXPR(r, c)          (codegen.py:74-92)
//   accu       : *out = sum EXPR, f64 / wrapping int     (codegen.py:94-114)
//   reduce_dim : sum / mean / max / min / index_max / index_min of EXPR per
//                column (dim 0) or per row (dim 1), several outputs per pass
//
// An evaluator E provides kV (elements per thread) and
//   static void eval(const fm_program&, const Chunk&, uint32_t (&lo)[kV], uint32_t (&hi)[kV])
// returning the result bits of V consecutive elements (the root's element
// type is P.result_etype).
#pragma once
#include <math_constants.h>

#include "vm.cuh"

namespace fm {

constexpr int kThreads = 256;

struct ReduceOuts {
  fm_reduce_out o[FM_MAX_REDUCE_OUT];
  int n;
};

// ---- typed helpers -----------------------------------------------------------------
FM_DEV bool is_float_etype(int e) { return e == FM_F32 || e == FM_F64 || e == FM_BF16; }

// value of element v as f64 (exact for every element type)
FM_DEV double as_double(int etype, uint32_t lo, uint32_t hi) {
  switch (etype) {
    case FM_F64: return u2d(lo, hi);
    case FM_U32: return (double)lo;
    case FM_I32: return (double)(int32_t)lo;
    default: return (double)u2f(lo);   // f32 and bf16 (held as f32)
  }
}

FM_DEV void st_v4(void *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

template <int V>
FM_DEV void store_chunk(void *out, int etype, int64_t base, int cnt, const uint32_t (&lo)[V],
                        const uint32_t (&hi)[V]) {
  if (etype == FM_F64) {
    unsigned long long *p = (unsigned long long *)out + base;
    if (cnt == V && (((uintptr_t)p) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < V / 2; ++q) st_v4(p + 2 * q, lo[2 * q], hi[2 * q], lo[2 * q + 1], hi[2 * q + 1]);
      return;
    }
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (v < cnt) p[v] = ((unsigned long long)hi[v] << 32) | lo[v];
  } else if (etype == FM_BF16) {
    uint16_t *p = (uint16_t *)out + base;
    if (V == 8 && cnt == V && (((uintptr_t)p) & 15) == 0) {
      uint32_t w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = (lo[(2 * q) % V] >> 16) | (lo[(2 * q + 1) % V] & 0xffff0000u);
      st_v4(p, w[0], w[1], w[2], w[3]);
      return;
    }
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (v < cnt) p[v] = (uint16_t)(lo[v] >> 16);
  } else {
    uint32_t *p = (uint32_t *)out + base;
    if (cnt == V && (((uintptr_t)p) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < V / 4; ++q) st_v4(p + 4 * q, lo[4 * q], lo[4 * q + 1], lo[4 * q + 2], lo[4 * q + 3]);
      return;
    }
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (v < cnt) p[v] = lo[v];
  }
}

// Chunk number c of the domain.  Flat programs chunk the flat index space;
// others chunk each column into runs of V rows.
template <int V>
FM_DEV Chunk make_chunk(const fm_program &P, int64_t c, int64_t n_rows, int64_t n_elem, int64_t nrb) {
  Chunk ch;
  if (P.flat) {
    ch.base = c * V;
    ch.cnt = (int)min((int64_t)V, n_elem - ch.base);
    ch.row0 = 0; ch.col = 0; ch.flat = true;
  } else {
    ch.col = c / nrb;
    ch.row0 = (c - ch.col * nrb) * V;
    ch.cnt = (int)min((int64_t)V, n_rows - ch.row0);
    ch.base = ch.row0 + ch.col * n_rows;
    ch.flat = false;
  }
  return ch;
}

template <int V>
FM_DEV int64_t chunk_count(const fm_program &P, int64_t n_rows, int64_t n_cols, int64_t &nrb) {
  nrb = (n_rows + V - 1) / V;
  return P.flat ? (n_rows * n_cols + V - 1) / V : nrb * n_cols;
}

// ---- copy ------------------------------------------------------------------------------
// Evaluators with kFast take a typed, branch-free path over whole warp tiles
// (32 x V elements, coalesced 512-byte vector accesses, the next tile's loads
// issued before the current tile's math) when the program is flat and
// 16-byte aligned; the ragged remainder (and every other program) uses the
// general chunk path.
// prefetch depth of the copy fast path (FM_COPY_DEPTH2_HEAVY=0 at build
// time keeps every chain at depth 1)
#ifndef FM_COPY_DEPTH2_HEAVY
#define FM_COPY_DEPTH2_HEAVY 1
#endif
template <class E>
constexpr int kCopyDepth() {
  // measured (bench.py --config c3 / suite): C3 (2 inputs, exp) 6.24 -> 6.44
  // TB/s at depth 2; single-input heavy chains (sigmoid, swish, gelu) lose
  // 2-4 % to the extra registers
  if constexpr (E::kFast) return (FM_COPY_DEPTH2_HEAVY && E::kHeavy && E::kNin >= 2) ? 2 : 1;
  else return 0;   // wide tiles: no tile prefetched ahead
}
template <class E, bool VM = E::kIsVm> struct WideTile { static constexpr bool v = false; };
template <class E> struct WideTile<E, false> { static constexpr bool v = E::kWideTile; };

template <class E>
__global__ void __launch_bounds__(kThreads, E::kMinBlocks) k_copy(const __grid_constant__ fm_program P, void *out,
                                                   int64_t n_rows, int64_t n_cols) {
  constexpr int V = E::kV;
  const int indep = P.reserved & 1;   // launch-window class (common.cuh)
  pdl_enter(indep);
  const int64_t n_elem = n_rows * n_cols;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if constexpr (E::kFast || WideTile<E>::v) {
    if (E::fast_ok(P, out)) {
      constexpr int kTile = E::kTile;
      const int lane = threadIdx.x & 31;
      const int64_t nwarp = stride >> 5;
      const int64_t ntile = n_elem / kTile;
      int64_t t = c >> 5;
      if constexpr (kCopyDepth<E>() == 0) {
        for (; t < ntile; t += nwarp) {
          typename E::Buf b;
          E::load_tile(P, t * kTile, lane, b);
          E::copy_tile(P, out, t * kTile, lane, b);
        }
      } else if constexpr (kCopyDepth<E>() == 2) {
        // long per-element math: two tiles in flight per warp
        typename E::Buf b0, b1;
        if (t < ntile) E::load_tile(P, t * kTile, lane, b0);
        if (t + nwarp < ntile) E::load_tile(P, (t + nwarp) * kTile, lane, b1);
        for (; t < ntile; t += nwarp) {
          const typename E::Buf cur = b0;
          b0 = b1;
          if (t + 2 * nwarp < ntile) E::load_tile(P, (t + 2 * nwarp) * kTile, lane, b1);
          E::copy_tile(P, out, t * kTile, lane, cur);
        }
      } else {
        typename E::Buf buf;
        if (t < ntile) E::load_tile(P, t * kTile, lane, buf);
        for (; t < ntile; t += nwarp) {
          const typename E::Buf cur = buf;
          if (t + nwarp < ntile) E::load_tile(P, (t + nwarp) * kTile, lane, buf);
          E::copy_tile(P, out, t * kTile, lane, cur);
        }
      }
      c += ntile * 32;   // ragged remainder: flat V-element chunks from here on
    }
  }
  int64_t nrb;
  const int64_t nch = chunk_count<V>(P, n_rows, n_cols, nrb);
  for (; c < nch; c += stride) {
    Chunk ch = make_chunk<V>(P, c, n_rows, n_elem, nrb);
    uint32_t lo[V], hi[V];
    E::eval(P, ch, lo, hi);
    store_chunk<V>(out, P.result_etype, ch.base, ch.cnt, lo, hi);
  }
  if (blockIdx.x == 0) pdl_exit(indep);
}

// ---- block reductions ------------------------------------------------------------------------
FM_DEV double warp_sum_d(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
FM_DEV uint32_t warp_sum_u(uint32_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// (value, index) candidate for max / min with numpy semantics: NaN wins
// (first NaN), ties keep the lowest index.
struct Cand {
  double v;
  int64_t i;
};
FM_DEV bool better_max(const Cand &a, const Cand &b) {
  const bool an = a.v != a.v, bn = b.v != b.v;
  if (an || bn) return an && (!bn || a.i < b.i);
  return a.v > b.v || (a.v == b.v && a.i < b.i);
}
FM_DEV bool better_min(const Cand &a, const Cand &b) {
  const bool an = a.v != a.v, bn = b.v != b.v;
  if (an || bn) return an && (!bn || a.i < b.i);
  return a.v < b.v || (a.v == b.v && a.i < b.i);
}
FM_DEV Cand shfl_cand(const Cand &c, int o) {
  Cand r;
  r.v = __shfl_xor_sync(0xffffffffu, c.v, o);
  r.i = __shfl_xor_sync(0xffffffffu, c.i, o);
  return r;
}
template <bool MAX>
FM_DEV Cand warp_best(Cand c) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Cand x = shfl_cand(c, o);
    if (MAX ? better_max(x, c) : better_min(x, c)) c = x;
  }
  return c;
}

// block-wide helpers (kThreads threads; result valid in thread 0)
FM_DEV double block_sum_d(double x, double *sm) {
  x = warp_sum_d(x);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm[w] = x;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = (l < kThreads / 32) ? sm[l] : 0.0;
    r = warp_sum_d(r);
  }
  return r;
}
FM_DEV uint32_t block_sum_u(uint32_t x, uint32_t *sm) {
  x = warp_sum_u(x);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm[w] = x;
  __syncthreads();
  uint32_t r = 0;
  if (threadIdx.x < 32) {
    r = (l < kThreads / 32) ? sm[l] : 0u;
    r = warp_sum_u(r);
  }
  return r;
}
template <bool MAX>
FM_DEV Cand block_best(Cand c, Cand *sm) {
  c = warp_best<MAX>(c);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm[w] = c;
  __syncthreads();
  if (threadIdx.x < 32) {
    c = (l < kThreads / 32) ? sm[l] : sm[0];
    c = warp_best<MAX>(c);
  }
  return c;
}

// ---- accu ------------------------------------------------------------------------------------
// Per-block partials then a last-block finish: ONE launch, deterministic for
// a given grid (fixed per-thread order, fixed tree).
template <class E>
__global__ void __launch_bounds__(kThreads) k_accu(const __grid_constant__ fm_program P, void *out,
                                                   int64_t n_rows, int64_t n_cols, int finalize,
                                                   double *part_d, uint32_t *part_u, unsigned *counter) {
  constexpr int V = E::kV;
  __shared__ double smd[kThreads / 32];
  __shared__ uint32_t smu[kThreads / 32];
  __shared__ bool last;
  const int rt = P.result_etype;
  const bool fl = is_float_etype(rt);
  const int indep = P.reserved & 1;   // launch-window class (common.cuh)
  pdl_enter(indep);
  int64_t nrb;
  const int64_t nch = chunk_count<V>(P, n_rows, n_cols, nrb);
  const int64_t n_elem = n_rows * n_cols;
  double accd = 0.0;
  uint32_t accu = 0;
  int64_t c = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  if constexpr (E::kFast) {
    if (E::fast_ok(P, nullptr)) {   // all-float flat program: warp tiles, one in flight
      constexpr int kTile = E::kTile;
      const int lane = threadIdx.x & 31;
      const int64_t nwarp = stride >> 5;
      const int64_t ntile = n_elem / kTile;
      int64_t t = c >> 5;
      typename E::Buf buf;
      if (t < ntile) E::load_tile(P, t * kTile, lane, buf);
      for (; t < ntile; t += nwarp) {
        const typename E::Buf cur = buf;
        if (t + nwarp < ntile) E::load_tile(P, (t + nwarp) * kTile, lane, buf);
        E::accu_tile(P, cur, accd);
      }
      c += ntile * 32;
    }
  }
  for (; c < nch; c += stride) {
    Chunk ch = make_chunk<V>(P, c, n_rows, n_elem, nrb);
    uint32_t lo[V], hi[V];
    E::eval(P, ch, lo, hi);
    if (fl) {
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (v < ch.cnt) accd += as_double(rt, lo[v], hi[v]);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (v < ch.cnt) accu += lo[v];
    }
  }
  double bd = block_sum_d(accd, smd);
  uint32_t bu = block_sum_u(accu, smu);
  if (threadIdx.x == 0) {
    part_d[blockIdx.x] = bd;
    part_u[blockIdx.x] = bu;
    __threadfence();
    unsigned t = atomicAdd(counter, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (blockIdx.x == 0) pdl_exit(indep);
  if (!last) return;
  __threadfence();
  double sd = 0.0;
  uint32_t su = 0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += kThreads) {
    sd += ((volatile double *)part_d)[i];
    su += ((volatile uint32_t *)part_u)[i];
  }
  sd = block_sum_d(sd, smd);
  su = block_sum_u(su, smu);
  if (threadIdx.x == 0) {
    if (fl) {
      if (finalize == FM_FINAL_SQRT) sd = sqrt_d(sd);
      *(double *)out = sd;
    } else {
      *(uint32_t *)out = su;
    }
    *counter = 0u;   // self-reset for the next launch on this stream
  }
}

// ---- reduce_dim ------------------------------------------------------------------------------------
struct Stats {
  double sum;
  uint32_t usum;
  Cand mx, mn;
};

FM_DEV void stats_init(Stats &s) {
  s.sum = 0.0; s.usum = 0;
  s.mx.v = __longlong_as_double(0xfff0000000000000ll); s.mx.i = INT64_MAX;   // -inf
  s.mn.v = __longlong_as_double(0x7ff0000000000000ll); s.mn.i = INT64_MAX;   // +inf
}

FM_DEV void stats_add(Stats &s, int rt, bool fl, uint32_t lo, uint32_t hi, int64_t idx, unsigned need) {
  if (fl || !(need & 1u)) {
    const double x = as_double(rt, lo, hi);
    if (need & 1u) s.sum += x;
    Cand c{x, idx};
    if ((need & 2u) && better_max(c, s.mx)) s.mx = c;
    if ((need & 4u) && better_min(c, s.mn)) s.mn = c;
  } else {
    s.usum += lo;
    const double x = as_double(rt, lo, hi);
    Cand c{x, idx};
    if ((need & 2u) && better_max(c, s.mx)) s.mx = c;
    if ((need & 4u) && better_min(c, s.mn)) s.mn = c;
  }
}

// write one reduced value of kind k at position pos
FM_DEV void emit_out(const fm_reduce_out &o, int64_t pos, const Stats &s, int rt, bool fl, int64_t n_along) {
  switch (o.kind) {
    case FM_RED_SUM:
    case FM_RED_MEAN: {
      if (!fl) {   // integer sum wraps in the element type
        ((uint32_t *)o.out)[pos] = s.usum;
        return;
      }
      double v = s.sum;
      if (o.kind == FM_RED_MEAN) v = div_d(v, (double)n_along);
      if (o.etype == FM_F64) ((double *)o.out)[pos] = v;
      else if (o.etype == FM_BF16) ((uint16_t *)o.out)[pos] = (uint16_t)(f2u(d_to_bf(v)) >> 16);
      else ((float *)o.out)[pos] = d_to_f(v);
      return;
    }
    case FM_RED_MAX:
    case FM_RED_MIN: {
      const double v = (o.kind == FM_RED_MAX) ? s.mx.v : s.mn.v;
      switch (o.etype) {
        case FM_F64: ((double *)o.out)[pos] = v; break;
        case FM_F32: ((float *)o.out)[pos] = (float)v; break;
        case FM_BF16: ((uint16_t *)o.out)[pos] = (uint16_t)(f2u((float)v) >> 16); break;
        case FM_U32: ((uint32_t *)o.out)[pos] = (uint32_t)v; break;
        default: ((int32_t *)o.out)[pos] = (int32_t)v; break;
      }
      return;
    }
    case FM_RED_IMAX: ((uint32_t *)o.out)[pos] = (uint32_t)s.mx.i; return;
    default: ((uint32_t *)o.out)[pos] = (uint32_t)s.mn.i; return;
  }
}

FM_DEV unsigned needed_stats(const ReduceOuts &R) {
  unsigned need = 0;
  for (int i = 0; i < R.n; ++i) {
    const int k = R.o[i].kind;
    if (k == FM_RED_SUM || k == FM_RED_MEAN) need |= 1u;
    else if (k == FM_RED_MAX || k == FM_RED_IMAX) need |= 2u;
    else need |= 4u;
  }
  return need;
}

// Typed per-thread column statistics for the fast path.  A thread visits its
// rows in strictly increasing order, so "first index wins" needs no index
// compare: a later element replaces the candidate only if strictly better,
// or if it is the first NaN (numpy semantics), or if there is no candidate
// yet.  Branch-free selects; 32-bit row indices (outputs are u32).
template <class T>
struct ColStats {
  static constexpr uint32_t kNone = 0xFFFFFFFFu;
  double sum;
  T mx, mn;
  uint32_t imx, imn;
  FM_DEV void init() {
    sum = 0.0;
    mx = -CUDART_INF_F; mn = CUDART_INF_F;   // converts exactly for T = double
    imx = imn = kNone;
  }
  FM_DEV void add(T x, uint32_t i, unsigned need) {
    if (need & 1u) sum = add_d(sum, (double)x);
    if (need & 2u) {
      const bool take = (!(x <= mx) || imx == kNone) && (mx == mx);
      mx = take ? x : mx;
      imx = take ? i : imx;
    }
    if (need & 4u) {
      const bool take = (!(x >= mn) || imn == kNone) && (mn == mn);
      mn = take ? x : mn;
      imn = take ? i : imn;
    }
  }
  FM_DEV void to_stats(Stats &s) const {
    s.sum += sum;
    if (imx != kNone) { s.mx.v = (double)mx; s.mx.i = imx; }
    if (imn != kNone) { s.mn.v = (double)mn; s.mn.i = imn; }
  }
};

// General chunk path of a column (ragged row remainder, or programs without
// the typed fast path).  Out of line so its register needs do not crowd the
// fast path's loop in the same kernel.
template <class E>
__device__ __noinline__ void cols_generic(const fm_program &P, Stats &s, int64_t col, int64_t row_start,
                                          int64_t n_rows, int rt, bool fl, unsigned need) {
  constexpr int V = E::kV;
  for (int64_t row0 = row_start + (int64_t)threadIdx.x * V; row0 < n_rows; row0 += (int64_t)kThreads * V) {
    Chunk ch;
    ch.row0 = row0; ch.col = col; ch.base = row0 + col * n_rows;
    ch.cnt = (int)min((int64_t)V, n_rows - row0);
    ch.flat = P.flat != 0;
    uint32_t lo[V], hi[V];
    E::eval(P, ch, lo, hi);
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (v < ch.cnt) stats_add(s, rt, fl, lo[v], hi[v], row0 + v, need);
  }
}

// dim 0: one block per column (grid-stride over columns).  Fast path (typed
// evaluator, flat program, 16-byte aligned columns): each warp streams warp
// tiles of its column with the next tile's loads in flight while the current
// tile's statistics are folded in; ragged row remainders and every other
// program use the general chunk path.
template <class E>
__global__ void __launch_bounds__(kThreads, 3) k_reduce_cols(const __grid_constant__ fm_program P,
                                                          const __grid_constant__ ReduceOuts R,
                                                          int64_t n_rows, int64_t n_cols) {
  constexpr int V = E::kV;
  __shared__ double smd[kThreads / 32];
  __shared__ uint32_t smu[kThreads / 32];
  __shared__ Cand smc[kThreads / 32];
  const int rt = P.result_etype;
  const bool fl = is_float_etype(rt);
  const unsigned need = needed_stats(R);
  const int indep = P.reserved & 1;   // launch-window class (common.cuh)
  pdl_enter(indep);
  bool fast = false;
  int64_t fast_rows = 0;
  if constexpr (E::kFast) {
    using T = typename E::Elem;
    fast = E::fast_ok(P, nullptr) && ((n_rows * (int64_t)sizeof(T)) & 15) == 0 && n_rows < 0xFFFFFFFFll;
    if (fast) fast_rows = (n_rows / E::kTile) * E::kTile;
  }
  for (int64_t col = blockIdx.x; col < n_cols; col += gridDim.x) {
    Stats s;
    stats_init(s);
    int64_t row_start = 0;
    if constexpr (E::kFast) {
      if (fast) {
        using T = typename E::Elem;
        constexpr int kTile = E::kTile, kW = E::kW;
        const int lane = threadIdx.x & 31;
        const int64_t ntile = fast_rows / kTile;
        const int64_t cbase = col * n_rows;
        ColStats<T> cs;
        cs.init();
        int64_t t = threadIdx.x >> 5;
        typename E::Buf buf;
        if (t < ntile) E::load_tile(P, cbase + t * kTile, lane, buf);
        for (; t < ntile; t += kThreads / 32) {
          const typename E::Buf cur = buf;
          if (t + kThreads / 32 < ntile) E::load_tile(P, cbase + (t + kThreads / 32) * kTile, lane, buf);
          T r[V];
          E::eval_tile(P, cur, r);
          const uint32_t r0 = (uint32_t)(t * kTile) + lane * kW;
#pragma unroll
          for (int q = 0; q < V / kW; ++q)
#pragma unroll
            for (int e = 0; e < kW; ++e) cs.add(r[q * kW + e], r0 + q * 32 * kW + e, need);
        }
        cs.to_stats(s);
        row_start = fast_rows;
      }
    }
    if (row_start < n_rows) cols_generic<E>(P, s, col, row_start, n_rows, rt, fl, need);
    Stats t = s;
    if (need & 1u) {
      t.sum = block_sum_d(s.sum, smd);
      t.usum = block_sum_u(s.usum, smu);
    }
    if (need & 2u) t.mx = block_best<true>(s.mx, smc);
    if (need & 4u) t.mn = block_best<false>(s.mn, smc);
    if (threadIdx.x == 0)
      for (int i = 0; i < R.n; ++i) emit_out(R.o[i], col, t, rt, fl, n_rows);
    __syncthreads();
  }
  if (blockIdx.x == 0) pdl_exit(indep);
}

// dim 0, typed fast path only: every column is a whole number of warp tiles
// (the host checks).  A kernel of its own so that no general-path code shares
// its register allocation (measured: with the chunk path in the same kernel
// ptxas spilled inside this loop, C4 7.46 -> 7.10 TB/s).
template <class E>
__global__ void __launch_bounds__(kThreads, 3) k_reduce_cols_fast(const __grid_constant__ fm_program P,
                                                               const __grid_constant__ ReduceOuts R,
                                                               int64_t n_rows, int64_t n_cols) {
  constexpr int V = E::kV;
  using T = typename E::Elem;
  constexpr int kTile = E::kTile, kW = E::kW;
  __shared__ double smd[kThreads / 32];
  __shared__ uint32_t smu[kThreads / 32];
  __shared__ Cand smc[kThreads / 32];
  const int rt = P.result_etype;
  const unsigned need = needed_stats(R);
  const int indep = P.reserved & 1;   // launch-window class (common.cuh)
  pdl_enter(indep);
  const int lane = threadIdx.x & 31;
  const int64_t ntile = n_rows / kTile;
  for (int64_t col = blockIdx.x; col < n_cols; col += gridDim.x) {
    Stats s;
    stats_init(s);
    const int64_t cbase = col * n_rows;
    ColStats<T> cs;
    cs.init();
    int64_t t = threadIdx.x >> 5;
    typename E::Buf buf;
    if (t < ntile) E::load_tile(P, cbase + t * kTile, lane, buf);
    for (; t < ntile; t += kThreads / 32) {
      const typename E::Buf cur = buf;
      if (t + kThreads / 32 < ntile) E::load_tile(P, cbase + (t + kThreads / 32) * kTile, lane, buf);
      T r[V];
      E::eval_tile(P, cur, r);
      const uint32_t r0 = (uint32_t)(t * kTile) + lane * kW;
#pragma unroll
      for (int q = 0; q < V / kW; ++q)
#pragma unroll
        for (int e = 0; e < kW; ++e) cs.add(r[q * kW + e], r0 + q * 32 * kW + e, need);
    }
    cs.to_stats(s);
    Stats tt = s;
    if (need & 1u) tt.sum = block_sum_d(s.sum, smd);
    if (need & 2u) tt.mx = block_best<true>(s.mx, smc);
    if (need & 4u) tt.mn = block_best<false>(s.mn, smc);
    (void)smu;
    if (threadIdx.x == 0)
      for (int i = 0; i < R.n; ++i) emit_out(R.o[i], col, tt, rt, true, n_rows);
    __syncthreads();
  }
  if (blockIdx.x == 0) pdl_exit(indep);
}

// General chunk path of a row run over columns [c0, c1): out of line so the
// typed fast path keeps its registers (as cols_generic).
template <class E>
__device__ __noinline__ void rows_generic(const fm_program &P, Stats (&s)[E::kV], int64_t row0, int cnt,
                                          int64_t c0, int64_t c1, int64_t n_rows, int rt, bool fl, unsigned need) {
  constexpr int V = E::kV;
  for (int64_t col = c0; col < c1; ++col) {
    Chunk ch;
    ch.row0 = row0; ch.col = col; ch.base = row0 + col * n_rows; ch.cnt = cnt;
    ch.flat = P.flat != 0;
    uint32_t lo[V], hi[V];
    E::eval(P, ch, lo, hi);
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (v < cnt) stats_add(s[v], rt, fl, lo[v], hi[v], col, need);
  }
}

// dim 1: each thread owns V consecutive rows; blockIdx.y splits the columns.
// With several splits, partial stats go to scratch and the last block of each
// row tile combines them in split order (one launch, deterministic).
struct RowPartial {
  double sum;
  uint32_t usum;
  uint32_t pad;
  Cand mx, mn;
};

// mbarrier + TMA bulk copy helpers of the staged row reduction
FM_DEV uint32_t smem_addr_rows(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
FM_DEV void mbar_init_rows(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr_rows(bar)), "r"(count));
}
FM_DEV void mbar_arrive_expect_tx_rows(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr_rows(bar)), "r"(bytes)
               : "memory");
}
FM_DEV void mbar_wait_rows(uint64_t *bar, uint32_t parity) {
  const uint32_t a = smem_addr_rows(bar);
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
FM_DEV void bulk_g2s_rows(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr_rows(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr_rows(bar))
      : "memory");
}

// `depth` > 0: the typed fast path streams its columns through a shared-
// memory ring of `depth` stages filled by TMA bulk copies (one per input and
// column: the block's rows of a column are contiguous), so `depth` columns
// are in flight without holding registers.  The register version (one
// column ahead) kept ~50 KB in flight per SM at 25 % occupancy and ran
// long-scoreboard-bound at 6.34 TB/s (profiles/r02/ncu_c4r_rowstats); a
// per-thread cp.async ring was MIO-throttled (3.8 TB/s).
template <class E>
__global__ void __launch_bounds__(kThreads) k_reduce_rows(const __grid_constant__ fm_program P,
                                                          const __grid_constant__ ReduceOuts R,
                                                          int64_t n_rows, int64_t n_cols,
                                                          RowPartial *part, unsigned *counters, int depth) {
  constexpr int V = E::kV;
  __shared__ bool last;
  const int rt = P.result_etype;
  const bool fl = is_float_etype(rt);
  const unsigned need = needed_stats(R);
  const int splits = gridDim.y;
  const int64_t cols_per = (n_cols + splits - 1) / splits;
  const int64_t c0 = (int64_t)blockIdx.y * cols_per;
  const int64_t c1 = min(n_cols, c0 + cols_per);
  const int64_t row0 = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * V;
  const bool active = row0 < n_rows;
  const int cnt = active ? (int)min((int64_t)V, n_rows - row0) : 0;
  Stats s[V];
#pragma unroll
  for (int v = 0; v < V; ++v) stats_init(s[v]);
  bool done_fast = false;
  if constexpr (E::kFast) {
    // Typed fast path: whole V-row runs of a flat, 16-byte aligned program.
    // The next column's vectors are loaded while the current one is folded
    // into branch-free per-row stats (columns visited in increasing order, so
    // a strictly-better test keeps the first index).
    using T = typename E::Elem;
    constexpr int NIN = E::kNin, kW = E::kW, NQ = V / kW;
    if (active && cnt == V && E::fast_ok(P, nullptr) && ((n_rows * (int64_t)sizeof(T)) & 15) == 0 &&
        n_cols < 0xFFFFFFFFll) {
      ColStats<T> cs[V];
#pragma unroll
      for (int v = 0; v < V; ++v) cs[v].init();
      auto fold = [&](const uint4 (&b)[NIN][NQ], int64_t col) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
          for (int e = 0; e < kW; ++e) {
            T x[NIN];
#pragma unroll
            for (int i = 0; i < NIN; ++i) {
              if constexpr (sizeof(T) == 8) x[i] = e == 0 ? u2d(b[i][q].x, b[i][q].y) : u2d(b[i][q].z, b[i][q].w);
              else x[i] = u2f(e == 0 ? b[i][q].x : e == 1 ? b[i][q].y : e == 2 ? b[i][q].z : b[i][q].w);
            }
            cs[q * kW + e].add(E::ev_elem(P, x), (uint32_t)col, need);
          }
      };
      if (depth > 0) {
        // ring of `depth` stages; stage d holds, per input, this CTA's
        // kThreads * V rows of one column (contiguous in HBM: one TMA bulk
        // copy each, completion counted on full[d]); thread 0 refills a
        // stage once the whole block has read it
        extern __shared__ __align__(128) unsigned char rring[];
        constexpr int kSeg = kThreads * V * (int)sizeof(T);      // bytes per input per column
        uint64_t *full = (uint64_t *)(rring + (size_t)depth * NIN * kSeg);
        const int64_t rows_here = min((int64_t)kThreads * V, n_rows - (int64_t)blockIdx.x * kThreads * V);
        const uint32_t seg_bytes = (uint32_t)(rows_here * (int64_t)sizeof(T));
        auto issue = [&](int64_t col, int d) {
          mbar_arrive_expect_tx_rows(&full[d], seg_bytes * NIN);
#pragma unroll
          for (int i = 0; i < NIN; ++i)
            bulk_g2s_rows(rring + (size_t)(d * NIN + i) * kSeg,
                          (const T *)P.slots[i].ptr + col * n_rows + (int64_t)blockIdx.x * kThreads * V, seg_bytes,
                          &full[d]);
        };
        if (threadIdx.x == 0) {
          for (int d = 0; d < depth; ++d) mbar_init_rows(&full[d], 1);
          asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
          for (int d = 0; d < depth; ++d)
            if (c0 + d < c1) issue(c0 + d, d);
        }
        __syncthreads();
        int d = 0;
        uint32_t ph = 0;
        for (int64_t col = c0; col < c1; ++col) {
          mbar_wait_rows(&full[d], ph);
          uint4 b[NIN][NQ];
#pragma unroll
          for (int i = 0; i < NIN; ++i)
#pragma unroll
            for (int q = 0; q < NQ; ++q)
              b[i][q] = *(const uint4 *)(rring + (size_t)(d * NIN + i) * kSeg + (size_t)threadIdx.x * V * sizeof(T) + 16 * q);
          __syncthreads();   // stage d read by the whole block
          if (threadIdx.x == 0 && col + depth < c1) issue(col + depth, d);
          fold(b, col);
          if (++d == depth) { d = 0; ph ^= 1u; }
        }
      } else {
      uint4 cur[NIN][NQ], nxt[NIN][NQ];
      auto load = [&](int64_t col, uint4 (&b)[NIN][NQ]) {
#pragma unroll
        for (int i = 0; i < NIN; ++i) {
          const T *p = (const T *)P.slots[i].ptr + col * n_rows + row0;
#pragma unroll
          for (int q = 0; q < NQ; ++q) b[i][q] = ldg_v4(p + q * kW);
        }
      };
      if (c0 < c1) load(c0, cur);
      for (int64_t col = c0; col < c1; ++col) {
        if (col + 1 < c1) load(col + 1, nxt);
        fold(cur, col);
#pragma unroll
        for (int i = 0; i < NIN; ++i)
#pragma unroll
          for (int q = 0; q < NQ; ++q) cur[i][q] = nxt[i][q];
      }
      }
#pragma unroll
      for (int v = 0; v < V; ++v) cs[v].to_stats(s[v]);
      done_fast = true;
    }
  }
  if (active && !done_fast) rows_generic<E>(P, s, row0, cnt, c0, c1, n_rows, rt, fl, need);
  if (splits == 1) {
    if (active)
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (v < cnt)
          for (int i = 0; i < R.n; ++i) emit_out(R.o[i], row0 + v, s[v], rt, fl, n_cols);
    return;
  }
  if (active) {
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (v < cnt) {
        RowPartial p;
        p.sum = s[v].sum; p.usum = s[v].usum; p.pad = 0; p.mx = s[v].mx; p.mn = s[v].mn;
        part[(int64_t)blockIdx.y * n_rows + row0 + v] = p;
      }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = atomicAdd(&counters[blockIdx.x], 1u);
    last = (t == (unsigned)splits - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (active) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      if (v >= cnt) continue;
      Stats t;
      stats_init(t);
      for (int y = 0; y < splits; ++y) {
        const RowPartial *pp = &part[(int64_t)y * n_rows + row0 + v];
        const double ps = ((volatile const double *)&pp->sum)[0];
        const uint32_t pu = ((volatile const uint32_t *)&pp->usum)[0];
        Cand pmx, pmn;
        pmx.v = ((volatile const double *)&pp->mx.v)[0];
        pmx.i = ((volatile const int64_t *)&pp->mx.i)[0];
        pmn.v = ((volatile const double *)&pp->mn.v)[0];
        pmn.i = ((volatile const int64_t *)&pp->mn.i)[0];
        t.sum += ps; t.usum += pu;
        if (better_max(pmx, t.mx)) t.mx = pmx;
        if (better_min(pmn, t.mn)) t.mn = pmn;
      }
      for (int i = 0; i < R.n; ++i) emit_out(R.o[i], row0 + v, t, rt, fl, n_cols);
    }
  }
  if (threadIdx.x == 0) counters[blockIdx.x] = 0u;
}

}  // namespace fm
