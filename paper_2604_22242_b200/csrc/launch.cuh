// launch.cuh -- host-side launchers of the skeletons for one evaluator type.
// Grid sizing follows the B200 measurements in profiles/: memory-bound
// grid-stride kernels want many resident warps and several waves, so grids
// are multiples of the SM count (148) capped where partial results must be
// combined.
#pragma once
#include <cstdlib>

#include "common.cuh"
#include "bulk.cuh"
#include "skeletons.cuh"
#include "tiled.cuh"
#include "pair.cuh"

namespace fm {

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline int etype_bytes(int e) { return e == FM_F64 ? 8 : (e == FM_BF16 ? 2 : 4); }

// Launch-window class of a PDL launch (common.cuh): the program's reads over
// the domain plus the given writes; returns the program to launch (bit 0 of
// `reserved` = independent) and the scratch slot.
struct Classified {
  fm_program P;
  int slot;
};
inline Classified classify(cudaStream_t s, const fm_program &P0, int64_t n_rows, int64_t n_cols,
                           const Footprint &writes) {
  Footprint fp = writes;
  program_reads(P0, n_rows, n_cols, fp);
  const PdlPlan pp = pdl_classify(s, fp);
  Classified c{P0, pp.slot};
  c.P.reserved = (P0.reserved & ~1) | pp.independent;
  return c;
}
inline Footprint writes_of(const void *out, size_t bytes) {
  Footprint fp;
  footprint_write(fp, out, bytes);
  return fp;
}
inline Footprint reduce_writes(const ReduceOuts &R, int64_t n) {
  Footprint fp;
  for (int i = 0; i < R.n; ++i) footprint_write(fp, R.o[i].out, (size_t)n * etype_bytes(R.o[i].etype));
  return fp;
}

// Resident blocks of `kernel` per SM at kThreads threads (queried once per
// kernel).  Streaming kernels launch exactly one full wave -- SMs x resident
// blocks -- and grid-stride: a fractional last wave would leave most SMs idle
// while a few finish (ncu showed 1.33 and 5.33 waves before this).
// `Tag` keys the cache: every k_copy<E> has the same function-pointer type.
template <class Tag, class K>
int resident_blocks(K kernel) {
  static int cached = 0;
  if (cached == 0) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, kThreads, 0) != cudaSuccess || n < 1) n = 1;
    cached = n;
  }
  return cached;
}
template <class Tag, class K>
int64_t wave_grid(K kernel, int64_t work_blocks) {
  const int64_t full = (int64_t)sm_count() * resident_blocks<Tag>(kernel);
  return std::max<int64_t>(1, std::min<int64_t>(work_blocks, full));
}
template <class E, int Skel> struct GridTag {};

// Streaming path choice for an eligible template (flat, 16-byte aligned):
// TMA-bulk staging with dynamically claimed chunks (bulk.cuh) once the
// working set is well beyond L2.  Measured on B200 (profiles/r01): light
// 2R+1W chain at 32768^2 7.03 TB/s bulk vs 5.47 on register tiles; C3 7.02
// vs 6.44; C2 reductions 7.15 step; at 4096^2 (1.5x L2) register tiles win
// (7.06 vs 6.89).  Chains flagged RegTiles (tanh, elementwise division) stay
// on register tiles.  FMB200_BULK=0 / 1 forces one path (A/B measurements).
inline int bulk_override() {
  static int v = [] {
    const char *e = getenv("FMB200_BULK");
    return (e && *e) ? atoi(e) : -1;
  }();
  return v;
}
constexpr int64_t kBulkMinBytes = 512ll << 20;
inline bool bulk_wanted(int64_t working_set_bytes, bool reg_tiles) {
  const int ov = bulk_override();
  return ov >= 0 ? ov == 1 : (!reg_tiles && working_set_bytes >= kBulkMinBytes);
}

template <class E>
bool host_fast_ok(const fm_program &P, const void *out) {
  if (!P.flat || P.result_etype != E::kEtype || (((uintptr_t)out) & 15)) return false;
  for (int i = 0; i < P.n_slots; ++i)
    if ((((uintptr_t)P.slots[i].ptr) & 15) || !(P.slots[i].etype == E::kEtype ||
        (sizeof(typename E::Elem) == 4 && (P.slots[i].etype == FM_U32 || P.slots[i].etype == FM_I32))))
      return false;
  return true;
}

template <class E>
int run_copy_bulk(const fm_program &P, void *out, int64_t n_elem, cudaStream_t s) {
  using G = bulk::Geometry<E, bulk::CopyWarps<E>::v>;
  static bool attr = false;
  if (!attr) {
    FM_CHECK(cudaFuncSetAttribute(bulk::k_copy_bulk<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::kSmem));
    attr = true;
  }
  const int64_t chunks = n_elem / G::kChunk;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(chunks, sm_count()));
  const Classified cl = classify(s, P, n_elem, 1, writes_of(out, (size_t)n_elem * etype_bytes(P.result_etype)));
  Scratch sc;
  int st = get_scratch((void *)s, 64, &sc, cl.slot);
  if (st) return st;
  FM_CHECK(launch_pdl(bulk::k_copy_bulk<E>, dim3((unsigned)grid), dim3(bulk::copy_bulk_threads<E>()), G::kSmem, s, cl.P, out,
                      n_elem, sc.counters));
  FM_CHECK_LAUNCH("fused copy kernel (bulk)");
  return 0;
}

// Register VM over bulk-staged chunks (bulk.cuh k_copy_bulk_vm): a flat
// program of <= 8 leaf slots, 16-byte aligned, large enough for a wave of
// chunks.  handled = false: not eligible.
template <class E>
int run_copy_bulk_vm(const fm_program &P0, void *out, int64_t n_elem, cudaStream_t s, bool &handled) {
  handled = false;
  if (!P0.flat || P0.n_slots < 1 || P0.n_slots > 8) return 0;
  fm_program P = P0;
  int bytes_per_elem = 0;
  for (int j = 0; j < P.n_slots; ++j) {
    const fm_slot &sl = P.slots[j];
    if (((uintptr_t)sl.ptr) & 15) return 0;
    bytes_per_elem += etype_bytes(sl.etype);
  }
  // 4 stages in <= 200 KiB; 256-element granules keep every slot's run a
  // 16-byte multiple (TMA bulk copies)
  const int chunk = (200 * 1024 / 4 / bytes_per_elem) / 256 * 256;
  if (chunk < 256 || n_elem < (int64_t)chunk * sm_count()) return 0;
  int off = 0;
  for (int j = 0; j < P.n_slots; ++j) {   // slot j's run inside a stage
    P.slots[j].reserved = off;
    off += chunk * etype_bytes(P.slots[j].etype);
  }
  const int stage_bytes = off, stages = 4;
  const size_t smem = (size_t)stages * stage_bytes + (size_t)stages * 24 + 64;
  static bool attr = false;
  if (!attr) {
    FM_CHECK(cudaFuncSetAttribute(bulk::k_copy_bulk_vm<typename NoPrefetch<E>::type>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
    attr = true;
  }
  const Classified cl = classify(s, P, n_elem, 1, writes_of(out, (size_t)n_elem * etype_bytes(P.result_etype)));
  Scratch sc;
  if (int st = get_scratch((void *)s, 64, &sc, cl.slot)) return st;
  const int64_t grid = std::min<int64_t>(n_elem / chunk, sm_count());
  using EV = typename NoPrefetch<E>::type;
  FM_CHECK(launch_pdl(bulk::k_copy_bulk_vm<EV>, dim3((unsigned)grid), dim3(bulk::VmGeo<EV>::kThreads), smem, s, cl.P,
                      out, n_elem, sc.counters, chunk, stages, stage_bytes));
  FM_CHECK_LAUNCH("fused copy kernel (VM, bulk-staged)");
  handled = true;
  return 0;
}

// Full reduction of a flat program on the VM over bulk-staged chunks
// (bulk.cuh k_accu_bulk_vm); eligibility as run_copy_bulk_vm.
template <class E>
int run_accu_bulk_vm(const fm_program &P0, void *out, int64_t n_elem, int finalize, cudaStream_t s, bool &handled) {
  handled = false;
  if (!P0.flat || P0.n_slots < 1 || P0.n_slots > 8) return 0;
  fm_program P = P0;
  int bytes_per_elem = 0;
  for (int j = 0; j < P.n_slots; ++j) {
    if (((uintptr_t)P.slots[j].ptr) & 15) return 0;
    bytes_per_elem += etype_bytes(P.slots[j].etype);
  }
  const int chunk = (200 * 1024 / 4 / bytes_per_elem) / 256 * 256;
  if (chunk < 256 || n_elem < (int64_t)chunk * sm_count()) return 0;
  int off = 0;
  for (int j = 0; j < P.n_slots; ++j) {
    P.slots[j].reserved = off;
    off += chunk * etype_bytes(P.slots[j].etype);
  }
  const int stage_bytes = off, stages = 4;
  const size_t smem = (size_t)stages * stage_bytes + (size_t)stages * 24 + 64;
  using EV = typename NoPrefetch<E>::type;
  static bool attr = false;
  if (!attr) {
    FM_CHECK(cudaFuncSetAttribute(bulk::k_accu_bulk_vm<EV>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
    attr = true;
  }
  const int64_t grid = std::min<int64_t>(n_elem / chunk, sm_count());
  const int64_t nfull = n_elem / chunk;
  const int64_t ndyn = nfull - (nfull * 3 / 4 / grid) * grid;
  const Classified cl = classify(s, P, n_elem, 1, writes_of(out, 8));
  Scratch sc;
  if (int st = get_scratch((void *)s, (size_t)(grid + ndyn) * (sizeof(double) + sizeof(uint32_t)) + 64, &sc, cl.slot))
    return st;
  double *pd = (double *)sc.payload;
  uint32_t *pu = (uint32_t *)(pd + grid + ndyn);
  FM_CHECK(launch_pdl(bulk::k_accu_bulk_vm<EV>, dim3((unsigned)grid), dim3(bulk::VmGeo<EV>::kThreads), smem, s, cl.P, out,
                      n_elem, finalize, pd, pu, sc.counters, chunk, stages, stage_bytes));
  FM_CHECK_LAUNCH("fused accu kernel (VM, bulk-staged)");
  handled = true;
  return 0;
}

// Tiled, shared-memory staged VM copy (tiled.cuh): the widest column tile
// whose double-buffered slot tiles fit in shared memory.
template <class E, int TC>
int launch_tiled(const fm_program &P, void *out, int64_t n_rows, int64_t n_cols, cudaStream_t s) {
  using G = tiled::Geo<E::kV, TC, E::kWide ? 8 : 4>;
  constexpr int kMaxSmem = 200 * 1024;
  static int occ_slots = -1, occ_blocks = 0;
  const int smem = (int)tiled::smem_bytes<E, TC>(P.n_slots);
  static bool attr = false;
  if (!attr) {
    FM_CHECK(cudaFuncSetAttribute(tiled::k_copy_tiled<E, TC>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    attr = true;
  }
  if (occ_slots != P.n_slots) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, tiled::k_copy_tiled<E, TC>, G::NT, smem) != cudaSuccess ||
        n < 1)
      n = 1;
    occ_slots = P.n_slots;
    occ_blocks = n;
  }
  const int64_t ntiles = cdiv(n_rows, G::TR) * cdiv(n_cols, TC);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)sm_count() * occ_blocks));
  tiled::k_copy_tiled<E, TC><<<(unsigned)grid, G::NT, smem, s>>>(P, out, n_rows, n_cols);
  FM_CHECK_LAUNCH("fused copy kernel (tiled)");
  return 0;
}

template <class E>
int run_copy_tiled(const fm_program &P, void *out, int64_t n_rows, int64_t n_cols, cudaStream_t s) {
  constexpr int64_t kMaxSmem = 200 * 1024;
  // (whole square matrices with transposed leaves take the tile-pair
  // skeleton, pair.cuh, before this)
  if (tiled::smem_bytes<E, 32>(P.n_slots) <= kMaxSmem) return launch_tiled<E, 32>(P, out, n_rows, n_cols, s);
  if (tiled::smem_bytes<E, 16>(P.n_slots) <= kMaxSmem) return launch_tiled<E, 16>(P, out, n_rows, n_cols, s);
  return launch_tiled<E, 8>(P, out, n_rows, n_cols, s);
}

// FMB200_TILED=0 disables the staged VM copy (A/B measurements)
inline bool tiled_enabled() {
  static int v = [] {
    const char *e = getenv("FMB200_TILED");
    return (e && *e) ? atoi(e) : 1;
  }();
  return v != 0;
}

template <class E>
int run_copy(const fm_program &P, void *out, int64_t n_rows, int64_t n_cols, cudaStream_t s) {
  constexpr int V = E::kV;
  if (n_rows == 0 || n_cols == 0) return 0;
  // views / transposes (VM or template): stage through shared memory (for
  // flat many-leaf programs on the VM, staging measured slower -- add8N 3.5
  // -> 1.6 TB/s, the VM's per-instruction cost dominates -- so the add-N
  // chains get AOT templates instead)
  if constexpr (E::kTiled) {
    // transposed leaves need the staged tile; views alone read their column
    // runs directly (vector loads in load_slot)
    bool transposed = false;
    for (int j = 0; j < P.n_slots; ++j) transposed |= P.slots[j].transposed != 0;
    // whole square matrices read plain and transposed: tile pairs, every
    // input block staged once by TMA (pair.cuh)
    if (transposed && pair_eligible(P, n_rows, n_cols)) {
      bool handled = false;
      if (int st = run_copy_pair<E>(P, out, n_rows, s, handled)) return st;
      if (handled) return 0;
    }
    if (tiled_enabled() && transposed && n_rows * n_cols >= 4096) return run_copy_tiled<E>(P, out, n_rows, n_cols, s);
  }
  if constexpr (E::kIsVm) {
    bool handled = false;
    if (int st = run_copy_bulk_vm<E>(P, out, n_rows * n_cols, s, handled)) return st;
    if (handled) return 0;
  }
  if constexpr (E::kFast) {
    if constexpr (bulk::Geometry<E>::kOk) {
      const int64_t n = n_rows * n_cols;
      if (bulk_wanted(n * (E::kNin + 1) * (int64_t)sizeof(typename E::Elem), E::kRegTiles) && P.n_slots == E::kNin &&
          host_fast_ok<E>(P, out) && n >= (int64_t)bulk::Geometry<E>::kChunk * sm_count())
        return run_copy_bulk<E>(P, out, n, s);
    }
  }
  const int64_t nrb = cdiv(n_rows, V);
  const int64_t nch = P.flat ? cdiv(n_rows * n_cols, V) : nrb * n_cols;
  const int64_t grid = wave_grid<GridTag<E, 0>>(k_copy<E>, cdiv(nch, kThreads));
  const Classified cl =
      classify(s, P, n_rows, n_cols, writes_of(out, (size_t)(n_rows * n_cols) * etype_bytes(P.result_etype)));
  FM_CHECK(launch_pdl(k_copy<E>, dim3((unsigned)grid), dim3(kThreads), 0, s, cl.P, out, n_rows, n_cols));
  FM_CHECK_LAUNCH("fused copy kernel");
  return 0;
}

template <class E>
int run_accu_bulk(const fm_program &P, void *out, int64_t n_elem, int finalize, cudaStream_t s) {
  using G = bulk::Geometry<E>;
  static bool attr = false;
  if (!attr) {
    FM_CHECK(cudaFuncSetAttribute(bulk::k_accu_bulk<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::kSmem));
    attr = true;
  }
  const int64_t chunks = n_elem / G::kChunk;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(chunks, sm_count()));
  // static head: 80 % of the chunks round-robin (summed per CTA), the rest
  // claimed dynamically with one partial slot each
  static const int64_t static_pct = [] {
    const char *e = getenv("FMB200_BULK_STATIC_PCT");
    return (int64_t)((e && *e) ? std::min(100, std::max(0, atoi(e))) : 80);
  }();
  const int64_t nstat = chunks * static_pct / 100 / grid;
  const int64_t ndyn = chunks - nstat * grid;
  const Classified cl = classify(s, P, n_elem, 1, writes_of(out, 8));
  Scratch sc;
  int st = get_scratch((void *)s, (grid + ndyn) * sizeof(double) + 64, &sc, cl.slot);
  if (st) return st;
  double *part_d = (double *)sc.payload;
  FM_CHECK(launch_pdl(bulk::k_accu_bulk<E>, dim3((unsigned)grid), dim3(bulk::kBulkThreads), G::kSmem, s, cl.P, out,
                      n_elem, finalize, part_d, part_d + grid, nstat, sc.counters));
  FM_CHECK_LAUNCH("fused accu kernel (bulk)");
  return 0;
}

template <class E>
int run_accu(const fm_program &P, void *out, int64_t n_rows, int64_t n_cols, int finalize,
             cudaStream_t s) {
  constexpr int V = E::kV;
  if constexpr (E::kIsVm) {
    bool handled = false;
    if (int st = run_accu_bulk_vm<E>(P, out, n_rows * n_cols, finalize, s, handled)) return st;
    if (handled) return 0;
  }
  if constexpr (E::kFast) {
    if constexpr (bulk::Geometry<E>::kOk) {
      const int64_t n = n_rows * n_cols;
      if (bulk_wanted(n * E::kNin * (int64_t)sizeof(typename E::Elem), E::kRegTiles) && P.n_slots == E::kNin &&
          host_fast_ok<E>(P, nullptr) && n >= (int64_t)bulk::Geometry<E>::kChunk * sm_count())
        return run_accu_bulk<E>(P, out, n, finalize, s);
    }
  }
  const int64_t nrb = cdiv(n_rows, V);
  const int64_t nch = P.flat ? cdiv(n_rows * n_cols, V) : nrb * n_cols;
  const int64_t grid = wave_grid<GridTag<E, 1>>(k_accu<E>, cdiv(nch, kThreads));
  const Classified cl = classify(s, P, n_rows, n_cols, writes_of(out, 8));
  Scratch sc;
  int st = get_scratch((void *)s, grid * (sizeof(double) + sizeof(uint32_t)) + 64, &sc, cl.slot);
  if (st) return st;
  double *pd = (double *)sc.payload;
  uint32_t *pu = (uint32_t *)(pd + grid);
  FM_CHECK(launch_pdl(k_accu<E>, dim3((unsigned)grid), dim3(kThreads), 0, s, cl.P, out, n_rows, n_cols, finalize, pd,
                      pu, sc.counters));
  FM_CHECK_LAUNCH("fused accu kernel");
  return 0;
}

template <class E>
int run_reduce_dim(const fm_program &P, int dim, int64_t n_rows, int64_t n_cols, const ReduceOuts &R,
                   cudaStream_t s) {
  constexpr int V = E::kV;
  if (n_rows == 0 || n_cols == 0) {
    return 0;
  }
  if (dim == 0) {
    if constexpr (E::kFast) {
      using T = typename E::Elem;
      if (host_fast_ok<E>(P, nullptr) && ((n_rows * (int64_t)sizeof(T)) & 15) == 0 && n_rows % E::kTile == 0 &&
          n_rows < 0xFFFFFFFFll) {
        // 3 CTAs per SM (C4, 65536 x 16384 f64: 2 -> 7.01, 3 -> 7.38, 4 -> 7.23,
        // 6 -> 7.24 TB/s); FMB200_COLS_BLOCKS_PER_SM overrides
        static const int per_sm = [] {
          const char *e = getenv("FMB200_COLS_BLOCKS_PER_SM");
          return (e && *e) ? std::max(1, atoi(e)) : 3;
        }();
        const int64_t grid = std::min<int64_t>(std::min<int64_t>(n_cols, (int64_t)sm_count() * per_sm),
                                               wave_grid<GridTag<E, 4>>(k_reduce_cols_fast<E>, n_cols));
        const fm_program Pc = classify(s, P, n_rows, n_cols, reduce_writes(R, n_cols)).P;
        FM_CHECK(launch_pdl(k_reduce_cols_fast<E>, dim3((unsigned)grid), dim3(kThreads), 0, s, Pc, R, n_rows, n_cols));
        FM_CHECK_LAUNCH("fused column-reduction kernel (typed)");
        return 0;
      }
    }
    // one persistent wave; columns are the work units (C4: 16384 / 444)
    const int64_t grid = wave_grid<GridTag<E, 2>>(k_reduce_cols<E>, n_cols);
    const fm_program Pc = classify(s, P, n_rows, n_cols, reduce_writes(R, n_cols)).P;
    FM_CHECK(launch_pdl(k_reduce_cols<E>, dim3((unsigned)grid), dim3(kThreads), 0, s, Pc, R, n_rows, n_cols));
    FM_CHECK_LAUNCH("fused column-reduction kernel");
    return 0;
  }
  const int64_t gx = cdiv(n_rows, (int64_t)kThreads * V);
  if (gx > 65535 * 1024LL) return fail_msg("reduce_dim: too many rows");
  // typed fast path: a TMA-bulk ring of `depth` columns per block (the
  // deepest of 8..3 that still fits two CTAs per SM)
  int depth = 0;
  size_t smem = 0;
  if constexpr (E::kFast) {
    using T = typename E::Elem;
    if (host_fast_ok<E>(P, nullptr) && ((n_rows * (int64_t)sizeof(T)) & 15) == 0 && n_rows % (kThreads * V) == 0) {
      const size_t per_col = (size_t)E::kNin * E::kV * sizeof(T) * kThreads;
      for (int d = 8; d >= 3; --d)
        if (d * per_col + 8 * d <= 100 * 1024) { depth = d; break; }
      smem = depth * per_col + 8 * (size_t)depth;
      static bool attr = false;
      if (depth && !attr) {
        FM_CHECK(cudaFuncSetAttribute(k_reduce_rows<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
        attr = true;
      }
    }
  }
  // column splits so enough CTAs per SM stream concurrently: c4r (65536 x
  // 16384 f64), register path 2 -> 4.74, 4 -> 5.80, 8 -> 6.13, 16 -> 6.37,
  // 32 -> 5.95 TB/s; staged path 2 -> 5.93, 4 -> 6.67, 6 -> 6.76,
  // 8 -> 6.79, 16 -> 6.44 (longer column runs per CTA)
  static const int64_t per_sm_env = [] {
    const char *e = getenv("FMB200_ROW_SPLITS_PER_SM");
    return (int64_t)((e && *e) ? std::max(1, atoi(e)) : 0);
  }();
  const int64_t per_sm = per_sm_env ? per_sm_env : (depth ? 8 : 16);
  int64_t splits = std::max<int64_t>(1, cdiv((int64_t)sm_count() * per_sm, gx));
  if (depth && !per_sm_env) {
    // staged path: keep >= ~384 columns per CTA (the ring's ramp and the
    // partial combine amortise over the run; 16384 x 8192 f64: 74 splits
    // 2.9 TB/s, 19 splits 5.1) while still filling two CTAs per SM
    const int64_t fill = cdiv(2 * (int64_t)sm_count(), gx);
    splits = std::min(splits, std::max(fill, n_cols / 384));
  }
  splits = std::max<int64_t>(1, std::min<int64_t>(splits, std::min<int64_t>(n_cols, 65535)));
  RowPartial *part = nullptr;
  unsigned *counters = nullptr;
  if (splits > 1) {
    Scratch sc;
    int st = get_scratch((void *)s, (size_t)(splits * n_rows) * sizeof(RowPartial), &sc);
    if (st) return st;
    if ((size_t)gx * sizeof(unsigned) > 64 * 1024) return fail_msg("reduce_dim: counter space exhausted");
    part = (RowPartial *)sc.payload;
    counters = sc.counters;
  }
  dim3 grid((unsigned)gx, (unsigned)splits);
  k_reduce_rows<E><<<grid, kThreads, smem, s>>>(P, R, n_rows, n_cols, part, counters, depth);
  FM_CHECK_LAUNCH("fused row-reduction kernel");
  return 0;
}

// Registry of ahead-of-time template kernels (templates.cu, generated).
enum { SK_COPY = 0, SK_ACCU = 1, SK_DIM0 = 2, SK_DIM1 = 3 };
struct TemplateEntry {
  const char *signature;   // bare expression signature (exprtree.signature_of)
  int (*copy)(const fm_program &, void *, int64_t, int64_t, cudaStream_t);
  int (*accu)(const fm_program &, void *, int64_t, int64_t, int, cudaStream_t);
  int (*reduce_dim)(const fm_program &, int, int64_t, int64_t, const ReduceOuts &, cudaStream_t);
  int n_inputs;
  int etype;
};
const TemplateEntry *template_table(int *n);

}  // namespace fm

#include "split.cuh"
