// bulk.cuh -- TMA-bulk-staged copy skeleton for compute-heavy fused chains.
//
// The register-tile copy path (k_copy fast path) keeps one warp tile in
// flight per warp, so its memory parallelism is bounded by registers and
// occupancy.  For chains whose per-element math is long (a transcendental,
// e.g. C3's exp), the warps spend most of their time computing and the loads
// in flight fall below what HBM3e needs (profiles/r01/ncu_c3_copy.txt:
// long-scoreboard stalls, 77 % DRAM throughput).  This skeleton decouples the
// two: one producer warp streams fixed-size chunks of every input into a
// ring of shared-memory stages with `cp.async.bulk` (TMA bulk copies,
// completion counted on an mbarrier), and the consumer warps evaluate the
// expression out of shared memory and store the results with 128-bit
// coalesced st.global.  Bytes in flight per SM = (stages-1) x chunk x inputs,
// independent of the consumers' register use.
//
// Persistent: one CTA per SM.  SMs drain HBM at visibly different rates
// (ncu, profiles/r01/ncu_c2_accu_f32: per-SM active cycles 175K..229K for
// equal static shares), so only a static head of the chunks is assigned
// round-robin; the rest are claimed dynamically (one atomicAdd per chunk,
// fetched a chunk ahead by the producer), so fast SMs take more.  Copies are
// deterministic regardless; reductions keep a fixed summation order by
// summing the static head per CTA and each dynamic chunk into its own
// partial slot, combined in chunk order.  The ragged tail (< one chunk) is
// evaluated by the consumers with the general chunk path.
#pragma once
#include "skeletons.cuh"

namespace fm {
namespace bulk {

constexpr int kConsumerWarps = 16;
constexpr int kBulkThreads = (kConsumerWarps + 1) * 32;
constexpr int kChunkBytesMax = 16384;     // per input per stage (<= 4 inputs)
constexpr int kSmemBudget = 192 * 1024;

FM_DEV uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
FM_DEV void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
FM_DEV void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
FM_DEV void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
FM_DEV void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
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
// global -> shared bulk copy (TMA, no tensor map), completion on `bar`;
// evict-first: every input byte is read exactly once.
FM_DEV void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
FM_DEV uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

template <class E, int NW = kConsumerWarps>
struct Geometry {
  using T = typename E::Elem;
  static constexpr int kWarps = NW;
  static constexpr int kNin = E::kNin;
  // 16 consumer warps: 32 / 16 / 8 KiB per input; other warp counts: whole
  // 16-byte vectors for every consumer lane (2 or 1 per lane per input)
  static constexpr int kChunkBytes =
      NW == kConsumerWarps ? (kNin <= 2 ? 2 * kChunkBytesMax : (kNin <= 4 ? kChunkBytesMax : kChunkBytesMax / 2))
                           : (kNin <= 2 ? 2 : 1) * 16 * 32 * NW;
  static constexpr int kChunk = kChunkBytes / (int)sizeof(T);               // elements per chunk
  static constexpr int kStagesRaw = kSmemBudget / (kChunkBytes * (kNin > 0 ? kNin : 1));
  static constexpr int kStages = kStagesRaw > 8 ? 8 : (kStagesRaw < 2 ? 2 : kStagesRaw);
  static constexpr int kSmem = kStages * kNin * kChunkBytes + 3 * kStages * 8 + 128;
  static constexpr int kW = 16 / (int)sizeof(T);                            // elements per vector
  static constexpr int kVecPerThread = kChunk / kW / (NW * 32);
  static_assert(kChunk % (kW * NW * 32) == 0, "chunk splits evenly over consumers");
  static constexpr bool kOk = kNin <= 8 && kSmem <= 200 * 1024;             // fits the ring
};

// shared-memory ring: [stage][input] chunks, then full[S] / empty[S] mbarriers
template <class E, int NW = kConsumerWarps>
struct Ring {
  using G = Geometry<E, NW>;
  unsigned char *base;
  uint64_t *full, *empty;
  int64_t *cid;          // chunk held by each stage (-1: no more chunks)
  FM_DEV explicit Ring(unsigned char *smem) {
    base = smem;
    full = (uint64_t *)(smem + G::kStages * G::kNin * G::kChunkBytes);
    empty = full + G::kStages;
    cid = (int64_t *)(empty + G::kStages);
  }
  FM_DEV const unsigned char *chunk(int s, int i) const { return base + (s * G::kNin + i) * G::kChunkBytes; }
  FM_DEV void init() {
    if (threadIdx.x == 0) {
      for (int s = 0; s < G::kStages; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], NW);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  // producer (one elected lane): the static head, chunks blockIdx.x + j*grid
  // for j < nstat, then dynamic chunks nstat*grid + atomicAdd(ctr, 1) until
  // nfull, then a sentinel stage (cid = -1, plain arrive).
  FM_DEV void produce(const fm_program &P, int64_t nfull, int64_t nstat, unsigned *ctr) {
    using T = typename E::Elem;
    constexpr int S = G::kStages;
    const uint64_t pol = evict_first_policy();
    int64_t k = 0;
    auto stage_for = [&](int64_t kk) {
      const int s = (int)(kk % S);
      if (kk >= S) mbar_wait(&empty[s], (uint32_t)(((kk / S) & 1) ^ 1));
      return s;
    };
    auto issue = [&](int64_t c) {
      const int s = stage_for(k++);
      cid[s] = c;
      mbar_expect_tx(&full[s], G::kNin * G::kChunkBytes);
#pragma unroll
      for (int i = 0; i < G::kNin; ++i)
        bulk_g2s((void *)chunk(s, i), (const T *)P.slots[i].ptr + c * G::kChunk, G::kChunkBytes, &full[s], pol);
    };
    for (int64_t j = 0; j < nstat; ++j) issue(blockIdx.x + j * gridDim.x);
    const int64_t dbase = nstat * gridDim.x;
    int64_t c = dbase + atomicAdd(ctr, 1u);
    while (c < nfull) {
      const int64_t next = dbase + atomicAdd(ctr, 1u);   // claim ahead: the atomic overlaps the slot wait
      issue(c);
      c = next;
    }
    const int s = stage_for(k);
    cid[s] = -1;
    mbar_arrive(&full[s]);
  }
  // consumer: evaluate the kVecPerThread x kW elements of this thread in chunk stage s
  FM_DEV void eval(const fm_program &P, int s, int ctid, typename E::Elem (&r)[G::kVecPerThread][G::kW]) const {
    using T = typename E::Elem;
    constexpr int NIN = G::kNin;
#pragma unroll
    for (int j = 0; j < G::kVecPerThread; ++j) {
      const int q = ctid + j * NW * 32;
      uint4 w[NIN];
#pragma unroll
      for (int i = 0; i < NIN; ++i) w[i] = *(const uint4 *)(chunk(s, i) + q * 16);
#pragma unroll
      for (int e = 0; e < G::kW; ++e) {
        T x[NIN];
#pragma unroll
        for (int i = 0; i < NIN; ++i) {
          if constexpr (sizeof(T) == 8) x[i] = e == 0 ? u2d(w[i].x, w[i].y) : u2d(w[i].z, w[i].w);
          else x[i] = u2f(e == 0 ? w[i].x : e == 1 ? w[i].y : e == 2 ? w[i].z : w[i].w);
        }
        r[j][e] = E::ev_elem(P, x);
      }
    }
  }
  FM_DEV void release(int s) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
  }
};

// Consumer warps of the bulk copy: transcendental f32 chains of <= 4 inputs
// (sigmoid, swish, gelu: one exp / tanh per element evaluated in f64) stall on
// the dependent FP64 chain ("wait" is the top stall at 16 warps,
// profiles/r02/ncu_suite_sigmoid.txt), so they run 31 (1024 threads with the
// producer warp, <= 64 registers, no spills): expr3 3.03 -> 3.72 TB/s (24
// warps: 3.39), sigmoid 4.74 -> 4.86, C3 unchanged.
template <class E>
struct CopyWarps {
  static constexpr int v = (E::kHeavy && sizeof(typename E::Elem) == 4 && E::kNin <= 4) ? 31 : kConsumerWarps;
};
template <class E> constexpr int copy_bulk_threads() { return (CopyWarps<E>::v + 1) * 32; }

template <class E>
__global__ void __launch_bounds__(copy_bulk_threads<E>(), 1)
    k_copy_bulk(const __grid_constant__ fm_program P, void *out, int64_t n_elem, unsigned *counters) {
  constexpr int NW = CopyWarps<E>::v;
  using G = Geometry<E, NW>;
  using T = typename E::Elem;
  constexpr int S = G::kStages, C = G::kChunk;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Ring<E, NW> ring(smem_raw);
  ring.init();
  const int indep = P.reserved & 1;   // launch-window class (common.cuh)
  pdl_enter(indep);
  const int warp = threadIdx.x >> 5;
  const int64_t nfull = n_elem / C;
  unsigned *ctr = counters, *done = counters + 1;
  if (warp == NW) {
    if ((threadIdx.x & 31) == 0) ring.produce(P, nfull, 0, ctr);   // all dynamic: copies are order-free
  } else {
  const int ctid = threadIdx.x;   // 0 .. NW*32-1
  for (int64_t k = 0;; ++k) {
    const int s = (int)(k % S);
    mbar_wait(&ring.full[s], (uint32_t)((k / S) & 1));
    const int64_t c = ring.cid[s];
    if (c < 0) break;
    T r[G::kVecPerThread][G::kW];
    ring.eval(P, s, ctid, r);
    ring.release(s);   // smem reads done: free the stage before the long-latency stores
    T *o = (T *)out + c * C;
#pragma unroll
    for (int j = 0; j < G::kVecPerThread; ++j) {
      const int q = ctid + j * NW * 32;
      if constexpr (sizeof(T) == 8) {
        uint32_t a0, a1, b0, b1;
        d2u(r[j][0], a0, a1);
        d2u(r[j][1], b0, b1);
        st_v4(o + q * 2, a0, a1, b0, b1);
      } else {
        st_v4(o + q * 4, f2u(r[j][0]), f2u(r[j][1]), f2u(r[j][2]), f2u(r[j][3]));
      }
    }
  }

  // ---- ragged tail: fewer than one chunk, general path, block 0 only ----
  if (blockIdx.x == 0) {
    constexpr int V = E::kV;
    const int64_t base = nfull * C;
    for (int64_t e0 = base + (int64_t)ctid * V; e0 < n_elem; e0 += (int64_t)NW * 32 * V) {
      Chunk ch;
      ch.base = e0;
      ch.cnt = (int)min((int64_t)V, n_elem - e0);
      ch.row0 = 0; ch.col = 0; ch.flat = true;
      uint32_t lo[V], hi[V];
      E::eval(P, ch, lo, hi);
      store_chunk<V>(out, P.result_etype, ch.base, ch.cnt, lo, hi);
    }
  }
  }
  // the last CTA out resets the chunk counter for the next launch on this stream
  __syncthreads();
  if (blockIdx.x == 0) pdl_exit(indep);
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      *ctr = 0u;
      *done = 0u;
    }
  }
}


// Fused full reduction over bulk-staged chunks: per-thread f64 accumulation
// (the reduce_accu accumulator type, codegen.py:47-49).  The static head is
// summed per CTA (warp trees + block tree -> part_d[cta]); every dynamic chunk
// gets its own partial (warp trees, then one thread over the warps in order
// -> part_c[chunk - head]).  The last CTA combines part_d in CTA order and
// part_c in chunk order: one launch, and the result does not depend on which
// CTA claimed which dynamic chunk.
template <class E>
__global__ void __launch_bounds__(kBulkThreads, 1)
    k_accu_bulk(const __grid_constant__ fm_program P, void *out, int64_t n_elem, int finalize,
                double *part_d, double *part_c, int64_t nstat, unsigned *counters) {
  using G = Geometry<E>;
  using T = typename E::Elem;
  constexpr int S = G::kStages, C = G::kChunk;
  constexpr int NW = kConsumerWarps;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double smd[NW];
  __shared__ double wsum[2][NW];
  __shared__ bool last;
  Ring<E> ring(smem_raw);
  ring.init();
  const int indep = P.reserved & 1;   // launch-window class (common.cuh)
  pdl_enter(indep);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nfull = n_elem / C;
  const int64_t dbase = nstat * gridDim.x;
  unsigned *done = counters, *ctr = counters + 1;
  double acc = 0.0;
  if (warp == NW) {
    if (lane == 0) ring.produce(P, nfull, nstat, ctr);
  } else {
    const int ctid = threadIdx.x;
    int par = 0;
    for (int64_t k = 0;; ++k) {
      const int s = (int)(k % S);
      mbar_wait(&ring.full[s], (uint32_t)((k / S) & 1));
      const int64_t c = ring.cid[s];
      if (c < 0) break;
      T r[G::kVecPerThread][G::kW];
      ring.eval(P, s, ctid, r);
      ring.release(s);
      if (c < dbase) {
#pragma unroll
        for (int j = 0; j < G::kVecPerThread; ++j)
#pragma unroll
          for (int e = 0; e < G::kW; ++e) acc = add_d(acc, (double)r[j][e]);
      } else {
        double a = 0.0;
#pragma unroll
        for (int j = 0; j < G::kVecPerThread; ++j)
#pragma unroll
          for (int e = 0; e < G::kW; ++e) a = add_d(a, (double)r[j][e]);
        a = warp_sum_d(a);
        if (lane == 0) wsum[par][warp] = a;
        asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");   // consumer warps only
        if (ctid == 0) {
          double t = 0.0;
#pragma unroll
          for (int w = 0; w < NW; ++w) t = add_d(t, wsum[par][w]);
          part_c[c - dbase] = t;
        }
        par ^= 1;
      }
    }
    if (blockIdx.x == gridDim.x - 1) {   // ragged tail (< one chunk): general path
      constexpr int V = E::kV;
      for (int64_t e0 = nfull * C + (int64_t)ctid * V; e0 < n_elem; e0 += (int64_t)NW * 32 * V) {
        Chunk ch;
        ch.base = e0;
        ch.cnt = (int)min((int64_t)V, n_elem - e0);
        ch.row0 = 0; ch.col = 0; ch.flat = true;
        uint32_t lo[V], hi[V];
        E::eval(P, ch, lo, hi);
#pragma unroll
        for (int v = 0; v < V; ++v)
          if (v < ch.cnt) acc = add_d(acc, as_double(P.result_etype, lo[v], hi[v]));
      }
    }
  }
  // block tree over the consumer warps (the producer contributes 0)
  acc = warp_sum_d(acc);
  __syncthreads();
  if (lane == 0 && warp < NW) smd[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < NW; ++w) b = add_d(b, smd[w]);
    part_d[blockIdx.x] = b;
    __threadfence();
    last = (atomicAdd(done, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (blockIdx.x == 0) pdl_exit(indep);
  if (!last) return;
  __threadfence();
  // combine: per-CTA partials then per-chunk partials, each thread over a
  // fixed strided subset, then fixed trees
  const int64_t ndyn = nfull - dbase;
  // The partials were written by other SMs: read them through L2 (ld.cg),
  // kU independent loads in flight per thread, then added in the same fixed
  // order (thread t: t, t + T, t + 2T, ...) -- the tail of the launch is
  // these loads' latency, so they must not serialise one per add.
  constexpr int kU = 8;
  double sd = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += kBulkThreads) sd = add_d(sd, __ldcg(part_d + i));
  double sc = 0.0;
  for (int64_t i0 = threadIdx.x; i0 < ndyn; i0 += (int64_t)kU * kBulkThreads) {
    double v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + (int64_t)u * kBulkThreads;
      v[u] = i < ndyn ? __ldcg(part_c + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i0 + (int64_t)u * kBulkThreads < ndyn) sc = add_d(sc, v[u]);
  }
  sd = warp_sum_d(sd);
  sc = warp_sum_d(sc);
  __shared__ double fin_d[kBulkThreads / 32], fin_c[kBulkThreads / 32];
  if (lane == 0) { fin_d[warp] = sd; fin_c[warp] = sc; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kBulkThreads / 32; ++w) { a = add_d(a, fin_d[w]); b = add_d(b, fin_c[w]); }
    double total = add_d(a, b);
    if (finalize == FM_FINAL_SQRT) total = sqrt_d(total);
    *(double *)out = total;
    *done = 0u;
    *ctr = 0u;
  }
}

// ---- register VM over bulk-staged chunks (flat programs) ----------------------
// The VM's chunk path keeps only its prefetched slots in flight per thread;
// with ~158 registers one 256-thread CTA fits an SM and C1 on the VM ran at
// 2.0 TB/s, 22 % DRAM, 23 % issue (profiles/r02/ncu_vm_c1).  Here a producer
// lane streams chunks of EVERY slot (any element widths, chunk_elems
// elements each) into a ring with TMA bulk copies, chunks claimed
// dynamically, and kVmWarps consumer warps run the VM out of shared memory
// (Chunk::bstage: slot j's data at stage + slot.reserved), storing straight
// to HBM.  Memory parallelism no longer depends on the VM's register use.
// consumer warps: 16 for 32-bit VMs (<= 120 registers each); the 64-bit
// VMs carry twice the stack and keep 8 (<= 224 registers, no spills)
template <class E> struct VmGeo {
  static constexpr int kWarps = E::kWide ? 8 : 16;
  static constexpr int kThreads = (kWarps + 1) * 32;
};

template <class E>
__global__ void __launch_bounds__(VmGeo<E>::kThreads, 1)
    k_copy_bulk_vm(const __grid_constant__ fm_program P, void *out, int64_t n_elem, unsigned *counters,
                   int chunk_elems, int stages, int stage_bytes) {
  constexpr int V = E::kV;
  extern __shared__ __align__(128) unsigned char vsm[];
  uint64_t *full = (uint64_t *)(vsm + (size_t)stages * stage_bytes);
  uint64_t *empty = full + stages;
  int64_t *cid = (int64_t *)(empty + stages);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], VmGeo<E>::kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int indep = P.reserved & 1;   // launch-window class (common.cuh)
  pdl_enter(indep);
  const int warp = threadIdx.x >> 5;
  const int64_t nfull = n_elem / chunk_elems;
  unsigned *ctr = counters, *done = counters + 1;
  if (warp == VmGeo<E>::kWarps) {
    if ((threadIdx.x & 31) == 0) {
      const uint64_t pol = evict_first_policy();
      int64_t k = 0;
      auto stage_for = [&](int64_t kk) {
        const int st = (int)(kk % stages);
        if (kk >= stages) mbar_wait(&empty[st], (uint32_t)(((kk / stages) & 1) ^ 1));
        return st;
      };
      auto issue = [&](int64_t c) {
        const int st = stage_for(k++);
        cid[st] = c;
        mbar_expect_tx(&full[st], (uint32_t)stage_bytes);
        for (int j = 0; j < P.n_slots; ++j) {
          const fm_slot &sl = P.slots[j];
          const int w = sl.etype == FM_F64 ? 8 : (sl.etype == FM_BF16 ? 2 : 4);
          bulk_g2s(vsm + (size_t)st * stage_bytes + sl.reserved, (const unsigned char *)sl.ptr + c * chunk_elems * w,
                   (uint32_t)chunk_elems * w, &full[st], pol);
        }
      };
      // a static head of the chunks round-robin (no claim round trip per
      // chunk: 148 producers on one counter made the claim the bottleneck),
      // the rest claimed dynamically so fast SMs take more
      const int64_t nstat = nfull * 3 / 4 / gridDim.x;
      for (int64_t j = 0; j < nstat; ++j) issue(blockIdx.x + j * gridDim.x);
      const int64_t dbase = nstat * gridDim.x;
      int64_t c = dbase + atomicAdd(ctr, 1u);
      while (c < nfull) {
        const int64_t next = dbase + atomicAdd(ctr, 1u);
        issue(c);
        c = next;
      }
      const int st = stage_for(k);
      cid[st] = -1;
      mbar_arrive(&full[st]);
    }
  } else {
    const int ctid = threadIdx.x;
    const int groups = chunk_elems / V;
    for (int64_t k = 0;; ++k) {
      const int st = (int)(k % stages);
      mbar_wait(&full[st], (uint32_t)((k / stages) & 1));
      const int64_t c = cid[st];
      if (c < 0) break;
      for (int g = ctid; g < groups; g += VmGeo<E>::kWarps * 32) {
        Chunk ch;
        ch.flat = true;
        ch.base = c * chunk_elems + (int64_t)g * V;
        ch.cnt = V;
        ch.row0 = 0;
        ch.col = 0;
        ch.bstage = vsm + (size_t)st * stage_bytes;
        ch.boff = g * V;
        uint32_t lo[V], hi[V];
        E::eval(P, ch, lo, hi);
        store_chunk<V>(out, P.result_etype, ch.base, V, lo, hi);
      }
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[st]);
    }
    // ragged tail (< one chunk): block 0, the VM's global-memory path
    if (blockIdx.x == 0) {
      for (int64_t e0 = nfull * chunk_elems + (int64_t)ctid * V; e0 < n_elem; e0 += (int64_t)VmGeo<E>::kWarps * 32 * V) {
        Chunk ch;
        ch.base = e0;
        ch.cnt = (int)min((int64_t)V, n_elem - e0);
        ch.row0 = 0; ch.col = 0; ch.flat = true;
        uint32_t lo[V], hi[V];
        E::eval(P, ch, lo, hi);
        store_chunk<V>(out, P.result_etype, ch.base, ch.cnt, lo, hi);
      }
    }
  }
  // the last CTA out resets the chunk counter for the next launch on this slot
  __syncthreads();
  if (blockIdx.x == 0) pdl_exit(indep);
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      *ctr = 0u;
      *done = 0u;
    }
  }
}

// Full reduction on the register VM over bulk-staged chunks (accu of a flat
// program with no template): the same producer / consumer ring as
// k_copy_bulk_vm; a static head of chunks round-robin summed per CTA, the
// rest claimed dynamically with one partial slot each (fixed summation order
// within a chunk), combined in chunk order by the last CTA -- deterministic
// for a given grid, like k_accu_bulk.  Floats accumulate in f64, integers
// wrap in 32 bits (codegen.py:47-49).
template <class E>
__global__ void __launch_bounds__(VmGeo<E>::kThreads, 1)
    k_accu_bulk_vm(const __grid_constant__ fm_program P, void *out, int64_t n_elem, int finalize, double *part_d,
                   uint32_t *part_u, unsigned *counters, int chunk_elems, int stages, int stage_bytes) {
  constexpr int V = E::kV;
  constexpr int NW = VmGeo<E>::kWarps;
  extern __shared__ __align__(128) unsigned char vsm[];
  uint64_t *full = (uint64_t *)(vsm + (size_t)stages * stage_bytes);
  uint64_t *empty = full + stages;
  int64_t *cid = (int64_t *)(empty + stages);
  __shared__ double wd[2][NW];
  __shared__ uint32_t wu[2][NW];
  __shared__ double smd[NW + 1];
  __shared__ uint32_t smu[NW + 1];
  __shared__ bool last;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int indep = P.reserved & 1;
  pdl_enter(indep);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rt = P.result_etype;
  const bool fl = is_float_etype(rt);
  const int64_t nfull = n_elem / chunk_elems;
  const int64_t nstat = nfull * 3 / 4 / gridDim.x;
  const int64_t dbase = nstat * gridDim.x;
  double *part_c = part_d + gridDim.x;       // one slot per dynamic chunk
  uint32_t *part_cu = part_u + gridDim.x;
  unsigned *done = counters, *ctr = counters + 1;
  double accd = 0.0;
  uint32_t accu = 0;
  if (warp == NW) {
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int64_t k = 0;
      auto stage_for = [&](int64_t kk) {
        const int st = (int)(kk % stages);
        if (kk >= stages) mbar_wait(&empty[st], (uint32_t)(((kk / stages) & 1) ^ 1));
        return st;
      };
      auto issue = [&](int64_t c) {
        const int st = stage_for(k++);
        cid[st] = c;
        mbar_expect_tx(&full[st], (uint32_t)stage_bytes);
        for (int j = 0; j < P.n_slots; ++j) {
          const fm_slot &sl = P.slots[j];
          const int w = sl.etype == FM_F64 ? 8 : (sl.etype == FM_BF16 ? 2 : 4);
          bulk_g2s(vsm + (size_t)st * stage_bytes + sl.reserved, (const unsigned char *)sl.ptr + c * chunk_elems * w,
                   (uint32_t)chunk_elems * w, &full[st], pol);
        }
      };
      for (int64_t j = 0; j < nstat; ++j) issue(blockIdx.x + j * gridDim.x);
      int64_t c = dbase + atomicAdd(ctr, 1u);
      while (c < nfull) {
        const int64_t next = dbase + atomicAdd(ctr, 1u);
        issue(c);
        c = next;
      }
      const int st = stage_for(k);
      cid[st] = -1;
      mbar_arrive(&full[st]);
    }
  } else {
    const int ctid = threadIdx.x;
    const int groups = chunk_elems / V;
    int par = 0;
    for (int64_t k = 0;; ++k) {
      const int st = (int)(k % stages);
      mbar_wait(&full[st], (uint32_t)((k / stages) & 1));
      const int64_t c = cid[st];
      if (c < 0) break;
      double cd = 0.0;
      uint32_t cu = 0;
      for (int g = ctid; g < groups; g += NW * 32) {
        Chunk ch;
        ch.flat = true;
        ch.base = c * chunk_elems + (int64_t)g * V;
        ch.cnt = V;
        ch.row0 = 0;
        ch.col = 0;
        ch.bstage = vsm + (size_t)st * stage_bytes;
        ch.boff = g * V;
        uint32_t lo[V], hi[V];
        E::eval(P, ch, lo, hi);
        if (fl) {
#pragma unroll
          for (int v = 0; v < V; ++v) cd = add_d(cd, as_double(rt, lo[v], hi[v]));
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) cu += lo[v];
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (c < dbase) {
        accd = add_d(accd, cd);
        accu += cu;
      } else {
        // dynamic chunk: its own partial, reduced in a fixed order
        cd = warp_sum_d(cd);
        cu = warp_sum_u(cu);
        if (lane == 0) { wd[par][warp] = cd; wu[par][warp] = cu; }
        asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");   // consumer warps only
        if (ctid == 0) {
          double t = 0.0;
          uint32_t tu = 0;
          for (int w = 0; w < NW; ++w) { t = add_d(t, wd[par][w]); tu += wu[par][w]; }
          part_c[c - dbase] = t;
          part_cu[c - dbase] = tu;
        }
        par ^= 1;
      }
    }
    if (blockIdx.x == gridDim.x - 1) {   // ragged tail (< one chunk): the VM's global-memory path
      for (int64_t e0 = nfull * chunk_elems + (int64_t)ctid * V; e0 < n_elem; e0 += (int64_t)NW * 32 * V) {
        Chunk ch;
        ch.base = e0;
        ch.cnt = (int)min((int64_t)V, n_elem - e0);
        ch.row0 = 0; ch.col = 0; ch.flat = true;
        uint32_t lo[V], hi[V];
        E::eval(P, ch, lo, hi);
        for (int v = 0; v < ch.cnt; ++v) {
          if (fl) accd = add_d(accd, as_double(rt, lo[v], hi[v]));
          else accu += lo[v];
        }
      }
    }
  }
  // per-CTA partial (the producer warp contributes 0)
  accd = warp_sum_d(accd);
  accu = warp_sum_u(accu);
  __syncthreads();
  if (lane == 0) { smd[warp] = accd; smu[warp] = accu; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    uint32_t bu = 0;
    for (int w = 0; w <= NW; ++w) { b = add_d(b, smd[w]); bu += smu[w]; }
    part_d[blockIdx.x] = b;
    part_u[blockIdx.x] = bu;
    __threadfence();
    last = (atomicAdd(done, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (blockIdx.x == 0) pdl_exit(indep);
  if (!last) return;
  __threadfence();
  // combine in a fixed order with every thread: thread t sums the partials
  // t, t + T, ... (8 loads in flight), then warp trees, then warps in order
  // (one thread walking ~2600 partials serially cost ~0.7 ms of L2 latency)
  const int64_t ndyn = nfull - dbase;
  constexpr int kT = VmGeo<E>::kThreads, kU = 8;
  double sd = 0.0;
  uint32_t su = 0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += kT) { sd = add_d(sd, __ldcg(part_d + i)); su += __ldcg(part_u + i); }
  double sc = 0.0;
  uint32_t scu = 0;
  for (int64_t i0 = threadIdx.x; i0 < ndyn; i0 += (int64_t)kU * kT) {
    double v[kU];
    uint32_t w[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + (int64_t)u * kT;
      v[u] = i < ndyn ? __ldcg(part_c + i) : 0.0;
      w[u] = i < ndyn ? __ldcg(part_cu + i) : 0u;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i0 + (int64_t)u * kT < ndyn) { sc = add_d(sc, v[u]); scu += w[u]; }
  }
  sd = warp_sum_d(sd);
  sc = warp_sum_d(sc);
  su = warp_sum_u(su);
  scu = warp_sum_u(scu);
  __shared__ double fd[VmGeo<E>::kWarps + 1], fc[VmGeo<E>::kWarps + 1];
  __shared__ uint32_t fu[VmGeo<E>::kWarps + 1], fcu[VmGeo<E>::kWarps + 1];
  if (lane == 0) { fd[warp] = sd; fc[warp] = sc; fu[warp] = su; fcu[warp] = scu; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    uint32_t au = 0;
    for (int w2 = 0; w2 <= VmGeo<E>::kWarps; ++w2) { a = add_d(a, fd[w2]); b = add_d(b, fc[w2]); au += fu[w2] + fcu[w2]; }
    a = add_d(a, b);
    if (fl) {
      if (finalize == FM_FINAL_SQRT) a = sqrt_d(a);
      *(double *)out = a;
    } else {
      *(uint32_t *)out = au;
    }
    *done = 0u;
    *ctr = 0u;
  }
}

}  // namespace bulk
}  // namespace fm
