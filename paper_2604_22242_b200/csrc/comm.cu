// comm.cu -- the cross-GPU exchange of the sharded path (include/fmb200.h,
// "collectives").  SURVEY.md section 8(e): column-sharded matrices need no
// exchange for elementwise work; only reduction partials (full and row-wise)
// and the GEMM's column shards of Y cross GPUs.
//
// Every collective is "gather in rank order, then combine in rank order":
// each rank ends with bit-identical results (the combine order does not
// depend on the transport or on NCCL's ring/tree choice), and the combine
// rules are the single-GPU kernels' (NaN-propagating max/min, first-index
// arg-select with NaN winning, f64 sums, wrapping integer sums).
//
// Two transports:
//  * PEER -- ONE kernel per collective over peer memory.  Each rank owns an
//    IPC-exported block [flag | counters | epoch | data[2][slot]]; the kernel
//    copies this rank's contribution into data[epoch & 1], publishes
//    flag = epoch + 1 with a system-scope release, waits for every peer's
//    flag, then reads the peers' data straight over NVLink (or the same HBM
//    when ranks share a GPU) and combines it in registers.  Two data parities
//    make the blocks reusable without a second handshake: a rank can only
//    overwrite parity p at epoch e+2 after every peer has published e+1,
//    i.e. finished reading epoch e.  The epoch lives in device memory, so
//    the kernels replay inside CUDA graphs.  Works when ranks share one GPU
//    (the only multi-rank setup a one-GPU box allows: NCCL rejects duplicate
//    devices), which is how the tests exercise it.
//  * NCCL -- ncclAllGather (libnccl loaded with dlopen, no link-time
//    dependency) into a comm-owned gather buffer, then the same combine
//    kernel reading the gathered rows.  The default when every rank has its
//    own GPU.
#include <dlfcn.h>

#include <cstddef>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace fm {

// ---- NCCL, resolved at run time ----------------------------------------------
// (the few declarations the shim needs; ABI-stable across NCCL 2.x)
typedef struct {
  char internal[128];
} nccl_unique_id;
typedef void *nccl_comm_t;
enum { kNcclUint8 = 1 };

struct NcclApi {
  void *lib = nullptr;
  int (*get_unique_id)(nccl_unique_id *) = nullptr;
  int (*comm_init_rank)(nccl_comm_t *, int, nccl_unique_id, int) = nullptr;
  int (*comm_destroy)(nccl_comm_t) = nullptr;
  int (*all_gather)(const void *, void *, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
  const char *(*error_string)(int) = nullptr;
  int (*get_version)(int *) = nullptr;
};
static NcclApi g_nccl;

static int nccl_fail(const char *what, int r) {
  std::string m = std::string(what) + ": NCCL error " + std::to_string(r);
  if (g_nccl.error_string) m += std::string(" (") + g_nccl.error_string(r) + ")";
  return fail_msg(m);
}

// ---- peer blocks ---------------------------------------------------------------
static constexpr int kMaxRanks = 16;
static constexpr size_t kHeader = 256;   // flag, error, counters, epoch; data starts here

struct BlockHeader {
  unsigned long long flag;     // epoch + 1 of the last published contribution
  unsigned long long error;    // nonzero: a wait on a peer timed out
  unsigned arrive;             // CTAs of this rank that finished writing data
  unsigned depart;             // CTAs of this rank that finished reading peers
  unsigned long long epoch;    // collectives completed by this rank
  unsigned long long slot;     // bytes per data parity (same on every rank)
};

struct PeerPtrs {
  char *block[kMaxRanks];      // every rank's block (own one included), mapped here
};

struct Comm {
  int transport;               // FM_COMM_NCCL / FM_COMM_PEER
  int nranks, rank, device;
  // peer
  char *own = nullptr;         // this rank's block (cudaMalloc, IPC-exported)
  bool own_block = false;
  size_t slot = 0;             // bytes per data parity
  PeerPtrs peers{};
  // nccl
  nccl_comm_t nccl = nullptr;
  char *gather = nullptr;      // gather buffer (nranks * gather_bytes)
  size_t gather_bytes = 0;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---- element combine rules (rank order, identical on every rank) ---------------
struct ArgElem {               // 16 B: value (f64, exact for f32) + global index
  double v;
  unsigned idx;
  unsigned pad;
};

template <class T> __device__ __forceinline__ bool is_nan(T v) { return v != v; }

template <class T> __device__ __forceinline__ T combine(T a, T b, int op) {
  if (op == FM_COMBINE_SUM) return a + b;          // f64: one IEEE add per rank; ints wrap
  if (is_nan(a)) return a;                          // max/min propagate NaN (numpy)
  if (is_nan(b)) return b;
  if (op == FM_COMBINE_MAX) return b > a ? b : a;
  return b < a ? b : a;
}
template <> __device__ __forceinline__ unsigned combine<unsigned>(unsigned a, unsigned b, int op) {
  if (op == FM_COMBINE_SUM) return a + b;
  if (op == FM_COMBINE_MAX) return b > a ? b : a;
  return b < a ? b : a;
}
template <> __device__ __forceinline__ int combine<int>(int a, int b, int op) {
  if (op == FM_COMBINE_SUM) return (int)((unsigned)a + (unsigned)b);
  if (op == FM_COMBINE_MAX) return b > a ? b : a;
  return b < a ? b : a;
}

// first index of the extreme, NaN wins (first NaN) -- the single-GPU
// index_max / index_min rule (numpy argmax / argmin)
__device__ __forceinline__ ArgElem combine_arg(ArgElem best, ArgElem c, bool maximize) {
  const bool cn = c.v != c.v, bn = best.v != best.v;
  bool better;
  if (cn || bn) better = cn && (!bn || c.idx < best.idx);
  else if (maximize) better = c.v > best.v || (c.v == best.v && c.idx < best.idx);
  else better = c.v < best.v || (c.v == best.v && c.idx < best.idx);
  return better ? c : best;
}

// peer data is written by another kernel (another process) during this one:
// read it through L2 only (ld.global.cg), never a possibly stale L1 line
__device__ __forceinline__ ArgElem load_arg(const ArgElem *p) {
  const double2 raw = __ldcg((const double2 *)p);
  ArgElem a;
  a.v = raw.x;
  a.idx = (unsigned)__double_as_longlong(raw.y);
  a.pad = 0;
  return a;
}

// ---- the peer kernel: publish, wait, combine -------------------------------------
enum { kModeGather = 0, kModeReduce = 1, kModeArg = 2 };

struct PeerJob {
  int mode, op, etype, nranks, rank;
  int64_t count;               // elements (reduce / arg) or bytes (gather) in this chunk
  size_t slot_off;             // byte offset inside the data parity
  const void *src;             // this rank's contribution (reduce / gather)
  const void *src_idx;         // arg: u32 indices
  void *dst;                   // reduce / arg: values; gather: base of rank 0's piece
  void *dst_idx;               // arg: u32 indices
  size_t dst_stride;           // gather: bytes between ranks' pieces in dst
  double divisor;              // reduce: result /= divisor when > 0 (mean)
  unsigned idx_offset;         // arg: added to this rank's indices (global column)
  int maximize;
  int vec;                     // gather: copy unit in bytes (16 / 4 / 1)
};

template <class T>
__device__ void pack_reduce(const PeerJob &J, char *data) {
  const T *src = (const T *)J.src;
  T *d = (T *)(data + J.slot_off);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < J.count;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = src[i];
}

template <class T>
__device__ void finish_reduce(const PeerJob &J, const PeerPtrs &P, size_t par_off) {
  T *dst = (T *)J.dst;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < J.count;
       i += (int64_t)gridDim.x * blockDim.x) {
    T acc = __ldcg((const T *)(P.block[0] + kHeader + par_off + J.slot_off) + i);
    for (int q = 1; q < J.nranks; ++q)
      acc = combine<T>(acc, __ldcg((const T *)(P.block[q] + kHeader + par_off + J.slot_off) + i), J.op);
    if (J.divisor > 0) acc = (T)((double)acc / J.divisor);    // mean (f64 partial sums)
    dst[i] = acc;
  }
}

// grid-stride byte copy in `vec`-byte units (16, 4 or 1: the widest that
// divides every address, length and stride of the job); `peer` reads go
// through L2 only
template <class V>
__device__ __forceinline__ void copy_units(char *dst, const char *src, int64_t n, bool peer) {
  V *d = (V *)dst;
  const V *s = (const V *)src;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = peer ? __ldcg(s + i) : s[i];
}
__device__ __forceinline__ void copy_bytes(char *dst, const char *src, int64_t bytes, int vec, bool peer) {
  if (vec == 16) copy_units<uint4>(dst, src, bytes / 16, peer);
  else if (vec == 4) copy_units<unsigned>(dst, src, bytes / 4, peer);
  else copy_units<unsigned char>(dst, src, bytes, peer);
}

__global__ void __launch_bounds__(256) k_peer_collective(PeerJob J, PeerPtrs P) {
  char *own = P.block[J.rank];
  BlockHeader *H = (BlockHeader *)own;
  const unsigned long long e = *(volatile unsigned long long *)&H->epoch;
  const size_t par_off = (e & 1) ? (size_t)H->slot : 0;
  char *data = own + kHeader + par_off;

  // 1. this rank's contribution -> own block
  if (J.mode == kModeGather) {
    copy_bytes(data + J.slot_off, (const char *)J.src, J.count, J.vec, false);
  } else if (J.mode == kModeArg) {
    ArgElem *d = (ArgElem *)(data + J.slot_off);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < J.count;
         i += (int64_t)gridDim.x * blockDim.x) {
      ArgElem a;
      a.v = J.etype == FM_F64 ? ((const double *)J.src)[i] : (double)((const float *)J.src)[i];
      a.idx = ((const unsigned *)J.src_idx)[i] + J.idx_offset;
      a.pad = 0;
      d[i] = a;
    }
  } else {
    switch (J.etype) {
      case FM_F64: pack_reduce<double>(J, data); break;
      case FM_F32: pack_reduce<float>(J, data); break;
      case FM_I32: pack_reduce<int>(J, data); break;
      default: pack_reduce<unsigned>(J, data); break;
    }
  }

  // 2. publish once every CTA of this rank has written (last-CTA-done)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(&H->arrive, 1u) == gridDim.x - 1) {
      H->arrive = 0;
      __threadfence_system();
      st_release_sys(&H->flag, e + 1);
    }
  }
  // 3. wait for every rank's contribution of this epoch (bounded: 30 s)
  if (threadIdx.x < J.nranks) {
    const unsigned long long *f = (const unsigned long long *)P.block[threadIdx.x];
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(f) < e + 1) {
      if (globaltimer() - t0 > 30ull * 1000000000ull) {
        atomicExch(&H->error, 1ull + threadIdx.x);
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();

  // 4. read the peers in rank order and combine
  if (J.mode == kModeGather) {
    for (int q = 0; q < J.nranks; ++q)
      copy_bytes((char *)J.dst + q * J.dst_stride, P.block[q] + kHeader + par_off + J.slot_off, J.count,
                 J.vec, true);
  } else if (J.mode == kModeArg) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < J.count;
         i += (int64_t)gridDim.x * blockDim.x) {
      ArgElem best = load_arg((const ArgElem *)(P.block[0] + kHeader + par_off + J.slot_off) + i);
      for (int q = 1; q < J.nranks; ++q)
        best = combine_arg(best, load_arg((const ArgElem *)(P.block[q] + kHeader + par_off + J.slot_off) + i),
                           J.maximize != 0);
      if (J.etype == FM_F64) ((double *)J.dst)[i] = best.v;
      else ((float *)J.dst)[i] = (float)best.v;
      ((unsigned *)J.dst_idx)[i] = best.idx;
    }
  } else {
    switch (J.etype) {
      case FM_F64: finish_reduce<double>(J, P, par_off); break;
      case FM_F32: finish_reduce<float>(J, P, par_off); break;
      case FM_I32: finish_reduce<int>(J, P, par_off); break;
      default: finish_reduce<unsigned>(J, P, par_off); break;
    }
  }

  // 5. the last CTA to finish reading advances the epoch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&H->depart, 1u) == gridDim.x - 1) {
      H->depart = 0;
      H->epoch = e + 1;
      __threadfence();
    }
  }
}

// ---- combine of NCCL-gathered rows (rank-major: row q = rank q's contribution) ----
template <class T>
__global__ void k_combine_rows(const T *g, int64_t count, int nranks, int op, double divisor, T *dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    T acc = g[i];
    for (int q = 1; q < nranks; ++q) acc = combine<T>(acc, g[q * count + i], op);
    if (divisor > 0) acc = (T)((double)acc / divisor);
    dst[i] = acc;
  }
}

__global__ void k_pack_arg(const void *vals, const unsigned *idx, int64_t count, int etype, unsigned off,
                           ArgElem *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    ArgElem a;
    a.v = etype == FM_F64 ? ((const double *)vals)[i] : (double)((const float *)vals)[i];
    a.idx = idx[i] + off;
    a.pad = 0;
    out[i] = a;
  }
}

__global__ void k_combine_arg(const ArgElem *g, int64_t count, int nranks, int maximize, int etype,
                              void *vals, unsigned *idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    ArgElem best = g[i];
    for (int q = 1; q < nranks; ++q) best = combine_arg(best, g[q * count + i], maximize != 0);
    if (etype == FM_F64) ((double *)vals)[i] = best.v;
    else ((float *)vals)[i] = (float)best.v;
    idx[i] = best.idx;
  }
}

static int elem_width(int etype) {
  switch (etype) {
    case FM_F64: return 8;
    case FM_F32: case FM_U32: case FM_I32: return 4;
    default: return 0;
  }
}

static int grid_for(int64_t n, int cap) {
  int64_t g = (n + 255) / 256;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// peer: CTAs spin on each other's flags, so they must all be resident; a
// small grid (<= 32 CTAs of 256 threads) always is on a 148-SM B200
static constexpr int kPeerGrid = 32;

static int peer_run(Comm *c, PeerJob J, cudaStream_t s) {
  J.nranks = c->nranks;
  J.rank = c->rank;
  k_peer_collective<<<grid_for(J.mode == kModeGather ? J.count / J.vec + 1 : J.count, kPeerGrid), 256, 0, s>>>(
      J, c->peers);
  FM_CHECK_LAUNCH("k_peer_collective");
  return 0;
}

static int gather_buffer(Comm *c, size_t bytes_per_rank) {
  if (c->gather_bytes >= bytes_per_rank) return 0;
  size_t want = bytes_per_rank < (1u << 20) ? (1u << 20) : bytes_per_rank;
  // the outgrown buffer is retired, not freed: a captured graph may hold it
  void *p = nullptr;
  int st = alloc_plain(&p, want * c->nranks);
  if (st) return st;
  c->gather = (char *)p;
  c->gather_bytes = want;
  return 0;
}

}  // namespace fm

using namespace fm;

extern "C" {

int fm_comm_nccl_load(const char *path) {
  if (g_nccl.lib) return 0;
  void *h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return fail_msg(std::string("dlopen libnccl: ") + dlerror());
  NcclApi a;
  a.lib = h;
  a.get_unique_id = (decltype(a.get_unique_id))dlsym(h, "ncclGetUniqueId");
  a.comm_init_rank = (decltype(a.comm_init_rank))dlsym(h, "ncclCommInitRank");
  a.comm_destroy = (decltype(a.comm_destroy))dlsym(h, "ncclCommDestroy");
  a.all_gather = (decltype(a.all_gather))dlsym(h, "ncclAllGather");
  a.error_string = (decltype(a.error_string))dlsym(h, "ncclGetErrorString");
  a.get_version = (decltype(a.get_version))dlsym(h, "ncclGetVersion");
  if (!a.get_unique_id || !a.comm_init_rank || !a.comm_destroy || !a.all_gather)
    return fail_msg("libnccl lacks ncclGetUniqueId / ncclCommInitRank / ncclAllGather");
  g_nccl = a;
  return 0;
}

int fm_comm_nccl_version(int *version) {
  if (!g_nccl.lib || !g_nccl.get_version) return fail_msg("NCCL not loaded (fm_comm_nccl_load)");
  int r = g_nccl.get_version(version);
  return r ? nccl_fail("ncclGetVersion", r) : 0;
}

int fm_comm_nccl_unique_id(uint8_t *id128) {
  if (!g_nccl.lib) return fail_msg("NCCL not loaded (fm_comm_nccl_load)");
  nccl_unique_id u;
  int r = g_nccl.get_unique_id(&u);
  if (r) return nccl_fail("ncclGetUniqueId", r);
  memcpy(id128, u.internal, 128);
  return 0;
}

int fm_comm_init_nccl(void **comm, int nranks, int rank, const uint8_t *id128) {
  if (!g_nccl.lib) return fail_msg("NCCL not loaded (fm_comm_nccl_load)");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail_msg("comm_init_nccl: bad rank");
  nccl_unique_id u;
  memcpy(u.internal, id128, 128);
  Comm *c = new Comm();
  c->transport = FM_COMM_NCCL;
  c->nranks = nranks;
  c->rank = rank;
  cudaGetDevice(&c->device);
  int r = g_nccl.comm_init_rank(&c->nccl, nranks, u, rank);
  if (r) {
    delete c;
    return nccl_fail("ncclCommInitRank", r);
  }
  *comm = c;
  return 0;
}

int fm_comm_peer_block(void **block, size_t slot_bytes, uint8_t *ipc_handle64) {
  if (slot_bytes < 4096 || slot_bytes % 256) return fail_msg("comm_peer_block: slot must be >= 4096, a multiple of 256");
  void *p = nullptr;
  int st = alloc_plain(&p, kHeader + 2 * slot_bytes);
  if (st) return st;
  unsigned long long sb = slot_bytes;
  FM_CHECK(cudaMemcpy((char *)p + offsetof(BlockHeader, slot), &sb, sizeof(sb), cudaMemcpyHostToDevice));
  cudaIpcMemHandle_t h;
  FM_CHECK(cudaIpcGetMemHandle(&h, p));
  memcpy(ipc_handle64, &h, sizeof(h));
  *block = p;
  return 0;
}

int fm_comm_init_peer(void **comm, int nranks, int rank, void *block, const uint8_t *handles,
                      size_t slot_bytes) {
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
    return fail_msg("comm_init_peer: bad rank / more than 16 ranks");
  Comm *c = new Comm();
  c->transport = FM_COMM_PEER;
  c->nranks = nranks;
  c->rank = rank;
  c->own = (char *)block;
  c->own_block = true;
  c->slot = slot_bytes;
  cudaGetDevice(&c->device);
  for (int q = 0; q < nranks; ++q) {
    if (q == rank) {
      c->peers.block[q] = (char *)block;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + 64 * q, sizeof(h));
    void *p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (int k = 0; k < q; ++k)
        if (k != rank) cudaIpcCloseMemHandle(c->peers.block[k]);
      delete c;
      return fail("cudaIpcOpenMemHandle", e);
    }
    c->peers.block[q] = (char *)p;
  }
  *comm = c;
  return 0;
}

int fm_comm_destroy(void *comm) {
  Comm *c = (Comm *)comm;
  if (!c) return 0;
  cudaDeviceSynchronize();
  if (c->transport == FM_COMM_PEER) {
    for (int q = 0; q < c->nranks; ++q)
      if (q != c->rank && c->peers.block[q]) cudaIpcCloseMemHandle(c->peers.block[q]);
    // the own block stays allocated: peers may still hold it open
  } else if (c->nccl && g_nccl.comm_destroy) {
    g_nccl.comm_destroy(c->nccl);
  }
  delete c;
  return 0;
}

int fm_comm_info(void *comm, int *nranks, int *rank, int *transport) {
  Comm *c = (Comm *)comm;
  if (!c) return fail_msg("comm_info: null comm");
  *nranks = c->nranks;
  *rank = c->rank;
  *transport = c->transport;
  return 0;
}

int fm_comm_status(void *comm, int64_t *error) {
  Comm *c = (Comm *)comm;
  if (!c) return fail_msg("comm_status: null comm");
  *error = 0;
  if (c->transport != FM_COMM_PEER) return 0;
  unsigned long long e = 0;
  FM_CHECK(cudaMemcpy(&e, c->own + offsetof(BlockHeader, error), sizeof(e), cudaMemcpyDeviceToHost));
  *error = (int64_t)e;
  return 0;
}

int fm_allreduce(void *comm, void *buf, int64_t count, int32_t etype, int32_t op, double divisor,
                 void *stream) {
  Comm *c = (Comm *)comm;
  if (!c) return fail_msg("allreduce: null comm");
  const int w = elem_width(etype);
  if (!w) return fail_msg("allreduce: element type must be f32, f64, u32 or i32");
  if (op < FM_COMBINE_SUM || op > FM_COMBINE_MIN) return fail_msg("allreduce: bad op");
  if (count <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (c->transport == FM_COMM_PEER) {
    const int64_t per = (int64_t)(c->slot / w);
    for (int64_t off = 0; off < count; off += per) {
      PeerJob J{};
      J.mode = kModeReduce;
      J.op = op;
      J.etype = etype;
      J.count = count - off < per ? count - off : per;
      J.src = (const char *)buf + off * w;
      J.dst = (char *)buf + off * w;
      J.divisor = divisor;
      int st = peer_run(c, J, s);
      if (st) return st;
    }
    return 0;
  }
  int st = gather_buffer(c, (size_t)count * w);
  if (st) return st;
  int r = g_nccl.all_gather(buf, c->gather, (size_t)count * w, kNcclUint8, c->nccl, s);
  if (r) return nccl_fail("ncclAllGather", r);
  const int g = grid_for(count, 1184);
  switch (etype) {
    case FM_F64: k_combine_rows<double><<<g, 256, 0, s>>>((const double *)c->gather, count, c->nranks, op, divisor, (double *)buf); break;
    case FM_F32: k_combine_rows<float><<<g, 256, 0, s>>>((const float *)c->gather, count, c->nranks, op, divisor, (float *)buf); break;
    case FM_I32: k_combine_rows<int><<<g, 256, 0, s>>>((const int *)c->gather, count, c->nranks, op, divisor, (int *)buf); break;
    default: k_combine_rows<unsigned><<<g, 256, 0, s>>>((const unsigned *)c->gather, count, c->nranks, op, divisor, (unsigned *)buf); break;
  }
  FM_CHECK_LAUNCH("k_combine_rows");
  return 0;
}

int fm_allreduce_arg(void *comm, void *vals, uint32_t *idx, int64_t count, int32_t etype,
                     uint32_t idx_offset, int32_t maximize, void *stream) {
  Comm *c = (Comm *)comm;
  if (!c) return fail_msg("allreduce_arg: null comm");
  if (etype != FM_F32 && etype != FM_F64) return fail_msg("allreduce_arg: values must be f32 or f64");
  if (count <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int w = etype == FM_F64 ? 8 : 4;
  if (c->transport == FM_COMM_PEER) {
    const int64_t per = (int64_t)(c->slot / sizeof(ArgElem));
    for (int64_t off = 0; off < count; off += per) {
      PeerJob J{};
      J.mode = kModeArg;
      J.etype = etype;
      J.count = count - off < per ? count - off : per;
      J.src = (const char *)vals + off * w;
      J.src_idx = idx + off;
      J.dst = (char *)vals + off * w;
      J.dst_idx = idx + off;
      J.idx_offset = idx_offset;
      J.maximize = maximize;
      int st = peer_run(c, J, s);
      if (st) return st;
    }
    return 0;
  }
  // NCCL: pack (value, global index) pairs in the upper half of the gather
  // buffer's own row, gather, select
  const size_t bytes = (size_t)count * sizeof(ArgElem);
  int st = gather_buffer(c, 2 * bytes);
  if (st) return st;
  ArgElem *packed = (ArgElem *)(c->gather + (size_t)c->nranks * bytes);   // past the gathered rows
  const int g = grid_for(count, 1184);
  k_pack_arg<<<g, 256, 0, s>>>(vals, idx, count, etype, idx_offset, packed);
  FM_CHECK_LAUNCH("k_pack_arg");
  int r = g_nccl.all_gather(packed, c->gather, bytes, kNcclUint8, c->nccl, s);
  if (r) return nccl_fail("ncclAllGather", r);
  k_combine_arg<<<g, 256, 0, s>>>((const ArgElem *)c->gather, count, c->nranks, maximize, etype, vals, idx);
  FM_CHECK_LAUNCH("k_combine_arg");
  return 0;
}

int fm_allgather(void *comm, const void *src, size_t bytes, void *dst, void *stream) {
  Comm *c = (Comm *)comm;
  if (!c) return fail_msg("allgather: null comm");
  if (bytes == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (c->transport == FM_COMM_PEER) {
    const size_t per = c->slot;
    for (size_t off = 0; off < bytes; off += per) {
      PeerJob J{};
      J.mode = kModeGather;
      J.count = (int64_t)(bytes - off < per ? bytes - off : per);
      J.src = (const char *)src + off;
      J.dst = (char *)dst + off;
      J.dst_stride = bytes;
      const uintptr_t a = (uintptr_t)J.src | (uintptr_t)J.dst | (uintptr_t)J.count | (uintptr_t)bytes;
      J.vec = (a % 16 == 0) ? 16 : (a % 4 == 0) ? 4 : 1;
      int st = peer_run(c, J, s);
      if (st) return st;
    }
    return 0;
  }
  int r = g_nccl.all_gather(src, dst, bytes, kNcclUint8, c->nccl, s);
  if (r) return nccl_fail("ncclAllGather", r);
  return 0;
}

}  // extern "C"
