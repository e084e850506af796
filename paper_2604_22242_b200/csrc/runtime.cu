// runtime.cu -- device, memory, stream, event entry points of the C ABI and
// the shared scratch / error plumbing (include/fmb200.h).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <string>

#include <vector>

#include "common.cuh"

namespace fm {

static thread_local std::string g_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string &msg) { g_error = msg; }
int fail(const char *what, cudaError_t e) {
  set_error(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
  return (int)e == 0 ? -1 : (int)e;
}
int fail_msg(const std::string &msg) {
  set_error(msg);
  return -1;
}
void count_launch(int64_t n) { g_launches += n; }

bool pdl_enabled() {
  static const bool on = [] {
    const char *e = getenv("FMB200_PDL");
    return !(e && *e && atoi(e) == 0);
  }();
  return on;
}

// cuTensorMapEncodeTiled from the driver through the runtime's entry-point
// query (no link-time libcuda dependency: the CPU suite loads this library)
void *tensor_map_encoder() {
  static void *fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return p;
  }();
  return fn;
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && cached[dev]) return cached[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev < 64) cached[dev] = n;
  return n;
}

static constexpr size_t kCounterBytes = 64 * 1024;
struct ScratchEntry {
  void *base = nullptr;
  size_t payload = 0;
};
static std::mutex g_scratch_mu;
static std::map<std::pair<int, void *>, ScratchEntry> g_scratch;

// A zero-filled device block allocated OUTSIDE any stream capture: plain
// cudaMalloc under a relaxed capture mode (so it is legal while this thread
// is capturing) and a memset on a private side stream that is synchronised
// before returning.  Used for memory whose address a CUDA graph may bake in
// (the scratch arena, allocations made while capturing): a graph memory node
// would be unmapped between replays and could not be relaunched unfreed.
// per-device non-blocking side stream for the setup copies below (never
// captured: no legacy-stream implicit synchronisation with a capture)
static cudaError_t side_stream(int dev, cudaStream_t *out) {
  static thread_local cudaStream_t side[64] = {nullptr};
  const int d = dev < 64 ? dev : 0;
  if (side[d] == nullptr) {
    cudaError_t e = cudaStreamCreateWithFlags(&side[d], cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
  }
  *out = side[d];
  return cudaSuccess;
}

// cudaMalloc + fill (zeros, or `host` bytes) outside any capture
static int alloc_filled(void **ptr, size_t bytes, const void *host) {
  int dev = 0;
  FM_CHECK(cudaGetDevice(&dev));
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  FM_CHECK(cudaThreadExchangeStreamCaptureMode(&mode));
  cudaStream_t side = nullptr;
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e == cudaSuccess) e = side_stream(dev, &side);
  if (e == cudaSuccess)
    e = host ? cudaMemcpyAsync(*ptr, host, bytes, cudaMemcpyHostToDevice, side) : cudaMemsetAsync(*ptr, 0, bytes, side);
  if (e == cudaSuccess) e = cudaStreamSynchronize(side);
  cudaThreadExchangeStreamCaptureMode(&mode);
  if (e != cudaSuccess) return fail("alloc_plain", e);
  return 0;
}

int alloc_plain(void **ptr, size_t bytes) { return alloc_filled(ptr, bytes, nullptr); }

// Tile-pair order tables (pair.cuh), one per (device, tile count); never
// freed -- CUDA graphs may hold the address.
int pair_order(int64_t n, const uint32_t **table) {
  static std::mutex mu;
  static std::map<std::pair<int, int64_t>, void *> tables;
  constexpr int kTile = 32, kStrip = 8;
  int dev = 0;
  FM_CHECK(cudaGetDevice(&dev));
  const int64_t nt = (n + kTile - 1) / kTile;
  std::lock_guard<std::mutex> lk(mu);
  void *&d = tables[{dev, nt}];
  if (d == nullptr) {
    std::vector<uint32_t> h;
    h.reserve((size_t)(nt * (nt + 1) / 2));
    for (int64_t j0 = 0; j0 < nt; j0 += kStrip) {
      const int64_t j1 = std::min<int64_t>(nt, j0 + kStrip);
      for (int64_t i = 0; i < j1; ++i)
        for (int64_t j = std::max(i, j0); j < j1; ++j) h.push_back((uint32_t)i | ((uint32_t)j << 16));
    }
    void *p = nullptr;
    if (int st = alloc_filled(&p, h.size() * sizeof(uint32_t), h.data())) return st;
    d = p;
  }
  *table = (const uint32_t *)d;
  return 0;
}

int get_scratch(void *stream, size_t payload_bytes, Scratch *out, int slot) {
  int dev = 0;
  FM_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_scratch_mu);
  ScratchEntry &e = g_scratch[{dev * kPdlWindow + slot, stream}];
  if (e.base == nullptr || e.payload < payload_bytes) {
    // grow geometrically; the outgrown block is retired, not freed, because a
    // CUDA graph captured earlier (fm_graph_*) may still hold its address.
    // Never a stream-ordered / graph allocation: the arena's address outlives
    // any capture that first needed it (eager launches and replays share it).
    size_t want = payload_bytes < (size_t)(1 << 20) ? (size_t)(1 << 20) : payload_bytes;
    if (want < 2 * e.payload) want = 2 * e.payload;
    void *base = nullptr;
    int st = alloc_plain(&base, kCounterBytes + want);
    if (st) return st;
    e.base = base;
    e.payload = want;
  }
  out->counters = (unsigned *)e.base;
  out->payload = (char *)e.base + kCounterBytes;
  out->payload_bytes = e.payload;
  return 0;
}

// ---- launch windows (common.cuh: overlap of independent launches) ----------
struct PdlWindow {
  std::vector<Footprint> fps;
};
static std::mutex g_pdl_mu;
static std::map<std::pair<int, void *>, PdlWindow> g_pdl;

static bool overlaps(const ByteRange *a, int na, const ByteRange *b, int nb) {
  for (int i = 0; i < na; ++i)
    for (int j = 0; j < nb; ++j)
      if (a[i].lo < b[j].hi && b[j].lo < a[i].hi) return true;
  return false;
}

// forget the stream's window (graph boundaries: the launches around a
// capture are not each other's neighbours when the graph replays)
static void pdl_reset(void *stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_pdl_mu);
  g_pdl.erase({dev, stream});
}

PdlPlan pdl_classify(cudaStream_t s, const Footprint &fp) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_pdl_mu);
  PdlWindow &w = g_pdl[{dev, (void *)s}];
  bool indep = pdl_enabled() && !w.fps.empty() && (int)w.fps.size() < kPdlWindow && fp.n_wr > 0;
  for (size_t i = 0; indep && i < w.fps.size(); ++i) {
    const Footprint &o = w.fps[i];
    if (overlaps(fp.rd, fp.n_rd, o.wr, o.n_wr) || overlaps(fp.wr, fp.n_wr, o.rd, o.n_rd) ||
        overlaps(fp.wr, fp.n_wr, o.wr, o.n_wr))
      indep = false;
  }
  if (!indep) w.fps.clear();
  w.fps.push_back(fp);
  return PdlPlan{indep ? 1 : 0, (int)w.fps.size() - 1};
}

void program_reads(const fm_program &P, int64_t n_rows, int64_t n_cols, Footprint &fp) {
  for (int j = 0; j < P.n_slots; ++j) {
    const fm_slot &sl = P.slots[j];
    const int w = sl.etype == FM_F64 ? 8 : (sl.etype == FM_BF16 ? 2 : 4);
    int64_t r = n_rows, c = n_cols;
    if (sl.transposed) std::swap(r, c);
    if (sl.map == FM_MAP_DIAG) c = r;
    const int64_t last = (sl.row_off + std::max<int64_t>(r, 1) - 1) + (sl.col_off + std::max<int64_t>(c, 1) - 1) * sl.ld;
    fp.rd[fp.n_rd++] = {(uintptr_t)sl.ptr, (uintptr_t)sl.ptr + (uintptr_t)((last + 1) * w)};
  }
}

// ---- graph-owned allocations ---------------------------------------------
// While a thread captures a stream (fm_graph_begin .. fm_graph_end), buffers
// it allocates are plain (non-graph) allocations and buffers it frees are not
// released: the graph's kernels reference both on every replay.  They stay
// alive until the last graph that captured them is destroyed AND the owner
// has freed them (a temp the planner freed at the end of a captured assign,
// or an output buffer swapped out by an aliasing assign).  A capture-time
// allocation that the caller keeps (e.g. the temp an aliasing assign swaps
// into the output) returns to normal ownership when the graph goes away.
struct Owned {
  int graphs = 0;            // live graphs (or the open capture) referencing it
  bool released = false;     // the owner called fm_free
  bool plain = false;        // cudaMalloc'ed (else stream-ordered pool memory)
};
static std::mutex g_owned_mu;
static std::map<void *, Owned> g_owned;
// plain (cudaMalloc) buffers that went back to their owner after the graphs
// that captured them were destroyed: freed with cudaFree, not cudaFreeAsync
static std::set<void *> g_plain;
struct CaptureState {
  bool active = false;
  std::vector<void *> ptrs;
};
static thread_local CaptureState g_capture;

static void owned_add_to_capture(void *p, bool released, bool plain) {
  Owned &o = g_owned[p];
  if (o.graphs == 0) o.plain = plain;
  o.graphs += 1;
  o.released = o.released || released;
  g_capture.ptrs.push_back(p);
}

static int owned_release_refs(const std::vector<void *> &ptrs) {
  std::vector<std::pair<void *, bool>> to_free;
  {
    std::lock_guard<std::mutex> lk(g_owned_mu);
    for (void *p : ptrs) {
      auto it = g_owned.find(p);
      if (it == g_owned.end()) continue;
      if (--it->second.graphs > 0) continue;
      if (it->second.released) to_free.push_back({p, it->second.plain});
      else if (it->second.plain) g_plain.insert(p);
      g_owned.erase(it);
    }
  }
  if (to_free.empty()) return 0;
  FM_CHECK(cudaDeviceSynchronize());   // replays still in flight may use them
  for (auto &f : to_free) {
    if (f.second) FM_CHECK(cudaFree(f.first));
    else FM_CHECK(cudaFreeAsync(f.first, (cudaStream_t)0));
  }
  return 0;
}

}  // namespace fm

using namespace fm;

extern "C" {

const char *fm_last_error(void) { return g_error.c_str(); }
int fm_abi_version(void) { return FMB200_ABI_VERSION; }
int64_t fm_launch_counter(void) { return g_launches.load(); }

int fm_device_count(int *count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    cudaGetLastError();
    return fail("cudaGetDeviceCount", e);
  }
  *count = n;
  return 0;
}

int fm_set_device(int device) {
  FM_CHECK(cudaSetDevice(device));
  return 0;
}

int fm_get_device(int *device) {
  FM_CHECK(cudaGetDevice(device));
  return 0;
}

int fm_device_info(int device, int *sm, int *major, int *minor, int64_t *l2, int64_t *hbm) {
  cudaDeviceProp p;
  FM_CHECK(cudaGetDeviceProperties(&p, device));
  *sm = p.multiProcessorCount;
  *major = p.major;
  *minor = p.minor;
  *l2 = p.l2CacheSize;
  *hbm = (int64_t)p.totalGlobalMem;
  return 0;
}

int fm_device_pci_bus_id(int device, char *buf, int len) {
  FM_CHECK(cudaDeviceGetPCIBusId(buf, len, device));
  return 0;
}

int fm_alloc(void **ptr, size_t bytes, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (bytes == 0) bytes = 1;
  if (g_capture.active) {
    // inside fm_graph_begin/end: a plain allocation owned by the graph
    int st = alloc_plain(ptr, bytes);
    if (st) return st;
    std::lock_guard<std::mutex> lk(g_owned_mu);
    owned_add_to_capture(*ptr, false, true);
    return 0;
  }
  FM_CHECK(cudaMallocAsync(ptr, bytes, s));
  FM_CHECK(cudaMemsetAsync(*ptr, 0, bytes, s));
  return 0;
}

int fm_free(void *ptr, void *stream) {
  if (!ptr) return 0;
  {
    std::lock_guard<std::mutex> lk(g_owned_mu);
    auto it = g_owned.find(ptr);
    if (it != g_owned.end()) {         // a live graph references it: defer
      if (g_capture.active) owned_add_to_capture(ptr, true, it->second.plain);
      else it->second.released = true;
      return 0;
    }
    bool plain = g_plain.count(ptr) > 0;
    if (g_capture.active) {            // freed while capturing: the graph keeps it
      if (plain) g_plain.erase(ptr);
      owned_add_to_capture(ptr, true, plain);
      return 0;
    }
    if (plain) {
      g_plain.erase(ptr);
      FM_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
      FM_CHECK(cudaFree(ptr));
      return 0;
    }
  }
  FM_CHECK(cudaFreeAsync(ptr, (cudaStream_t)stream));
  return 0;
}

int64_t fm_graph_owned_count(void) {
  std::lock_guard<std::mutex> lk(g_owned_mu);
  return (int64_t)g_owned.size();
}

int fm_host_alloc(void **ptr, size_t bytes) {
  FM_CHECK(cudaHostAlloc(ptr, bytes ? bytes : 1, cudaHostAllocPortable));
  return 0;
}

int fm_host_free(void *ptr) {
  FM_CHECK(cudaFreeHost(ptr));
  return 0;
}

int fm_memcpy_h2d(void *dst, const void *src, size_t bytes, void *stream) {
  FM_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream));
  return 0;
}

int fm_memcpy_d2h(void *dst, const void *src, size_t bytes, void *stream) {
  FM_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  return 0;
}

int fm_memcpy_d2d(void *dst, const void *src, size_t bytes, void *stream) {
  FM_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return 0;
}

int fm_memset(void *dst, int value, size_t bytes, void *stream) {
  FM_CHECK(cudaMemsetAsync(dst, value, bytes, (cudaStream_t)stream));
  return 0;
}

int fm_stream_create(void **stream) {
  cudaStream_t s;
  FM_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  // keep freed blocks in the pool: cudaMallocAsync then costs ~1 us
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *stream = (void *)s;
  return 0;
}

int fm_stream_destroy(void *stream) {
  FM_CHECK(cudaStreamDestroy((cudaStream_t)stream));
  return 0;
}

int fm_stream_sync(void *stream) {
  FM_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
  return 0;
}

int fm_event_create(void **event) {
  cudaEvent_t e;
  FM_CHECK(cudaEventCreate(&e));
  *event = (void *)e;
  return 0;
}

int fm_event_destroy(void *event) {
  FM_CHECK(cudaEventDestroy((cudaEvent_t)event));
  return 0;
}

int fm_event_record(void *event, void *stream) {
  // Under stream capture a plain record is only a capture-internal
  // dependency; an external record becomes an event-record node of the graph,
  // so the event still times the replayed kernels.
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  FM_CHECK(cudaStreamIsCapturing((cudaStream_t)stream, &cs));
  if (cs == cudaStreamCaptureStatusActive)
    FM_CHECK(cudaEventRecordWithFlags((cudaEvent_t)event, (cudaStream_t)stream, cudaEventRecordExternal));
  else
    FM_CHECK(cudaEventRecord((cudaEvent_t)event, (cudaStream_t)stream));
  return 0;
}

int fm_event_elapsed_ms(void *start, void *stop, float *ms) {
  FM_CHECK(cudaEventSynchronize((cudaEvent_t)stop));
  FM_CHECK(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)stop));
  return 0;
}

// ---- CUDA graphs: capture a sequence of launches on a stream, replay it ----
// Replaces per-step host work (planning, binding, ctypes) with one
// cudaGraphLaunch; the captured kernels are exactly the ones the eager calls
// enqueue.  The launch counter advances by the graph's kernel count per replay.
struct FmGraph {
  cudaGraphExec_t exec;
  int64_t kernels;
  std::vector<void *> owned;   // allocations the captured launches reference
};

int fm_graph_begin(void *stream) {
  if (g_capture.active) return fail_msg("graph_begin: this thread is already capturing");
  FM_CHECK(cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeThreadLocal));
  pdl_reset(stream);
  g_capture.active = true;
  g_capture.ptrs.clear();
  return 0;
}

int fm_graph_end(void *stream, void **graph, int64_t *kernels) {
  cudaGraph_t g;
  g_capture.active = false;
  std::vector<void *> owned;
  owned.swap(g_capture.ptrs);
  cudaError_t ce = cudaStreamEndCapture((cudaStream_t)stream, &g);
  pdl_reset(stream);
  if (ce != cudaSuccess) {
    owned_release_refs(owned);
    return fail("cudaStreamEndCapture", ce);
  }
  size_t n = 0;
  cudaGraphGetNodes(g, nullptr, &n);
  std::vector<cudaGraphNode_t> nodes(n);
  if (n) cudaGraphGetNodes(g, nodes.data(), &n);
  int64_t k = 0;
  for (size_t i = 0; i < n; ++i) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nodes[i], &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
  }
  cudaGraphExec_t exec;
  cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    owned_release_refs(owned);
    return fail("cudaGraphInstantiate", e);
  }
  FmGraph *fg = new FmGraph{exec, k, std::move(owned)};
  *graph = fg;
  if (kernels) *kernels = k;
  return 0;
}

int fm_graph_launch(void *graph, void *stream) {
  if (!graph) return fail_msg("graph_launch: null graph");
  FmGraph *fg = (FmGraph *)graph;
  FM_CHECK(cudaGraphLaunch(fg->exec, (cudaStream_t)stream));
  pdl_reset(stream);
  count_launch(fg->kernels);
  return 0;
}

int fm_graph_destroy(void *graph) {
  if (!graph) return 0;
  FmGraph *fg = (FmGraph *)graph;
  cudaError_t e = cudaGraphExecDestroy(fg->exec);
  std::vector<void *> owned = std::move(fg->owned);
  delete fg;
  if (e != cudaSuccess) return fail("cudaGraphExecDestroy", e);
  return owned_release_refs(owned);
}

}  // extern "C"
