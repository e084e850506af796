// common.cuh -- error plumbing, per-stream scratch and the launch counter
// shared by every translation unit of libfmb200.so.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>

#include "fmb200.h"

namespace fm {

// thread-local last error (fm_last_error)
void set_error(const std::string &msg);
int fail(const char *what, cudaError_t e);
int fail_msg(const std::string &msg);
void count_launch(int64_t n = 1);

// Stream-ordered scratch owned by the library, one per (device, stream).
// Layout: [counters: 64 KiB, zero-filled once, self-resetting][payload ...]
struct Scratch {
  unsigned *counters;
  void *payload;
  size_t payload_bytes;
};
int get_scratch(void *stream, size_t payload_bytes, Scratch *out, int slot = 0);

// ---- overlap of independent launches (programmatic dependent launch) ------
// A launch whose byte ranges neither read what an in-flight launch writes
// nor write what one reads or writes is INDEPENDENT of it.  The library
// keeps, per stream, the window of launches that may still be running (all
// launches since the last dependent one, at most kPdlWindow); each PDL launch
// is classified against it (pdl_classify) and told so through bit 0 of
// fm_program.reserved:
//   dependent   -- griddepcontrol.wait, then launch_dependents: everything
//                  before it has completed before its CTAs do any work, and
//                  its successor cannot start before that (the window resets);
//   independent -- launch_dependents at once and NO wait before its work, so
//                  its CTAs fill SMs the previous kernel's tail leaves idle;
//                  it waits only before exiting, so its completion still
//                  implies its predecessors' (later dependent launches stay
//                  correctly ordered).
// Each launch in a window gets its own scratch slot (window position), so
// concurrently running reductions never share partials or counters.
constexpr int kPdlWindow = 4;
struct ByteRange {
  uintptr_t lo, hi;   // [lo, hi)
};
struct Footprint {
  ByteRange rd[FM_MAX_SLOTS];
  int n_rd = 0;
  ByteRange wr[FM_MAX_REDUCE_OUT];
  int n_wr = 0;
};
struct PdlPlan {
  int independent;   // 1: skip the initial wait (fm_program.reserved bit 0)
  int slot;          // scratch slot of this launch
};
PdlPlan pdl_classify(cudaStream_t s, const Footprint &fp);
// read footprint of a program's slots over an n_rows x n_cols domain
void program_reads(const fm_program &P, int64_t n_rows, int64_t n_cols, Footprint &fp);
inline void footprint_write(Footprint &fp, const void *p, size_t bytes) {
  if (fp.n_wr < FM_MAX_REDUCE_OUT) fp.wr[fp.n_wr++] = {(uintptr_t)p, (uintptr_t)p + bytes};
}

// kernel side: bit 0 of P.reserved (see above)
__device__ __forceinline__ void pdl_enter(int independent);
__device__ __forceinline__ void pdl_exit(int independent);
// zero-filled plain cudaMalloc made outside any stream capture (safe to call
// while this thread captures; the address can be baked into a graph)
int alloc_plain(void **ptr, size_t bytes);

int sm_count();

// fused.cu: run a validated program through the generic (VM) kernels --
// the GEMM operand prologue (split into bf16 planes, split.cuh) or a plain
// copy into a buffer (operands of the exact GEMM path)
int validate_program(const fm_program *P);
int launch_split_program(const fm_program &P, uint16_t *planes, int64_t n_rows, int64_t n_cols, int64_t ld_out,
                         int64_t plane_off, const unsigned *amax, cudaStream_t s);
int launch_amax_program(const fm_program &P, int64_t n_rows, int64_t n_cols, unsigned *amax, cudaStream_t s,
                        bool *handled);
int launch_copy_program(const fm_program &P, void *out, int64_t n_rows, int64_t n_cols, cudaStream_t s);

// Programmatic dependent launch: kernels launched through launch_pdl may
// start while the previous kernel on the stream drains; they call
// pdl_wait() before touching global memory (it returns once the previous
// grid has completed and its writes are visible) and pdl_trigger() early so
// their own successor can do the same.  FMB200_PDL=0 disables it.
bool pdl_enabled();
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter(int independent) {
  if (independent) {
    pdl_trigger();
  } else {
    pdl_wait();
    pdl_trigger();
  }
}
__device__ __forceinline__ void pdl_exit(int independent) {
  if (independent) pdl_wait();
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace fm

#define FM_CHECK(call)                                                   \
  do {                                                                   \
    cudaError_t fm_e_ = (call);                                          \
    if (fm_e_ != cudaSuccess) return ::fm::fail(#call, fm_e_);            \
  } while (0)

#define FM_CHECK_LAUNCH(what)                                            \
  do {                                                                   \
    cudaError_t fm_e_ = cudaGetLastError();                              \
    if (fm_e_ != cudaSuccess) return ::fm::fail(what, fm_e_);             \
    ::fm::count_launch();                                                \
  } while (0)
