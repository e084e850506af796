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
int get_scratch(void *stream, size_t payload_bytes, Scratch *out);
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
