// common.cuh -- error plumbing, per-stream scratch and the launch counter
// shared by every translation unit of libfmb200.so.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

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

int sm_count();

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
