// rng.cu -- device-side synthetic inputs and utility kernels.
//
// fm_randu / fm_randi reproduce the reference's counter-based splitmix64
// stream bit for bit (/root/reference/pkg/src/fusemat/rng.py:35-72):
//   x_k = mix64(seed + (k+1) * 0x9E3779B97F4A7C15)
//   f32: (x_k >> 40) * 2^-24      f64: (x_k >> 11) * 2^-53
//   int: (x_k >> 32) mod high
// `offset` shifts k so a column shard generates exactly its slice of the
// global stream.  bf16 rounds the f32 value to nearest even.
#include "common.cuh"
#include "ops.cuh"

namespace fm {

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

__device__ __forceinline__ unsigned long long word(unsigned long long seed, long long k) {
  return mix64(seed + (unsigned long long)(k + 1) * 0x9E3779B97F4A7C15ull);
}

__global__ void k_randu(void *out, int etype, long long n, unsigned long long seed, long long offset) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long w = word(seed, offset + i);
    if (etype == FM_F64) {
      ((double *)out)[i] = (double)(w >> 11) * 0x1.0p-53;
    } else {
      const float f = (float)(unsigned)(w >> 40) * 0x1.0p-24f;
      if (etype == FM_BF16) ((uint16_t *)out)[i] = f_to_bf16_bits(f);
      else ((float *)out)[i] = f;
    }
  }
}

__global__ void k_randi(uint32_t *out, long long n, uint32_t high, unsigned long long seed, long long offset) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long w = word(seed, offset + i);
    out[i] = (uint32_t)((w >> 32) % (unsigned long long)high);
  }
}

__global__ void k_fill(void *out, int width, long long n, unsigned long long bits) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if (width == 8) ((unsigned long long *)out)[i] = bits;
    else if (width == 4) ((uint32_t *)out)[i] = (uint32_t)bits;
    else ((uint16_t *)out)[i] = (uint16_t)bits;
  }
}

__global__ void k_copy16(uint4 *dst, const uint4 *src, long long n16) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void k_touch(uint4 *p, long long n16, unsigned salt) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x)
    p[i] = make_uint4(salt, (unsigned)i, salt ^ 0x5bd1e995u, (unsigned)(i >> 32));
}

// Read pass over the flush buffer: after k_touch evicted every input line,
// reading the (now written-back) scratch leaves L2 holding only clean lines,
// so the timed kernel neither hits its inputs in L2 nor pays for write-backs
// of the flush's dirty lines.
__global__ void k_read_sink(const uint4 *p, long long n16, unsigned *sink) {
  unsigned acc = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (long long)gridDim.x * blockDim.x) {
    uint4 w = __ldcg(p + i);
    acc ^= w.x ^ w.y ^ w.z ^ w.w;
  }
  if (acc == 0x9e3779b9u && sink) *sink = acc;   // practically never taken; keeps the loads live
}

static unsigned grid_for(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  long long cap = (long long)sm_count() * 32;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (unsigned)g;
}

static int width_of(int etype) {
  switch (etype) {
    case FM_F64: return 8;
    case FM_BF16: return 2;
    default: return 4;
  }
}

}  // namespace fm

using namespace fm;

extern "C" {

int fm_randu(void *out, int32_t etype, int64_t n, uint64_t seed, int64_t offset, void *stream) {
  if (etype != FM_F32 && etype != FM_F64 && etype != FM_BF16) return fail_msg("randu: float element types only");
  if (n <= 0) return 0;
  k_randu<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(out, etype, n, seed, offset);
  FM_CHECK_LAUNCH("randu kernel");
  return 0;
}

int fm_randi(void *out, int32_t etype, int64_t n, uint32_t high, uint64_t seed, int64_t offset, void *stream) {
  if (etype != FM_U32 && etype != FM_I32) return fail_msg("randi: integer element types only");
  if (high == 0) return fail_msg("randi: high must be positive");
  if (n <= 0) return 0;
  k_randi<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>((uint32_t *)out, n, high, seed, offset);
  FM_CHECK_LAUNCH("randi kernel");
  return 0;
}

int fm_fill(void *out, int32_t etype, int64_t n, uint64_t bits, void *stream) {
  if (n <= 0) return 0;
  k_fill<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(out, width_of(etype), n, bits);
  FM_CHECK_LAUNCH("fill kernel");
  return 0;
}

int fm_copy(void *dst, const void *src, size_t bytes, void *stream) {
  if (bytes % 16 || ((uintptr_t)dst | (uintptr_t)src) % 16) {
    FM_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return 0;
  }
  long long n16 = (long long)(bytes / 16);
  if (n16 == 0) return 0;
  k_copy16<<<grid_for(n16, 512), 512, 0, (cudaStream_t)stream>>>((uint4 *)dst, (const uint4 *)src, n16);
  FM_CHECK_LAUNCH("copy kernel");
  return 0;
}

int fm_flush_l2(void *scratch, size_t bytes, void *stream) {
  static unsigned salt = 1;
  long long n16 = (long long)(bytes / 16);
  if (n16 == 0) return 0;
  k_touch<<<grid_for(n16, 512), 512, 0, (cudaStream_t)stream>>>((uint4 *)scratch, n16, salt++);
  FM_CHECK_LAUNCH("l2 flush kernel");
  k_read_sink<<<grid_for(n16, 512), 512, 0, (cudaStream_t)stream>>>((const uint4 *)scratch, n16,
                                                                    (unsigned *)scratch);
  FM_CHECK_LAUNCH("l2 clean-read kernel");
  return 0;
}

}  // extern "C"
