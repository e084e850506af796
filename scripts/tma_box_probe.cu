// tma_box_probe.cu -- how fast can 2-D TMA boxes stream a column-major
// matrix on B200, by access order?  (Design probe for csrc/pair.cuh.)
//
// A persistent grid; per CTA one producer lane issues boxes of {128 B rows,
// BC columns} into a ring of S stages and the consumer warps only wait on
// the full barrier, touch one word, and release the stage.  Orders:
//   col   -- consecutive row blocks of one column stripe (contiguous runs)
//   row   -- consecutive column blocks of one row stripe (128 B per column)
//   pair  -- the tile-pair order: block (I,J) then (J,I), strips of 8
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_box_probe scripts/tma_box_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));            \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(su32(bar)), "r"(parity) : "memory");
  } while (!done);
}

__global__ void __launch_bounds__(160) k_probe(const __grid_constant__ CUtensorMap map, const uint32_t *order,
                                               int nitems, int boxes_per_item, int box_bytes, int stages,
                                               int bc, unsigned *sink) {
  extern __shared__ unsigned char raw[];
  unsigned char *sm = raw + ((1024u - (su32(raw) & 1023u)) & 1023u);
  const int stage_bytes = boxes_per_item * box_bytes;
  uint64_t *full = (uint64_t *)(sm + stages * stage_bytes);
  uint64_t *empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(4));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 4) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int s = 0;
      uint32_t use = 0;
      for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                     "r"(stage_bytes) : "memory");
        for (int b = 0; b < boxes_per_item; ++b) {
          const uint32_t c = order[(size_t)it * boxes_per_item + b];
          const int x = (int)(c & 0xffffu) * 32, y = (int)(c >> 16) * bc;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
              " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(su32(sm + s * stage_bytes + b * box_bytes)),
              "l"(&map), "r"(x), "r"(y), "r"(su32(&full[s])), "l"(pol)
              : "memory");
        }
        if (++s == stages) { s = 0; ++use; }
      }
    }
    return;
  }
  unsigned acc = 0;
  int s = 0;
  uint32_t ph = 0;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    mbar_wait(&full[s], ph);
    acc += *(const unsigned *)(sm + s * stage_bytes + threadIdx.x * 4);
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    if (++s == stages) { s = 0; ph ^= 1u; }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main(int argc, char **argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 16384;   // n x n f32
  float *d;
  CK(cudaMalloc(&d, (size_t)n * n * 4));
  CK(cudaMemset(d, 0, (size_t)n * n * 4));
  unsigned *sink;
  CK(cudaMalloc(&sink, 4));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
  const int nt = n / 32;
  for (int bc : {32, 64, 128}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
    cuuint64_t str[1] = {(cuuint64_t)n * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)bc};
    cuuint32_t es[2] = {1, 1};
    if (cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, d, dims, str, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode failed\n");
      return 1;
    }
    const int ncb = n / bc;   // column blocks
    const int box_bytes = 128 * bc;
    for (const char *mode : {"col", "row", "pair"}) {
      std::vector<uint32_t> ord;
      int bpi = 1;
      if (mode[0] == 'c') {
        for (int j = 0; j < ncb; ++j)
          for (int i = 0; i < nt; ++i) ord.push_back((uint32_t)i | ((uint32_t)j << 16));
      } else if (mode[0] == 'r') {
        for (int i = 0; i < nt; ++i)
          for (int j = 0; j < ncb; ++j) ord.push_back((uint32_t)i | ((uint32_t)j << 16));
      } else {
        if (bc != 32) continue;
        bpi = 2;
        for (int j0 = 0; j0 < nt; j0 += 8)
          for (int i = 0; i < j0 + 8 && i < nt; ++i)
            for (int j = i > j0 ? i : j0; j < j0 + 8 && j < nt; ++j) {
              ord.push_back((uint32_t)i | ((uint32_t)j << 16));
              ord.push_back((uint32_t)j | ((uint32_t)i << 16));
            }
      }
      uint32_t *dord;
      CK(cudaMalloc(&dord, ord.size() * 4));
      CK(cudaMemcpy(dord, ord.data(), ord.size() * 4, cudaMemcpyHostToDevice));
      const int nitems = (int)ord.size() / bpi;
      for (int stages : {2, 3, 4, 6, 8}) {
        const int smem = stages * bpi * box_bytes + 1024 + 256;
        if (smem > 210 * 1024) continue;
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_probe, 160, smem));
        if (occ < 1) continue;
        const int grid = sms * occ;
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        for (int w = 0; w < 2; ++w) k_probe<<<grid, 160, smem>>>(map, dord, nitems, bpi, box_bytes, stages, bc, sink);
        CK(cudaEventRecord(a));
        const int reps = 5;
        for (int r = 0; r < reps; ++r) k_probe<<<grid, 160, smem>>>(map, dord, nitems, bpi, box_bytes, stages, bc, sink);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        const double bytes = (double)nitems * bpi * box_bytes;
        printf("box 128Bx%-3d %-4s stages %d ctas/SM %d inflight/SM %6.0f KB: %7.1f GB/s\n", bc, mode, stages, occ,
               (double)occ * stages * bpi * box_bytes / 1024, bytes / (ms / reps * 1e-3) / 1e9);
      }
      CK(cudaFree(dord));
    }
  }
  return 0;
}
