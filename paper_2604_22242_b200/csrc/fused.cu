// fused.cu -- C-ABI launch entry points of the fused path and the generic
// register-VM kernels (include/fmb200.h: fm_launch_copy / fm_launch_accu /
// fm_launch_reduce_dim / fm_kernel_lookup).
//
// Replaces the reference's compile-and-launch path (cjit.py:113-154): a
// kernel id from fm_kernel_lookup selects an ahead-of-time template kernel;
// id -1 runs the same program on the VM.  Either way one launch per fused
// step.
#include <algorithm>
#include <cstring>
#include <string>

#include "vm_variants.cuh"

namespace fm {

int validate_program(const fm_program *P) {
  if (!P) return fail_msg("null program");
  if (P->n_instr <= 0 || P->n_instr > FM_MAX_INSTR) return fail_msg("program: bad instruction count");
  if (P->n_slots < 0 || P->n_slots > FM_MAX_SLOTS) return fail_msg("program: bad slot count");
  if (P->depth <= 0 || P->depth > FM_MAX_DEPTH) return fail_msg("program: bad stack depth");
  for (int i = 0; i < P->n_instr; ++i) {
    const int op = P->code[i].key >> 3;
    const int d = P->code[i].key & 7;
    if (op >= FM_OP_COUNT) return fail_msg("program: unknown opcode " + std::to_string(op));
    if (d >= P->depth) return fail_msg("program: instruction writes above the declared depth");
    if ((op == FM_OP_PUSH32 || op == FM_OP_PUSH64) && P->code[i].arg >= P->n_slots)
      return fail_msg("program: push of an unbound slot");
  }
  for (int j = 0; j < P->n_slots; ++j)
    if (!P->slots[j].ptr) return fail_msg("program: slot " + std::to_string(j) + " has no buffer");
  return 0;
}

template <template <class> class F, class... A>
static int vm_dispatch(const fm_program &P, A... a) {
  if (P.wide) {
    if (P.depth <= 4) return F<Vm64s>::run(P, a...);
    return F<Vm64d>::run(P, a...);
  }
  if (P.depth <= 4) return F<Vm32s>::run(P, a...);
  return F<Vm32d>::run(P, a...);
}

template <class E> struct CopyF {
  static int run(const fm_program &P, void *out, int64_t r, int64_t c, cudaStream_t s) {
    return run_copy<E>(P, out, r, c, s);
  }
};
template <class E> struct AccuF {
  static int run(const fm_program &P, void *out, int64_t r, int64_t c, int fin, cudaStream_t s) {
    return run_accu<E>(P, out, r, c, fin, s);
  }
};
template <class E> struct DimF {
  static int run(const fm_program &P, int dim, int64_t r, int64_t c, ReduceOuts R, cudaStream_t s) {
    return run_reduce_dim<E>(P, dim, r, c, R, s);
  }
};

template <class E> struct SplitF {
  static int run(const fm_program &P, uint16_t *o, int64_t r, int64_t c, int64_t ld, int64_t po, const unsigned *am,
                 cudaStream_t s) {
    return run_split<E>(P, o, r, c, ld, po, am, s);
  }
};

int launch_split_program(const fm_program &P, uint16_t *planes, int64_t n_rows, int64_t n_cols, int64_t ld_out,
                         int64_t plane_off, const unsigned *amax, cudaStream_t s) {
  return vm_dispatch<SplitF>(P, planes, n_rows, n_cols, ld_out, plane_off, amax, s);
}

// max |EXPR| over the domain as f32 bits, atomically max-ed into *amax:
// the program with one ABS appended, column maxima (dim-0 MAX reduction,
// NaN propagates), then the maximum of those.  handled = false when the
// program has no room for the extra instruction.
__global__ void k_amax_vec(const float *v, int64_t n, unsigned *amax) {
  unsigned m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, __float_as_uint(v[i]) & 0x7fffffffu);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(amax, m);
}

int launch_amax_program(const fm_program &P0, int64_t n_rows, int64_t n_cols, unsigned *amax, cudaStream_t s,
                        bool *handled) {
  *handled = false;
  if (P0.n_instr >= FM_MAX_INSTR || P0.result_etype != FM_F32 || n_rows == 0 || n_cols == 0) return 0;
  fm_program P = P0;
  P.code[P.n_instr].key = (uint16_t)(FM_OP_ABS_F << 3);
  P.code[P.n_instr].arg = 0;
  ++P.n_instr;
  float *colmax = nullptr;
  FM_CHECK(cudaMallocAsync((void **)&colmax, (size_t)n_cols * sizeof(float), s));
  ReduceOuts R;
  R.n = 1;
  R.o[0].kind = FM_RED_MAX;
  R.o[0].etype = FM_F32;
  R.o[0].out = colmax;
  int st = vm_dispatch<DimF>(P, 0, n_rows, n_cols, R, s);
  if (!st) {
    k_amax_vec<<<(unsigned)std::min<int64_t>((n_cols + 255) / 256, 148), 256, 0, s>>>(colmax, n_cols, amax);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) st = fail("operand max |x| kernel", e);
    else count_launch();
  }
  cudaFreeAsync(colmax, s);
  if (!st) *handled = true;
  return st;
}
int launch_copy_program(const fm_program &P, void *out, int64_t n_rows, int64_t n_cols, cudaStream_t s) {
  return vm_dispatch<CopyF>(P, out, n_rows, n_cols, s);
}

static const TemplateEntry *entry_for(int kernel_id, int skeleton) {
  if (kernel_id < 0) return nullptr;
  int n = 0;
  const TemplateEntry *t = template_table(&n);
  const int idx = kernel_id / 4;
  if (idx >= n || kernel_id % 4 != skeleton) return nullptr;
  return &t[idx];
}

}  // namespace fm

using namespace fm;

extern "C" {

int fm_kernel_count(int *count) {
  int n = 0;
  template_table(&n);
  *count = n;
  return 0;
}

int fm_kernel_signature(int kernel_id, const char **signature) {
  int n = 0;
  const TemplateEntry *t = template_table(&n);
  if (kernel_id < 0 || kernel_id / 4 >= n) return fail_msg("no such kernel id");
  *signature = t[kernel_id / 4].signature;
  return 0;
}

// qualified signature: "copy|SIG", "reduce_accu|SIG[|finalN]", "reduce_dim{D:kinds}|SIG"
int fm_kernel_lookup(const char *qsig, int *kernel_id) {
  *kernel_id = -1;
  if (!qsig) return fail_msg("null signature");
  std::string q(qsig);
  const size_t bar = q.find('|');
  if (bar == std::string::npos) return 0;
  const std::string sk = q.substr(0, bar);
  std::string sig = q.substr(bar + 1);
  const size_t fin = sig.find("|final");
  if (fin != std::string::npos) sig = sig.substr(0, fin);
  int skel = -1;
  if (sk == "copy") skel = SK_COPY;
  else if (sk == "reduce_accu") skel = SK_ACCU;
  else if (sk.rfind("reduce_dim{0", 0) == 0) skel = SK_DIM0;
  else if (sk.rfind("reduce_dim{1", 0) == 0) skel = SK_DIM1;
  if (skel < 0) return 0;
  int n = 0;
  const TemplateEntry *t = template_table(&n);
  for (int i = 0; i < n; ++i)
    if (sig == t[i].signature) {
      *kernel_id = i * 4 + skel;
      return 0;
    }
  return 0;
}

int fm_launch_copy(int kernel_id, const fm_program *prog, void *out, int64_t n_rows, int64_t n_cols,
                   void *stream) {
  int st = validate_program(prog);
  if (st) return st;
  if (!out && n_rows * n_cols > 0) return fail_msg("copy: null output");
  cudaStream_t s = (cudaStream_t)stream;
  if (kernel_id >= 0) {
    const TemplateEntry *e = entry_for(kernel_id, SK_COPY);
    if (!e || e->n_inputs != prog->n_slots) return fail_msg("copy: kernel id does not match the program");
    return e->copy(*prog, out, n_rows, n_cols, s);
  }
  return vm_dispatch<CopyF>(*prog, out, n_rows, n_cols, s);
}

int fm_launch_accu(int kernel_id, const fm_program *prog, void *out, int64_t n_rows, int64_t n_cols,
                   int32_t finalize, void *stream) {
  int st = validate_program(prog);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (kernel_id >= 0) {
    const TemplateEntry *e = entry_for(kernel_id, SK_ACCU);
    if (!e || e->n_inputs != prog->n_slots) return fail_msg("accu: kernel id does not match the program");
    return e->accu(*prog, out, n_rows, n_cols, finalize, s);
  }
  return vm_dispatch<AccuF>(*prog, out, n_rows, n_cols, (int)finalize, s);
}

int fm_launch_reduce_dim(int kernel_id, const fm_program *prog, int32_t dim, int64_t n_rows,
                         int64_t n_cols, const fm_reduce_out *outs, int32_t n_outs, void *stream) {
  int st = validate_program(prog);
  if (st) return st;
  if (dim != 0 && dim != 1) return fail_msg("reduce_dim: dim must be 0 or 1");
  if (n_outs <= 0 || n_outs > FM_MAX_REDUCE_OUT) return fail_msg("reduce_dim: bad output count");
  ReduceOuts R;
  R.n = n_outs;
  for (int i = 0; i < n_outs; ++i) {
    if (!outs[i].out) return fail_msg("reduce_dim: null output");
    R.o[i] = outs[i];
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (kernel_id >= 0) {
    const TemplateEntry *e = entry_for(kernel_id, dim == 0 ? SK_DIM0 : SK_DIM1);
    if (!e || e->n_inputs != prog->n_slots) return fail_msg("reduce_dim: kernel id does not match the program");
    return e->reduce_dim(*prog, dim, n_rows, n_cols, R, s);
  }
  return vm_dispatch<DimF>(*prog, (int)dim, n_rows, n_cols, R, s);
}

}  // extern "C"
