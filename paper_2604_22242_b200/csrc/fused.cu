// fused.cu -- C-ABI launch entry points of the fused path and the generic
// register-VM kernels (include/fmb200.h: fm_launch_copy / fm_launch_accu /
// fm_launch_reduce_dim / fm_kernel_lookup).
//
// Replaces the reference's compile-and-launch path (cjit.py:113-154): a
// kernel id from fm_kernel_lookup selects an ahead-of-time template kernel;
// id -1 runs the same program on the VM.  Either way one launch per fused
// step.
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
  static int run(const fm_program &P, uint16_t *o, int64_t r, int64_t c, int64_t ld, int64_t po, cudaStream_t s) {
    return run_split<E>(P, o, r, c, ld, po, s);
  }
};

int launch_split_program(const fm_program &P, uint16_t *planes, int64_t n_rows, int64_t n_cols, int64_t ld_out,
                         int64_t plane_off, cudaStream_t s) {
  return vm_dispatch<SplitF>(P, planes, n_rows, n_cols, ld_out, plane_off, s);
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
