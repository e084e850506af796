// vm_inst.cu -- explicit instantiation of one register-VM variant for one
// skeleton (see vm_variants.cuh).  Compiled once per
//   FM_VM_VARIANT  in 0..3  (Vm32s, Vm32d, Vm64s, Vm64d)
//   FM_VM_SKELETON in 0..3  (copy, accu, reduce_dim, gemm operand split)
#ifndef FM_VM_VARIANT
#error "build.py compiles this file with -DFM_VM_VARIANT=<0..3> -DFM_VM_SKELETON=<0..3>"
#endif
#include "vm_variants.cuh"

namespace fm {

#if FM_VM_VARIANT == 0
using VmT = Vm32s;
#elif FM_VM_VARIANT == 1
using VmT = Vm32d;
#elif FM_VM_VARIANT == 2
using VmT = Vm64s;
#else
using VmT = Vm64d;
#endif

#if FM_VM_SKELETON == 0
template int run_copy<VmT>(const fm_program &, void *, int64_t, int64_t, cudaStream_t);
#elif FM_VM_SKELETON == 1
template int run_accu<VmT>(const fm_program &, void *, int64_t, int64_t, int, cudaStream_t);
#elif FM_VM_SKELETON == 2
template int run_reduce_dim<VmT>(const fm_program &, int, int64_t, int64_t, const ReduceOuts &, cudaStream_t);
#else
template int run_split<VmT>(const fm_program &, uint16_t *, int64_t, int64_t, int64_t, int64_t, const unsigned *,
                            cudaStream_t);
#endif

}  // namespace fm
