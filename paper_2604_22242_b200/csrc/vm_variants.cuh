// vm_variants.cuh -- the four register-VM instantiations and their explicit
// instantiation declarations.  The VM kernels are large (one specialised
// case per (opcode, stack slot)), so each (variant, skeleton) pair is
// compiled in its own object from vm_inst.cu (build.py passes
// -DFM_VM_VARIANT / -DFM_VM_SKELETON) and the objects build in parallel;
// fused.cu only sees these declarations.
#pragma once
#include "launch.cuh"

namespace fm {

// 64-bit registers only when the program touches f64; a shallower stack when
// the program allows (fewer live registers).
using Vm32s = Vm<false, 4, 8, 4>;
using Vm32d = Vm<false, 8, 8, 4>;
using Vm64s = Vm<true, 4, 4, 4>;
using Vm64d = Vm<true, 8, 4, 4>;

#define FM_VM_DECLARE(E)                                                                          \
  extern template int run_copy<E>(const fm_program &, void *, int64_t, int64_t, cudaStream_t);    \
  extern template int run_accu<E>(const fm_program &, void *, int64_t, int64_t, int, cudaStream_t); \
  extern template int run_reduce_dim<E>(const fm_program &, int, int64_t, int64_t, const ReduceOuts &, \
                                        cudaStream_t);                                                  \
  extern template int run_split<E>(const fm_program &, uint16_t *, int64_t, int64_t, int64_t, int64_t,  \
                                   const unsigned *, cudaStream_t);
#ifndef FM_VM_VARIANT
FM_VM_DECLARE(Vm32s)
FM_VM_DECLARE(Vm32d)
FM_VM_DECLARE(Vm64s)
FM_VM_DECLARE(Vm64d)
#endif
#undef FM_VM_DECLARE

}  // namespace fm
