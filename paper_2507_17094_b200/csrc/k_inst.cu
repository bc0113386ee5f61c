// k_inst.cu -- one specialisation of K1 per translation unit, compiled once
// per dimension with -DPW_DIM=<d> (0 = generic d) so the instantiations build
// in parallel; pw_abi.cu reaches each through pw_kernel_<d>().
#include "beam_search.cuh"

#ifndef PW_DIM
#error "compile with -DPW_DIM=<dimension>"
#endif
#define PW_CAT2(a, b) a##b
#define PW_CAT(a, b) PW_CAT2(a, b)

pw::KernelFn PW_CAT(pw_kernel_, PW_DIM)() { return pw::beam_search_kernel<PW_DIM>; }
