// k_inst.cu -- one specialisation of K1 per translation unit, compiled once
// per dimension with -DPW_DIM=<d> (0 = generic d) -- and -DPW_U8 for uint8
// rows, -DPW_IP for the inner-product metric -- so the instantiations build in parallel; pw_abi.cu reaches each
// through pw_kernel_<d>() / pw_kernel_u8_<d>().
#include "beam_search.cuh"

#ifndef PW_DIM
#error "compile with -DPW_DIM=<dimension>"
#endif
#define PW_CAT2(a, b) a##b
#define PW_CAT(a, b) PW_CAT2(a, b)

#if defined(PW_U8)
pw::KernelFn PW_CAT(pw_kernel_u8_, PW_DIM)() { return pw::beam_search_kernel<PW_DIM, uint8_t, 0>; }
#elif defined(PW_IP)
pw::KernelFn PW_CAT(pw_kernel_ip_, PW_DIM)() { return pw::beam_search_kernel<PW_DIM, float, 1>; }
#else
pw::KernelFn PW_CAT(pw_kernel_, PW_DIM)() { return pw::beam_search_kernel<PW_DIM, float, 0>; }
#endif
