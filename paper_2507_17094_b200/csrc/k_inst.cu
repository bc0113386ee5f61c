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

// -DPW_FAST: the FAST instance (cold paths compiled out, beam_search.cuh)
// -DPW_FAST -DPW_WIDE: its 20-warp build (kWideWarps x 32 threads)
#if defined(PW_FAST) && defined(PW_WIDE)
#define PW_FAST_V true, pw::kWideWarps * 32
#define PW_SFX(name) PW_CAT(name, fw_)
#elif defined(PW_FAST)
#define PW_FAST_V true
#define PW_SFX(name) PW_CAT(name, f_)
#else
#define PW_FAST_V false
#define PW_SFX(name) name
#endif
#if defined(PW_U8)
pw::KernelFn PW_CAT(PW_SFX(pw_kernel_u8_), PW_DIM)() { return pw::beam_search_kernel<PW_DIM, uint8_t, 0, PW_FAST_V>; }
#elif defined(PW_IP)
pw::KernelFn PW_CAT(PW_SFX(pw_kernel_ip_), PW_DIM)() { return pw::beam_search_kernel<PW_DIM, float, 1, PW_FAST_V>; }
#else
pw::KernelFn PW_CAT(PW_SFX(pw_kernel_), PW_DIM)() { return pw::beam_search_kernel<PW_DIM, float, 0, PW_FAST_V>; }
#endif
