// fbf_kernel_inst.cu -- explicit instantiations of the fused kernel for
// radii [FBF_R_LO, FBF_R_HI] (built several times with different ranges so
// the 32 radius specialisations compile in parallel).
#include "fbf_kernel.cuh"

#ifndef FBF_R_LO
#define FBF_R_LO 1
#endif
#ifndef FBF_R_HI
#define FBF_R_HI 32
#endif

#include "fbf_kernel_inst_list.inc"
