// bsim_step_large.cu -- the fused step kernel for large articulations.
//
// Same source as bsim_step.cu, compiled with a CTA of 4 envs x 32 threads
// (fp32; fp64: 2 envs x 32) and its own namespace so the two instantiations
// never collide.  The per-env workspace is item-major / env-minor with stride
// NE + 1 = 5, so a 22-body / 21-joint / 22-slot humanoid (2,207 items, 8.8 KB
// per env in fp32) fits 5 CTAs (20 envs, 20 warps) per SM instead of one
// 16-env CTA (4 warps) with the default shape.  bsim_step.cu dispatches here
// when its default CTA would leave fewer than 2 CTAs per SM.
#define BSIM_LARGE_TU 1
#define BSIM_NE32 4
#define BSIM_NTH32 128
#define BSIM_NE64 2
#define BSIM_NTH64 64
#define BSIM_MINB 5   // 5 x 128 threads: the 20-env-per-SM occupancy the record size allows
#ifndef BSIM_LARGE_SUBGROUPS
#define BSIM_LARGE_SUBGROUPS 1   // 4 = one warp per env with its own named barrier: measured 1804 -> 2417 us
#endif                           // per 16384-env humanoid step, so the CTA stays whole
#define BSIM_SUBGROUPS BSIM_LARGE_SUBGROUPS
#define bsim bsim_large
#include "bsim_step.cu"
