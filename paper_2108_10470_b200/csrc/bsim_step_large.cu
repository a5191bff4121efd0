// bsim_step_large.cu -- the fused step kernel for large articulations.
//
// Same source as bsim_step.cu, compiled with a CTA of 8 envs x 32 threads
// (fp32; fp64: 2 envs x 32) and its own namespace so the two instantiations
// never collide.  A 22-body / 21-joint / 22-slot humanoid (8.8 KB of
// workspace per env in fp32) then runs 2 CTAs (16 envs, 16 warps) per SM
// instead of one 16-env CTA (4 warps) with the default shape.  bsim_step.cu
// dispatches here when its default CTA's workspace exceeds 113 KB.
#define BSIM_LARGE_TU 1
// fp32 CTA: 8 envs x 32 threads, >= 2 CTAs per SM (<= 128 registers).  The
// sweep warp then carries 8 envs (4 lanes each) instead of 4: measured at
// 16384 envs, humanoid 1804 -> 1490 us per control step, Franka cube-stack
// 7.46 -> 8.70 M, Shadow Hand 3.92 -> 4.26 M env-steps/s, against 4 x 32
// with 5 CTAs/SM (the round-1 shape); 8 x 32 at 3 CTAs/SM spills, 6 x 32,
// 12 x 32 and 16 x 32 are slower.
#ifndef BSIM_LARGE_NE
#define BSIM_LARGE_NE 8
#endif
#ifndef BSIM_LARGE_MINB
#define BSIM_LARGE_MINB 2
#endif
#undef BSIM_NE32
#undef BSIM_NTH32
#undef BSIM_NE64
#undef BSIM_NTH64
#undef BSIM_MINB
#define BSIM_NE32 BSIM_LARGE_NE
#define BSIM_NTH32 (32 * BSIM_LARGE_NE)
#define BSIM_NE64 2
#define BSIM_NTH64 64
#define BSIM_MINB BSIM_LARGE_MINB
#ifndef BSIM_LARGE_SUBGROUPS
#define BSIM_LARGE_SUBGROUPS 1   // 4 = one warp per env with its own named barrier: measured 1804 -> 2417 us
#endif                           // per 16384-env humanoid step, so the CTA stays whole
#define BSIM_SUBGROUPS BSIM_LARGE_SUBGROUPS
#ifndef BSIM_LARGE_SCHED_WARPS   // the row-schedule sweep on 4 warps (16 lanes per env): measured
#define BSIM_LARGE_SCHED_WARPS 4    // humanoid 16384 envs 1610 -> 1541 us per control step (phased
#endif                              // schedule; 2 warps 1586), Shadow Hand / Franka unchanged
#undef BSIM_SCHED_WARPS
#define BSIM_SCHED_WARPS BSIM_LARGE_SCHED_WARPS
#define bsim bsim_large
#include "bsim_step.cu"
