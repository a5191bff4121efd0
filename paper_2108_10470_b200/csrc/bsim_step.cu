// bsim_step.cu -- sm_100a kernels for the batched TGS step, forward kinematics,
// indexed state setters, contact queries, and their C-ABI entry points
// (declared in include/batchsim_b200.h).
//
// Step kernel mapping: one CTA owns up to NE envs (Shape<R>
// in bsim_step.cuh: 16 fp32 / 8 fp64; the launch plan picks `epc` <= NE for
// whole waves) with 8 threads per env for the lane-parallel phase A and one
// thread (two for the Ant's star sweep) per env for the Gauss-Seidel sweep.
// The CTA's workspace is dynamic shared memory: one env-major record per env
// (16-byte aligned vector items, PAD = 4 mod 8 words apart) followed by a
// padded copy of the joint table.  Body state moves HBM <-> shared memory
// with coalesced loads / stores of the CTA's contiguous [envs x B bodies x 13]
// slab; all substeps of a control step run on the resident workspace, so HBM
// sees the state once per control step.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "bsim_step.cuh"
#include "bsim_topologies.cuh"
#include "bsim_kin.cuh"
#include "bsim_tasks.cuh"

using namespace bsim;

#ifndef BSIM_LARGE_TU
extern "C" {
int bsim_large_step_f32(const bsim_layout_t *, const bsim_params_t *, const bsim_state_t *, int32_t,
                        const bsim_actions_t *, const bsim_task_t *, int32_t, int32_t, void *);
int bsim_large_step_f64(const bsim_layout_t *, const bsim_params64_t *, const bsim_state64_t *, int32_t,
                        const bsim_actions_t *, const bsim_task_t *, int32_t, int32_t, void *);
int bsim_large_envs_per_wave(const bsim_layout_t *, int32_t, int32_t *);
const char *bsim_large_last_error(void);
}
#endif

namespace {

std::string g_err;

int set_err(const char *what, cudaError_t e) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return BSIM_E_CUDA;
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(what, e);
    return BSIM_OK;
}

// the env workspace records, then a copy of the joint table (phase A reads
// its frames every pass; from L1/L2 they were a top long-scoreboard stall)
template <class R> __host__ __device__ size_t step_ws_bytes(const Dims &d, int n_envs = Shape<R>::NE) {
    return ((size_t)d.pad * n_envs * sizeof(R) + 15) & ~(size_t)15;
}
template <class R> size_t step_smem_bytes(const Dims &d, int n_envs = Shape<R>::NE) {
    return step_ws_bytes<R>(d, n_envs) + (size_t)d.J * jtab_stride_smem<R>();
}

// ------------------------------------------------------------------ step
// Sub-partition placement of the serial sweep.  A warp's SM sub-partition
// (scheduler) is its hardware warp slot % 4; the co-resident CTAs of an SM
// must not all run their one-warp Gauss-Seidel sweep on the same scheduler.
// Each CTA claims a free sub-partition in a per-SM bitmask (released at
// exit) and runs its sweep on its warp that lives there.  Placement only:
// which lanes execute an env's sweep never changes its arithmetic.
__device__ unsigned int g_sweep_smsp[1024];

__device__ __forceinline__ unsigned hw_warp_slot() {
    unsigned w;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(w));
    return w;
}
__device__ __forceinline__ unsigned hw_sm_id() {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    return s;
}

// thread 0: claim a sub-partition among those this CTA's warps occupy;
// returns the claimed bit (0 = none free) and the warp to sweep on.
template <int NW> __device__ unsigned claim_sweep_smsp(const int *warp_smsp, unsigned *sm_slot, int &warp) {
    unsigned avail = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) avail |= 1u << warp_smsp[w];
    unsigned *m = &g_sweep_smsp[*sm_slot = hw_sm_id() & 1023];
    unsigned old = *(volatile unsigned *)m, bit = 0;
    for (int tries = 0; tries < 8; ++tries) {
        unsigned free_ = avail & ~old;
        if (!free_) break;
        unsigned b = free_ & (0u - free_);
        unsigned prev = atomicCAS(m, old, old | b);
        if (prev == old) {
            bit = b;
            break;
        }
        old = prev;
    }
    warp = 0;
    if (bit)
#pragma unroll
        for (int w = 0; w < NW; ++w)
            if ((1u << warp_smsp[w]) == bit) warp = w;
    return bit;
}

template <class R>
__device__ __noinline__ void task_step_env_call(const Ctx<R> &c, const bsim_task_t &t, R *stage, int e0, int e, int sl,
                                                R *scratch) {
    TaskView<R> tv{t, stage, e0};
    tv.scratch = scratch;
    tv.scratch_stride = (13 * c.d.B + 2 * c.d.D + 3) & ~3;
    task_step_env_g<R, BSIM_TASK_G>(c, tv, e, sl);
}

#ifndef BSIM_SUBGROUPS
#define BSIM_SUBGROUPS 1
#endif
static_assert(BSIM_SUBGROUPS >= 1 && BSIM_SUBGROUPS <= 8, "1..8 sub-CTA env groups");
#ifndef BSIM_MINB
#define BSIM_MINB 4   // 4 x 128 threads at <= 128 registers: matches the shared-memory limit
#endif
// `epc` envs per CTA (<= NE): chosen by the launcher so the grid is a whole
// number of waves of resident CTAs (148 SMs x CTAs/SM).  The grid covers envs
// [e_begin, e_end) -- all of them, or one wave-sized chunk of the pipelined
// host-buffer step (bsim_env_step_range).
#ifdef BSIM_EXP_PHASE_CLOCKS
// timing experiment only: thread-0 cycles per step_kernel phase summed over CTAs ([7] = CTAs),
// and per CTA of the last launch: SM id, %globaltimer at entry, before the task tail, at exit
__device__ unsigned long long g_phase_clk[8];
__device__ unsigned long long g_cta_times[4096][4];
__device__ unsigned long long g_last_end;        // latest CTA exit %globaltimer (previous launches)
__device__ unsigned long long g_gap_sum, g_gap_n;   // first-CTA start - previous launch's last exit
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif
template <class R, class T, bool SCHED>
__global__ void __launch_bounds__(Shape<R>::NTH, BSIM_MINB)
    step_kernel(const __grid_constant__ Ctx<R> c, int n_substeps, bsim_actions_t act, int epc, int e_begin,
                int e_end, const __grid_constant__ bsim_task_t task, int with_task) {
    constexpr int NTH = Shape<R>::NTH;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Dims &d = c.d;
    R *ws = reinterpret_cast<R *>(smem_raw);
    const int tid = threadIdx.x;
    const int e0 = e_begin + blockIdx.x * epc;   // envs [e_begin, e_end) of the scene's E
#ifdef BSIM_EXP_PHASE_CLOCKS
    unsigned long long pc_prev = clock64();
    if (tid == 0) atomicAdd(&g_phase_clk[7], 1ull);
    if (tid == 0 && blockIdx.x < 4096) {
        g_cta_times[blockIdx.x][0] = hw_sm_id();
        g_cta_times[blockIdx.x][1] = gtimer();
    }
    if (tid == 0 && blockIdx.x == 0) {   // block 0 starts first: the gap since the previous launch's last CTA
        const unsigned long long prev = *(volatile unsigned long long *)&g_last_end, now = gtimer();
        if (prev && now > prev && now - prev < 1000000ull) {
            atomicAdd(&g_gap_sum, now - prev);
            atomicAdd(&g_gap_n, 1ull);
        }
    }
#define BSIM_PCLK(i)                                                             \
    do {                                                                         \
        if (tid == 0) {                                                          \
            unsigned long long t_ = clock64();                                   \
            atomicAdd(&g_phase_clk[i], t_ - pc_prev);                            \
            pc_prev = t_;                                                        \
        }                                                                        \
    } while (0)
#else
#define BSIM_PCLK(i) \
    do {             \
    } while (0)
#endif
    const int ne = min(epc, e_end - e0);
    const int per_env = 13 * d.B;
    constexpr int NW = NTH / 32;
    __shared__ int s_warp_smsp[NW], s_sweep_warp;
    __shared__ unsigned s_sweep_bit, s_sm_slot;
    if ((tid & 31) == 0) s_warp_smsp[tid >> 5] = hw_warp_slot() & 3;

    // coalesced load of the CTA's contiguous [ne x B x 13] body slab
    {
        const R *src = c.s.body_q + (size_t)e0 * per_env;
        for (int i = tid; i < ne * per_env; i += NTH) {
            int el = i / per_env, item = i - el * per_env;
            int b = item / 13, k = item - b * 13;
            ws[(size_t)el * d.pad + d.o_body + b * BODY_ITEMS + body_item13(k)] = src[i];
        }
        // the joint table (sizeof(Joint) is a multiple of 16 bytes)
        constexpr int rec16 = (int)(sizeof(typename Abi<R>::Joint) / 16), str16 = jtab_stride_smem<R>() / 16;
        const float4 *js = reinterpret_cast<const float4 *>(c.joints);
        float4 *jd = reinterpret_cast<float4 *>(smem_raw + step_ws_bytes<R>(d, epc));
        for (int i = tid; i < d.J * rec16; i += NTH) jd[(i / rec16) * str16 + i % rec16] = js[i];
    }
    // the per-env inputs and the fused action mapping (envs.py:180, 421-424)
    // in the same phase as the slab load: their global loads overlap instead
    // of waiting behind a barrier (they write workspace items the slab does
    // not, and the targets are read after the barriers below)
    {
        const Grp<R> g0{ws, e0, ne, tid, NTH, 0, d.pad, JTab<R>{nullptr, 0}};
        stage_group(c, g0);
        if (act.actions) {
            BS_ITEMS(g0, d.D, el, k) {
                size_t o = (size_t)(e0 + el) * d.D + k;
                R a = clampr(reinterpret_cast<const R *>(act.actions)[o], R(-1), R(1));
                if (act.actions_clipped) reinterpret_cast<R *>(act.actions_clipped)[o] = a;
                R v = R(act.scale) * a;
                if (act.mode == BSIM_MODE_POSITION)
                    c.s.ctrl_dof_pos_target[o] = v;
                else
                    c.s.ctrl_dof_force[o] = v;
            }
        }
    }
    __syncthreads();
    BSIM_PCLK(0);
    if (tid == 0) {
        int w;
        s_sweep_bit = claim_sweep_smsp<NW>(s_warp_smsp, &s_sm_slot, w);
        s_sweep_warp = w;
    }
    __syncthreads();
    const Grp<R> g{ws, e0, ne, tid, NTH, 32 * s_sweep_warp, d.pad,
                   JTab<R>{smem_raw + step_ws_bytes<R>(d, epc), jtab_stride_smem<R>()}};
    BSIM_PCLK(1);
    // BSIM_SUBGROUPS = K > 1: the substeps run on K independent groups of
    // NTH / K threads (envs split evenly, each group with its own named
    // barrier and sweep warp), so one group's phase A overlaps another's
    // sweep instead of the whole CTA waiting at every barrier.  Measured
    // slower on both CTAs, so K = 1: the default CTA with K = 2
    // (Ant 234 -> 252 us), the large CTA with K = 4 (humanoid 1804 -> 2417 us)
    constexpr int K = NTH / 32 < BSIM_SUBGROUPS ? NTH / 32 : BSIM_SUBGROUPS;   // named barriers: >= 1 warp each
    constexpr bool halves = K > 1;
    Grp<R> gs = g;
    if (halves) {
        constexpr int TG = NTH / K;
        const int h = tid / TG, per = (ne + K - 1) / K, first = min(ne, h * per);
        gs.ws = ws + (size_t)first * d.pad;
        gs.e0 = e0 + first;
        gs.ne = min(ne, first + per) - first;
        gs.tid = tid % TG;
        gs.nth = TG;
        gs.lane0 = 0;
        gs.bar = 1 + h;
    }
    for (int s = 0; s < n_substeps; ++s) {
        group_step<R, T, SCHED>(c, gs, s == n_substeps - 1, s);
        if (d.T && s != n_substeps - 1) {  // fixed tendons read dof_state next substep
            if (halves) __syncthreads();
            readout_group(c, g);
            __syncthreads();
        }
    }
    if (halves) __syncthreads();
    BSIM_PCLK(2);
    readout_group(c, g);
    BS_ITEMS(g, d.P, el, i) {
        for (int k = 0; k < 3; ++k)
            c.s.friction_anchor[3 * ((size_t)i * d.E + e0 + el) + k] =
                g.env(el).at(d.o_anchor + ANCHOR_ITEMS * i + k);
    }
    // (no barrier: the readout above and the stores below only read the
    // workspace, final since group_step's last barrier)
    // coalesced stores: canonical env-local state, world-frame body_state / root_state
    {
        R *dq = c.s.body_q + (size_t)e0 * per_env;
        R *db = c.s.body_state + (size_t)e0 * per_env;
        for (int i = tid; i < ne * per_env; i += NTH) {
            int el = i / per_env, item = i - el * per_env;
            int b = item / 13, k = item - b * 13;
            R x = ws[(size_t)el * d.pad + d.o_body + b * BODY_ITEMS + body_item13(k)];
            dq[i] = x;
            db[i] = k < 3 ? x + c.s.env_origins[3 * (size_t)(e0 + el) + k] : x;
        }
        const int per_root = d.A * 13;
        R *dr = c.s.root_state + (size_t)e0 * per_root;
        for (int i = tid; i < ne * per_root; i += NTH) {
            int el = i / per_root, item = i - el * per_root;
            int a = item / 13, k = item - a * 13;
            int b = c.L.actor_body_offset[a];
            R x = ws[(size_t)el * d.pad + d.o_body + b * BODY_ITEMS + body_item13(k)];
            dr[i] = k < 3 ? x + c.s.env_origins[3 * (size_t)(e0 + el) + k] : x;
        }
    }
    if (tid == 0 && s_sweep_bit) atomicAnd(&g_sweep_smsp[s_sm_slot], ~s_sweep_bit);
    if (with_task) {   // EnvBatch.step tail for this CTA's envs (bsim_env_step)
        __syncthreads();   // the CTA's state stores above are visible; the workspace is dead
        BSIM_PCLK(3);
#ifdef BSIM_EXP_PHASE_CLOCKS
        if (tid == 0 && blockIdx.x < 4096) g_cta_times[blockIdx.x][2] = gtimer();
#endif
        // observation rows are staged in the dead workspace and leave as one
        // coalesced block (task.obs may be mapped host memory: bsim_env_step_host
        // zero-copy mode, where a scattered row store would be a PCIe write each)
        R *stage = ws;
        // the resets' FK scratch rows follow the obs rows in the dead workspace
        const size_t obs_words = ((size_t)ne * task.obs_dim + 3) & ~(size_t)3;
        const size_t scr_words = (size_t)ne * ((13 * d.B + 2 * d.D + 3) & ~3);
        R *scratch = obs_words + scr_words <= (size_t)epc * d.pad ? ws + obs_words : nullptr;
#ifndef BSIM_EXP_SKIP_TAIL   // timing experiment only: the launch without the tail's work
        if (tid < BSIM_TASK_G * ne)
            task_step_env_call(c, task, stage, e0, e0 + tid / BSIM_TASK_G, tid % BSIM_TASK_G, scratch);
#endif
        __syncthreads();
        BSIM_PCLK(4);
        R *dst = reinterpret_cast<R *>(task.obs) + (size_t)e0 * task.obs_dim;
        for (int i = tid; i < ne * task.obs_dim; i += NTH) dst[i] = stage[i];
        BSIM_PCLK(5);
    }
#ifdef BSIM_EXP_PHASE_CLOCKS
    if (tid == 0 && blockIdx.x < 4096) {
        if (!with_task) g_cta_times[blockIdx.x][2] = gtimer();
        g_cta_times[blockIdx.x][3] = gtimer();
    }
    if (tid == 0) {
        __threadfence();
        atomicMax(&g_last_end, gtimer());
    }
#endif
#undef BSIM_PCLK
}

// Scene.forward_kinematics(env_mask, actors) + the buffers' repack
// (physics.py:366-425, buffers.py:109-123): a group of FK_G lanes per env on
// a shared-memory copy of the env's rows and DOF state (fk_group walks the
// tree level by level), FK_EPC envs per CTA; bodies >= 64 (fk_group's mask)
// fall back to one lane per env on global memory.
constexpr int FK_G = 8, FK_EPC = 16;
template <class R> __host__ __device__ int fk_stride(const Dims &d) { return (13 * d.B + 2 * d.D + 3) & ~3; }
template <class R>
__global__ void __launch_bounds__(FK_G * FK_EPC)
    fk_kernel(Ctx<R> c, const uint8_t *env_mask, const uint32_t *amask_dev, uint32_t amask) {
    extern __shared__ __align__(16) unsigned char fk_smem[];
    const Dims &d = c.d;
    const int el = threadIdx.x / FK_G, sl = threadIdx.x % FK_G;
    const int e = blockIdx.x * FK_EPC + el;
    if (e >= d.E || (env_mask && !env_mask[e])) return;   // whole groups leave together
    const uint32_t m = amask_dev ? *amask_dev : amask;
    if (d.B > 64) {
        if (sl == 0) {
            fk_env(c, e, m);
            repack_env(c, e, m);
        }
        return;
    }
    constexpr unsigned gm_base = (1u << FK_G) - 1u;
    const unsigned gm = gm_base << ((threadIdx.x & 31u) & ~(unsigned)(FK_G - 1));
    R *__restrict__ bq = reinterpret_cast<R *>(fk_smem) + (size_t)el * fk_stride<R>(d);
    R *__restrict__ dq = bq + 13 * d.B;
    const R *__restrict__ gq = c.s.body_q + (size_t)e * d.B * 13;
    const R *__restrict__ gd = c.s.dof_state + 2 * (size_t)e * d.D;
#pragma unroll 4
    for (int i = sl; i < 13 * d.B; i += FK_G) bq[i] = gq[i];
#pragma unroll 4
    for (int i = sl; i < 2 * d.D; i += FK_G) dq[i] = gd[i];
    __syncwarp(gm);
    fk_group<FK_G>(c, bq, dq, sl, gm, m);
    const R *__restrict__ o = c.s.env_origins + 3 * (size_t)e;
    const R ox = o[0], oy = o[1], oz = o[2];
    for (int a = 0; a < d.A; ++a) {               // rows of the masked actors (fk_env + repack_env)
        if (!((m >> a) & 1u)) continue;
        const int b0 = c.L.actor_body_offset[a], n = 13 * (c.L.actor_body_offset[a + 1] - b0);
        R *__restrict__ dst_q = c.s.body_q + 13 * ((size_t)e * d.B + b0);
        R *__restrict__ dst_s = c.s.body_state + 13 * ((size_t)e * d.B + b0);
        const R *src = bq + 13 * b0;
        for (int i = sl; i < n; i += FK_G) {
            const int k = i % 13;
            const R v = src[i];
            dst_q[i] = v;
            dst_s[i] = v + (k == 0 ? ox : k == 1 ? oy : k == 2 ? oz : R(0));
        }
        R *__restrict__ rr = c.s.root_state + 13 * ((size_t)e * d.A + a);
        for (int k = sl; k < 13; k += FK_G) rr[k] = src[k] + (k == 0 ? ox : k == 1 ? oy : k == 2 ? oz : R(0));
    }
}

// refresh_buffers without a contact context (physics.py:1037-1046): DOF
// readout and body / root packing for REF_EPC envs per CTA.  The CTA's
// contiguous [envs x B x 13] slab of body_q is staged in shared memory with
// one coalesced pass, body_state / root_state leave coalesced from it, and
// the DOF readout runs one thread per (env, joint) on the staged rows.
constexpr int REF_EPC = 16, REF_NTH = 256;
template <class R> __global__ void __launch_bounds__(REF_NTH) refresh_kernel(Ctx<R> c) {
    extern __shared__ __align__(16) unsigned char ref_smem[];
    const Dims &d = c.d;
    const int e0 = blockIdx.x * REF_EPC, ne = min(REF_EPC, d.E - e0), per = 13 * d.B;
    R *__restrict__ sq = reinterpret_cast<R *>(ref_smem);
    const R *__restrict__ gq = c.s.body_q + (size_t)e0 * per;
    R *__restrict__ gs = c.s.body_state + (size_t)e0 * per;
    const R *__restrict__ org = c.s.env_origins + 3 * (size_t)e0;
    for (int i = threadIdx.x; i < ne * per; i += REF_NTH) {
        const R v = gq[i];
        const int el = i / per, k = (i - el * per) % 13;
        sq[i] = v;
        gs[i] = k < 3 ? v + org[3 * el + k] : v;
    }
    __syncthreads();
    R *__restrict__ gr = c.s.root_state + (size_t)e0 * d.A * 13;
    for (int i = threadIdx.x; i < ne * d.A * 13; i += REF_NTH) {
        const int el = i / (13 * d.A), rem = i - el * 13 * d.A, a = rem / 13, k = rem - a * 13;
        const R v = sq[el * per + 13 * c.L.actor_body_offset[a] + k];
        gr[i] = k < 3 ? v + org[3 * el + k] : v;
    }
    for (int i = threadIdx.x; i < ne * d.J; i += REF_NTH) {
        const int el = i / d.J, j = i - el * d.J;
        readout_joint(c, c.joints[j], sq + (size_t)el * per, c.s.dof_state + 2 * (size_t)(e0 + el) * d.D);
    }
}

// set_root_state: write the root bodies of the listed actors (env-local), renormalise quats
template <class R>
__global__ void set_root_kernel(Ctx<R> c, const R *values, const int64_t *idx, int n, uint8_t *env_mask,
                                uint32_t *amask) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t a_glob = idx[i];
    int e = (int)(a_glob / c.d.A), a = (int)(a_glob % c.d.A);
    const R *v = values + 13 * a_glob;
    R nq = r_sqrt(v[3] * v[3] + v[4] * v[4] + v[5] * v[5] + v[6] * v[6]);
    R *dst = c.s.body_q + 13 * ((size_t)e * c.d.B + c.L.actor_body_offset[a]);
    const R *o = c.s.env_origins + 3 * (size_t)e;
    for (int k = 0; k < 3; ++k) dst[k] = v[k] - o[k];
    for (int k = 3; k < 7; ++k) dst[k] = v[k] / nq;
    for (int k = 7; k < 13; ++k) dst[k] = v[k];
    env_mask[e] = 1;
    atomicOr(amask, 1u << a);
}

template <class R>
__global__ void set_dof_kernel(Ctx<R> c, const R *values, const int64_t *idx, int n, uint8_t *env_mask,
                               uint32_t *amask) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t a_glob = idx[i];
    int e = (int)(a_glob / c.d.A), a = (int)(a_glob % c.d.A);
    int d0 = c.L.actor_dof_offset[a], d1 = c.L.actor_dof_offset[a + 1];
    if (d1 == d0) return;
    for (int k = d0; k < d1; ++k) {
        size_t r = (size_t)e * c.d.D + k;
        c.s.dof_state[2 * r] = values[2 * r];
        c.s.dof_state[2 * r + 1] = values[2 * r + 1];
    }
    env_mask[e] = 1;
    atomicOr(amask, 1u << a);
}

// contact candidate per (slot, env) (physics.py:463-498); world-frame point
template <class R>
__device__ void slot_geometry(const Ctx<R> &c, int i, int e, bool &active, R &depth, V3<R> &point, V3<R> &n) {
    const Dims &d = c.d;
    const size_t E = (size_t)d.E;
    const R *bq = c.s.body_q + (size_t)e * d.B * 13;
    V3<R> org = jv3(c.s.env_origins + 3 * (size_t)e);
    if (i < d.P) {
        int b = c.L.plane_body[i];
        const R *B_ = bq + 13 * b;
        const R *off = c.s.plane_off + 3 * ((size_t)i * E + e);
        R rad = c.s.plane_rad[(size_t)i * E + e];
        V3<R> arm = qrot(Q4<R>{B_[3], B_[4], B_[5], B_[6]}, jv3(off));
        V3<R> pos = V3<R>{B_[0], B_[1], B_[2]};
        R gap = (pos.z + arm.z) - rad;
        depth = c.p.rest_offset - gap;
        point = pos + v3(arm.x, arm.y, arm.z - rad) + org;
        n = v3(R(0), R(0), R(1));
    } else {
        int q = i - d.P;
        const R *A_ = bq + 13 * c.L.pair_body[2 * q], *B_ = bq + 13 * c.L.pair_body[2 * q + 1];
        const R *off = c.s.pair_off + 6 * ((size_t)q * E + e);
        const R *rr = c.s.pair_rad + 2 * ((size_t)q * E + e);
        V3<R> pa = V3<R>{A_[0], A_[1], A_[2]};
        V3<R> ra;
        R gap;
        pair_shape_contact(c.L.pair_kind[q], Q4<R>{A_[3], A_[4], A_[5], A_[6]}, Q4<R>{B_[3], B_[4], B_[5], B_[6]},
                           V3<R>{B_[0], B_[1], B_[2]} - pa, off, rr, c.pair_ext() + 4 * q, n, gap, ra);
        depth = c.p.rest_offset - gap;
        point = pa + ra + org;
    }
    active = depth > -c.p.solver_offset_slop;
}

template <class R>
__global__ void contact_geometry_kernel(Ctx<R> c, uint8_t *active, R *depth, R *point, R *normal) {
    size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    size_t total = (size_t)(c.d.P + c.d.Q) * c.d.E;
    if (t >= total) return;
    int i = (int)(t / c.d.E), e = (int)(t % c.d.E);
    bool a;
    R dp;
    V3<R> pt, n;
    slot_geometry(c, i, e, a, dp, pt, n);
    active[t] = a;
    depth[t] = dp;
    point[3 * t] = pt.x; point[3 * t + 1] = pt.y; point[3 * t + 2] = pt.z;
    normal[3 * t] = n.x; normal[3 * t + 1] = n.y; normal[3 * t + 2] = n.z;
}

// collide(): warp-aggregated compaction in (slot, env) order (physics.py:500-517).
constexpr int CT = 256;
template <class R> __global__ void collide_count_kernel(Ctx<R> c, int32_t *block_counts) {
    size_t t = (size_t)blockIdx.x * CT + threadIdx.x;
    size_t total = (size_t)(c.d.P + c.d.Q) * c.d.E;
    bool a = false;
    if (t < total) {
        R dp;
        V3<R> pt, n;
        slot_geometry(c, (int)(t / c.d.E), (int)(t % c.d.E), a, dp, pt, n);
    }
    unsigned m = __ballot_sync(0xffffffffu, a);
    __shared__ int wc[CT / 32];
    if ((threadIdx.x & 31) == 0) wc[threadIdx.x >> 5] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int k = 0; k < CT / 32; ++k) s += wc[k];
        block_counts[blockIdx.x] = s;
    }
}

// single-CTA exclusive scan of the per-CTA counts; total -> *total
__global__ void scan_kernel(int32_t *counts, int n, int32_t *total) {
    __shared__ int32_t carry;
    __shared__ int ws_[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int base = 0; base < n; base += blockDim.x) {
        int i = base + threadIdx.x;
        int v = i < n ? counts[i] : 0;
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) ws_[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int s = lane < (int)(blockDim.x >> 5) ? ws_[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            ws_[lane] = s;
        }
        __syncthreads();
        int excl = x - v + (wid ? ws_[wid - 1] : 0) + carry;
        if (i < n) counts[i] = excl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

template <class R>
__global__ void collide_write_kernel(Ctx<R> c, const int32_t *block_offsets, int32_t capacity, int32_t *body_a,
                                     int32_t *body_b, R *depth, R *point, R *normal) {
    size_t t = (size_t)blockIdx.x * CT + threadIdx.x;
    size_t total = (size_t)(c.d.P + c.d.Q) * c.d.E;
    bool a = false;
    R dp = R(0);
    V3<R> pt = zero3<R>(), n = zero3<R>();
    int i = 0, e = 0;
    if (t < total) {
        i = (int)(t / c.d.E);
        e = (int)(t % c.d.E);
        slot_geometry(c, i, e, a, dp, pt, n);
    }
    unsigned m = __ballot_sync(0xffffffffu, a);
    __shared__ int wc[CT / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) wc[wid] = __popc(m);
    __syncthreads();
    int woff = 0;
    for (int k = 0; k < wid; ++k) woff += wc[k];
    if (a) {
        int slot = block_offsets[blockIdx.x] + woff + __popc(m & ((1u << lane) - 1u));
        if (slot < capacity) {
            const Dims &d = c.d;
            if (i < d.P) {
                body_a[slot] = -1;
                body_b[slot] = e * d.B + c.L.plane_body[i];
            } else {
                body_a[slot] = e * d.B + c.L.pair_body[2 * (i - d.P)];
                body_b[slot] = e * d.B + c.L.pair_body[2 * (i - d.P) + 1];
            }
            depth[slot] = dp;
            point[3 * slot] = pt.x; point[3 * slot + 1] = pt.y; point[3 * slot + 2] = pt.z;
            normal[3 * slot] = n.x; normal[3 * slot + 1] = n.y; normal[3 * slot + 2] = n.z;
        }
    }
}

template <class R>
Ctx<R> make_ctx(const bsim_layout_t *L, const typename Abi<R>::Params *p, const typename Abi<R>::State *s) {
    Ctx<R> c;
    c.L = *L;
    if (p) c.p = *p; else std::memset(&c.p, 0, sizeof c.p);
    c.s = *s;
    c.d = make_dims(*L, sizeof(R) == 8);
    c.joints = reinterpret_cast<const typename Abi<R>::Joint *>(L->joints);
    return c;
}

bool bad_layout(const bsim_layout_t *L) {
    return !L || L->num_envs < 0 || L->bodies_per_env < 0 || L->actors_per_env < 1 ||
           L->actors_per_env > 32 || (L->joints_per_env && !L->joints);
}

// ------------------------------------------------------------ launchers
// Launch plan of step_kernel<R, T> for a layout and batch size E: the CTA's
// env count n <= NE fixes its shared memory (n workspace records + the joint
// table) and so the resident CTAs per SM; take the n needing the fewest waves
// of resident CTAs (largest n on ties), then spread the envs evenly over those
// waves (whole waves, no partial last one) -- `epc` envs per CTA.  Chunks of
// a pipelined step (bsim_env_step_host) use the plan of the scene's whole E,
// so n concurrent chunk grids fill the same waves.  Cached per (layout, E);
// host-side state, not thread-safe (one host thread drives a scene).
struct Plan {
    int epc;
    size_t smem;
    long capacity;   // resident envs of one wave (SMs x CTAs/SM x envs/CTA)
};
template <class R, class T, bool SCHED> int plan_launch(const Dims &d, int E, Plan *out) {
    constexpr int NE = Shape<R>::NE;
    struct Entry {
        int dev, pad, J, E;
        Plan p;
    };
    // keyed by device: the function attribute and the SM count are per device
    constexpr int MAX_DEV = 64;
    static Entry cache[16];
    static int n_cache = 0;
    static size_t configured[MAX_DEV] = {};
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= MAX_DEV) return set_err("plan_launch: device ordinal", cudaErrorInvalidDevice);
    for (int i = 0; i < n_cache && i < 16; ++i)
        if (cache[i].dev == dev && cache[i].pad == d.pad && cache[i].J == d.J && cache[i].E == E) {
            *out = cache[i].p;
            return BSIM_OK;
        }
    const size_t smax = step_smem_bytes<R>(d, NE);
    if (smax > 48 * 1024 && smax > configured[dev]) {
        cudaError_t e = cudaFuncSetAttribute(step_kernel<R, T, SCHED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smax);
        if (e != cudaSuccess) return set_err("cudaFuncSetAttribute(step_kernel)", e);
        configured[dev] = smax;
    }
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long En = E > 0 ? E : 1;
    long best_waves = -1, best_slots = 0;
    int best_n = 0;
    for (int n = NE; n >= 1; --n) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, step_kernel<R, T, SCHED>, Shape<R>::NTH,
                                                      step_smem_bytes<R>(d, n));
        if (per_sm < 1) continue;
        const long slots = (long)sms * per_sm, waves = (En + slots * n - 1) / (slots * n);
        if (best_waves < 0 || waves < best_waves) {
            best_waves = waves;
            best_slots = slots;
            best_n = n;
        }
    }
    if (!best_n) return set_err("step_kernel occupancy", cudaErrorInvalidConfiguration);
    int epc = best_n;
#ifndef BSIM_NO_BALANCE
    epc = (int)((En + best_waves * best_slots - 1) / (best_waves * best_slots));
    if (epc < 1) epc = 1;
    if (epc > best_n) epc = best_n;
#endif
    Plan p{epc, step_smem_bytes<R>(d, epc), best_slots * best_n};
    cache[n_cache % 16] = Entry{dev, d.pad, d.J, E, p};
    ++n_cache;
    *out = p;
    return BSIM_OK;
}

// the sweep a layout runs on topology T: the row schedule when it has one
// (and T is neither a star nor a register-sweep topology)
template <class T> constexpr bool sched_capable() { return !topo_register_sweep<T>() && !topo_star<T>(); }

template <class R, class T, bool SCHED>
int launch_step_tt(const Ctx<R> &c, int n_substeps, const bsim_actions_t &act, const bsim_task_t *task,
                   int e_begin, int e_count, cudaStream_t st) {
    Plan pl;
    if (int rc = plan_launch<R, T, SCHED>(c.d, c.d.E, &pl)) return rc;
    const int epc = pl.epc;
    const int grid = (e_count + epc - 1) / epc;
    bsim_task_t tk;
    if (task) tk = *task; else std::memset(&tk, 0, sizeof tk);
    if (task && (size_t)epc * task->obs_dim * sizeof(R) > step_ws_bytes<R>(c.d, epc)) {
        g_err = "bsim_env_step: observation rows do not fit the CTA workspace";
        return BSIM_E_TOO_LARGE;
    }
    step_kernel<R, T, SCHED><<<grid, Shape<R>::NTH, pl.smem, st>>>(c, n_substeps, act, epc, e_begin,
                                                                  e_begin + e_count, tk, task != nullptr);
    return check_launch("step_kernel");
}
template <class R, class T>
int launch_step_t(const Ctx<R> &c, size_t smem, int n_substeps, const bsim_actions_t &act, const bsim_task_t *task,
                  int e_begin, int e_count, cudaStream_t st) {
    (void)smem;
    if constexpr (sched_capable<T>())
        if (c.L.sched_stages > 0) return launch_step_tt<R, T, true>(c, n_substeps, act, task, e_begin, e_count, st);
    return launch_step_tt<R, T, false>(c, n_substeps, act, task, e_begin, e_count, st);
}
template <class R, class T> int plan_launch_for(const bsim_layout_t *l, const Dims &d, Plan *out) {
    if constexpr (sched_capable<T>())
        if (l->sched_stages > 0) return plan_launch<R, T, true>(d, d.E, out);
    return plan_launch<R, T, false>(d, d.E, out);
}

// the task-layer argument rules of bsim_task_step (bsim_tasks.cu)
bool task_ok(const bsim_layout_t *L, const bsim_task_t *t) { return task_args_ok(L, t); }

#ifndef BSIM_LARGE_TU
// The large-articulation variant (bsim_step_large.cu: this source with a
// 4-env x 32-thread CTA) is used when the default 16-env CTA's workspace
// leaves fewer than 2 CTAs per SM (e.g. the 22-body humanoid: 150 KB).
template <class R> bool use_large_variant(const Dims &d) {
    return step_ws_bytes<R>(d) > 113 * 1024;
}
int call_large(const bsim_layout_t *l, const bsim_params_t *p, const bsim_state_t *s, int32_t n,
               const bsim_actions_t *a, const bsim_task_t *t, int32_t eb, int32_t en, void *st) {
    return bsim_large_step_f32(l, p, s, n, a, t, eb, en, st);
}
int call_large(const bsim_layout_t *l, const bsim_params64_t *p, const bsim_state64_t *s, int32_t n,
               const bsim_actions_t *a, const bsim_task_t *t, int32_t eb, int32_t en, void *st) {
    return bsim_large_step_f64(l, p, s, n, a, t, eb, en, st);
}
#endif

template <class R>
int launch_step(const bsim_layout_t *layout, const typename Abi<R>::Params *params,
                const typename Abi<R>::State *state, int32_t n_substeps, const bsim_actions_t *actions,
                void *stream, const bsim_task_t *task = nullptr, int32_t env_begin = 0, int32_t env_count = -1) {
    if (bad_layout(layout) || !params || !state || n_substeps < 1) {
        g_err = "bsim_step: invalid arguments";
        return BSIM_E_INVALID;
    }
    if (env_count < 0) env_count = layout->num_envs - env_begin;
    if (env_begin < 0 || env_begin + env_count > layout->num_envs) {
        g_err = "bsim_step: env range out of bounds";
        return BSIM_E_INVALID;
    }
    if (task && !task_ok(layout, task)) {
        g_err = "bsim_env_step: invalid task";
        return BSIM_E_INVALID;
    }
    Ctx<R> c = make_ctx<R>(layout, params, state);
    if (c.d.E == 0 || env_count == 0) return BSIM_OK;
    size_t smem = step_smem_bytes<R>(c.d);
    bsim_actions_t act;
    if (actions) act = *actions; else std::memset(&act, 0, sizeof act);
    cudaStream_t st = (cudaStream_t)stream;
#ifdef BSIM_LARGE_TU
    if (smem > 227 * 1024) {
        g_err = "bsim_step: model too large for the step kernel's shared-memory workspace";
        return BSIM_E_TOO_LARGE;
    }
    switch (layout->topology_id) {
#define BSIM_LAUNCH_TOPO(ID, TYPE)                                      \
    case ID:                                                            \
        return launch_step_t<R, TYPE>(c, smem, n_substeps, act, task, env_begin, env_count, st);
        BSIM_TOPOLOGIES_LARGE(BSIM_LAUNCH_TOPO)
#undef BSIM_LAUNCH_TOPO
    default:
        return launch_step_t<R, TopoGeneric>(c, smem, n_substeps, act, task, env_begin, env_count, st);
    }
#else
    if (use_large_variant<R>(c.d)) {   // big articulations: 4 envs x 32 threads per CTA
        int rc = call_large(layout, params, state, n_substeps, actions, task, env_begin, env_count, stream);
        if (rc != BSIM_OK) g_err = bsim_large_last_error();
        return rc;
    }
    if (smem > 227 * 1024) {
        g_err = "bsim_step: model too large for the step kernel's shared-memory workspace";
        return BSIM_E_TOO_LARGE;
    }
    switch (layout->topology_id) {
#define BSIM_LAUNCH_TOPO(ID, TYPE)                                      \
    case ID:                                                            \
        return launch_step_t<R, TYPE>(c, smem, n_substeps, act, task, env_begin, env_count, st);
        BSIM_TOPOLOGIES(BSIM_LAUNCH_TOPO)
#undef BSIM_LAUNCH_TOPO
    default:
        return launch_step_t<R, TopoGeneric>(c, smem, n_substeps, act, task, env_begin, env_count, st);
    }
#endif
}

// dynamic shared memory above the default 48 KB needs the kernel's opt-in (once per size and device)
template <class K> int allow_smem(K *kernel, size_t bytes) {
    if (bytes <= 48 * 1024) return BSIM_OK;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    return e == cudaSuccess ? BSIM_OK : set_err("cudaFuncSetAttribute(aux kernel)", e);
}

template <class R>
int launch_fk(const bsim_layout_t *layout, const typename Abi<R>::State *state, const uint8_t *env_mask,
              uint32_t actor_mask, void *stream) {
    if (bad_layout(layout) || !state) return BSIM_E_INVALID;
    Ctx<R> c = make_ctx<R>(layout, nullptr, state);
    if (c.d.E == 0) return BSIM_OK;
    const size_t smem = FK_EPC * fk_stride<R>(c.d) * sizeof(R);
    if (int rc = allow_smem(fk_kernel<R>, smem)) return rc;
    fk_kernel<R><<<(c.d.E + FK_EPC - 1) / FK_EPC, FK_G * FK_EPC, smem, (cudaStream_t)stream>>>(c, env_mask, nullptr,
                                                                                             actor_mask);
    return check_launch("fk_kernel");
}

template <class R> int launch_refresh(const bsim_layout_t *layout, const typename Abi<R>::State *state, void *stream) {
    if (bad_layout(layout) || !state) return BSIM_E_INVALID;
    Ctx<R> c = make_ctx<R>(layout, nullptr, state);
    if (c.d.E == 0) return BSIM_OK;
    const size_t smem = REF_EPC * 13 * c.d.B * sizeof(R);
    if (int rc = allow_smem(refresh_kernel<R>, smem)) return rc;
    refresh_kernel<R><<<(c.d.E + REF_EPC - 1) / REF_EPC, REF_NTH, smem, (cudaStream_t)stream>>>(c);
    return check_launch("refresh_kernel");
}

template <class R>
int launch_set(bool root, const bsim_layout_t *layout, const typename Abi<R>::State *state, const R *values,
               const int64_t *idx, int32_t n, uint8_t *env_mask, uint32_t *amask, void *stream) {
    if (bad_layout(layout) || !state || !values || !idx || n < 0 || !env_mask || !amask) return BSIM_E_INVALID;
    Ctx<R> c = make_ctx<R>(layout, nullptr, state);
    if (n == 0 || c.d.E == 0) return BSIM_OK;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e1 = cudaMemsetAsync(env_mask, 0, (size_t)c.d.E, st);
    if (e1 != cudaSuccess) return set_err("memset env_mask", e1);
    cudaError_t e2 = cudaMemsetAsync(amask, 0, sizeof(uint32_t), st);
    if (e2 != cudaSuccess) return set_err("memset actor mask", e2);
    if (root)
        set_root_kernel<R><<<(n + 127) / 128, 128, 0, st>>>(c, values, idx, n, env_mask, amask);
    else
        set_dof_kernel<R><<<(n + 127) / 128, 128, 0, st>>>(c, values, idx, n, env_mask, amask);
    int r = check_launch(root ? "set_root_kernel" : "set_dof_kernel");
    if (r) return r;
    // FK over (touched envs) x (touched actors), then repack (buffers.py:151-152, 177-178)
    const size_t smem = FK_EPC * fk_stride<R>(c.d) * sizeof(R);
    if (int rc = allow_smem(fk_kernel<R>, smem)) return rc;
    fk_kernel<R><<<(c.d.E + FK_EPC - 1) / FK_EPC, FK_G * FK_EPC, smem, st>>>(c, env_mask, amask, 0u);
    return check_launch("fk_kernel");
}

template <class R>
int launch_contact_geometry(const bsim_layout_t *layout, const typename Abi<R>::Params *params,
                            const typename Abi<R>::State *state, uint8_t *active, R *depth, R *point, R *normal,
                            void *stream) {
    if (bad_layout(layout) || !params || !state) return BSIM_E_INVALID;
    Ctx<R> c = make_ctx<R>(layout, params, state);
    size_t total = (size_t)(c.d.P + c.d.Q) * c.d.E;
    if (!total) return BSIM_OK;
    contact_geometry_kernel<R><<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        c, active, depth, point, normal);
    return check_launch("contact_geometry_kernel");
}

template <class R>
int launch_collide(const bsim_layout_t *layout, const typename Abi<R>::Params *params,
                   const typename Abi<R>::State *state, int32_t capacity, int32_t *count, int32_t *body_a,
                   int32_t *body_b, R *depth, R *point, R *normal, int32_t *scratch, void *stream) {
    if (bad_layout(layout) || !params || !state || !count || !scratch) return BSIM_E_INVALID;
    Ctx<R> c = make_ctx<R>(layout, params, state);
    size_t total = (size_t)(c.d.P + c.d.Q) * c.d.E;
    cudaStream_t st = (cudaStream_t)stream;
    if (!total) {
        cudaError_t e = cudaMemsetAsync(count, 0, sizeof(int32_t), st);
        return e == cudaSuccess ? BSIM_OK : set_err("memset count", e);
    }
    int nb = (int)((total + CT - 1) / CT);
    collide_count_kernel<R><<<nb, CT, 0, st>>>(c, scratch);
    int r = check_launch("collide_count_kernel");
    if (r) return r;
    scan_kernel<<<1, 1024, 0, st>>>(scratch, nb, count);
    if ((r = check_launch("scan_kernel"))) return r;
    collide_write_kernel<R><<<nb, CT, 0, st>>>(c, scratch, capacity, body_a, body_b, depth, point, normal);
    return check_launch("collide_write_kernel");
}

// resident envs of one full wave of step_kernel CTAs for this layout (the
// chunk size of the pipelined host-buffer step)
template <class R> int envs_per_wave(const bsim_layout_t *l, int32_t *envs) {
    Dims d = make_dims(*l, sizeof(R) == 8);
    if (step_smem_bytes<R>(d, 1) > 227 * 1024) return BSIM_E_TOO_LARGE;
    Plan pl{0, 0, 0};
    int rc = BSIM_OK;
    switch (l->topology_id) {
#define BSIM_WAVE_TOPO(ID, TYPE) \
    case ID:                     \
        rc = plan_launch_for<R, TYPE>(l, d, &pl); break;
#ifdef BSIM_LARGE_TU
        BSIM_TOPOLOGIES_LARGE(BSIM_WAVE_TOPO)
#else
        BSIM_TOPOLOGIES(BSIM_WAVE_TOPO)
#endif
#undef BSIM_WAVE_TOPO
    default:
        rc = plan_launch_for<R, TopoGeneric>(l, d, &pl);
    }
    *envs = (int32_t)pl.capacity;
    return rc;
}

}  // namespace

#ifdef BSIM_LARGE_TU
extern "C" {
int bsim_large_step_f32(const bsim_layout_t *l, const bsim_params_t *p, const bsim_state_t *s, int32_t n,
                        const bsim_actions_t *a, const bsim_task_t *t, int32_t eb, int32_t en, void *st) {
    return launch_step<float>(l, p, s, n, a, st, t, eb, en);
}
int bsim_large_step_f64(const bsim_layout_t *l, const bsim_params64_t *p, const bsim_state64_t *s, int32_t n,
                        const bsim_actions_t *a, const bsim_task_t *t, int32_t eb, int32_t en, void *st) {
    return launch_step<double>(l, p, s, n, a, st, t, eb, en);
}
int bsim_large_envs_per_wave(const bsim_layout_t *l, int32_t fp64, int32_t *envs) {
    return fp64 ? envs_per_wave<double>(l, envs) : envs_per_wave<float>(l, envs);
}
const char *bsim_large_last_error(void) { return g_err.c_str(); }
}
#else
extern "C" {

int bsim_abi_version(void) { return BSIM_ABI_VERSION; }
const char *bsim_last_error(void) { return g_err.c_str(); }

int bsim_step_smem_per_env(const bsim_layout_t *layout, int32_t fp64, int32_t *bytes_per_env,
                           int32_t *envs_per_cta) {
    if (bad_layout(layout)) return BSIM_E_INVALID;
    Dims d = make_dims(*layout, fp64 != 0);
    const bool large = fp64 ? use_large_variant<double>(d) : use_large_variant<float>(d);
    // the large-articulation TU's CTA (bsim_step_large.cu): 8 envs (fp32) / 2 envs (fp64)
    const int ne = large ? (fp64 ? 2 : 8) : (fp64 ? Shape<double>::NE : Shape<float>::NE);
    // too large only when ONE env's workspace and the joint table exceed the
    // shared memory: the launch plan lowers the envs per CTA to what fits
    size_t one_env = (size_t)d.pad * (fp64 ? 8 : 4) + 16 +
                     (size_t)d.J * (fp64 ? sizeof(bsim_joint64_t) + 16 : sizeof(bsim_joint_t) + 16);
    if (bytes_per_env) *bytes_per_env = (int32_t)(d.pad * (fp64 ? 8 : 4));
    if (envs_per_cta) *envs_per_cta = ne;
    return one_env > 227 * 1024 ? BSIM_E_TOO_LARGE : BSIM_OK;
}

int bsim_step(const bsim_layout_t *l, const bsim_params_t *p, const bsim_state_t *s, int32_t n,
              const bsim_actions_t *a, void *st) {
    return launch_step<float>(l, p, s, n, a, st);
}
}  // extern "C"
// Domain randomisation at the auto-resets is deferred to one env-parallel
// launch right after the step (its mask: the step's done flags, which are
// exactly the reset envs; its step count: the one the reset would have used).
// Inside the fused tail it ran on one lane of the env's group and a late CTA
// with a randomised reset held the whole launch (Shadow Hand, 67 resets per
// step: 4652 -> ~3800 us).  Nothing the step returns depends on the
// randomised parameters (the post-reset observation reads state, not
// masses / gains / friction), and the next step sees them, so the results are
// the in-tail ones.  The CUDA-graph path (step count on the device) keeps the
// in-tail form.
template <class R, class P, class S, class F>
int env_step_dr_deferred(const bsim_layout_t *l, const P *p, const S *s, int32_t n, const bsim_actions_t *a,
                         const bsim_task_t *t, void *st, F randomize) {
    if (!t) return BSIM_E_INVALID;
    if (!t->dr.enabled || t->step_count_dev || !t->done) return launch_step<R>(l, p, s, n, a, st, t);
    bsim_task_t t2 = *t;
    t2.dr.enabled = 0;
    if (int rc = launch_step<R>(l, p, s, n, a, st, &t2)) return rc;
    return randomize(l, s, &t->dr, t->done, t->step_count, st);
}
extern "C" {
int bsim_env_step(const bsim_layout_t *l, const bsim_params_t *p, const bsim_state_t *s, int32_t n,
                  const bsim_actions_t *a, const bsim_task_t *t, void *st) {
    return env_step_dr_deferred<float>(l, p, s, n, a, t, st, bsim_randomize);
}
int bsim_env_step_f64(const bsim_layout_t *l, const bsim_params64_t *p, const bsim_state64_t *s, int32_t n,
                      const bsim_actions_t *a, const bsim_task_t *t, void *st) {
    return env_step_dr_deferred<double>(l, p, s, n, a, t, st, bsim_randomize_f64);
}
int bsim_step_f64(const bsim_layout_t *l, const bsim_params64_t *p, const bsim_state64_t *s, int32_t n,
                  const bsim_actions_t *a, void *st) {
    return launch_step<double>(l, p, s, n, a, st);
}
int bsim_step_range(const bsim_layout_t *l, const bsim_params_t *p, const bsim_state_t *s, int32_t n,
                    const bsim_actions_t *a, int32_t env_begin, int32_t env_count, void *st) {
    if (env_count < 0) return BSIM_E_INVALID;
    return launch_step<float>(l, p, s, n, a, st, nullptr, env_begin, env_count);
}
int bsim_step_range_f64(const bsim_layout_t *l, const bsim_params64_t *p, const bsim_state64_t *s, int32_t n,
                        const bsim_actions_t *a, int32_t env_begin, int32_t env_count, void *st) {
    if (env_count < 0) return BSIM_E_INVALID;
    return launch_step<double>(l, p, s, n, a, st, nullptr, env_begin, env_count);
}
int bsim_env_step_range(const bsim_layout_t *l, const bsim_params_t *p, const bsim_state_t *s, int32_t n,
                        const bsim_actions_t *a, const bsim_task_t *t, int32_t env_begin, int32_t env_count,
                        void *st) {
    if (!t || env_count < 0) return BSIM_E_INVALID;
    return launch_step<float>(l, p, s, n, a, st, t, env_begin, env_count);
}
int bsim_env_step_range_f64(const bsim_layout_t *l, const bsim_params64_t *p, const bsim_state64_t *s, int32_t n,
                            const bsim_actions_t *a, const bsim_task_t *t, int32_t env_begin, int32_t env_count,
                            void *st) {
    if (!t || env_count < 0) return BSIM_E_INVALID;
    return launch_step<double>(l, p, s, n, a, st, t, env_begin, env_count);
}
int bsim_step_envs_per_wave(const bsim_layout_t *l, int32_t fp64, int32_t *envs) {
    if (bad_layout(l) || !envs) return BSIM_E_INVALID;
    Dims d = make_dims(*l, fp64 != 0);
    const bool large = fp64 ? use_large_variant<double>(d) : use_large_variant<float>(d);
    if (large) return bsim_large_envs_per_wave(l, fp64, envs);
    return fp64 ? envs_per_wave<double>(l, envs) : envs_per_wave<float>(l, envs);
}
int bsim_forward_kinematics(const bsim_layout_t *l, const bsim_state_t *s, const uint8_t *m, uint32_t am,
                            void *st) {
    return launch_fk<float>(l, s, m, am, st);
}
int bsim_forward_kinematics_f64(const bsim_layout_t *l, const bsim_state64_t *s, const uint8_t *m, uint32_t am,
                                void *st) {
    return launch_fk<double>(l, s, m, am, st);
}
int bsim_refresh_buffers(const bsim_layout_t *l, const bsim_state_t *s, void *st) {
    return launch_refresh<float>(l, s, st);
}
int bsim_refresh_buffers_f64(const bsim_layout_t *l, const bsim_state64_t *s, void *st) {
    return launch_refresh<double>(l, s, st);
}
int bsim_set_root_state_indexed(const bsim_layout_t *l, const bsim_state_t *s, const float *v, const int64_t *i,
                                int32_t n, uint8_t *em, uint32_t *am, void *st) {
    return launch_set<float>(true, l, s, v, i, n, em, am, st);
}
int bsim_set_root_state_indexed_f64(const bsim_layout_t *l, const bsim_state64_t *s, const double *v,
                                    const int64_t *i, int32_t n, uint8_t *em, uint32_t *am, void *st) {
    return launch_set<double>(true, l, s, v, i, n, em, am, st);
}
int bsim_set_dof_state_indexed(const bsim_layout_t *l, const bsim_state_t *s, const float *v, const int64_t *i,
                               int32_t n, uint8_t *em, uint32_t *am, void *st) {
    return launch_set<float>(false, l, s, v, i, n, em, am, st);
}
int bsim_set_dof_state_indexed_f64(const bsim_layout_t *l, const bsim_state64_t *s, const double *v,
                                   const int64_t *i, int32_t n, uint8_t *em, uint32_t *am, void *st) {
    return launch_set<double>(false, l, s, v, i, n, em, am, st);
}
int bsim_contact_geometry(const bsim_layout_t *l, const bsim_params_t *p, const bsim_state_t *s, uint8_t *a,
                          float *d, float *pt, float *n, void *st) {
    return launch_contact_geometry<float>(l, p, s, a, d, pt, n, st);
}
int bsim_contact_geometry_f64(const bsim_layout_t *l, const bsim_params64_t *p, const bsim_state64_t *s,
                              uint8_t *a, double *d, double *pt, double *n, void *st) {
    return launch_contact_geometry<double>(l, p, s, a, d, pt, n, st);
}
int bsim_collide(const bsim_layout_t *l, const bsim_params_t *p, const bsim_state_t *s, int32_t cap, int32_t *cnt,
                 int32_t *ba, int32_t *bb, float *d, float *pt, float *n, int32_t *scr, void *st) {
    return launch_collide<float>(l, p, s, cap, cnt, ba, bb, d, pt, n, scr, st);
}
int bsim_collide_f64(const bsim_layout_t *l, const bsim_params64_t *p, const bsim_state64_t *s, int32_t cap,
                     int32_t *cnt, int32_t *ba, int32_t *bb, double *d, double *pt, double *n, int32_t *scr,
                     void *st) {
    return launch_collide<double>(l, p, s, cap, cnt, ba, bb, d, pt, n, scr, st);
}

}  // extern "C"
#endif  // BSIM_LARGE_TU

#if defined(BSIM_EXP_RESET_CLOCKS) && !defined(BSIM_LARGE_TU)
// timing experiment only (tools/reset_clocks.py): read and clear the reset phase counters
extern "C" int bsim_exp_reset_clocks(unsigned long long *out8) {
    if (cudaMemcpyFromSymbol(out8, bsim::bsim_reset_clk, sizeof(unsigned long long) * 8) != cudaSuccess) return -1;
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    return cudaMemcpyToSymbol(bsim::bsim_reset_clk, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
#endif

#if defined(BSIM_EXP_PHASE_CLOCKS) && !defined(BSIM_LARGE_TU)
// timing experiment only (tools/phase_clocks.py): read and clear the step_kernel phase counters
extern "C" int bsim_exp_phase_clocks(unsigned long long *out8) {
    if (cudaMemcpyFromSymbol(out8, g_phase_clk, sizeof(unsigned long long) * 8) != cudaSuccess) return -1;
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    return cudaMemcpyToSymbol(g_phase_clk, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
extern "C" int bsim_exp_cta_times(unsigned long long *out) {   // [4096][4]
    return cudaMemcpyFromSymbol(out, g_cta_times, sizeof(unsigned long long) * 4096 * 4) == cudaSuccess ? 0 : -1;
}
extern "C" int bsim_exp_launch_gap(unsigned long long *out2) {   // (sum ns, count); read and clear
    if (cudaMemcpyFromSymbol(out2, g_gap_sum, 8) != cudaSuccess) return -1;
    if (cudaMemcpyFromSymbol(out2 + 1, g_gap_n, 8) != cudaSuccess) return -1;
    unsigned long long z = 0;
    cudaMemcpyToSymbol(g_gap_sum, &z, 8);
    cudaMemcpyToSymbol(g_gap_n, &z, 8);
    return cudaMemcpyToSymbol(g_last_end, &z, 8) == cudaSuccess ? 0 : -1;
}
#endif

#if defined(BSIM_EXP_PASS_CLOCKS) && !defined(BSIM_LARGE_TU)
// timing experiment only (tools/pass_clocks.py): read and clear the solver-pass phase counters
extern "C" int bsim_exp_pass_clocks(unsigned long long *out8) {
    if (cudaMemcpyFromSymbol(out8, bsim::bsim_pass_clk, sizeof(unsigned long long) * 8) != cudaSuccess) return -1;
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    return cudaMemcpyToSymbol(bsim::bsim_pass_clk, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
#endif

#if defined(BSIM_EXP_PASS_CLOCKS) && defined(BSIM_LARGE_TU)
// the large-articulation TU's own counters (timing experiment only)
extern "C" int bsim_exp_pass_clocks_large(unsigned long long *out8) {
    if (cudaMemcpyFromSymbol(out8, bsim::bsim_pass_clk, sizeof(unsigned long long) * 8) != cudaSuccess) return -1;
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    return cudaMemcpyToSymbol(bsim::bsim_pass_clk, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
#endif
