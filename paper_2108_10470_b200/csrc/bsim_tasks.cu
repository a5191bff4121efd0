// bsim_tasks.cu -- the fused task-layer kernels (one thread per env) and their
// C-ABI entry points: EnvBatch.step's reward / done / obs / auto-reset tail
// and EnvBatch.reset (reference envs.py:145-200, 359-565).
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "bsim_tasks.cuh"

using namespace bsim;

namespace {

std::string t_err;

int t_set_err(const char *what, cudaError_t e) {
    t_err = std::string(what) + ": " + cudaGetErrorString(e);
    return BSIM_E_CUDA;
}

// One thread per env over envs [e_begin, e_end).  The CTA's observation rows
// are built in shared memory and leave with one coalesced copy (a thread-per-
// env row store is a 240-348 B stride across the warp).
template <class R> __device__ void obs_copy_out(const bsim_task_t &t, const R *stage, int cta_e0, int e_end) {
    __syncthreads();
    const int n = max(0, e_end - cta_e0) * t.obs_dim;
    R *dst = reinterpret_cast<R *>(t.obs) + (size_t)cta_e0 * t.obs_dim;
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = stage[i];
}

// TASK_G lanes per env (bsim_tasks.cuh group form; the fused tail of
// bsim_env_step uses the same G, so both paths agree bitwise)
constexpr int TASK_G = BSIM_TASK_G;

template <class R>
__global__ void task_step_kernel(const __grid_constant__ Ctx<R> c, const __grid_constant__ bsim_task_t t, int e_begin,
                                 int e_end) {
    extern __shared__ __align__(16) unsigned char task_smem[];
    R *stage = reinterpret_cast<R *>(task_smem);
    const int epc = blockDim.x / TASK_G;
    const int cta_e0 = e_begin + blockIdx.x * epc, e = cta_e0 + threadIdx.x / TASK_G;
    if (e < e_end) task_step_env_g<R, TASK_G>(c, TaskView<R>{t, stage, cta_e0}, e, threadIdx.x % TASK_G);
    obs_copy_out(t, stage, cta_e0, min(e_end, cta_e0 + epc));
}

// EnvBatch.reset(env_indices) (envs.py:141-166) + the post-reset observation:
// TASK_G lanes per env, 128 / TASK_G envs per CTA.  Locomotion / ANYmal envs
// reset on the whole group (task_reset_env_g: parallel draws by PCG64
// jump-ahead, level-parallel FK on the env's shared-memory scratch after the
// CTA's obs rows); the other tasks, or models over 64 bodies, on lane 0.
template <class R>
__global__ void task_reset_kernel(const __grid_constant__ Ctx<R> c, const __grid_constant__ bsim_task_t t,
                                  const uint8_t *mask) {
    extern __shared__ __align__(16) unsigned char task_smem[];
    constexpr int G = TASK_G, EPC = 128 / TASK_G;
    R *stage = reinterpret_cast<R *>(task_smem);
    const int cta_e0 = blockIdx.x * EPC, e = cta_e0 + threadIdx.x / G, sl = threadIdx.x % G;
    if (e < c.d.E) {
        TaskView<R> tv{t, stage, cta_e0};
        tv.scratch = stage + (((size_t)EPC * t.obs_dim + 3) & ~(size_t)3);
        tv.scratch_stride = (13 * c.d.B + 2 * c.d.D + 3) & ~3;
        const bool group = c.d.B <= 64 && (t.kind == BSIM_TASK_QUADRUPED || t.kind == BSIM_TASK_ANYMAL ||
                                          t.kind == BSIM_TASK_HUMANOID);
        if (!mask || mask[e]) {
            if (group)
                task_reset_env_g<R, G>(c, tv, e, sl);
            else if (sl == 0)
                task_reset_env(c, tv, e);
        }
        __syncwarp(group_mask<G>());
        task_obs_g<R, G>(c, tv, e, sl);
    }
    obs_copy_out(t, stage, cta_e0, min(c.d.E, cta_e0 + EPC));
}

template <class R>
__global__ void randomize_kernel(const Ctx<R> c, const bsim_dr_t dr, const uint8_t *mask, int64_t step) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= c.d.E || (mask && !mask[e])) return;
    dr_randomize_env(c, dr, e, step);
}

template <class R>
Ctx<R> task_ctx(const bsim_layout_t *L, const typename Abi<R>::State *s) {
    Ctx<R> c;
    c.L = *L;
    std::memset(&c.p, 0, sizeof c.p);
    c.s = *s;
    c.d = make_dims(*L);
    c.joints = reinterpret_cast<const typename Abi<R>::Joint *>(L->joints);
    return c;
}

bool bad(const bsim_layout_t *L, const void *s, const bsim_task_t *t) {
    return !L || !s || !t || !task_args_ok(L, t);
}

template <class R>
int launch_task(const bsim_layout_t *L, const typename Abi<R>::State *s, const bsim_task_t *t, bool reset,
                const uint8_t *mask, int env_begin, int env_count, void *stream) {
    if (bad(L, s, t)) {
        t_err = "bsim_task: invalid arguments";
        return BSIM_E_INVALID;
    }
    if (env_count < 0) env_count = L->num_envs - env_begin;
    if (env_begin < 0 || env_begin + env_count > L->num_envs) {
        t_err = "bsim_task: env range out of bounds";
        return BSIM_E_INVALID;
    }
    Ctx<R> c = task_ctx<R>(L, s);
    if (env_count == 0) return BSIM_OK;
    // obs staging rows: up to 128 envs per CTA within the default 48 KB
    const size_t row = (size_t)t->obs_dim * sizeof(R);
    int tpb = 128;
    while (tpb > 32 && tpb * row > 48 * 1024) tpb -= 32;
    if (tpb * row > 48 * 1024) {
        t_err = "bsim_task: observation too wide";
        return BSIM_E_TOO_LARGE;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (reset) {   // TASK_G lanes per env; the obs rows, then each env's reset scratch
        const int epc = 128 / TASK_G;
        const size_t smem = ((((size_t)epc * t->obs_dim + 3) & ~(size_t)3) +
                             (size_t)epc * ((13 * c.d.B + 2 * c.d.D + 3) & ~3)) * sizeof(R);
        if (smem > 48 * 1024) {
            cudaError_t ea = cudaFuncSetAttribute(task_reset_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)smem);
            if (ea != cudaSuccess) return t_set_err("cudaFuncSetAttribute(task_reset_kernel)", ea);
        }
        bsim_task_t tr = *t;
        if (tr.dr.enabled && !tr.step_count_dev) {
            // domain randomisation of the reset envs first, one thread per env (full warps; inside the
            // group reset it would run on one lane of eight), then the resets without it -- the DR
            // draws are keyed apart from the reset draws, so the order does not change a value
            randomize_kernel<R><<<(c.d.E + 127) / 128, 128, 0, st>>>(c, tr.dr, mask, tr.step_count);
            cudaError_t ed = cudaGetLastError();
            if (ed != cudaSuccess) return t_set_err("randomize_kernel", ed);
            tr.dr.enabled = 0;
        }
        task_reset_kernel<R><<<(c.d.E + epc - 1) / epc, 128, smem, st>>>(c, tr, mask);
    } else {   // TASK_G lanes per env: 128 / TASK_G envs per CTA
        const int epc = 128 / TASK_G;
        task_step_kernel<R><<<(env_count + epc - 1) / epc, 128, epc * row, st>>>(c, *t, env_begin,
                                                                               env_begin + env_count);
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BSIM_OK : t_set_err(reset ? "task_reset_kernel" : "task_step_kernel", e);
}

template <class R>
int launch_randomize(const bsim_layout_t *L, const typename Abi<R>::State *s, const bsim_dr_t *dr,
                     const uint8_t *mask, int64_t step, void *stream) {
    if (!L || !s || !dr) {
        t_err = "bsim_randomize: invalid arguments";
        return BSIM_E_INVALID;
    }
    Ctx<R> c = task_ctx<R>(L, s);
    if (c.d.E == 0) return BSIM_OK;
    randomize_kernel<R><<<(c.d.E + 127) / 128, 128, 0, (cudaStream_t)stream>>>(c, *dr, mask, step);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BSIM_OK : t_set_err("randomize_kernel", e);
}

}  // namespace

extern "C" {

int bsim_randomize(const bsim_layout_t *l, const bsim_state_t *s, const bsim_dr_t *dr, const uint8_t *m,
                   int64_t step, void *st) {
    return launch_randomize<float>(l, s, dr, m, step, st);
}
int bsim_randomize_f64(const bsim_layout_t *l, const bsim_state64_t *s, const bsim_dr_t *dr, const uint8_t *m,
                       int64_t step, void *st) {
    return launch_randomize<double>(l, s, dr, m, step, st);
}

int bsim_task_step(const bsim_layout_t *l, const bsim_state_t *s, const bsim_task_t *t, void *st) {
    return launch_task<float>(l, s, t, false, nullptr, 0, -1, st);
}
int bsim_task_step_f64(const bsim_layout_t *l, const bsim_state64_t *s, const bsim_task_t *t, void *st) {
    return launch_task<double>(l, s, t, false, nullptr, 0, -1, st);
}
int bsim_task_reset(const bsim_layout_t *l, const bsim_state_t *s, const bsim_task_t *t, const uint8_t *m,
                    void *st) {
    return launch_task<float>(l, s, t, true, m, 0, -1, st);
}
int bsim_task_reset_f64(const bsim_layout_t *l, const bsim_state64_t *s, const bsim_task_t *t, const uint8_t *m,
                        void *st) {
    return launch_task<double>(l, s, t, true, m, 0, -1, st);
}
int bsim_task_step_range(const bsim_layout_t *l, const bsim_state_t *s, const bsim_task_t *t, int32_t env_begin,
                         int32_t env_count, void *st) {
    if (env_count < 0) return BSIM_E_INVALID;
    return launch_task<float>(l, s, t, false, nullptr, env_begin, env_count, st);
}
int bsim_task_step_range_f64(const bsim_layout_t *l, const bsim_state64_t *s, const bsim_task_t *t,
                             int32_t env_begin, int32_t env_count, void *st) {
    if (env_count < 0) return BSIM_E_INVALID;
    return launch_task<double>(l, s, t, false, nullptr, env_begin, env_count, st);
}
const char *bsim_task_last_error(void) { return t_err.c_str(); }

}  // extern "C"
