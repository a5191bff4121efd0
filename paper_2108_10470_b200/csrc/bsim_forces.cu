// bsim_forces.cu -- random object disturbance forces on the device
// (reference randomize.py:192-221, RandomForceState / random_object_force).
// One thread per env; draws come from per-env numpy-PCG64 streams keyed
// (seed, tag, global env id, counter) so results do not depend on how the
// env batch is partitioned over GPUs.
#include <cuda_runtime.h>

#include <cmath>

#include "bsim_dr.cuh"

using namespace bsim;

namespace {

constexpr uint32_t TAG_PROB = 0xF0u, TAG_FORCE = 0xF1u;

// RandomForceState.__init__ / resample_probability (randomize.py:204-212)
template <class R> __global__ void force_resample_kernel(bsim_force_t f, const uint8_t *mask) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= f.num_envs || (mask && !mask[e])) return;
    uint32_t key[4] = {f.seed, TAG_PROB, (uint32_t)(f.env_offset + e), (uint32_t)f.epoch[e]};
    NpRng r = np_rng(key, 4);
    reinterpret_cast<R *>(f.probability)[e] = R(exp(np_uniform(r, log(f.p_lo), log(f.p_hi))));
    R *F = reinterpret_cast<R *>(f.force) + 3 * (size_t)e;
    F[0] = F[1] = F[2] = R(0);
    f.epoch[e] += 1;
}

// random_object_force (randomize.py:215-221)
template <class R>
__global__ void random_force_kernel(bsim_force_t f, const R *mass, double decay, R *body_force, int B, int body) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= f.num_envs) return;
    uint32_t key[4] = {f.seed, TAG_FORCE, (uint32_t)(f.env_offset + e), (uint32_t)f.count[e]};
    NpRng r = np_rng(key, 4);
    R *F = reinterpret_cast<R *>(f.force) + 3 * (size_t)e;
    const double u = np_uniform(r, 0.0, 1.0);   // Generator.random
    if (u < (double)reinterpret_cast<const R *>(f.probability)[e]) {
        const double m = (double)mass[e];
        for (int k = 0; k < 3; ++k) F[k] = R(np_std_normal(r) * m);
    } else {
        for (int k = 0; k < 3; ++k) F[k] = R(F[k] * R(decay));
    }
    f.count[e] += 1;
    if (body_force) {
        R *o = body_force + 3 * ((size_t)e * B + body);
        o[0] = F[0]; o[1] = F[1]; o[2] = F[2];
    }
}

bool bad(const bsim_force_t *f) {
    return !f || f->num_envs < 0 || (f->num_envs > 0 && (!f->probability || !f->force || !f->epoch || !f->count));
}

int launched() { return cudaGetLastError() == cudaSuccess ? BSIM_OK : BSIM_E_CUDA; }

}  // namespace

extern "C" {

int bsim_force_resample(const bsim_force_t *f, const uint8_t *mask, void *st) {
    if (bad(f) || !(f->p_lo > 0.0) || !(f->p_hi >= f->p_lo)) return BSIM_E_INVALID;
    if (f->num_envs == 0) return BSIM_OK;
    const int grid = (f->num_envs + 127) / 128;
    if (f->fp64)
        force_resample_kernel<double><<<grid, 128, 0, (cudaStream_t)st>>>(*f, mask);
    else
        force_resample_kernel<float><<<grid, 128, 0, (cudaStream_t)st>>>(*f, mask);
    return launched();
}

int bsim_random_object_force(const bsim_force_t *f, const void *mass, double dt, void *body_force, int32_t B,
                             int32_t body, void *st) {
    if (bad(f) || !mass || (body_force && (B < 1 || body < 0 || body >= B))) return BSIM_E_INVALID;
    if (f->num_envs == 0) return BSIM_OK;
    const double decay = std::pow(0.99, dt / 0.05);
    const int grid = (f->num_envs + 127) / 128;
    if (f->fp64)
        random_force_kernel<double><<<grid, 128, 0, (cudaStream_t)st>>>(
            *f, (const double *)mass, decay, (double *)body_force, B, body);
    else
        random_force_kernel<float><<<grid, 128, 0, (cudaStream_t)st>>>(
            *f, (const float *)mass, decay, (float *)body_force, B, body);
    return launched();
}

}  // extern "C"
