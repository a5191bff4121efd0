// bsim_dr.cuh -- domain randomisation and observation noise on the device
// (reference randomize.py:86-237), bit-compatible with numpy's draws.
#pragma once

#include "bsim_rng.cuh"
#include "bsim_step.cuh"
#include "bsim_ziggurat.cuh"

namespace bsim {

// Generator.standard_normal: numpy's 256-level ziggurat
// (random_standard_normal, numpy/random/src/distributions/distributions.c)
__device__ inline double np_std_normal(NpRng &r) {
    for (;;) {
        uint64_t u = np_next64(r);
        int idx = (int)(u & 0xff);
        u >>= 8;
        int sign = (int)(u & 1);
        uint64_t rabs = (u >> 1) & 0x000fffffffffffffull;
        double x = (double)rabs * ZIG_WI[idx];
        if (sign) x = -x;
        if (rabs < ZIG_KI[idx]) return x;
        if (idx == 0) {
            for (;;) {
                double xx = -ZIG_NOR_INV_R * log1p(-np_uniform(r, 0.0, 1.0));
                double yy = -log1p(-np_uniform(r, 0.0, 1.0));
                if (yy + yy > xx * xx) return ((rabs >> 8) & 1) ? -(ZIG_NOR_R + xx) : ZIG_NOR_R + xx;
            }
        } else if ((ZIG_FI[idx - 1] - ZIG_FI[idx]) * np_uniform(r, 0.0, 1.0) + ZIG_FI[idx] < exp(-0.5 * x * x)) {
            return x;
        }
    }
}

// RandomizationEntry.sample (randomize.py:38-46), one draw
__device__ inline double dr_sample(NpRng &r, int dist, double a, double b) {
    if (dist == 0) return np_uniform(r, a, b);
    if (dist == 1) return exp(np_uniform(r, log(a), log(b)));
    return a + b * np_std_normal(r);
}

// DomainRandomizer._restore_env + randomize for one env (randomize.py:116-189)
template <class R>
__device__ void dr_randomize_env(const Ctx<R> &c, const bsim_dr_t &dr, int e, int64_t step) {
    if (!dr.enabled) return;
    if (step - (int64_t)dr.last_step[e] < (int64_t)dr.min_interval) return;
    const Dims &d = c.d;
    const size_t E = (size_t)d.E;
    const auto &s = c.s;
    auto base = [](const void *p) { return reinterpret_cast<const R *>(p); };
    // restore the base values of every watched array row of env e
    for (int b = 0; b < d.B; ++b) {
        size_t g = (size_t)e * d.B + b;
        s.inv_mass[g] = base(dr.inv_mass)[g];
        for (int k = 0; k < 3; ++k) {
            s.inertia_local[3 * g + k] = base(dr.inertia_local)[3 * g + k];
            s.inv_inertia_local[3 * g + k] = base(dr.inv_inertia_local)[3 * g + k];
        }
    }
    for (int k = 0; k < 3; ++k) s.gravity[3 * e + k] = base(dr.gravity)[3 * e + k];
    s.mu_static[e] = base(dr.mu_static)[e];
    s.mu_dynamic[e] = base(dr.mu_dynamic)[e];
    for (int j = 0; j < d.J; ++j) {
        size_t o = (size_t)j * E + e;
        s.joint_stiffness[o] = base(dr.joint_stiffness)[o];
        s.joint_damping[o] = base(dr.joint_damping)[o];
        s.joint_limit_lo[o] = base(dr.joint_limit_lo)[o];
        s.joint_limit_hi[o] = base(dr.joint_limit_hi)[o];
    }
    for (int i = 0; i < d.P; ++i) {
        size_t o = (size_t)i * E + e;
        s.plane_rad[o] = base(dr.plane_rad)[o];
        for (int k = 0; k < 3; ++k) s.plane_off[3 * o + k] = base(dr.plane_off)[3 * o + k];
    }
    for (int i = 0; i < d.Q; ++i) {
        size_t o = (size_t)i * E + e;
        for (int k = 0; k < 2; ++k) s.pair_rad[2 * o + k] = base(dr.pair_rad)[2 * o + k];
        for (int k = 0; k < 6; ++k) s.pair_off[6 * o + k] = base(dr.pair_off)[6 * o + k];
    }
    uint32_t key[3] = {dr.seed, (uint32_t)(c.L.env_offset + e), (uint32_t)dr.epoch[e]};
    NpRng r = np_rng(key, 3);
    for (int t = 0; t < 7; ++t) {
        if (!dr.use[t]) continue;
        const int dist = dr.dist[t];
        const double a = dr.a[t], b = dr.b[t];
        if (t == 0) {           // dims: scale every contact radius / offset of the env
            R sc = R(dr_sample(r, dist, a, b));
            for (int i = 0; i < d.P; ++i) {
                size_t o = (size_t)i * E + e;
                s.plane_rad[o] *= sc;
                for (int k = 0; k < 3; ++k) s.plane_off[3 * o + k] *= sc;
            }
            for (int i = 0; i < d.Q; ++i) {
                size_t o = (size_t)i * E + e;
                for (int k = 0; k < 2; ++k) s.pair_rad[2 * o + k] *= sc;
                for (int k = 0; k < 6; ++k) s.pair_off[6 * o + k] *= sc;
            }
        } else if (t == 1) {    // masses
            for (int bb = 0; bb < d.B; ++bb) {
                R m = R(dr_sample(r, dist, a, b));
                size_t g = (size_t)e * d.B + bb;
                s.inv_mass[g] /= m;
                for (int k = 0; k < 3; ++k) {
                    s.inertia_local[3 * g + k] *= m;
                    s.inv_inertia_local[3 * g + k] /= m;
                }
            }
        } else if (t == 2) {    // friction
            R f = R(dr_sample(r, dist, a, b));
            s.mu_static[e] *= f;
            s.mu_dynamic[e] *= f;
        } else if (t == 3 || t == 4) {   // damping / gains
            R *arr = t == 3 ? s.joint_damping : s.joint_stiffness;
            for (int j = 0; j < d.J; ++j) arr[(size_t)j * E + e] *= R(dr_sample(r, dist, a, b));
        } else if (t == 5) {    // joint limits: n draws for lo then n for hi
            for (int j = 0; j < d.J; ++j) s.joint_limit_lo[(size_t)j * E + e] += R(dr_sample(r, dist, a, b));
            for (int j = 0; j < d.J; ++j) s.joint_limit_hi[(size_t)j * E + e] += R(dr_sample(r, dist, a, b));
        } else {                // gravity
            for (int k = 0; k < 3; ++k) {
                R gk = R(dr_sample(r, dist, a, b));
                if (dr.mode[t] == 0) s.gravity[3 * e + k] *= gk;
                else s.gravity[3 * e + k] += gk;
            }
        }
    }
    dr.epoch[e] += 1;
    dr.last_step[e] = (int32_t)step;
}

}  // namespace bsim
