// bsim_rewards.cu -- batched reward kernels (reference rewards.py:78-219),
// one thread per env, float and double.  Used directly by the task layer's
// callers for tasks whose env is assembled in Python (Humanoid-style
// locomotion, Shadow-Hand cube reorientation, Franka cube stacking).
#include <cuda_runtime.h>

#include <cstdint>

#include "bsim_math.cuh"
#include "../../include/batchsim_b200.h"

using namespace bsim;

namespace {

template <class R> __device__ R sq(R x) { return x * x; }
template <class R> __device__ R norm3(const R *a, const R *b) {
    return r_sqrt(sq(a[0] - b[0]) + sq(a[1] - b[1]) + sq(a[2] - b[2]));
}
template <class R> __device__ bool fin(R x) { return x - x == R(0); }

// locomotion_reward (rewards.py:78-112)
template <class R>
__global__ void loco_kernel(int n, int D, const R *torso, const R *target, const R *up, const R *heading,
                            const R *act, const R *qpos, const R *qvel, const R *lo, const R *hi, const R *strength,
                            const R *prev, bsim_loco_params_t p, R *out, R *pot) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    R potential = -norm3(target + 3 * i, torso + 3 * i) / R(p.dt);
    R r = potential - prev[i];
    R hgt = torso[3 * i + 2];
    r = r + (hgt >= R(p.termination_height) ? R(p.alive_bonus) : R(0));
    r = r + (hgt <= R(p.termination_height) ? R(p.death_penalty) : R(0));
    r = r + (up[i] > R(p.upright_threshold) ? R(p.upright_weight) : R(0));
    R hp = heading[i];
    r = r + R(p.heading_weight) * (hp >= R(0.8) ? R(1) : hp / R(0.8));
    R sa = 0, se = 0, near_ = 0;
    for (int k = 0; k < D; ++k) {
        R a = act[(size_t)i * D + k];
        sa = sa + a * a;
        se = se + a * strength[k] * qvel[(size_t)i * D + k];
        if (fin(lo[k]) && fin(hi[k])) {
            R frac = (qpos[(size_t)i * D + k] - lo[k]) / (hi[k] - lo[k]);
            if (frac < R(0.01) || frac > R(0.99)) near_ = near_ + R(1);
        }
    }
    r = r - R(p.action_cost_weight) * sa + R(p.effort_weight) * se - R(p.dof_limit_weight) * near_;
    out[i] = r;
    pot[i] = potential;
}

// anymal_reward (rewards.py:129-158); rough adds the nine-term sum
template <class R>
__global__ void anymal_kernel(int n, int D, int A, int F, const R *lin, const R *ang, const R *cmd, const R *qvel,
                              const R *qacc, const R *torques, const R *arate, const R *coll, const R *air,
                              bsim_anymal_params_t p, int rough, R *out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const R dt = R(p.dt);
    const R *l = lin + 3 * i, *w = ang + 3 * i, *c = cmd + 3 * i;
    R exy = sq(c[0] - l[0]) + sq(c[1] - l[1]);
    R eyaw = sq(c[2] - w[2]);
    R tq = 0;
    for (int k = 0; k < D; ++k) tq = tq + sq(torques[(size_t)i * D + k]);
    R r = R(p.w_vel_xy) * dt * exp_r(-exy / R(0.25)) + R(p.w_vel_yaw) * dt * exp_r(-eyaw / R(0.25)) -
          R(p.w_torque) * dt * tq;
    if (rough) {
        r = r - R(p.w_vel_z) * dt * sq(l[2]);
        r = r - R(p.w_pitch_roll) * dt * (sq(w[0]) + sq(w[1]));
        R jm = 0, jv = 0, ar = 0, at = 0;
        for (int k = 0; k < D; ++k) {
            jm = jm + sq(qacc[(size_t)i * D + k]);
            jv = jv + sq(qvel[(size_t)i * D + k]);
        }
        for (int k = 0; k < A; ++k) ar = ar + sq(arate[(size_t)i * A + k]);
        for (int k = 0; k < F; ++k) at = at + (air[(size_t)i * F + k] - R(0.5));
        r = r - R(p.w_joint_motion) * dt * (jm + jv);
        r = r - R(p.w_action_rate) * dt * ar;
        r = r - R(p.w_collision) * dt * coll[i];
        r = r + R(p.w_air_time) * dt * at;
    }
    out[i] = r;
}

// rot_dist (spatial.py:125-132): 2 asin(clip(|vec(qa (x) conj(qb))|, 0, 1))
template <class R> __device__ R rot_dist(const R *a, const R *b) {
    Q4<R> d = qmul(Q4<R>{a[0], a[1], a[2], a[3]}, qconj(Q4<R>{b[0], b[1], b[2], b[3]}));
    R nn = r_sqrt(d.x * d.x + d.y * d.y + d.z * d.z);
    nn = nn < R(0) ? R(0) : (nn > R(1) ? R(1) : nn);
    return R(2) * asin(nn);
}

// cube_reorientation_reward (rewards.py:161-176)
template <class R>
__global__ void cube_kernel(int n, int A, const R *opos, const R *oq, const R *tpos, const R *tq, const R *act,
                            bsim_cube_params_t p, R *out, uint8_t *reset, uint8_t *success) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    R gd = norm3(opos + 3 * i, tpos + 3 * i);
    R rd = rot_dist(oq + 4 * i, tq + 4 * i);
    R sa = 0;
    for (int k = 0; k < A; ++k) sa = sa + sq(act[(size_t)i * A + k]);
    R r = gd * R(p.dist_reward_scale) + (R(1) / (fabs(rd) + R(p.rot_eps))) * R(p.rot_reward_scale) +
          sa * R(p.action_penalty_scale);
    bool ok = fabs(rd) <= R(p.success_tolerance);
    if (ok) r = r + R(p.reach_goal_bonus);
    if (gd >= R(p.fall_dist)) r = r + R(p.fall_penalty);
    out[i] = r;
    reset[i] = ok;
    success[i] = ok;
}

// franka_stack_reward (rewards.py:200-219)
template <class R>
__global__ void franka_kernel(int n, const R *ca, const R *cb, const R *gp, const R *lf, const R *rf,
                              bsim_franka_params_t p, R *out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const R *a = ca + 3 * i, *b = cb + 3 * i, *g = gp + 3 * i;
    R xy = r_sqrt(sq(a[0] - b[0]) + sq(a[1] - b[1]));
    bool lifted = a[2] > R(p.lift_height);
    bool aligned = xy < R(p.align_tolerance);
    R dg = norm3(g, a);
    bool away = dg > R(p.away_distance);
    bool stacked = (a[2] > b[2]) && aligned && away;
    R rs = stacked ? R(p.w_stack) : R(0);
    R ral = lifted ? R(p.w_align) * (R(1) - tanh(R(10) * xy)) : R(0);
    R rl = lifted ? R(p.w_lift) : R(0);
    R ds = dg + norm3(lf + 3 * i, a) + norm3(rf + 3 * i, a);
    R rr = R(p.w_reach) * (R(1) - tanh((R(10) / R(3)) * ds));
    R alt = ral + rl + rr;
    out[i] = rs > alt ? rs : alt;
}

// trifinger_reward (rewards.py:179-197): logistic position kernel + rotation
// term, fingertip-to-cube progress (until the cutoff) and fingertip speed
template <class R>
__global__ void trifinger_kernel(int n, int F, const R *cp, const R *pcp, const R *cq, const R *tp, const R *tq,
                                 const R *ft, const R *pft, const R *fv, const int64_t *ts,
                                 bsim_trifinger_params_t p, R *out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const R *c = cp + 3 * i, *pc = pcp + 3 * i;
    R x = norm3(c, tp + 3 * i);
    R ka = R(p.kernel_a) * x;
    R kern = R(1) / (exp(ka) + R(p.kernel_b) + exp(-ka));
    R rd = rot_dist(cq + 4 * i, tq + 4 * i);
    R rog = kern + R(1) / (R(3) * fabs(rd) + R(0.01));
    R delta = 0, speed = 0;
    for (int f = 0; f < F; ++f) {
        size_t o = ((size_t)i * F + f) * 3;
        delta = delta + (norm3(ft + o, c) - norm3(pft + o, pc));
        speed = speed + sq(fv[o]) + sq(fv[o + 1]) + sq(fv[o + 2]);
    }
    R rfo = (double)ts[i] <= p.fingertip_term_cutoff ? delta : R(0);
    out[i] = R(p.w_og) * rog + R(p.w_fo) * rfo + R(p.w_fv) * speed;
}

// ingenuity_reward (rewards.py:115-121): R_pos (1 + R_upright + R_spin)
template <class R>
__global__ void ingenuity_kernel(int n, int S, const R *pos, const R *tgt, const R *upz, const R *spin, R *out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const R *a = pos + 3 * i, *b = tgt + 3 * i;
    R d2 = sq(a[0] - b[0]) + sq(a[1] - b[1]) + sq(a[2] - b[2]);
    R s2 = 0;
    for (int k = 0; k < S; ++k) s2 = s2 + sq(spin[(size_t)i * S + k]);
    R rpos = R(1) / (R(1) + d2);
    R rspin = R(1) / (R(1) + s2);
    R rup = R(1) / (R(1) + sq(upz[i]));
    out[i] = rpos * (R(1) + rup + rspin);
}

// amp_imitation_reward (rewards.py:222-225)
template <class R>
__global__ void amp_kernel(int n, const R *d, R *out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    R v = d[i];
    const R lo = R(1e-4), hi = R(1) - R(1e-4);
    v = v < lo ? lo : (v > hi ? hi : v);  // np.clip; NaN passes through
    out[i] = -log(R(1) - v);
}

int done(const char *) { return cudaGetLastError() == cudaSuccess ? 0 : -2; }
constexpr int TPB = 256;
inline int grid(int n) { return (n + TPB - 1) / TPB; }

}  // namespace


extern "C" {

int bsim_reward_locomotion(int n, int D, int fp64, const void *torso, const void *target, const void *up,
                           const void *heading, const void *act, const void *qpos, const void *qvel, const void *lo,
                           const void *hi, const void *strength, const void *prev, const bsim_loco_params_t *p,
                           void *out, void *pot, void *stream) {
    if (n <= 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (fp64)
        loco_kernel<double><<<grid(n), TPB, 0, s>>>(n, D, (const double *)torso, (const double *)target,
            (const double *)up, (const double *)heading, (const double *)act, (const double *)qpos,
            (const double *)qvel, (const double *)lo, (const double *)hi, (const double *)strength,
            (const double *)prev, *p, (double *)out, (double *)pot);
    else
        loco_kernel<float><<<grid(n), TPB, 0, s>>>(n, D, (const float *)torso, (const float *)target,
            (const float *)up, (const float *)heading, (const float *)act, (const float *)qpos,
            (const float *)qvel, (const float *)lo, (const float *)hi, (const float *)strength,
            (const float *)prev, *p, (float *)out, (float *)pot);
    return done("loco");
}

int bsim_reward_anymal(int n, int D, int A, int F, int fp64, const void *lin, const void *ang, const void *cmd,
                       const void *qvel, const void *qacc, const void *torques, const void *arate, const void *coll,
                       const void *air, const bsim_anymal_params_t *p, int rough, void *out, void *stream) {
    if (n <= 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (fp64)
        anymal_kernel<double><<<grid(n), TPB, 0, s>>>(n, D, A, F, (const double *)lin, (const double *)ang,
            (const double *)cmd, (const double *)qvel, (const double *)qacc, (const double *)torques,
            (const double *)arate, (const double *)coll, (const double *)air, *p, rough, (double *)out);
    else
        anymal_kernel<float><<<grid(n), TPB, 0, s>>>(n, D, A, F, (const float *)lin, (const float *)ang,
            (const float *)cmd, (const float *)qvel, (const float *)qacc, (const float *)torques,
            (const float *)arate, (const float *)coll, (const float *)air, *p, rough, (float *)out);
    return done("anymal");
}

int bsim_reward_cube(int n, int A, int fp64, const void *opos, const void *oq, const void *tpos, const void *tq,
                     const void *act, const bsim_cube_params_t *p, void *out, uint8_t *reset, uint8_t *success,
                     void *stream) {
    if (n <= 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (fp64)
        cube_kernel<double><<<grid(n), TPB, 0, s>>>(n, A, (const double *)opos, (const double *)oq,
            (const double *)tpos, (const double *)tq, (const double *)act, *p, (double *)out, reset, success);
    else
        cube_kernel<float><<<grid(n), TPB, 0, s>>>(n, A, (const float *)opos, (const float *)oq,
            (const float *)tpos, (const float *)tq, (const float *)act, *p, (float *)out, reset, success);
    return done("cube");
}

int bsim_reward_franka(int n, int fp64, const void *ca, const void *cb, const void *gp, const void *lf,
                       const void *rf, const bsim_franka_params_t *p, void *out, void *stream) {
    if (n <= 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (fp64)
        franka_kernel<double><<<grid(n), TPB, 0, s>>>(n, (const double *)ca, (const double *)cb,
            (const double *)gp, (const double *)lf, (const double *)rf, *p, (double *)out);
    else
        franka_kernel<float><<<grid(n), TPB, 0, s>>>(n, (const float *)ca, (const float *)cb, (const float *)gp,
            (const float *)lf, (const float *)rf, *p, (float *)out);
    return done("franka");
}

int bsim_reward_trifinger(int n, int F, int fp64, const void *cp, const void *pcp, const void *cq, const void *tp,
                          const void *tq, const void *ft, const void *pft, const void *fv, const int64_t *ts,
                          const bsim_trifinger_params_t *p, void *out, void *stream) {
    if (n <= 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (fp64)
        trifinger_kernel<double><<<grid(n), TPB, 0, s>>>(n, F, (const double *)cp, (const double *)pcp,
            (const double *)cq, (const double *)tp, (const double *)tq, (const double *)ft, (const double *)pft,
            (const double *)fv, ts, *p, (double *)out);
    else
        trifinger_kernel<float><<<grid(n), TPB, 0, s>>>(n, F, (const float *)cp, (const float *)pcp,
            (const float *)cq, (const float *)tp, (const float *)tq, (const float *)ft, (const float *)pft,
            (const float *)fv, ts, *p, (float *)out);
    return done("trifinger");
}

int bsim_reward_ingenuity(int n, int S, int fp64, const void *pos, const void *tgt, const void *upz,
                          const void *spin, void *out, void *stream) {
    if (n <= 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (fp64)
        ingenuity_kernel<double><<<grid(n), TPB, 0, s>>>(n, S, (const double *)pos, (const double *)tgt,
            (const double *)upz, (const double *)spin, (double *)out);
    else
        ingenuity_kernel<float><<<grid(n), TPB, 0, s>>>(n, S, (const float *)pos, (const float *)tgt,
            (const float *)upz, (const float *)spin, (float *)out);
    return done("ingenuity");
}

int bsim_reward_amp(int n, int fp64, const void *d, void *out, void *stream) {
    if (n <= 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    if (fp64)
        amp_kernel<double><<<grid(n), TPB, 0, s>>>(n, (const double *)d, (double *)out);
    else
        amp_kernel<float><<<grid(n), TPB, 0, s>>>(n, (const float *)d, (float *)out);
    return done("amp");
}

}  // extern "C"
