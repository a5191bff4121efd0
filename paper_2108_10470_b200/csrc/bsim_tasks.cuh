// bsim_tasks.cuh -- per-env task logic of the locomotion tasks: reward,
// termination, observation and reset, fused so one group of G lanes per env
// (task_step_env_g) finishes a whole EnvBatch.step() tail.
//
// QuadrupedEnv: reference envs.py:359-478, locomotion_reward rewards.py:78-112.
// AnymalObsEnv: reference envs.py:484-565, anymal_reward (flat) rewards.py:129-158.
#pragma once

#ifndef BSIM_TASK_G
#define BSIM_TASK_G 8   // lanes per env of the task tail (task_step_env_g)
#endif

#include "bsim_dr.cuh"
#include "bsim_kin.cuh"
#include "bsim_rng.cuh"

namespace bsim {

// the task-layer argument rules shared by bsim_task_* and bsim_env_step*
inline bool task_args_ok(const bsim_layout_t *L, const bsim_task_t *t) {
    if (t->kind == BSIM_TASK_CUBE)
        return t->goals && t->act_dim == L->dofs_per_env && L->actors_per_env == 2 &&
               t->obs_dim == 2 * L->dofs_per_env + 24 + t->act_dim;
    if (t->kind == BSIM_TASK_STACK)
        return t->goals && t->act_dim == L->dofs_per_env && L->actors_per_env == 3 && L->bodies_per_env >= 5 &&
               t->obs_dim == 2 * L->dofs_per_env + 27 + t->act_dim;
    const bool kind_ok = t->kind == BSIM_TASK_QUADRUPED || t->kind == BSIM_TASK_ANYMAL || t->kind == BSIM_TASK_HUMANOID;
    return kind_ok && t->act_dim == L->dofs_per_env && L->actors_per_env == 1 &&
           t->obs_dim == 12 + 2 * t->act_dim + (t->kind == BSIM_TASK_ANYMAL ? 0 : 6 * L->sensors_per_env) + t->act_dim;
}

template <class R> struct TaskView {
    const bsim_task_t &t;
    R *stage = nullptr;   // optional shared-memory obs rows of envs [stage_e0, ...) (coalesced copy-out)
    int stage_e0 = 0;
    R *scratch = nullptr; // optional per-env shared-memory scratch of envs [stage_e0, ...): 13 B body-row
    int scratch_stride = 0;   // words + 2 D DOF words each (the group reset, task_reset_env_g)
    BS_HD R *obs(int e) const {
        return stage ? stage + (size_t)(e - stage_e0) * t.obs_dim : reinterpret_cast<R *>(t.obs) + (size_t)e * t.obs_dim;
    }
    BS_HD R &reward(int e) const { return reinterpret_cast<R *>(t.reward)[e]; }
    BS_HD R *act(int e) const { return reinterpret_cast<R *>(t.actions) + (size_t)e * t.act_dim; }
    BS_HD double &potential(int e) const { return t.potentials[e]; }
    BS_HD R *cmd(int e) const { return reinterpret_cast<R *>(t.commands) + 3 * (size_t)e; }
    BS_HD R *goal(int e) const { return reinterpret_cast<R *>(t.goals) + 8 * (size_t)e; }
    BS_HD R lo(int k) const { return reinterpret_cast<const R *>(t.dof_lower)[k]; }
    BS_HD R hi(int k) const { return reinterpret_cast<const R *>(t.dof_upper)[k]; }
};

// env-local root pose / velocity of actor 0
template <class R> struct Root {
    V3<R> p, v, w;
    Q4<R> q;
};
template <class R> BS_HD Root<R> root_of(const Ctx<R> &c, int e) {
    const R *b = c.s.body_q + (size_t)e * c.d.B * 13;
    return Root<R>{V3<R>{b[0], b[1], b[2]}, V3<R>{b[7], b[8], b[9]}, V3<R>{b[10], b[11], b[12]},
                   Q4<R>{b[3], b[4], b[5], b[6]}};
}
template <class R> BS_HD V3<R> rot_inv(Q4<R> q, V3<R> v) { return qrot(qconj(q), v); }

// ------------------------------------------------------------ quadruped
constexpr double QUAD_TARGET_X = 1000.0;

// heading / up projections shared by obs and reward (envs.py:426-439)
template <class R> struct Frame {
    V3<R> lin_b, ang_b;
    R up_z, heading_proj;
};
template <class R> BS_HD Frame<R> quad_frame(const Root<R> &r) {
    Frame<R> f;
    f.lin_b = rot_inv(r.q, r.v);
    f.ang_b = rot_inv(r.q, r.w);
    f.up_z = qrot(r.q, v3(R(0), R(0), R(1))).z;
    V3<R> heading = qrot(r.q, v3(R(1), R(0), R(0)));
    R tx = R(QUAD_TARGET_X) - r.p.x, ty = R(0) - r.p.y;
    R nrm = r_max(r_sqrt(tx * tx + ty * ty), R(1e-9));
    f.heading_proj = heading.x * (tx / nrm) + heading.y * (ty / nrm);
    return f;
}

// ------------------------------------------------------------ cube reorientation
// The env's last body is the cube (actor 1); tv.goal(e) = goal pos 3, quat 4, successes.
template <class R> BS_HD const R *cube_row(const Ctx<R> &c, int e) {
    return c.s.body_q + ((size_t)e * c.d.B + c.d.B - 1) * 13;
}

// hand DOFs U(+-0.1) clamped into their limits, zero rates; the cube at the
// goal position (its spawn point above the palm) with a random yaw, at rest
template <class R> __device__ void arm_reset_dofs(const Ctx<R> &c, const TaskView<R> &tv, int e, NpRng &rng) {
    R *root = c.s.body_q + (size_t)e * c.d.B * 13;  // fixed-base root: the pose stays, the twist is zeroed
    for (int k = 7; k < 13; ++k) root[k] = R(0);
    R *dof = c.s.dof_state + 2 * (size_t)e * c.d.D;
    for (int k = 0; k < tv.t.act_dim; ++k) {
        double q = np_uniform(rng, -0.1, 0.1);
        const double lo = (double)tv.lo(k), hi = (double)tv.hi(k);
        dof[2 * k] = R(q < lo ? lo : (q > hi ? hi : q));
        dof[2 * k + 1] = R(0);
    }
}
// a single-body actor at rest at `p` (+ U(+-jitter) in x, y) with a random yaw
template <class R> __device__ void place_box(R *row, const R *p, double jitter, NpRng &rng) {
    const double jx = jitter > 0.0 ? np_uniform(rng, -jitter, jitter) : 0.0;
    const double jy = jitter > 0.0 ? np_uniform(rng, -jitter, jitter) : 0.0;
    const double yaw = np_uniform(rng, -3.141592653589793, 3.141592653589793);
    row[0] = R((double)p[0] + jx); row[1] = R((double)p[1] + jy); row[2] = p[2];
    row[3] = R(0); row[4] = R(0); row[5] = R(sin(yaw / 2.0)); row[6] = R(cos(yaw / 2.0));
    for (int k = 7; k < 13; ++k) row[k] = R(0);
}
template <class R> __device__ void cube_reset_state(const Ctx<R> &c, const TaskView<R> &tv, int e, NpRng &rng) {
    arm_reset_dofs(c, tv, e, rng);
    place_box(c.s.body_q + ((size_t)e * c.d.B + c.d.B - 1) * 13, tv.goal(e), 0.0, rng);
}
// Franka stacking: arm DOFs as above, cube A / B near their spawn points
template <class R> __device__ void stack_reset_state(const Ctx<R> &c, const TaskView<R> &tv, int e, NpRng &rng) {
    arm_reset_dofs(c, tv, e, rng);
    R *rows = c.s.body_q + (size_t)e * c.d.B * 13;
    place_box(rows + (size_t)(c.d.B - 2) * 13, tv.goal(e), 0.05, rng);
    place_box(rows + (size_t)(c.d.B - 1) * 13, tv.goal(e) + 3, 0.05, rng);
}

// a new goal orientation, uniform on SO(3) (Shoemake), from the stream keyed
// (seed, global env, reset count, successes)
template <class R> __device__ void cube_new_goal(const Ctx<R> &c, const TaskView<R> &tv, int e) {
    R *g = tv.goal(e);
    uint32_t key[4] = {tv.t.seed, (uint32_t)(c.L.env_offset + e), (uint32_t)tv.t.reset_count[e],
                       0xD000u + (uint32_t)g[7]};
    NpRng r = np_rng(key, 4);
    const double u1 = np_uniform(r, 0.0, 1.0), u2 = np_uniform(r, 0.0, 1.0), u3 = np_uniform(r, 0.0, 1.0);
    const double a = sqrt(1.0 - u1), b = sqrt(u1), tp = 6.283185307179586;
    g[3] = R(a * sin(tp * u2)); g[4] = R(a * cos(tp * u2)); g[5] = R(b * sin(tp * u3)); g[6] = R(b * cos(tp * u3));
}

// ------------------------------------------------------------ reset
// EnvBatch.reset for one env (envs.py:145-166) with the task's _reset_envs
// (404-419 / 517-531) and _post_reset (385-397 / 506-515).
#if defined(BSIM_EXP_RESET_CLOCKS) && defined(__CUDACC__)
// timing experiment only: cycles per reset phase summed over all resets ([7] = count)
__device__ unsigned long long bsim_reset_clk[8];
#define BSIM_RCLK(i)                                              \
    do {                                                          \
        unsigned long long t_ = clock64();                        \
        atomicAdd(&bsim_reset_clk[i], t_ - t_prev_);              \
        t_prev_ = t_;                                             \
    } while (0)
#else
#define BSIM_RCLK(i) \
    do {             \
    } while (0)
#endif

template <class R> __device__ void task_reset_env(const Ctx<R> &c, const TaskView<R> &tv, int e) {
#if defined(BSIM_EXP_RESET_CLOCKS) && defined(__CUDACC__)
    unsigned long long t_prev_ = clock64();
    atomicAdd(&bsim_reset_clk[7], 1ull);
#endif
    const bsim_task_t &t = tv.t;
    const Dims &d = c.d;
    if (c.s.nonfinite[e]) c.s.nonfinite[e] = 0;   // clear_nonfinite (physics.py:1090)
    const int64_t step_count = t.step_count_dev ? *t.step_count_dev : t.step_count;
    dr_randomize_env(c, t.dr, e, step_count);     // randomizer.randomize (envs.py:154-155)
    BSIM_RCLK(0);
    const uint32_t genv = (uint32_t)(c.L.env_offset + e);
    uint32_t key[4] = {t.seed, genv, (uint32_t)t.reset_count[e], 0xCu};
    NpRng rng = np_rng(key, 3);
    const bool cube = t.kind == BSIM_TASK_CUBE, stack = t.kind == BSIM_TASK_STACK;
    const bool loco = t.kind != BSIM_TASK_ANYMAL && !cube && !stack;
    if (cube) {
        cube_reset_state(c, tv, e, rng);
    } else if (stack) {
        stack_reset_state(c, tv, e, rng);
    } else {
        double qx = 0.0, qy = 0.0, qz = 0.0, qw = 1.0;
        if (loco) {
            double yaw = np_uniform(rng, -0.1, 0.1);
            qz = sin(yaw / 2.0);
            qw = cos(yaw / 2.0);
        }
        double n = sqrt(qx * qx + qy * qy + qz * qz + qw * qw);  // set_root_state renormalises (buffers.py:145)
        R *root = c.s.body_q + (size_t)e * d.B * 13;
        root[0] = R(0); root[1] = R(0); root[2] = R(t.rest_height + 0.02);
        root[3] = R(qx / n); root[4] = R(qy / n); root[5] = R(qz / n); root[6] = R(qw / n);
        for (int k = 7; k < 13; ++k) root[k] = R(0);
        R *dof = c.s.dof_state + 2 * (size_t)e * d.D;
        for (int k = 0; k < t.act_dim; ++k) {
            dof[2 * k] = R(np_uniform(rng, -0.1, 0.1));
            dof[2 * k + 1] = R(0);
        }
    }
    BSIM_RCLK(1);
    if (t.obs_noise) {  // per-episode correlated noise continues the reset stream (envs.py:161-164)
        R *cn = reinterpret_cast<R *>(t.corr_noise) + (size_t)e * t.obs_dim;
        for (int k = 0; k < t.obs_dim; ++k)
            cn[k] = t.obs_noise_corr > 0.0 ? R(0.0 + t.obs_noise_corr * np_std_normal(rng)) : R(0);
    }
    BSIM_RCLK(2);
    fk_env(c, e, 0xffffffffu);
    BSIM_RCLK(3);
    repack_env(c, e, 0xffffffffu);
    BSIM_RCLK(4);
    t.episode_steps[e] = 0;
    t.reset_count[e] += 1;
    R *a = tv.act(e);
    for (int k = 0; k < t.act_dim; ++k) a[k] = R(0);
    if (cube) {
        tv.goal(e)[7] = R(0);
        cube_new_goal(c, tv, e);
    } else if (loco) {
        const double z = (double)R(t.rest_height + 0.02);   // the stored root height
        tv.potential(e) = -sqrt(QUAD_TARGET_X * QUAD_TARGET_X + z * z) / t.control_dt;
    } else if (!stack) {   // anymal velocity commands
        key[2] = (uint32_t)t.reset_count[e];
        NpRng cr = np_rng(key, 4);
        R *cmd = tv.cmd(e);
        for (int k = 0; k < 3; ++k) cmd[k] = R(np_uniform(cr, -1.0, 1.0));
    }
    BSIM_RCLK(5);
}

// ------------------------------------------------------------ group form
// The same tail with G lanes per env (an aligned group of a warp, s = lane
// in the group): the per-DOF / per-sensor loops are strided over the group
// and the reward's DOF sums reduced with a fixed xor tree; everything else is
// computed redundantly by the group's lanes (one SIMT instruction stream) and
// written by lane 0.  Resets and observation noise (sequential RNG streams)
// run on lane 0.  G = 1 is the serial form.  Device only.
#if defined(__CUDACC__)
template <int G> __device__ __forceinline__ unsigned group_mask() {
    if constexpr (G >= 32) return 0xffffffffu;
    else return ((1u << G) - 1u) << ((threadIdx.x & 31u) & ~(unsigned)(G - 1));
}
template <int G, class R> __device__ __forceinline__ R group_sum(R v) {
    const unsigned m = group_mask<G>();
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(m, v, o);
    return v;
}

// task_reset_env for the locomotion / ANYmal tasks by the G lanes of the env's
// group, on the env's shared-memory scratch (TaskView::scratch): draw k of the
// env's reset stream is taken by lane k % G after np_advance(k) -- the same
// doubles in the same roles as the sequential draws -- the DOF rows and the
// root row are set in the scratch copy, forward kinematics walks the tree
// level by level (fk_group), and the rows go back to HBM in parallel.  The
// arithmetic per value is task_reset_env's, so results are bitwise equal; the
// latency of one reset (on the critical path of the CTA that holds it) drops
// from ~20 us of dependent single-lane global round trips.
template <class R, int G>
__device__ void task_reset_env_g(const Ctx<R> &c, const TaskView<R> &tv, int e, int sl) {
#if defined(BSIM_EXP_RESET_CLOCKS)
    unsigned long long t_prev_ = clock64();
    if (sl == 0) atomicAdd(&bsim_reset_clk[7], 1ull);
#define BSIM_GRCLK(i)                                                \
    do {                                                             \
        if (sl == 0) {                                               \
            unsigned long long t_ = clock64();                       \
            atomicAdd(&bsim_reset_clk[i], t_ - t_prev_);             \
            t_prev_ = t_;                                            \
        }                                                            \
    } while (0)
#else
#define BSIM_GRCLK(i) \
    do {              \
    } while (0)
#endif
    const bsim_task_t &t = tv.t;
    const Dims &d = c.d;
    const unsigned gm = group_mask<G>();
    const bool loco = t.kind != BSIM_TASK_ANYMAL;
    const uint32_t genv = (uint32_t)(c.L.env_offset + e);
    const uint32_t rc = (uint32_t)t.reset_count[e];
    R *__restrict__ bq = tv.scratch + (size_t)(e - tv.stage_e0) * tv.scratch_stride;
    R *__restrict__ dq = bq + 13 * d.B;
    // the env's rows into the scratch (actor roots keep theirs unless reset below)
    const R *__restrict__ gq = c.s.body_q + (size_t)e * d.B * 13;
#pragma unroll 8
    for (int i = sl; i < 13 * d.B; i += G) bq[i] = gq[i];   // unrolled: the loads issue back to back
    __syncwarp(gm);                                   // the copy lands before lane 0 rewrites the root row
    if (sl == 0) {
        if (c.s.nonfinite[e]) c.s.nonfinite[e] = 0;   // clear_nonfinite (physics.py:1090)
        const int64_t step_count = t.step_count_dev ? *t.step_count_dev : t.step_count;
        dr_randomize_env(c, t.dr, e, step_count);     // randomizer.randomize (envs.py:154-155)
    }
    BSIM_GRCLK(0);
    uint32_t key[4] = {t.seed, genv, rc, 0xCu};
    const NpRng rng = np_rng(key, 3);                 // every lane: the stream's start
    const int first = loco ? 1 : 0;                   // draw 0 = the locomotion yaw
    for (int k = sl; k < t.act_dim; k += G) {         // draw first + k -> DOF k (envs.py:404-419 / 536-549)
        NpRng r = rng;
        np_advance(r, (uint64_t)(first + k));
        dq[2 * k] = R(np_uniform(r, -0.1, 0.1));
        dq[2 * k + 1] = R(0);
    }
    for (int k = t.act_dim + sl; k < d.D; k += G) {   // (no other DOFs in these tasks; keep the state)
        dq[2 * k] = c.s.dof_state[2 * ((size_t)e * d.D + k)];
        dq[2 * k + 1] = c.s.dof_state[2 * ((size_t)e * d.D + k) + 1];
    }
    if (sl == 0) {
        double qx = 0.0, qy = 0.0, qz = 0.0, qw = 1.0;
        if (loco) {
            NpRng r = rng;
            double yaw = np_uniform(r, -0.1, 0.1);
            qz = sin(yaw / 2.0);
            qw = cos(yaw / 2.0);
        }
        double n = sqrt(qx * qx + qy * qy + qz * qz + qw * qw);  // set_root_state renormalises (buffers.py:145)
        bq[0] = R(0); bq[1] = R(0); bq[2] = R(t.rest_height + 0.02);
        bq[3] = R(qx / n); bq[4] = R(qy / n); bq[5] = R(qz / n); bq[6] = R(qw / n);
        for (int k = 7; k < 13; ++k) bq[k] = R(0);
        if (t.obs_noise) {  // per-episode correlated noise continues the reset stream (envs.py:161-164)
            NpRng r = rng;
            np_advance(r, (uint64_t)(first + t.act_dim));
            R *cn = reinterpret_cast<R *>(t.corr_noise) + (size_t)e * t.obs_dim;
            for (int k = 0; k < t.obs_dim; ++k)
                cn[k] = t.obs_noise_corr > 0.0 ? R(0.0 + t.obs_noise_corr * np_std_normal(r)) : R(0);
        }
    }
    __syncwarp(gm);
    BSIM_GRCLK(1);
    fk_group<G>(c, bq, dq, sl, gm);
    BSIM_GRCLK(3);
    // rows back to HBM: body_q (env-local), body_state (world), root_state, dof_state
    const R *__restrict__ o = c.s.env_origins + 3 * (size_t)e;
    R *__restrict__ dst_q = c.s.body_q + (size_t)e * d.B * 13;
    R *__restrict__ dst_s = c.s.body_state + (size_t)e * d.B * 13;
    const R ox = o[0], oy = o[1], oz = o[2];
#pragma unroll 8
    for (int i = sl; i < 13 * d.B; i += G) {
        const int k = i % 13;
        const R v = bq[i];
        dst_q[i] = v;
        dst_s[i] = v + (k == 0 ? ox : k == 1 ? oy : k == 2 ? oz : R(0));
    }
    for (int i = sl; i < 13 * d.A; i += G) {
        const int a = i / 13, k = i - 13 * a;
        const R v = bq[13 * c.L.actor_body_offset[a] + k];
        c.s.root_state[13 * ((size_t)e * d.A + a) + k] = v + (k == 0 ? ox : k == 1 ? oy : k == 2 ? oz : R(0));
    }
#pragma unroll 4
    for (int i = sl; i < 2 * d.D; i += G) c.s.dof_state[2 * (size_t)e * d.D + i] = dq[i];
    R *a = tv.act(e);
    for (int k = sl; k < t.act_dim; k += G) a[k] = R(0);
    BSIM_GRCLK(4);
    __syncwarp(gm);                                   // every lane read reset_count before it moves
    if (sl == 0) {
        t.episode_steps[e] = 0;
        t.reset_count[e] = (int32_t)(rc + 1u);
        if (loco) {
            const double z = (double)R(t.rest_height + 0.02);   // the stored root height
            tv.potential(e) = -sqrt(QUAD_TARGET_X * QUAD_TARGET_X + z * z) / t.control_dt;
        } else {                                      // anymal velocity commands
            key[2] = rc + 1u;
            NpRng cr = np_rng(key, 4);
            R *cmd = tv.cmd(e);
            for (int k = 0; k < 3; ++k) cmd[k] = R(np_uniform(cr, -1.0, 1.0));
        }
    }
    BSIM_GRCLK(5);
#undef BSIM_GRCLK
}

// locomotion_reward (rewards.py:78-112); returns the reward, lane 0 writes the new potential
template <class R, int G>
__device__ R quad_reward_g(const Ctx<R> &c, const TaskView<R> &tv, int e, int sl, const Root<R> &r, const Frame<R> &f,
                           bool &done) {
    const R dt = R(tv.t.control_dt), term = R(tv.t.termination_height);
    // the progress term in float64: |target - torso| ~ 1000 m, so -dist/dt in
    // fp32 would carry a 4e-3 rounding step; one double sqrt per env
    const double dx = QUAD_TARGET_X - (double)r.p.x, dy = -(double)r.p.y, dz = -(double)r.p.z;
    const double potential = -sqrt(dx * dx + dy * dy + dz * dz) / tv.t.control_dt;
    R rew = R(potential - tv.potential(e));
    R height = r.p.z;
    rew = rew + (height >= term ? R(0.5) : R(0));
    rew = rew + (height <= term ? R(-1) : R(0));
    rew = rew + (f.up_z > R(0.93) ? R(0.1) : R(0));
    rew = rew + R(0.5) * (f.heading_proj >= R(0.8) ? R(1) : f.heading_proj / R(0.8));
    const R *a = tv.act(e);
    const R *dof = c.s.dof_state + 2 * (size_t)e * c.d.D;
    R sa = R(0), se = R(0), near_ = R(0);
    #pragma unroll 4
    for (int k = sl; k < tv.t.act_dim; k += G) {
        sa = sa + a[k] * a[k];
        se = se + a[k] * R(1) * dof[2 * k + 1];
        R lo = tv.lo(k), hi = tv.hi(k);
        if (finite_r(lo) && finite_r(hi)) {
            R frac = (dof[2 * k] - lo) / (hi - lo);
            if (frac < R(0.01) || frac > R(0.99)) near_ = near_ + R(1);
        }
    }
    sa = group_sum<G>(sa);
    se = group_sum<G>(se);
    near_ = group_sum<G>(near_);
    rew = rew - R(0.005) * sa;
    rew = rew + R(0.05) * se;
    rew = rew - R(0.1) * near_;
    __syncwarp(group_mask<G>());           // every lane read the old potential
    if (sl == 0) tv.potential(e) = potential;
    done = height <= term;
    return rew;
}

// 60-dim observation (envs.py:441-461)
template <class R, int G> __device__ void quad_obs_g(const Ctx<R> &c, const TaskView<R> &tv, int e, int sl) {
    Root<R> r = root_of(c, e);
    R *__restrict__ o = tv.obs(e);   // the obs row aliases no input: loads may run ahead of the stores
    if (sl == 0) {
        Frame<R> f = quad_frame(r);
        R x = r.q.x, y = r.q.y, z = r.q.z, w = r.q.w;
        R yaw = r_atan2(R(2) * (w * z + x * y), R(1) - R(2) * (y * y + z * z));
        R roll = r_atan2(R(2) * (w * x + y * z), R(1) - R(2) * (x * x + y * y));
        R ang = r_atan2(-r.p.y, R(QUAD_TARGET_X) - r.p.x) - yaw;
        ang = r_atan2(r_sin(ang), r_cos(ang));
        o[0] = r.p.z;
        o[1] = f.lin_b.x; o[2] = f.lin_b.y; o[3] = f.lin_b.z;
        o[4] = f.ang_b.x; o[5] = f.ang_b.y; o[6] = f.ang_b.z;
        o[7] = yaw; o[8] = roll; o[9] = ang; o[10] = f.up_z; o[11] = f.heading_proj;
    }
    const int A = tv.t.act_dim, S = c.d.S;
    const R *dof = c.s.dof_state + 2 * (size_t)e * c.d.D;
    #pragma unroll 4
    for (int k = sl; k < A; k += G) {
        o[12 + k] = R(2) * (dof[2 * k] - tv.lo(k)) / (tv.hi(k) - tv.lo(k)) - R(1);
        o[12 + A + k] = dof[2 * k + 1] * R(0.05);
    }
    const R *sf = c.s.sensor_forces + 6 * (size_t)e * S;
    #pragma unroll 4
    for (int k = sl; k < 6 * S; k += G) o[12 + 2 * A + k] = sf[k] * R(0.01);
    const R *a = tv.act(e);
    #pragma unroll 4
    for (int k = sl; k < A; k += G) o[12 + 2 * A + 6 * S + k] = a[k];
}

// anymal_reward, flat terrain (rewards.py:129-158)
template <class R, int G>
__device__ R anymal_reward_g(const Ctx<R> &c, const TaskView<R> &tv, int e, int sl, const Root<R> &r, bool &done) {
    const R dt = R(tv.t.control_dt);
    V3<R> lin_b = rot_inv(r.q, r.v), ang_b = rot_inv(r.q, r.w);
    const R *cmd = tv.cmd(e);
    R ex = cmd[0] - lin_b.x, ey = cmd[1] - lin_b.y, ez = cmd[2] - ang_b.z;
    R err_xy = ex * ex + ey * ey, err_yaw = ez * ez;
    R tq = R(0);
    const R *df = c.s.dof_force + (size_t)e * c.d.D;
    #pragma unroll 4
    for (int k = sl; k < tv.t.act_dim; k += G) tq = tq + df[k] * df[k];
    tq = group_sum<G>(tq);
    R rew = R(1) * dt * exp_r(-err_xy / R(0.25)) + R(0.5) * dt * exp_r(-err_yaw / R(0.25)) - R(0.00002) * dt * tq;
    R up_z = qrot(r.q, v3(R(0), R(0), R(1))).z;
    done = up_z < R(0.3) || r.p.z < R(0.18);
    return rew;
}

// 48-dim observation (envs.py:538-550)
template <class R, int G> __device__ void anymal_obs_g(const Ctx<R> &c, const TaskView<R> &tv, int e, int sl) {
    Root<R> r = root_of(c, e);
    R *__restrict__ o = tv.obs(e);   // the obs row aliases no input: loads may run ahead of the stores
    if (sl == 0) {
        V3<R> lin_b = rot_inv(r.q, r.v), ang_b = rot_inv(r.q, r.w), gb = rot_inv(r.q, v3(R(0), R(0), R(-1)));
        o[0] = lin_b.x; o[1] = lin_b.y; o[2] = lin_b.z;
        o[3] = ang_b.x; o[4] = ang_b.y; o[5] = ang_b.z;
        o[6] = gb.x; o[7] = gb.y; o[8] = gb.z;
        const R *cmd = tv.cmd(e);
        o[9] = cmd[0]; o[10] = cmd[1]; o[11] = cmd[2];
    }
    const int A = tv.t.act_dim;
    const R *dof = c.s.dof_state + 2 * (size_t)e * c.d.D;
    #pragma unroll 4
    for (int k = sl; k < A; k += G) {
        o[12 + k] = dof[2 * k];
        o[12 + A + k] = dof[2 * k + 1] * R(0.05);
    }
    const R *a = tv.act(e);
    #pragma unroll 4
    for (int k = sl; k < A; k += G) o[12 + 2 * A + k] = a[k];
}

// cube_reorientation_reward (rewards.py:161-176) with the CubeRewardParams
// defaults (rewards.py:31-40); done = the cube fell (goal distance >= fall_dist)
template <class R, int G>
__device__ R cube_reward_g(const Ctx<R> &c, const TaskView<R> &tv, int e, int sl, bool &done, bool &success) {
    const R *cb = cube_row(c, e), *g = tv.goal(e);
    R dx = cb[0] - g[0], dy = cb[1] - g[1], dz = cb[2] - g[2];
    R gd = r_sqrt(dx * dx + dy * dy + dz * dz);
    Q4<R> dq = qmul(Q4<R>{cb[3], cb[4], cb[5], cb[6]}, qconj(Q4<R>{g[3], g[4], g[5], g[6]}));
    R nn = r_sqrt(dq.x * dq.x + dq.y * dq.y + dq.z * dq.z);
    nn = nn > R(1) ? R(1) : nn;
    R rd = R(2) * asin(nn);                   // rot_dist (spatial.py:125-132)
    const R *a = tv.act(e);
    R sa = R(0);
    #pragma unroll 4
    for (int k = sl; k < tv.t.act_dim; k += G) sa = sa + a[k] * a[k];
    sa = group_sum<G>(sa);
    R rew = gd * R(-10.0) + (R(1) / (fabs(rd) + R(0.1))) * R(1.0) + sa * R(-0.0002);
    success = fabs(rd) <= R(0.4);
    if (success) rew = rew + R(250.0);
    done = gd >= R(0.24);                     // + fall_penalty 0
    return rew;
}

// cube task observation (layout in include/batchsim_b200.h, BSIM_TASK_CUBE)
template <class R, int G> __device__ void cube_obs_g(const Ctx<R> &c, const TaskView<R> &tv, int e, int sl) {
    const int D = c.d.D, A = tv.t.act_dim;
    R *__restrict__ o = tv.obs(e);   // the obs row aliases no input: loads may run ahead of the stores
    const R *dof = c.s.dof_state + 2 * (size_t)e * D;
    #pragma unroll 4
    for (int k = sl; k < D; k += G) {
        R lo = tv.lo(k), hi = tv.hi(k), q = dof[2 * k];
        o[k] = finite_r(lo) && finite_r(hi) ? R(2) * (q - lo) / (hi - lo) - R(1) : q;
        o[D + k] = dof[2 * k + 1] * R(0.2);
    }
    if (sl == 0) {
        const R *cb = cube_row(c, e), *g = tv.goal(e);
        R *__restrict__ p = o + 2 * D;
        for (int k = 0; k < 10; ++k) p[k] = cb[k];
        for (int k = 10; k < 13; ++k) p[k] = cb[k] * R(0.2);
        for (int k = 0; k < 7; ++k) p[13 + k] = g[k];
        Q4<R> dq = qmul(Q4<R>{cb[3], cb[4], cb[5], cb[6]}, qconj(Q4<R>{g[3], g[4], g[5], g[6]}));
        p[20] = dq.x; p[21] = dq.y; p[22] = dq.z; p[23] = dq.w;
    }
    const R *a = tv.act(e);
    #pragma unroll 4
    for (int k = sl; k < A; k += G) o[2 * D + 24 + k] = a[k];
}

// franka_stack_reward (rewards.py:200-219) with the FrankaStackParams
// defaults (rewards.py:68-75); done = stacked (the r_stack condition)
template <class R> BS_HD const R *body_row(const Ctx<R> &c, int e, int b) {
    return c.s.body_q + ((size_t)e * c.d.B + b) * 13;
}
template <class R> __device__ R stack_reward(const Ctx<R> &c, int e, bool &done) {
    const int B = c.d.B;
    const R *a = body_row(c, e, B - 2), *b = body_row(c, e, B - 1), *g = body_row(c, e, B - 5);
    const R *lf = body_row(c, e, B - 4), *rf = body_row(c, e, B - 3);
    auto d3 = [](const R *x, const R *y) {
        R dx = x[0] - y[0], dy = x[1] - y[1], dz = x[2] - y[2];
        return r_sqrt(dx * dx + dy * dy + dz * dz);
    };
    R xy = r_sqrt((a[0] - b[0]) * (a[0] - b[0]) + (a[1] - b[1]) * (a[1] - b[1]));
    const bool lifted = a[2] > R(0.04), aligned = xy < R(0.02);
    R dg = d3(g, a);
    const bool stacked = a[2] > b[2] && aligned && dg > R(0.04);
    R rs = stacked ? R(16.0) : R(0);
    R ral = lifted ? R(2.0) * (R(1) - tanh(R(10) * xy)) : R(0);
    R rl = lifted ? R(1.5) : R(0);
    R ds = dg + d3(lf, a) + d3(rf, a);
    R rr = R(0.1) * (R(1) - tanh((R(10) / R(3)) * ds));
    R alt = ral + rl + rr;
    done = stacked;
    return rs > alt ? rs : alt;
}

// stacking observation (layout in include/batchsim_b200.h, BSIM_TASK_STACK)
template <class R, int G> __device__ void stack_obs_g(const Ctx<R> &c, const TaskView<R> &tv, int e, int sl) {
    const int D = c.d.D, A = tv.t.act_dim, B = c.d.B;
    R *__restrict__ o = tv.obs(e);   // the obs row aliases no input: loads may run ahead of the stores
    const R *dof = c.s.dof_state + 2 * (size_t)e * D;
    #pragma unroll 4
    for (int k = sl; k < D; k += G) {
        R lo = tv.lo(k), hi = tv.hi(k), q = dof[2 * k];
        o[k] = finite_r(lo) && finite_r(hi) ? R(2) * (q - lo) / (hi - lo) - R(1) : q;
        o[D + k] = dof[2 * k + 1] * R(0.1);
    }
    if (sl == 0) {
        const R *h = body_row(c, e, B - 5), *a = body_row(c, e, B - 2), *b = body_row(c, e, B - 1);
        R *__restrict__ p = o + 2 * D;
        for (int k = 0; k < 7; ++k) p[k] = h[k];
        for (int k = 0; k < 7; ++k) p[7 + k] = a[k];
        for (int k = 0; k < 3; ++k) p[14 + k] = a[k] - h[k];
        for (int k = 0; k < 7; ++k) p[17 + k] = b[k];
        for (int k = 0; k < 3; ++k) p[24 + k] = a[k] - b[k];
    }
    const R *a = tv.act(e);
    #pragma unroll 4
    for (int k = sl; k < A; k += G) o[2 * D + 27 + k] = a[k];
}

template <class R, int G> __device__ void task_obs_g(const Ctx<R> &c, const TaskView<R> &tv, int e, int sl) {
    const bsim_task_t &t = tv.t;
    if (t.kind == BSIM_TASK_CUBE) cube_obs_g<R, G>(c, tv, e, sl);
    else if (t.kind == BSIM_TASK_STACK) stack_obs_g<R, G>(c, tv, e, sl);
    else if (t.kind != BSIM_TASK_ANYMAL) quad_obs_g<R, G>(c, tv, e, sl);
    else anymal_obs_g<R, G>(c, tv, e, sl);
    if (t.obs_noise) {  // perturb_observations (randomize.py:231-237): one sequential stream per env
        __syncwarp(group_mask<G>());
        if (sl == 0) {
            R *__restrict__ o = tv.obs(e);   // the obs row aliases no input: loads may run ahead of the stores
            const R *cn = reinterpret_cast<const R *>(t.corr_noise) + (size_t)e * t.obs_dim;
            if (t.obs_noise_uncorr > 0.0) {
                uint32_t key[4] = {t.seed, 0xE7u, (uint32_t)(c.L.env_offset + e), (uint32_t)t.noise_count[e]};
                NpRng rr = np_rng(key, 4);
                for (int k = 0; k < t.obs_dim; ++k) o[k] = o[k] + R(0.0 + t.obs_noise_uncorr * np_std_normal(rr));
                t.noise_count[e] += 1;
            }
            for (int k = 0; k < t.obs_dim; ++k) o[k] = o[k] + cn[k];
        }
    }
}

// the reset path out of line: the tail's hot path stays small (inlined, the
// FK / DR / RNG code made instruction-fetch stalls the tail's top stall)
template <class R> __device__ __noinline__ void task_reset_env_call(const Ctx<R> &c, const TaskView<R> &tv, int e) {
    task_reset_env(c, tv, e);
}
template <class R, int G>
__device__ __noinline__ void task_reset_env_g_call(const Ctx<R> &c, const TaskView<R> &tv, int e, int sl) {
    task_reset_env_g<R, G>(c, tv, e, sl);
}
// goal reset after a success (cube task): successes + 1, a new goal orientation
template <class R> __device__ __noinline__ void cube_goal_call(const Ctx<R> &c, const TaskView<R> &tv, int e) {
    tv.goal(e)[7] = tv.goal(e)[7] + R(1);
    cube_new_goal(c, tv, e);
}

// EnvBatch.step tail after the decimated physics (envs.py:188-199), G lanes per env
template <class R, int G> __device__ void task_step_env_g(const Ctx<R> &c, const TaskView<R> &tv, int e, int sl) {
    const bsim_task_t &t = tv.t;
    const int steps = t.episode_steps[e] + 1;
    Root<R> r = root_of(c, e);
    bool done, success = false;
    R rew;
    if (t.kind == BSIM_TASK_CUBE) rew = cube_reward_g<R, G>(c, tv, e, sl, done, success);
    else if (t.kind == BSIM_TASK_STACK) rew = stack_reward(c, e, done);
    else if (t.kind != BSIM_TASK_ANYMAL) rew = quad_reward_g<R, G>(c, tv, e, sl, r, quad_frame(r), done);
    else rew = anymal_reward_g<R, G>(c, tv, e, sl, r, done);
    const bool timeout = steps >= t.episode_length;
    const bool pois = c.s.nonfinite[e] != 0;
    done = done || timeout || pois;
    __syncwarp(group_mask<G>());           // every lane read the pre-step state
    // locomotion / ANYmal resets run on the whole group (task_reset_env_g)
    const bool group_reset = tv.scratch && c.d.B <= 64 &&
                             (t.kind == BSIM_TASK_QUADRUPED || t.kind == BSIM_TASK_ANYMAL || t.kind == BSIM_TASK_HUMANOID);
    if (sl == 0) {
        t.episode_steps[e] = steps;
        tv.reward(e) = pois ? R(0) : rew;
        t.done[e] = done;
        t.timeout[e] = timeout;
        t.poisoned[e] = pois;
        if (done && !group_reset) task_reset_env_call(c, tv, e);
        else if (!done && success) cube_goal_call(c, tv, e);
    }
    if (done && group_reset) task_reset_env_g_call<R, G>(c, tv, e, sl);   // done is uniform over the group
    __syncwarp(group_mask<G>());           // the reset state is visible to the group
    task_obs_g<R, G>(c, tv, e, sl);        // reset rows get the post-reset observation (envs.py:195-198)
}
#endif

}  // namespace bsim
