/*
 * batchsim_b200.h -- C ABI of the B200 batched rigid-body step.
 *
 * The reference has no native ABI: its drop-in boundary is the duck-typed
 * Python `Scene` protocol plus the `SimBuffers` facade
 * (/root/reference/pkg/src/batchsim/physics.py:140-1091,
 *  /root/reference/pkg/src/batchsim/buffers.py:47-225).  Every entry point
 * below replaces one method of that boundary (cited per function) and takes
 * only plain pointers and sizes.  All state pointers are DEVICE pointers to
 * float32 arrays in the reference's shapes; `stream` is a cudaStream_t passed
 * as void*.  Every call is asynchronous on `stream` and returns 0 or a
 * negative BSIM_E* code; nothing is returned through device memory except
 * where stated.
 *
 * Precision / frame contract (B200 design): the canonical body state
 * `body_q` is float32 *env-local* (world position minus env origin); the
 * tensor-API outputs `root_state` / `body_state` are world frame like the
 * reference.  See DESIGN.md "Data layout in HBM".
 */
#ifndef BATCHSIM_B200_H
#define BATCHSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSIM_ABI_VERSION 2

enum bsim_status {
    BSIM_OK = 0,
    BSIM_E_INVALID = -1,   /* bad sizes / null pointers                          */
    BSIM_E_CUDA = -2,      /* a CUDA launch or API call failed (bsim_last_error) */
    BSIM_E_TOO_LARGE = -3, /* model does not fit the kernel's shared memory     */
};

enum bsim_joint_kind { BSIM_FIXED = 0, BSIM_REVOLUTE = 1, BSIM_PRISMATIC = 2, BSIM_SPHERICAL = 3 };
enum bsim_dof_mode { BSIM_MODE_FORCE = 0, BSIM_MODE_POSITION = 1, BSIM_MODE_VELOCITY = 2 };

/* Every real-valued table and array exists in two precisions: float (the
   fast path) and double (the exact-parity path, run on B200's FP64 units).
   The *64 structs are field-for-field the same with double in place of
   float; entry points with the _f64 suffix take them. */

/* One joint slot (reference physics.py:262-287).  parent/child are body
   indices local to the env; dof is the env-local first DOF or -1. */
#define BSIM_JOINT_FIELDS(REAL)                                             \
    int32_t kind, parent, child, dof, actor, has_limits, pad0, pad1;        \
    REAL axis[3], origin_pos[3], origin_quat[4], child_pos[3], child_quat[4]; \
    REAL pad[7];
typedef struct bsim_joint_t { BSIM_JOINT_FIELDS(float) } bsim_joint_t;      /* 128 B */
typedef struct bsim_joint64_t { BSIM_JOINT_FIELDS(double) } bsim_joint64_t; /* 224 B */

/* One tendon (reference model.py:123-134, tendons.py).  kind 0 fixed, 1 spatial;
   elements [first, first+count) of the element table. */
#define BSIM_TENDON_FIELDS(REAL)                                                       \
    int32_t kind, first, count, has_limits, reaction_body, actor, path_offset, pad;    \
    REAL rest_length, stiffness, damping, limit_lo, limit_hi, limit_stiffness, pad2[2];
typedef struct bsim_tendon_t { BSIM_TENDON_FIELDS(float) } bsim_tendon_t;
typedef struct bsim_tendon64_t { BSIM_TENDON_FIELDS(double) } bsim_tendon64_t;

/* fixed: index = env-local dof, joint = joint slot, v[0] = coefficient;
   spatial: index = env-local body, v[0..2] = offset, v[3] = weight. */
#define BSIM_TELEM_FIELDS(REAL) int32_t index, parent, joint, pad; REAL v[4];
typedef struct bsim_tendon_elem_t { BSIM_TELEM_FIELDS(float) } bsim_tendon_elem_t;
typedef struct bsim_tendon_elem64_t { BSIM_TELEM_FIELDS(double) } bsim_tendon_elem64_t;

/* Solver scalars (reference SimParams, physics.py:54-73). */
#define BSIM_PARAMS_FIELDS(REAL)                                                        \
    REAL dt;                                                                            \
    int32_t position_iterations, velocity_iterations;                                   \
    REAL max_bias, restitution, bounce_threshold, rest_offset, friction_offset_threshold, \
         solver_offset_slop, max_force, linear_damping, angular_damping,                \
         max_linear_velocity, max_angular_velocity;
typedef struct bsim_params_t { BSIM_PARAMS_FIELDS(float) } bsim_params_t;
typedef struct bsim_params64_t { BSIM_PARAMS_FIELDS(double) } bsim_params64_t;

/* Static per-env tables, replicated over envs (reference physics.py:216-355).
   Table pointers are DEVICE pointers; joints / tendons / tendon_elems point at
   the float or double struct variant matching the entry point's precision. */
typedef struct bsim_layout_t {
    int32_t num_envs, actors_per_env, bodies_per_env, dofs_per_env, joints_per_env,
            planes_per_env, pairs_per_env, sensors_per_env, tendons_per_env, env_offset;
    int32_t topology_id;   /* 0 = generic; k > 0 = the AOT-specialised topology k
                              (paper_2108_10470_b200/csrc/bsim_topologies.cuh) */
    int32_t sched_stages, sched_width;     /* the Gauss-Seidel row schedule below (0 = none:
                                              one lane per env in reference order) */
    int32_t sched_flags;                   /* bit 0: the schedule holds the joint rows only; the
                                              contact rows follow in reference order on one lane */
    const void *joints;                    /* [J]    */
    const int32_t *plane_body;             /* [P]    */
    const int32_t *pair_body;              /* [Q][2] */
    const int32_t *sensor_body;            /* [S]    */
    const int32_t *actor_body_offset;      /* [A+1]  */
    const int32_t *actor_dof_offset;       /* [A+1]  */
    const void *tendons;                   /* [T]    */
    const void *tendon_elems;
    const int32_t *spatial_paths;          /* per tendon at path_offset: npaths, {len, idx...}* */
    const int32_t *pair_kind;              /* [Q] BSIM_PAIR_* */
    const void *pair_ext;                  /* [Q][4] real: PB box half extents of b; PC (0, hh_b);
                                              CC (hh_a, hh_b); SS unused */
    const int32_t *sweep_sched;            /* [sched_stages][sched_width] rows of one solver pass
                                              (physics.py:760-775): r < J joint r, r < J + P plane
                                              slot r - J, else pair slot r - J - P; -1 = idle lane.
                                              Rows of one stage touch disjoint bodies, and every
                                              row comes after each earlier row (reference order)
                                              that shares a body with it, so running a stage's rows
                                              side by side gives the reference's sequential result
                                              (paper_2108_10470_b200/layout.py sweep_schedule). */
} bsim_layout_t;

/* Pair-slot narrow phase kinds.  SS is the reference's only pair type
   (physics.py:481-497); PB / PC / CC extend the slot model to box and capsule
   pairs (a sphere, capsule end sphere or box corner against a box; a sphere
   against a capsule segment; capsule against capsule). */
enum bsim_pair_kind { BSIM_PAIR_SS = 0, BSIM_PAIR_PB = 1, BSIM_PAIR_PC = 2, BSIM_PAIR_CC = 3 };

/* All per-env state, parameters, controls and tensor-API outputs
   (reference parallel.py:24-42 `_SHARED` working set).  DEVICE pointers. */
#define BSIM_STATE_FIELDS(REAL)                                                      \
    REAL *body_q;            /* [E*B][13] env-local pos3 quat4 linvel3 angvel3     */ \
    REAL *friction_anchor;   /* [P][E][3] env-local, NaN = none                    */ \
    uint8_t *nonfinite;      /* [E] sticky poison flags                            */ \
    const REAL *env_origins; /* [E][3]                                             */ \
    REAL *inv_mass;          /* [E*B]      (domain randomization writes these)     */ \
    REAL *inertia_local;     /* [E*B][3]                                           */ \
    REAL *inv_inertia_local; /* [E*B][3]                                           */ \
    REAL *gravity;           /* [E][3]                                             */ \
    REAL *mu_static, *mu_dynamic;              /* [E]                               */ \
    REAL *joint_stiffness, *joint_damping, *joint_armature, *joint_friction,          \
         *joint_limit_lo, *joint_limit_hi;     /* [J][E]                            */ \
    REAL *plane_off;         /* [P][E][3]                                          */ \
    REAL *plane_rad;         /* [P][E]                                             */ \
    REAL *pair_off;          /* [Q][E][2][3]                                       */ \
    REAL *pair_rad;          /* [Q][E][2]                                          */ \
    REAL *ctrl_dof_force, *ctrl_dof_pos_target, *ctrl_dof_vel_target; /* [E*D]      */ \
    REAL *ctrl_body_force, *ctrl_body_torque;                         /* [E*B][3]   */ \
    int8_t *dof_mode;                                                  /* [E*D]      */ \
    REAL *root_state;        /* [E*A][13] world frame                              */ \
    REAL *body_state;        /* [E*B][13] world frame                              */ \
    REAL *dof_state;         /* [E*D][2]                                           */ \
    REAL *net_contact;       /* [E*B][3]                                           */ \
    REAL *dof_force;         /* [E*D]                                              */ \
    REAL *sensor_forces;     /* [E*S][6]                                           */
typedef struct bsim_state_t { BSIM_STATE_FIELDS(float) } bsim_state_t;
typedef struct bsim_state64_t { BSIM_STATE_FIELDS(double) } bsim_state64_t;

/* Optional fused action mapping applied before the first substep:
   target = scale * clip(actions, -1, 1) written to ctrl_dof_pos_target
   (mode 1) or ctrl_dof_force (mode 0) -- reference envs.py:180, 421-424.
   Arrays have the entry point's precision. */
typedef struct bsim_actions_t {
    const void *actions;      /* [E][D] device, or NULL */
    void *actions_clipped;    /* [E][D] device copy of the clipped actions, or NULL */
    double scale;
    int32_t mode, pad;
} bsim_actions_t;

int bsim_abi_version(void);
const char *bsim_last_error(void);
/* Bytes of dynamic shared memory one env needs in the step kernel, and the
   envs per CTA the launcher picks; returns BSIM_E_TOO_LARGE if it cannot fit. */
int bsim_step_smem_per_env(const bsim_layout_t *layout, int32_t fp64, int32_t *bytes_per_env,
                           int32_t *envs_per_cta);

/* Scene.step() x n_substeps (physics.py:538-592; envs.py:186-187 decimation),
   fused in one launch.  actions may be NULL. */
int bsim_step(const bsim_layout_t *layout, const bsim_params_t *params, const bsim_state_t *state,
              int32_t n_substeps, const bsim_actions_t *actions, void *stream);

/* Scene.forward_kinematics(env_mask, actors) (physics.py:366-425) followed by
   the body/root repack of the touched rows (buffers.py:109-123).
   env_mask: [E] uint8 device or NULL (= all); actor_mask: bit a = actor a. */
int bsim_forward_kinematics(const bsim_layout_t *layout, const bsim_state_t *state,
                            const uint8_t *env_mask, uint32_t actor_mask, void *stream);

/* Scene.refresh_buffers() without a solver context (physics.py:1037-1046):
   dof readout + body/root packing for every env. */
int bsim_refresh_buffers(const bsim_layout_t *layout, const bsim_state_t *state, void *stream);

/* SimBuffers.set_root_state(values, indices) (buffers.py:127-152).
   values: [E*A][13] world frame device array (only rows at `actor_idx` are
   read); actor_idx: [n] int64 device, unique.  Validation (finite values,
   |quat| >= 0.5, index range) is the caller's (the Python facade raises the
   reference's BufferApiError family first).  The kernels renormalise quats,
   write the root bodies, then run FK over (touched envs) x (touched actors)
   and repack those rows, exactly the reference's cross product.
   env_mask_scratch: [E] uint8 device; actor_mask_scratch: [1] uint32 device. */
int bsim_set_root_state_indexed(const bsim_layout_t *layout, const bsim_state_t *state,
                                const float *values, const int64_t *actor_idx, int32_t n,
                                uint8_t *env_mask_scratch, uint32_t *actor_mask_scratch,
                                void *stream);

/* SimBuffers.set_dof_state(values, indices) (buffers.py:154-178); values
   [E*D][2].  Same scratch contract as above. */
int bsim_set_dof_state_indexed(const bsim_layout_t *layout, const bsim_state_t *state,
                               const float *values, const int64_t *actor_idx, int32_t n,
                               uint8_t *env_mask_scratch, uint32_t *actor_mask_scratch,
                               void *stream);

/* Scene._contact_geometry() (physics.py:463-498) for every (slot, env),
   planes then pairs, env-minor: active [(P+Q)*E] uint8, depth, point [..][3],
   normal [..][3] (world frame points).  Together with a prefix sum this
   yields the collide() list order (physics.py:500-517). */
int bsim_contact_geometry(const bsim_layout_t *layout, const bsim_params_t *params,
                          const bsim_state_t *state, uint8_t *active, float *depth,
                          float *point, float *normal, void *stream);

/* Compacted contact list in collide() order (slot-major, env-ascending,
   planes then pairs): warp-aggregated compaction.  Writes count[0] and up to
   `capacity` entries of body_a (-1 ground), body_b, depth, point, normal.
   scratch: [ceil((P+Q)*E/256)] int32 device. */
int bsim_collide(const bsim_layout_t *layout, const bsim_params_t *params,
                 const bsim_state_t *state, int32_t capacity, int32_t *count,
                 int32_t *body_a, int32_t *body_b, float *depth, float *point, float *normal,
                 int32_t *scratch, void *stream);

/* ------------------------------------------------------------------------
   Fused task layer (reference envs.py:145-200, 359-565; rewards.py:78-158):
   after the physics launch, one thread per env computes reward / done /
   timeout / poison handling, the observation, and -- for finished envs --
   the reset (numpy-identical PCG64 draws keyed (seed, global env, count)),
   forward kinematics of the new state and the post-reset observation.
   ------------------------------------------------------------------------ */
/* QUADRUPED: Ant analog (envs.py:359-478); ANYMAL: envs.py:484-565;
   HUMANOID: the same locomotion task (obs layout, locomotion_reward, reset
   law) on the authored 21-DOF humanoid with its own termination height.
   CUBE: in-hand cube reorientation (BASELINE.json config "Shadow Hand"; the
   reference has the reward, rewards.py:161-176, but no env): a fixed-base
   hand (actor 0) and a single-body cube (actor 1, the env's last body);
   obs = [2(q-lo)/(hi-lo)-1 (D), 0.2 qd (D), cube pos 3, quat 4, linvel 3,
   0.2 angvel 3, goal pos 3, goal quat 4, cube quat (x) conj(goal quat) 4,
   actions (A)]; reward = cube_reorientation_reward with the reference's
   CubeRewardParams defaults; done = cube farther than fall_dist from the
   goal | timeout | poisoned; a success draws a new goal orientation.
   STACK: Franka cube stacking (BASELINE.json config "Franka cube-stack"; the
   reference has franka_stack_reward, rewards.py:200-219, but no env): the
   arm (actor 0; its last five bodies are hand, left finger, right finger)
   then cube A and cube B (single-body actors, the env's last two bodies);
   obs = [2(q-lo)/(hi-lo)-1 (D), 0.1 qd (D), hand pos 3, hand quat 4, A pos 3,
   A quat 4, A - hand 3, B pos 3, B quat 4, A - B 3, actions (A)]; reward =
   franka_stack_reward with the reference's FrankaStackParams defaults;
   done = stacked | timeout | poisoned. */
enum bsim_task_kind { BSIM_TASK_QUADRUPED = 1, BSIM_TASK_ANYMAL = 2, BSIM_TASK_HUMANOID = 3, BSIM_TASK_CUBE = 4,
                      BSIM_TASK_STACK = 5 };

/* Domain randomisation (reference randomize.py:86-189).  Targets in the
   reference's order: 0 dims, 1 masses, 2 friction, 3 damping, 4 gains,
   5 joint_limits, 6 gravity.  dist: 0 uniform, 1 loguniform, 2 gaussian;
   mode: 0 scaling, 1 additive.  Draws use numpy-identical PCG64 streams keyed
   (seed, global env, epoch) and numpy's normal ziggurat. */
typedef struct bsim_dr_t {
    int32_t enabled;
    uint32_t seed;
    int32_t min_interval, pad;
    int32_t use[7], dist[7], mode[7], pad2;
    double a[7], b[7];
    int32_t *epoch, *last_step;     /* [E] */
    /* base snapshots (same shapes / precision as the state arrays) */
    const void *inv_mass, *inertia_local, *inv_inertia_local, *gravity, *mu_static, *mu_dynamic,
               *joint_stiffness, *joint_damping, *joint_limit_lo, *joint_limit_hi,
               *plane_rad, *plane_off, *pair_rad, *pair_off;
} bsim_dr_t;

typedef struct bsim_task_t {
    int32_t kind, obs_dim, act_dim, episode_length;
    uint32_t seed;
    int32_t obs_noise;          /* 1: correlated + uncorrelated observation noise on */
    double control_dt, rest_height;
    double obs_noise_uncorr, obs_noise_corr;
    int64_t step_count;         /* scene.step_count, for the DR interval (envs.py:155) */
    /* device buffers; real arrays have the entry point's precision */
    void *obs;                  /* [E][obs_dim]                                  */
    void *reward;               /* [E]                                           */
    uint8_t *done, *timeout, *poisoned;   /* [E] info flags of the last step      */
    int32_t *episode_steps, *reset_count; /* [E]                                  */
    void *actions;              /* [E][act_dim] clipped actions (zeroed by reset) */
    double *potentials;         /* [E] locomotion progress potential, float64 in both precisions:
                                   -dist/control_dt ~ -6e4 has an fp32 ulp of 4e-3, above the
                                   reward tolerance (envs.py:383-391, rewards.py:89-91) */
    void *commands;             /* [E][3] anymal velocity commands                */
    const void *dof_lower, *dof_upper;    /* [D] static joint limits              */
    void *corr_noise;           /* [E][obs_dim] per-episode correlated noise      */
    int32_t *noise_count;       /* [E] uncorrelated-noise stream counter          */
    bsim_dr_t dr;
    double termination_height;  /* locomotion tasks: done when torso z <= this (rewards.py:25) */
    const int64_t *step_count_dev;  /* optional device copy of step_count (CUDA-graph replay);
                                       NULL: use step_count */
    void *goals;                /* CUBE: [E][8] goal pos xyz (the cube's spawn point, set by the
                                   caller), goal quat xyzw, consecutive successes;
                                   STACK: [E][8] spawn points of cube A and cube B (set by the
                                   caller; resets add U(+-0.05) in x and y); NULL otherwise */
} bsim_task_t;

/* DomainRandomizer.randomize(env_indices, step) on its own (randomize.py:116-134). */
int bsim_randomize(const bsim_layout_t *layout, const bsim_state_t *state, const bsim_dr_t *dr,
                   const uint8_t *env_mask, int64_t step, void *stream);
int bsim_randomize_f64(const bsim_layout_t *layout, const bsim_state64_t *state, const bsim_dr_t *dr,
                       const uint8_t *env_mask, int64_t step, void *stream);

/* RandomForceState / random_object_force (randomize.py:192-221) on the
   device.  Per env: a firing probability p ~ logU[p_lo, p_hi] drawn per
   randomisation episode (bsim_force_resample, which also zeroes the force),
   and per call a fire test u < p: on a hit the force is resampled from
   N(0, mass^2) per axis, otherwise it decays by 0.99^(dt / 0.05).  The
   reference draws from one batch-wide stream; here each env has its own
   numpy-PCG64 stream keyed (seed, global env, counter) -- same law,
   independent of the env partition. */
typedef struct bsim_force_t {
    int32_t num_envs, env_offset;
    uint32_t seed;
    int32_t fp64;               /* real arrays are double when 1, float when 0 */
    double p_lo, p_hi;
    void *probability;          /* [E]    firing probability                    */
    void *force;                /* [E][3] current force                         */
    int32_t *epoch;             /* [E]    probability-draw counter               */
    int32_t *count;             /* [E]    per-call draw counter                  */
} bsim_force_t;

/* RandomForceState.__init__ / resample_probability(env_indices)
   (randomize.py:200-212): masked envs (NULL = all). */
int bsim_force_resample(const bsim_force_t *force, const uint8_t *env_mask, void *stream);
/* random_object_force(state, mass, dt) (randomize.py:215-221).  mass: [E]
   real.  body_force (nullable): the scene's ctrl_body_force [E*B][3]; when
   given, row e*bodies_per_env + body receives the new force (the object the
   disturbance acts on). */
int bsim_random_object_force(const bsim_force_t *force, const void *mass, double dt, void *body_force,
                             int32_t bodies_per_env, int32_t body, void *stream);

/* error text of the last failed task / randomisation call */
const char *bsim_task_last_error(void);

/* EnvBatch.step() tail (envs.py:188-199): call after bsim_step(). */
int bsim_task_step(const bsim_layout_t *layout, const bsim_state_t *state, const bsim_task_t *task,
                   void *stream);
/* EnvBatch.step() in ONE launch (envs.py:178-200): the fused physics step
   (bsim_step) followed, inside the same kernel, by the task tail of
   bsim_task_step for the CTA's envs -- reward / done / obs / auto-reset read
   the state the CTA just wrote, so the task layer costs no extra launch and no
   state re-read from HBM.  task->step_count must be the post-step count. */
int bsim_env_step(const bsim_layout_t *layout, const bsim_params_t *params, const bsim_state_t *state,
                  int32_t n_substeps, const bsim_actions_t *actions, const bsim_task_t *task, void *stream);
int bsim_env_step_f64(const bsim_layout_t *layout, const bsim_params64_t *params,
                      const bsim_state64_t *state, int32_t n_substeps, const bsim_actions_t *actions,
                      const bsim_task_t *task, void *stream);
/* EnvBatch.reset(idx) (envs.py:145-176): reset the masked envs (NULL = all)
   and write the observation of every env. */
int bsim_task_reset(const bsim_layout_t *layout, const bsim_state_t *state, const bsim_task_t *task,
                    const uint8_t *env_mask, void *stream);
int bsim_task_step_f64(const bsim_layout_t *layout, const bsim_state64_t *state, const bsim_task_t *task,
                       void *stream);
int bsim_task_reset_f64(const bsim_layout_t *layout, const bsim_state64_t *state, const bsim_task_t *task,
                        const uint8_t *env_mask, void *stream);

/* Env-range forms for the pipelined host-buffer step (EnvBatch.step with
   host arrays, envs.py:178-200 called with numpy actions): the same launches
   restricted to envs [env_begin, env_begin + env_count) of the scene, so a
   wave-sized chunk's device->host copy overlaps the next chunk's step.
   Every per-env result equals the whole-batch launch's (envs are independent). */
int bsim_step_range(const bsim_layout_t *layout, const bsim_params_t *params, const bsim_state_t *state,
                    int32_t n_substeps, const bsim_actions_t *actions, int32_t env_begin, int32_t env_count,
                    void *stream);
int bsim_step_range_f64(const bsim_layout_t *layout, const bsim_params64_t *params, const bsim_state64_t *state,
                        int32_t n_substeps, const bsim_actions_t *actions, int32_t env_begin, int32_t env_count,
                        void *stream);
int bsim_env_step_range(const bsim_layout_t *layout, const bsim_params_t *params, const bsim_state_t *state,
                        int32_t n_substeps, const bsim_actions_t *actions, const bsim_task_t *task,
                        int32_t env_begin, int32_t env_count, void *stream);
int bsim_env_step_range_f64(const bsim_layout_t *layout, const bsim_params64_t *params,
                            const bsim_state64_t *state, int32_t n_substeps, const bsim_actions_t *actions,
                            const bsim_task_t *task, int32_t env_begin, int32_t env_count, void *stream);
int bsim_task_step_range(const bsim_layout_t *layout, const bsim_state_t *state, const bsim_task_t *task,
                         int32_t env_begin, int32_t env_count, void *stream);
int bsim_task_step_range_f64(const bsim_layout_t *layout, const bsim_state64_t *state, const bsim_task_t *task,
                             int32_t env_begin, int32_t env_count, void *stream);
/* Host buffers of one pipelined host-buffer control step (EnvBatch.step with
   numpy arrays, envs.py:178-200).  Host arrays should be page-locked (pinned)
   for the copies to be asynchronous. */
typedef struct bsim_host_io_t {
    const void *actions;        /* [E][act_dim] host, the entry point's precision */
    void *obs, *reward;         /* [E][obs_dim], [E] host                          */
    uint8_t *done, *timeout, *poisoned;   /* [E] host                             */
    int32_t n_chunks;           /* env chunks; <= 0: one per step-kernel wave     */
    int32_t fused;              /* 1: one bsim_env_step_range launch per chunk;
                                   0: bsim_step_range + bsim_task_step_range;
                                   2: zero-copy -- ONE bsim_env_step launch that reads
                                   the actions from and writes obs / reward / done /
                                   timeout / poisoned straight to the (page-locked,
                                   device-mapped) host buffers; n_chunks unused, the
                                   device obs / reward / flag buffers are not written */
} bsim_host_io_t;
/* One control step from and to host memory, pipelined in ONE call: the envs
   are split into n_chunks ranges; every chunk's actions go host->device on a
   copy stream, chunk c steps (physics + task tail) on its own stream once its
   actions landed, and its obs / reward / done / timeout / poisoned go
   device->host on the copy stream while chunk c+1 is still stepping.  The
   work is ordered after everything already queued on `stream`, and `stream`
   waits for all of it, so synchronising `stream` makes the host buffers valid.
   actions->actions is the DEVICE staging array the uploaded actions land in
   ([E][act_dim]); scale / mode / actions_clipped as for bsim_step.
   task->step_count must be the post-step count (as for bsim_env_step). */
int bsim_env_step_host(const bsim_layout_t *layout, const bsim_params_t *params, const bsim_state_t *state,
                       int32_t n_substeps, const bsim_actions_t *actions, const bsim_task_t *task,
                       const bsim_host_io_t *io, void *stream);
/* error text of the last failed bsim_env_step_host call */
const char *bsim_host_last_error(void);
int bsim_env_step_host_f64(const bsim_layout_t *layout, const bsim_params64_t *params,
                           const bsim_state64_t *state, int32_t n_substeps, const bsim_actions_t *actions,
                           const bsim_task_t *task, const bsim_host_io_t *io, void *stream);
/* The pipelined host step captured once as a CUDA graph (one launch per
   control step).  task->step_count_dev must point at a device int64 the
   graph fills from *count_host (a pinned host slot) before the step, so the
   DR interval keeps advancing; the graph bakes every other pointer and the
   params, so rebuild it if any of them change.  Launch: re-points the action
   uploads at `host_actions` (same size and layout as io->actions), writes
   step_count (the post-step count) to *count_host, and launches on `stream`;
   the previous launch must have completed. */
typedef struct bsim_host_graph bsim_host_graph_t;
int bsim_env_step_host_graph(const bsim_layout_t *layout, const bsim_params_t *params, const bsim_state_t *state,
                             int32_t n_substeps, const bsim_actions_t *actions, const bsim_task_t *task,
                             const bsim_host_io_t *io, int64_t *count_host, bsim_host_graph_t **graph);
int bsim_env_step_host_graph_f64(const bsim_layout_t *layout, const bsim_params64_t *params,
                                 const bsim_state64_t *state, int32_t n_substeps, const bsim_actions_t *actions,
                                 const bsim_task_t *task, const bsim_host_io_t *io, int64_t *count_host,
                                 bsim_host_graph_t **graph);
int bsim_host_graph_launch(bsim_host_graph_t *graph, const void *host_actions, int64_t step_count, void *stream);
void bsim_host_graph_destroy(bsim_host_graph_t *graph);
/* Envs one full wave of the step kernel keeps resident on the current device
   (SMs x CTAs/SM x envs/CTA) -- the chunk size of the pipelined step. */
int bsim_step_envs_per_wave(const bsim_layout_t *layout, int32_t fp64, int32_t *envs);

/* ------------------------------------------------------------------------
   Batched reward kernels (reference rewards.py:78-219), one thread per env.
   Arrays are float (fp64 = 0) or double (fp64 = 1) device arrays. */
typedef struct bsim_loco_params_t {
    double heading_weight, alive_bonus, death_penalty, termination_height, upright_threshold,
        upright_weight, action_cost_weight, effort_weight, dof_limit_weight, dt;
} bsim_loco_params_t;
typedef struct bsim_anymal_params_t {
    double w_vel_xy, w_vel_yaw, w_vel_z, w_pitch_roll, w_joint_motion, w_torque, w_action_rate,
        w_collision, w_air_time, dt;
} bsim_anymal_params_t;
typedef struct bsim_cube_params_t {
    double dist_reward_scale, rot_reward_scale, rot_eps, action_penalty_scale, success_tolerance,
        reach_goal_bonus, fall_dist, fall_penalty;
} bsim_cube_params_t;
typedef struct bsim_franka_params_t {
    double w_stack, w_align, w_lift, w_reach, lift_height, align_tolerance, away_distance;
} bsim_franka_params_t;

/* locomotion_reward (rewards.py:78-112): writes reward[n] and the new potential[n] */
int bsim_reward_locomotion(int n, int D, int fp64, const void *torso, const void *target, const void *up,
                           const void *heading, const void *actions, const void *dof_pos,
                           const void *dof_vel, const void *dof_lower, const void *dof_upper,
                           const void *motor_strength, const void *prev_potential,
                           const bsim_loco_params_t *params, void *reward, void *potential, void *stream);
/* anymal_reward (rewards.py:129-158), rough = 1 for the nine-term variant */
int bsim_reward_anymal(int n, int D, int A, int F, int fp64, const void *lin_vel, const void *ang_vel,
                       const void *commands, const void *dof_vel, const void *dof_acc, const void *torques,
                       const void *action_rate, const void *collisions, const void *feet_air_time,
                       const bsim_anymal_params_t *params, int rough, void *reward, void *stream);
/* cube_reorientation_reward (rewards.py:161-176) */
int bsim_reward_cube(int n, int A, int fp64, const void *object_pos, const void *object_quat,
                     const void *target_pos, const void *target_quat, const void *actions,
                     const bsim_cube_params_t *params, void *reward, uint8_t *goal_reset,
                     uint8_t *success, void *stream);
/* franka_stack_reward (rewards.py:200-219) */
int bsim_reward_franka(int n, int fp64, const void *cubeA_pos, const void *cubeB_pos,
                       const void *gripper_pos, const void *lfinger_pos, const void *rfinger_pos,
                       const bsim_franka_params_t *params, void *reward, void *stream);
typedef struct bsim_trifinger_params_t {
    double w_og, w_fo, w_fv, kernel_a, kernel_b, fingertip_term_cutoff;
} bsim_trifinger_params_t;
/* trifinger_reward (rewards.py:179-197): F fingertips per env, positions /
   velocities [n][F][3]; timestep is int64 [n] */
int bsim_reward_trifinger(int n, int F, int fp64, const void *cube_pos, const void *prev_cube_pos,
                          const void *cube_quat, const void *target_pos, const void *target_quat,
                          const void *fingertip_pos, const void *prev_fingertip_pos,
                          const void *fingertip_vel, const int64_t *timestep,
                          const bsim_trifinger_params_t *params, void *reward, void *stream);
/* ingenuity_reward (rewards.py:115-121): S spin-rate components per env */
int bsim_reward_ingenuity(int n, int S, int fp64, const void *pos, const void *target,
                          const void *local_up_z, const void *spin_rate, void *reward, void *stream);
/* amp_imitation_reward (rewards.py:222-225): r = -ln(1 - clip(D, 1e-4, 1 - 1e-4)) elementwise */
int bsim_reward_amp(int n, int fp64, const void *d_score, void *reward, void *stream);

/* float64 variants (same semantics, double tables / params / state). */
int bsim_step_f64(const bsim_layout_t *layout, const bsim_params64_t *params,
                  const bsim_state64_t *state, int32_t n_substeps, const bsim_actions_t *actions,
                  void *stream);
int bsim_forward_kinematics_f64(const bsim_layout_t *layout, const bsim_state64_t *state,
                                const uint8_t *env_mask, uint32_t actor_mask, void *stream);
int bsim_refresh_buffers_f64(const bsim_layout_t *layout, const bsim_state64_t *state, void *stream);
int bsim_set_root_state_indexed_f64(const bsim_layout_t *layout, const bsim_state64_t *state,
                                    const double *values, const int64_t *actor_idx, int32_t n,
                                    uint8_t *env_mask_scratch, uint32_t *actor_mask_scratch,
                                    void *stream);
int bsim_set_dof_state_indexed_f64(const bsim_layout_t *layout, const bsim_state64_t *state,
                                   const double *values, const int64_t *actor_idx, int32_t n,
                                   uint8_t *env_mask_scratch, uint32_t *actor_mask_scratch,
                                   void *stream);
int bsim_contact_geometry_f64(const bsim_layout_t *layout, const bsim_params64_t *params,
                              const bsim_state64_t *state, uint8_t *active, double *depth,
                              double *point, double *normal, void *stream);
int bsim_collide_f64(const bsim_layout_t *layout, const bsim_params64_t *params,
                     const bsim_state64_t *state, int32_t capacity, int32_t *count,
                     int32_t *body_a, int32_t *body_b, double *depth, double *point,
                     double *normal, int32_t *scratch, void *stream);

#ifdef __cplusplus
}
#endif
#endif
