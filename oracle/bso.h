/*
 * bso.h -- CPU ORACLE for the batched TGS rigid-body step.  TEST INFRASTRUCTURE ONLY.
 *
 * A float64, one-environment-at-a-time C restatement of the reference
 * `Scene.step()` (/root/reference/pkg/src/batchsim/physics.py:538-592) and
 * of the pieces it calls (forward kinematics 366-425, DOF readout 427-459,
 * contact geometry 463-498, freeze 657-716, refresh 718-756, rows 777-1019,
 * friction anchors 1021-1033, readout 1037-1071, NaN containment 1073-1088,
 * tendons 598-653 + tendons.py:52-188).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the timed CPU baseline.  The product (paper_2108_10470_b200) never links it.
 *
 * Pinned against golden vectors produced by running the reference itself
 * (tests/golden/make_golden.py writes the npz fixtures).
 *
 * State is world-frame float64 in the reference's array layouts.
 */
#ifndef BSO_H
#define BSO_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t kind, parent, child, dof, actor, has_limits;
    double axis[3], origin_pos[3], origin_quat[4], child_pos[3], child_quat[4];
} bso_joint;

typedef struct {
    /* tendon row: kind 0 fixed / 1 spatial; elements [first, first+count) */
    int32_t kind, first, count, has_limits, reaction_body, actor;
    double rest_length, stiffness, damping, limit_lo, limit_hi, limit_stiffness;
} bso_tendon;

typedef struct {
    /* fixed: index = local dof, joint = joint slot, v[0] = coefficient
       spatial: index = local body, v[0..2] = offset, v[3] = weight        */
    int32_t index, parent, joint;
    double v[4];
} bso_telem;

typedef struct {
    double dt;
    int32_t position_iterations, velocity_iterations;
    double max_bias, restitution, bounce_threshold, rest_offset,
           friction_offset_threshold, solver_offset_slop, max_force,
           linear_damping, angular_damping, max_linear_velocity, max_angular_velocity;
} bso_params;

typedef struct {
    int32_t E, A, B, D, J, P, Q, S, T;
    const bso_joint *joints;          /* [J] */
    const int32_t *plane_body;        /* [P] */
    const int32_t *pair_body;         /* [Q][2] */
    const int32_t *pair_kind;         /* [Q] 0 SS (reference), 1 PB, 2 PC, 3 CC (extension) */
    const double *pair_ext;           /* [Q][4] box half extents / capsule half heights */
    const int32_t *sensor_body;       /* [S] */
    const int32_t *actor_body_offset; /* [A] */
    const bso_tendon *tendons;        /* [T] */
    const bso_telem *telems;
    const int32_t *spatial_paths;     /* flattened: per tendon [npaths][len, idx...] see oracle.py */
    const int32_t *spatial_path_off;  /* [T] offset into spatial_paths, -1 if none */
    bso_params params;

    /* canonical state, world frame */
    double *pos, *quat, *linvel, *angvel;        /* [E*B][3|4] */
    double *friction_anchor;                      /* [P][E][3], NaN = none */
    uint8_t *nonfinite;                           /* [E] */
    /* per-body parameters (randomizable) */
    double *inv_mass, *inertia_local, *inv_inertia_local;  /* [E*B], [E*B][3] */
    /* per-env parameters */
    double *gravity, *mu_static, *mu_dynamic;     /* [E][3], [E] */
    double *joint_stiffness, *joint_damping, *joint_armature, *joint_friction,
           *joint_limit_lo, *joint_limit_hi;      /* [J][E] */
    double *plane_off, *plane_rad;                /* [P][E][3], [P][E] */
    double *pair_off, *pair_rad;                  /* [Q][E][2][3], [Q][E][2] */
    /* controls */
    double *ctrl_dof_force, *ctrl_dof_pos_target, *ctrl_dof_vel_target; /* [E*D] */
    double *ctrl_body_force, *ctrl_body_torque;   /* [E*B][3] */
    int8_t *dof_mode;                             /* [E*D] */
    /* outputs */
    double *root_state, *body_state, *dof_state, *net_contact, *dof_force, *sensor_forces;
    /* test instrumentation (NULL = off): per env, the smallest distance of a
       discrete decision of the step from its threshold, min-accumulated over
       calls: [0] joint limit |q - lo|, |q - hi| (relative to max(1, |limit|)); [1] contact activation /
       friction-anchor depth margins; [2] stick / slip |v_t| - 1e-3;
       [3] restitution vn + bounce_threshold */
    double *margin;                                /* [E][4] */
    /* test instrumentation (seed 0 = off): a joint-limit decision with
       |q - limit| <= limit_jitter max(1, |limit|) is taken at q + u
       limit_jitter max(1, |limit|), u uniform in [-1, 1] from a hash of
       (seed, env, joint, call): the reference's own spread when such
       knife-edge decisions are re-decided at random */
    uint64_t limit_jitter_seed;
    double limit_jitter;
} bso_scene;

/* One Scene.step() for every env (OpenMP over envs when threads > 1). */
void bso_step(const bso_scene *s, int threads);
/* Scene.forward_kinematics(env_mask, actors); env_mask may be NULL (= all),
   actor_mask bit a selects actor a. */
void bso_forward_kinematics(const bso_scene *s, const uint8_t *env_mask, uint32_t actor_mask);
/* Scene.read_dof_states() */
void bso_read_dof_states(const bso_scene *s);
/* Scene.refresh_buffers() without a solver context (state packing only). */
void bso_refresh_buffers(const bso_scene *s);
/* Contact candidates evaluated at current poses (physics.py:463-498):
   plane slot-major then pair slot-major, env-minor.  Arrays sized
   (P+Q)*E: active, depth, point[3], normal[3]. */
void bso_contact_geometry(const bso_scene *s, uint8_t *active, double *depth,
                          double *point, double *normal);
int bso_version(void);

#ifdef __cplusplus
}
#endif
#endif
