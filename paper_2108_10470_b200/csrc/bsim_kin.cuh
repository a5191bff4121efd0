// bsim_kin.cuh -- forward kinematics, DOF readout and body/root repacking on
// global memory (host+device).  Reset / setter path, not the step's hot loop.
#pragma once

#include "bsim_step.cuh"

namespace bsim {

// --------------------------------------------------------- kinematics
// Scene.forward_kinematics (physics.py:366-425) for one env directly on
// global memory (reset path; not the hot loop).  Positions env-local.
template <class R, class J>
BS_HD void fk_joint(const J &jt_ref, R *__restrict__ bq, const R *__restrict__ dof) {
    const J jt = jt_ref;   // the whole record at once (vector loads), not field by field behind the stores
    R *P = bq + 13 * jt.parent, *Cc = bq + 13 * jt.child;
    Q4<R> qp = Q4<R>{P[3], P[4], P[5], P[6]};
    V3<R> pp = V3<R>{P[0], P[1], P[2]};
    Q4<R> jq = qmul(qp, jq4(jt.origin_quat));
    V3<R> jrel = qrot(qp, jv3(jt.origin_pos));   // joint origin relative to the parent body
    Q4<R> mq = Q4<R>{0, 0, 0, 1};
    V3<R> mp = zero3<R>(), qda = zero3<R>(), qdl = zero3<R>();
    if (jt.kind == BSIM_REVOLUTE) {
        R q = dof[2 * jt.dof], qd = dof[2 * jt.dof + 1];
        R sh = r_sin(R(0.5) * q), ch = r_cos(R(0.5) * q);
        mq = Q4<R>{jt.axis[0] * sh, jt.axis[1] * sh, jt.axis[2] * sh, ch};
        qda = qrot(jq, jv3(jt.axis)) * qd;
    } else if (jt.kind == BSIM_PRISMATIC) {
        R q = dof[2 * jt.dof], qd = dof[2 * jt.dof + 1];
        mp = jv3(jt.axis) * q;
        qdl = qrot(jq, jv3(jt.axis)) * qd;
    } else if (jt.kind == BSIM_SPHERICAL) {
        V3<R> q3 = v3(dof[2 * jt.dof], dof[2 * jt.dof + 2], dof[2 * jt.dof + 4]);
        V3<R> qd3 = v3(dof[2 * jt.dof + 1], dof[2 * jt.dof + 3], dof[2 * jt.dof + 5]);
        mq = qexp(q3);
        qda = qrot(jq, qd3);
    }
    Q4<R> qcf = qmul(jq, mq);
    V3<R> arel = jrel + qrot(jq, mp);                   // anchor relative to the parent body
    Q4<R> qc = qnormalize(qmul(qcf, qconj(jq4(jt.child_quat))));
    V3<R> crel = arel - qrot(qc, jv3(jt.child_pos));    // child body relative to the parent body
    V3<R> pc = pp + crel;
    V3<R> wp = V3<R>{P[10], P[11], P[12]}, vp = V3<R>{P[7], P[8], P[9]};
    V3<R> wc = wp + qda;
    V3<R> vc = vp + cross(wp, arel) + qdl + cross(wc, crel - arel);
    Cc[0] = pc.x; Cc[1] = pc.y; Cc[2] = pc.z;
    Cc[3] = qc.x; Cc[4] = qc.y; Cc[5] = qc.z; Cc[6] = qc.w;
    Cc[7] = vc.x; Cc[8] = vc.y; Cc[9] = vc.z;
    Cc[10] = wc.x; Cc[11] = wc.y; Cc[12] = wc.z;
}

template <class R> BS_HD void fk_env(const Ctx<R> &c, int e, uint32_t amask) {
    const Dims &d = c.d;
    R *bq = c.s.body_q + (size_t)e * d.B * 13;
    const R *dof = c.s.dof_state + 2 * (size_t)e * d.D;
    for (int j = 0; j < d.J; ++j) {
        const auto &jt = c.joints[j];
        if (!((amask >> jt.actor) & 1u)) continue;
        fk_joint(jt, bq, dof);
    }
}

#if defined(__CUDACC__)
// Forward kinematics of all actors of one env by the G lanes of its group,
// on a shared-memory copy of the env's rows (`bq`, 13 B words) and DOF
// state (`dof`): in each round every lane takes the not-yet-placed joints
// (j = lane, lane + G, ...) whose parent body is placed, so the tree is
// walked level by level (the Ant analog's 8 joints in 2 rounds, not 8 in
// sequence).  A child's pose depends only on its parent's final pose, so the
// result equals fk_env's joint-index order.  B <= 64 (the placed-body mask).
template <int G, class R>
__device__ void fk_group(const Ctx<R> &c, R *bq, const R *dof, int sl, unsigned gmask, uint32_t amask = ~0u) {
    const Dims &d = c.d;
    uint64_t placed = d.B >= 64 ? ~0ull : ((1ull << d.B) - 1);
    for (int j = 0; j < d.J; ++j)                 // actor roots, and every link of an actor not in amask
        if ((amask >> c.joints[j].actor) & 1u) placed &= ~(1ull << c.joints[j].child);
    uint32_t mine_done = 0;                       // this lane's joints placed (j = sl + G i -> bit i)
    for (int round = 0; round < d.J; ++round) {
        uint64_t grown = 0;
        int i = 0;
        for (int j = sl; j < d.J; j += G, ++i) {
            const auto &jt = c.joints[j];
            if (!((amask >> jt.actor) & 1u)) continue;
            if (!((mine_done >> i) & 1u) && ((placed >> jt.parent) & 1ull)) {
                fk_joint(jt, bq, dof);
                mine_done |= 1u << i;
                grown |= 1ull << jt.child;
            }
        }
        __syncwarp(gmask);                        // the new rows are visible to the group
        const uint32_t lo = __reduce_or_sync(gmask, (uint32_t)grown), hi = __reduce_or_sync(gmask, (uint32_t)(grown >> 32));
        const uint64_t all = ((uint64_t)hi << 32) | lo;
        if (!all) break;                          // every joint placed (uniform over the group)
        placed |= all;
    }
}
#endif

// repack body_state/root_state rows of the masked actors (buffers.py:109-123)
// The four arrays are distinct allocations (__restrict__): without it every
// load of the element-wise copy had to wait behind the previous element's
// store (may-alias), i.e. one L2 round trip per element of the env's rows --
// the auto-reset's dominant latency.
template <class R> BS_HD void repack_env(const Ctx<R> &c, int e, uint32_t amask) {
    const Dims &d = c.d;
    const R *__restrict__ o = c.s.env_origins + 3 * (size_t)e;
    const R ox = o[0], oy = o[1], oz = o[2];
    for (int a = 0; a < d.A; ++a) {
        if (!((amask >> a) & 1u)) continue;
        int b0 = c.L.actor_body_offset[a], b1 = c.L.actor_body_offset[a + 1];
        const R *__restrict__ src = c.s.body_q + 13 * ((size_t)e * d.B + b0);
        R *__restrict__ dst = c.s.body_state + 13 * ((size_t)e * d.B + b0);
        R *__restrict__ rr = c.s.root_state + 13 * ((size_t)e * d.A + a);
#pragma unroll 3
        for (int b = 0; b < b1 - b0; ++b) {   // a whole 13-word row per batch of independent loads
            R v[13];
#pragma unroll
            for (int k = 0; k < 13; ++k) v[k] = src[13 * b + k];
            v[0] += ox; v[1] += oy; v[2] += oz;
#pragma unroll
            for (int k = 0; k < 13; ++k) dst[13 * b + k] = v[k];
            if (b == 0) {
#pragma unroll
                for (int k = 0; k < 13; ++k) rr[k] = v[k];
            }
        }
    }
}

// dof readout for one env straight from global memory (physics.py:427-459)
template <class R, class J> BS_HD void readout_joint(const Ctx<R> &c, const J &jt, const R *bq, R *dof_env) {
    (void)c;
    if (jt.dof < 0) return;
    {
        const R *P = bq + 13 * jt.parent, *Cc = bq + 13 * jt.child;
        Q4<R> qp = Q4<R>{P[3], P[4], P[5], P[6]}, qc = Q4<R>{Cc[3], Cc[4], Cc[5], Cc[6]};
        Q4<R> jqp = qmul(qp, jq4(jt.origin_quat)), jqc = qmul(qc, jq4(jt.child_quat));
        V3<R> wp = V3<R>{P[10], P[11], P[12]}, wc = V3<R>{Cc[10], Cc[11], Cc[12]};
        R *o = dof_env + 2 * jt.dof;
        if (jt.kind == BSIM_REVOLUTE) {
            Q4<R> qr = qmul(qconj(jqp), jqc);
            V3<R> ax = jv3(jt.axis);
            o[0] = wrap_pi(R(2) * r_atan2(dot(qvec(qr), ax), qr.w));
            o[1] = dot(qrot(jqp, ax), wc - wp);
        } else if (jt.kind == BSIM_PRISMATIC) {
            V3<R> rp = qrot(qp, jv3(jt.origin_pos)), rc = qrot(qc, jv3(jt.child_pos));
            V3<R> sep = (V3<R>{Cc[0], Cc[1], Cc[2]} - V3<R>{P[0], P[1], P[2]}) + (rc - rp);
            V3<R> aw = qrot(jqp, jv3(jt.axis));
            o[0] = dot(aw, sep);
            V3<R> vap = V3<R>{P[7], P[8], P[9]} + cross(wp, rp), vac = V3<R>{Cc[7], Cc[8], Cc[9]} + cross(wc, rc);
            o[1] = dot(aw, vac - vap);
        } else if (jt.kind == BSIM_SPHERICAL) {
            Q4<R> qr = qmul(qconj(jqp), jqc);
            V3<R> rv = qlog(qr), wr = qrot(qconj(jqp), wc - wp);
            o[0] = rv.x; o[1] = wr.x; o[2] = rv.y; o[3] = wr.y; o[4] = rv.z; o[5] = wr.z;
        }
    }
}
template <class R> BS_HD void readout_env(const Ctx<R> &c, int e) {
    const Dims &d = c.d;
    const R *bq = c.s.body_q + (size_t)e * d.B * 13;
    for (int j = 0; j < d.J; ++j) readout_joint(c, c.joints[j], bq, c.s.dof_state + 2 * (size_t)e * d.D);
}

}  // namespace bsim
