// bsim_step.cuh -- the batched Temporal-Gauss-Seidel step for a group of
// environments (host+device), templated on the scalar type R (float fast
// path / double exact-parity path).
//
// B200 mapping: one CTA owns NE environments and
// NTH = NE * 8 threads.  Every TGS pass is split in two:
//
//   phase A (lane-parallel over (env, body|joint|contact) items): effective
//     poses, world inverse inertias, joint anchors/errors/axes and every
//     row's velocity-independent constants;
//   phase B (one thread per env): the Gauss-Seidel sweep itself, which only
//     reads/writes body velocities and applies precomputed constants -- the
//     part of the algorithm that is inherently sequential within an env
//     (environments are disjoint islands, reference physics.py:5-9).
//
// All per-env working state lives in shared memory, item-major / env-minor
// with a compile-time odd stride NE + 1 (conflict-free per-thread columns and
// conflict-free cooperative row loads; every field access is a register base
// plus an immediate offset).  The arithmetic follows the reference
// Scene.step (/root/reference/pkg/src/batchsim/physics.py:538-592) row for
// row; each function cites the lines it restates.  Positions are env-local.
#pragma once

#include "bsim_math.cuh"
#include "../../include/batchsim_b200.h"

#if defined(__CUDA_ARCH__)
// the step's barrier: the group's named barrier (g.bar > 0: a sub-CTA env
// group of g.nth threads, bsim_step.cu BSIM_HALVES) or the CTA's
#define BS_SYNC() bsim::bs_bar(g.bar, g.nth)
#else
#define BS_SYNC() ((void)0)
#endif

namespace bsim {

// float / double variants of the C structs
template <class R> struct Abi;
template <> struct Abi<float> {
    using Joint = bsim_joint_t;
    using Tendon = bsim_tendon_t;
    using TElem = bsim_tendon_elem_t;
    using Params = bsim_params_t;
    using State = bsim_state_t;
};
template <> struct Abi<double> {
    using Joint = bsim_joint64_t;
    using Tendon = bsim_tendon64_t;
    using TElem = bsim_tendon_elem64_t;
    using Params = bsim_params64_t;
    using State = bsim_state64_t;
};

// CTA shape of the step kernel: NE environments, NTH threads; the envs'
// workspace records are PAD words apart (make_dims).
template <class R> struct Shape;
#ifndef BSIM_NE32
#define BSIM_NE32 16
#endif
#ifndef BSIM_NTH32
#define BSIM_NTH32 128
#endif
template <> struct Shape<float> {
    static constexpr int NE = BSIM_NE32, NTH = BSIM_NTH32;
};
#ifndef BSIM_NE64
#define BSIM_NE64 8
#endif
#ifndef BSIM_NTH64
#define BSIM_NTH64 64
#endif
template <> struct Shape<double> {
    static constexpr int NE = BSIM_NE64, NTH = BSIM_NTH64;
};

// ---------------------------------------------------------------- items
// Per-env workspace items.  v8 layout: ENV-MAJOR records (one env's items are
// contiguous, envs PAD words apart) with every vector field 16-byte aligned,
// so a 3-vector / quaternion / symmetric 3x3 moves with one or two 128 / 64-bit
// shared-memory accesses (LDS.128 / STS.64) instead of 3-6 scalar ones.  PAD
// is = 4 (mod 8) words for fp32: the 8 lanes of each quarter-warp phase of a
// 128-bit access hit distinct 16-byte bank groups; odd for fp64 (scalar).
// Scalars live in the spare .w slots of the 3-vectors.
//
// per body: pose (+ inverse mass), velocity, TGS deltas, world inverse
// inertia (sym), effective orientation scratch
enum { BP = 0, BM = 3, BQ = 4, BV_ = 8, BW = 12, BDP = 16, BDA = 20, BI = 24, BQE = 32, BODY_ITEMS = 36 };
// per joint: geometry and the row constants of phase A
enum {
    JRP = 0,              // parent anchor arm (.w unused: q0 lives in registers)
    JRC = 4, JMEFF = 7,   // child anchor arm  | axis-row effective mass
    JPE = 8, JDA = 11,    // perr0 after geometry, the linear target -perr0/h after pass constants |
                          // PD impulse = DA - DB * qd  (812-848, implicit discretisation)
    JRE = 12, JDB = 15,   // rerr0 after geometry, the angular target -rerr0/h after pass constants
    JAX = 16, JLF = 19,   // world joint axis | direct-actuation impulse (FORCE mode)
    JKI = 20,             // point-3: K^-1 ; prismatic-perp: T^T K^-1 T            (sym, 6)
    JFRH = 26,            // joint friction bound fr * h (0 = off)
    JLV = 27,             // limit state this pass: 0 none, 1 below lo, 2 above hi
    JG = 28,              // angular rows: T^T (T Isum T^T)^-1 T                   (sym, 6)
    JLB = 34,             // limit bias velocity this pass
    JY1 = 36, JY2 = 40,   // axis rows: I_c x1 / I_p x2 per unit impulse
    JOINT_ITEMS = 44
};
// per plane contact slot (normal z, tangents (0,-1,0) and (1,0,0): every
// jacobian is a permutation of the arm r, so only r is stored)
enum { CR = 0, CACT = 3, CIXN = 4, CMN = 7, CIX1 = 8, CM1 = 11, CIX2 = 12, CM2 = 15, CLN = 16, CLT = 17,
       CTGT = 19, CST1 = 20, CST2 = 21, CD0 = 22, CREST = 23, CTE = 24, PLANE_ITEMS = 28 };
// per pair slot
enum { QR = 0, QD0 = 3, QRA = 4, QREST = 7, QN = 8, QLN = 11, QT1 = 12, QACT = 15, QT2 = 16, QMN = 19,
       QPT = 20, QM1 = 23, QXN = 24, QM2 = 27, QX1 = 28, QTGT = 31, QX2 = 32, QYN = 36, QY1 = 40, QY2 = 44,
       QIXN = 48, QIX1 = 52, QIX2 = 56, QIYN = 60, QIY1 = 64, QIY2 = 68, QLT = 72, PAIR_ITEMS = 76 };
// per dof: impulse accumulator, start-of-step readout
enum { DIMP = 0, DQ0 = 1, DOF_ITEMS = 2 };
// per env
// EBAD / EBAD + 1: the per-env non-finite flag of even / odd substeps (each
// cleared during the following substep, so no barrier-separated clear)
enum { EMUS = 0, EMUD = 1, EGX = 2, EGY = 3, EGZ = 4, EBAD = 5, ENV_ITEMS = 8 };
// per friction anchor (xyz + pad)
enum { ANCHOR_ITEMS = 4 };

// canonical 13-float body row (pos3 quat4 linvel3 angvel3) -> body item
BS_HD int body_item13(int k) { return k < 3 ? BP + k : (k < 7 ? BQ + k - 3 : (k < 10 ? BV_ + k - 7 : BW + k - 10)); }

struct Dims {
    int E, A, B, D, J, P, Q, S, T;
    int o_body, o_joint, o_plane, o_pair, o_anchor, o_dof, o_env, items, pad;
};

BS_HD int round4(int x) { return (x + 3) & ~3; }

// pad_mod8: fp32 -> PAD = 4 (mod 8); fp64 -> PAD odd
BS_HD Dims make_dims(const bsim_layout_t &L, bool fp64 = false) {
    Dims d;
    d.E = L.num_envs; d.A = L.actors_per_env; d.B = L.bodies_per_env; d.D = L.dofs_per_env;
    d.J = L.joints_per_env; d.P = L.planes_per_env; d.Q = L.pairs_per_env;
    d.S = L.sensors_per_env; d.T = L.tendons_per_env;
    d.o_body = 0;
    d.o_joint = d.o_body + BODY_ITEMS * d.B;
    d.o_plane = d.o_joint + JOINT_ITEMS * d.J;
    d.o_pair = d.o_plane + PLANE_ITEMS * d.P;
    d.o_anchor = d.o_pair + PAIR_ITEMS * d.Q;
    d.o_dof = d.o_anchor + ANCHOR_ITEMS * d.P;
    d.o_env = round4(d.o_dof + DOF_ITEMS * d.D);
    d.items = d.o_env + ENV_ITEMS;
    if (fp64) {
        d.pad = d.items | 1;
    } else {
        d.pad = d.items;
        while ((d.pad & 7) != 4) ++d.pad;
    }
    return d;
}

// One env's record of the shared workspace.  Vector accessors use 128 / 64-bit
// shared-memory accesses on the fp32 device path (every vector item offset is
// a multiple of 4 and the record base is 16-byte aligned: PAD = 4 mod 8).
template <class R> struct Ws {
    R *base;
    BS_HD R &at(int i) const { return base[i]; }
    BS_HD V3<R> l3(int i) const { return V3<R>{at(i), at(i + 1), at(i + 2)}; }
    BS_HD void s3(int i, V3<R> v) const { at(i) = v.x; at(i + 1) = v.y; at(i + 2) = v.z; }
    BS_HD Q4<R> l4(int i) const { return Q4<R>{at(i), at(i + 1), at(i + 2), at(i + 3)}; }
    BS_HD void s4(int i, Q4<R> q) const { at(i) = q.x; at(i + 1) = q.y; at(i + 2) = q.z; at(i + 3) = q.w; }
    BS_HD S3<R> lS(int i) const { return S3<R>{at(i), at(i + 1), at(i + 2), at(i + 3), at(i + 4), at(i + 5)}; }
    BS_HD void sS(int i, const S3<R> &m) const {
        at(i) = m.xx; at(i + 1) = m.xy; at(i + 2) = m.xz; at(i + 3) = m.yy; at(i + 4) = m.yz; at(i + 5) = m.zz;
    }
};
#if defined(__CUDA_ARCH__)
template <> struct Ws<float> {
    float *base;
    __device__ __forceinline__ float &at(int i) const { return base[i]; }
    __device__ __forceinline__ V3<float> l3(int i) const {
        float4 v = *reinterpret_cast<const float4 *>(base + i);
        return V3<float>{v.x, v.y, v.z};
    }
    __device__ __forceinline__ void s3(int i, V3<float> v) const {
        *reinterpret_cast<float2 *>(base + i) = make_float2(v.x, v.y);
        base[i + 2] = v.z;
    }
    __device__ __forceinline__ Q4<float> l4(int i) const {
        float4 v = *reinterpret_cast<const float4 *>(base + i);
        return Q4<float>{v.x, v.y, v.z, v.w};
    }
    __device__ __forceinline__ void s4(int i, Q4<float> q) const {
        *reinterpret_cast<float4 *>(base + i) = make_float4(q.x, q.y, q.z, q.w);
    }
    __device__ __forceinline__ S3<float> lS(int i) const {
        float4 a = *reinterpret_cast<const float4 *>(base + i);
        float2 b = *reinterpret_cast<const float2 *>(base + i + 4);
        return S3<float>{a.x, a.y, a.z, a.w, b.x, b.y};
    }
    __device__ __forceinline__ void sS(int i, const S3<float> &m) const {
        *reinterpret_cast<float4 *>(base + i) = make_float4(m.xx, m.xy, m.xz, m.yy);
        *reinterpret_cast<float2 *>(base + i + 4) = make_float2(m.yz, m.zz);
    }
};
#endif

// Arithmetic of the joint geometry (perr / rerr, joint_item) on the fp32
// path.  Default: fp32 with the position error summed by cancel_sum (TwoSum:
// accurate to ulp(perr) instead of ulp(pose)).  Measurement variants
// (profiles/r02_parity_fp32.md): BSIM_GEOM_F64 = orientations /
// rerr in double, BSIM_GEOMP_F64 = positions / perr in double,
// BSIM_RERR_PROJ = revolute rerr projected normal to the axis before rounding,
// BSIM_PERR_TWOSUM=0 = round 1's plain fp32 sums.
#ifndef BSIM_GEOM_F64
#define BSIM_GEOM_F64 0
#endif
#ifndef BSIM_GEOMP_F64
#define BSIM_GEOMP_F64 BSIM_GEOM_F64
#endif
#ifndef BSIM_RERR_PROJ
#define BSIM_RERR_PROJ 0
#endif
#ifndef BSIM_PERR_TWOSUM
#define BSIM_PERR_TWOSUM 1
#endif
// BSIM_EXP_I64 / BSIM_EXP_G64 / BSIM_EXP_K64 (off): world inverse inertias /
// revolute angular blocks / point blocks in double on the fp32 path --
// measurement variants for the Shadow Hand's fp32 error (tools/
// hand_fp32_probe.py: no change), kept so the finding can be re-measured
// contact slots that are inactive this substep (depth <= -slop at the freeze)
// skip their row constants and rows (measurement variant: BSIM_SKIP_INACTIVE=0)
#ifndef BSIM_SEQ_ACT_MASK
#define BSIM_SEQ_ACT_MASK 1   // the sequential sweep's contact rows from an activity mask (Franka +5 %)
#endif
#ifndef BSIM_SCHED_WARPS
#define BSIM_SCHED_WARPS 1   // warps running the row-schedule sweep (bsim_step_large.cu sets its own)
#endif
#ifndef BSIM_SKIP_INACTIVE
#define BSIM_SKIP_INACTIVE 1
#endif
#ifndef BSIM_DRIVE_POINT_OVERLAP   // revolute: the point row's impulse beside the drive row -- measured
#define BSIM_DRIVE_POINT_OVERLAP 0    // 3 % slower (Ant 235 -> 242 us) and looser in fp32: off
#endif
#ifndef BSIM_LIMIT_VOTE   // warp-vote skip of inactive limit rows: measured 0.4-2 % slower, off
#define BSIM_LIMIT_VOTE 0
#endif
template <class R> struct GeomT { using type = R; };
template <class R> struct GeomPT { using type = R; };
#if BSIM_GEOM_F64
template <> struct GeomT<float> { using type = double; };
#endif
#if BSIM_GEOMP_F64
template <> struct GeomPT<float> { using type = double; };
#endif

#if defined(BSIM_EXP_PASS_CLOCKS) && defined(__CUDACC__)
// timing experiment only: thread-0 cycles of each solver pass's phases summed
// over CTAs and passes -- [0] phase A, [1] sweep, [2] tail items, [7] passes
__device__ unsigned long long bsim_pass_clk[8];
#endif
#if defined(BSIM_EXP_PASS_CLOCKS) && defined(__CUDA_ARCH__)
#define BSIM_PASSCLK(i)                                                       \
    do {                                                                      \
        if (g.tid == 0) {                                                     \
            unsigned long long t_ = clock64();                                \
            atomicAdd(&bsim_pass_clk[i], t_ - pass_t0_);                      \
            pass_t0_ = t_;                                                    \
        }                                                                     \
    } while (0)
#else
#define BSIM_PASSCLK(i) \
    do {                \
    } while (0)
#endif

template <class R> struct Ctx {
    using Joint = typename Abi<R>::Joint;
    using Tendon = typename Abi<R>::Tendon;
    using TElem = typename Abi<R>::TElem;
    bsim_layout_t L;
    typename Abi<R>::Params p;
    typename Abi<R>::State s;
    Dims d;
    const Joint *joints;
    BS_HD const Tendon &tendon(int i) const { return reinterpret_cast<const Tendon *>(L.tendons)[i]; }
    BS_HD const TElem *elems() const { return reinterpret_cast<const TElem *>(L.tendon_elems); }
    BS_HD const R *pair_ext() const { return reinterpret_cast<const R *>(L.pair_ext); }
};

BS_HD int ib(const Dims &d, int b, int item) { return d.o_body + b * BODY_ITEMS + item; }
BS_HD int ij(const Dims &d, int j, int item) { return d.o_joint + j * JOINT_ITEMS + item; }
BS_HD int ipl(const Dims &d, int i, int item) { return d.o_plane + i * PLANE_ITEMS + item; }
BS_HD int ipr(const Dims &d, int i, int item) { return d.o_pair + i * PAIR_ITEMS + item; }
BS_HD int idf(const Dims &d, int k, int item) { return d.o_dof + k * DOF_ITEMS + item; }

template <class R> BS_HD V3<R> jv3(const R *a) { return V3<R>{a[0], a[1], a[2]}; }
template <class R> BS_HD Q4<R> jq4(const R *a) { return Q4<R>{a[0], a[1], a[2], a[3]}; }

// CTA-level view: thread `tid` of `nth`, envs [e0, e0 + ne) in the workspace;
// per-env serial work (the sweep) runs on threads [lane0, lane0 + ne).
// A joint table with a byte stride: the device copy in shared memory pads
// each 128 / 224-byte record by 16 bytes so the different joints a warp's
// lanes read fall in different banks.
template <class R> struct JTab {
    const unsigned char *base;
    int stride;
    BS_HD const typename Abi<R>::Joint &operator[](int j) const {
        return *reinterpret_cast<const typename Abi<R>::Joint *>(base + (size_t)j * stride);
    }
};
template <class R> constexpr int jtab_stride_smem() { return (int)sizeof(typename Abi<R>::Joint) + 16; }

template <class R> struct Grp {
    R *ws;
    int e0, ne, tid, nth, lane0, pad;
    JTab<R> jt;   // the joint table: a shared-memory copy on the device
    int bar = 0;  // 0: the CTA barrier; k > 0: named barrier k over the group's nth threads
    BS_HD Ws<R> env(int el) const { return Ws<R>{ws + (size_t)el * pad}; }
};
#if defined(__CUDA_ARCH__)
__device__ __forceinline__ void bs_bar(int id, int n) {
    if (id == 0)
        __syncthreads();
    else
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
#endif

// ====================================================== phase A pieces
template <class R> BS_HD void stage_env(const Ctx<R> &c, const Ws<R> &w, int e) {
    const Dims &d = c.d;
    const auto &s = c.s;
    w.at(d.o_env + EMUS) = s.mu_static[e];
    w.at(d.o_env + EMUD) = s.mu_dynamic[e];
    w.at(d.o_env + EGX) = s.gravity[3 * (size_t)e];
    w.at(d.o_env + EGY) = s.gravity[3 * (size_t)e + 1];
    w.at(d.o_env + EGZ) = s.gravity[3 * (size_t)e + 2];
    w.at(d.o_env + EBAD) = R(0);
    w.at(d.o_env + EBAD + 1) = R(0);
}

// world inverse inertia of body b from orientation item qitem (physics.py:594-596)
// The local inverse inertia diagonal is staged once per launch into spare
// record slots (BI + 6, BI + 7, BW.w; stage_group) -- refreshed every pass,
// it was a per-pass global load.
template <class R> BS_HD void body_inertia(const Ctx<R> &c, const Ws<R> &w, int e, int b, int qitem) {
    (void)e;
    const int bi = ib(c.d, b, BI);
    V3<R> d{w.at(bi + 6), w.at(bi + 7), w.at(ib(c.d, b, BW) + 3)};
#if BSIM_EXP_I64   // experiment: the world inverse inertia in double
    w.sS(bi, cs3<R>(world_inertia(cq4<double>(w.l4(ib(c.d, b, qitem))), cv3<double>(d))));
#else
    w.sS(bi, world_inertia(w.l4(ib(c.d, b, qitem)), d));
#endif
}

// external forces on body b (physics.py:545-552)
template <class R> BS_HD void body_external(const Ctx<R> &c, const Ws<R> &w, int e, int b) {
    const Dims &d = c.d;
    const R dt = c.p.dt, mf = c.p.max_force;
    R im = w.at(ib(d, b, BM));
    const R *f = c.s.ctrl_body_force + 3 * ((size_t)e * d.B + b);
    const R *tq = c.s.ctrl_body_torque + 3 * ((size_t)e * d.B + b);
    V3<R> v = w.l3(ib(d, b, BV_));
    if (im > R(0)) v = v + v3(w.at(d.o_env + EGX), w.at(d.o_env + EGY), w.at(d.o_env + EGZ)) * dt;
    v = v + v3(clampr(f[0], -mf, mf) * dt * im, clampr(f[1], -mf, mf) * dt * im, clampr(f[2], -mf, mf) * dt * im);
    w.s3(ib(d, b, BV_), v);
    V3<R> t = v3(clampr(tq[0], -mf, mf), clampr(tq[1], -mf, mf), clampr(tq[2], -mf, mf));
    w.s3(ib(d, b, BW), w.l3(ib(d, b, BW)) + smul(w.lS(ib(d, b, BI)), t) * dt);
}

// Reduced coordinates of joint j from the pose/velocity in the workspace
// (physics.py:427-459).  Writes q[k], qd[k] for its 1 or 3 DOFs.
// REV = every joint of the scene is revolute (a compile-time property of the
// AOT topology): the joint kind folds to a constant and the other kinds' code
// leaves the binary (smaller kernel, fewer instruction-cache misses).
// IDF = every joint frame has identity orientation (origin / child quats):
// the frame products fold away.
// a joint's topology fields (joint_meta below)
struct JMeta {
    int kind, parent, child, dof, limits;
};

template <class R, bool REV = false, bool IDF = false>
BS_HD int joint_dofs(const Ctx<R> &c, const Ws<R> &w, int j, R *q, R *qd, const JMeta *jm = nullptr,
                     const JTab<R> *jtab = nullptr) {
    const auto &jt = jtab ? (*jtab)[j] : c.joints[j];
    const int kind = REV ? (int)BSIM_REVOLUTE : (jm ? jm->kind : jt.kind);
    const Dims &d = c.d;
    int p = jm ? jm->parent : jt.parent, ch = jm ? jm->child : jt.child;
    Q4<R> qp = w.l4(ib(d, p, BQ)), qc = w.l4(ib(d, ch, BQ));
    Q4<R> jqp = IDF ? qp : qmul(qp, jq4(jt.origin_quat)), jqc = IDF ? qc : qmul(qc, jq4(jt.child_quat));
    V3<R> wp = w.l3(ib(d, p, BW)), wc = w.l3(ib(d, ch, BW));
    if (kind == BSIM_REVOLUTE) {
        Q4<R> qr = qmul(qconj(jqp), jqc);
        V3<R> ax = jv3(jt.axis);
        q[0] = wrap_pi(R(2) * r_atan2(dot(qvec(qr), ax), qr.w));
        qd[0] = dot(qrot(jqp, ax), wc - wp);
        return 1;
    }
    if (kind == BSIM_PRISMATIC) {
        V3<R> rp = qrot(qp, jv3(jt.origin_pos)), rc = qrot(qc, jv3(jt.child_pos));
        V3<R> sep = (w.l3(ib(d, ch, BP)) - w.l3(ib(d, p, BP))) + (rc - rp);
        V3<R> aw = qrot(jqp, jv3(jt.axis));
        q[0] = dot(aw, sep);
        V3<R> vap = w.l3(ib(d, p, BV_)) + cross(wp, rp), vac = w.l3(ib(d, ch, BV_)) + cross(wc, rc);
        qd[0] = dot(aw, vac - vap);
        return 1;
    }
    if (kind == BSIM_SPHERICAL) {
        Q4<R> qr = qmul(qconj(jqp), jqc);
        V3<R> rv = qlog(qr);
        V3<R> wr = qrot(qconj(jqp), wc - wp);
        q[0] = rv.x; q[1] = rv.y; q[2] = rv.z;
        qd[0] = wr.x; qd[1] = wr.y; qd[2] = wr.z;
        return 3;
    }
    return 0;
}

// Joint j's topology fields.  AOT topologies unpack them from the bit-packed
// compile-time tables of bsim_topologies.cuh (a shift and a mask, no memory
// access); the generic kernel reads the joint table (a dependent global load
// the slot's geometry has to wait for).
enum { TF_PARENT = 0, TF_CHILD = 1, TF_DOF1 = 2, TF_KL = 3, TF_PLANE = 4 };
template <class T, int F, int K> BS_HD unsigned long long topo_word() {
    if constexpr (F == TF_PARENT) { constexpr unsigned long long v = T::parent_w[K]; return v; }
    else if constexpr (F == TF_CHILD) { constexpr unsigned long long v = T::child_w[K]; return v; }
    else if constexpr (F == TF_DOF1) { constexpr unsigned long long v = T::dof1_w[K]; return v; }
    else if constexpr (F == TF_KL) { constexpr unsigned long long v = T::kl_w[K]; return v; }
    else { constexpr unsigned long long v = T::plane_body_w[K]; return v; }
}
template <class T, int F> constexpr int topo_words() {
    if constexpr (F == TF_PARENT) return sizeof(T::parent_w) / 8;
    else if constexpr (F == TF_CHILD) return sizeof(T::child_w) / 8;
    else if constexpr (F == TF_DOF1) return sizeof(T::dof1_w) / 8;
    else if constexpr (F == TF_KL) return sizeof(T::kl_w) / 8;
    else return sizeof(T::plane_body_w) / 8;
}
template <class T, int F, int K = 0> BS_HD unsigned long long topo_select(int word) {
    if constexpr (K + 1 >= topo_words<T, F>()) return topo_word<T, F, K>();
    else return word == K ? topo_word<T, F, K>() : topo_select<T, F, K + 1>(word);
}
template <class T, int F> BS_HD int topo_entry(int i) {
    return (int)((topo_select<T, F>(i >> 3) >> ((i & 7) << 3)) & 0xffull);
}
template <class T> constexpr bool topo_packed() {
    if constexpr (T::is_static) return T::packed_meta; else return false;
}
// (more than two words per field measured slower for the 21-joint humanoid:
// the select chain and its registers cost more than the load it replaces)
template <class T, class R> BS_HD JMeta joint_meta(const Ctx<R> &c, int j) {
    if constexpr (topo_packed<T>()) {
        const int kl = topo_entry<T, TF_KL>(j);
        return JMeta{kl & 3, topo_entry<T, TF_PARENT>(j), topo_entry<T, TF_CHILD>(j), topo_entry<T, TF_DOF1>(j) - 1,
                     kl >> 2};
    } else {
        const auto &jt = c.joints[j];
        return JMeta{jt.kind, jt.parent, jt.child, jt.dof, jt.has_limits};
    }
}
template <class T, class R> BS_HD int plane_body_of(const Ctx<R> &c, int i) {
    if constexpr (topo_packed<T>()) return topo_entry<T, TF_PLANE>(i);
    else return c.L.plane_body[i];
}

// Phase A of joint j for one pass, fused: geometry (freeze physics.py:660-680,
// refresh 733-756; `deltas`: the effective pose pos + dpos / BQE), the
// velocity-independent row constants (the algebra of physics.py:777-928 with
// everything that does not involve a velocity hoisted out of the serial
// sweep), and the per-pass constants (targets -perr/h, -rerr/h, the PD
// drive's affine impulse law, limit activation and bias).  Everything stays
// in registers and leaves as eleven whole 16-byte record groups (one STS.128
// each on the fp32 device path).  At freeze the reduced coordinates
// (read_dof_states, physics.py:557) seed q0, the unbiased limit rows' q and
// the DOF impulse accumulators.  Per-env gains / limits / controls are read
// from HBM (L1/L2 resident).
// The joint kinds a compile-time topology contains (bit k = kind k; every
// kind for a run-time layout), and a joint's kind folded onto them: code for
// kinds the scene does not have is then dead (the Franka scene: revolute and
// prismatic only), without a second copy of the rows.
template <class T> constexpr unsigned topo_kinds() {
    if constexpr (T::is_static) {
        unsigned m = 0;
        for (int j = 0; j < T::J; ++j) m |= 1u << T::kind[j];
        return m;
    } else {
        return 0xfu;
    }
}
template <class T> BS_HD int fold_kind(int k) {
    constexpr unsigned m = topo_kinds<T>();
    if constexpr (m == (1u << BSIM_REVOLUTE)) return BSIM_REVOLUTE;
    else if constexpr (m == ((1u << BSIM_REVOLUTE) | (1u << BSIM_PRISMATIC)))
        return k == BSIM_PRISMATIC ? BSIM_PRISMATIC : BSIM_REVOLUTE;
    else return k;
}
template <class R, class T, bool REV = false, bool IDF = false>
BS_HD void joint_item(const Ctx<R> &c, const Ws<R> &w, int e, int j, R h, bool biased, bool freeze, bool deltas,
                      const JTab<R> &jtab) {
    const Dims &d = c.d;
    const auto &jt = jtab[j];
    const JMeta jm = joint_meta<T>(c, j);
    const int kind = REV ? (int)BSIM_REVOLUTE : fold_kind<T>(jm.kind);
    const int p = jm.parent, ch = jm.child, jdof = jm.dof;
    R q0 = R(0);
    // per-env gains / limits / controls: issued first so their L1/L2 latency
    // hides behind the geometry below (they were the kernel's top long-
    // scoreboard stalls when loaded at their use)
    const bool axis = jdof >= 0 && kind != BSIM_SPHERICAL;
    const bool lim = axis && jm.limits;
    int g_mode = 0;
    R g_arm = R(0), g_tau = R(0), g_kp = R(0), g_kd = R(0), g_tgt = R(0), g_vt = R(0), g_fr = R(0);
    R g_lo = R(0), g_hi = R(0);
    if (axis) {
        const size_t pj = (size_t)j * d.E + e, pd = (size_t)e * d.D + jdof;
        if (biased) {
            g_mode = (int)c.s.dof_mode[pd];
            g_arm = c.s.joint_armature[pj];
            g_tau = c.s.ctrl_dof_force[pd];
            g_kp = c.s.joint_stiffness[pj];
            g_kd = c.s.joint_damping[pj];
            g_tgt = c.s.ctrl_dof_pos_target[pd];
            g_vt = c.s.ctrl_dof_vel_target[pd];
            g_fr = c.s.joint_friction[pj];
        }
        if (lim) {
            g_lo = c.s.joint_limit_lo[pj];
            g_hi = c.s.joint_limit_hi[pj];
        }
    }
    if (freeze) {
        R q[3], qd[3];
        int n = joint_dofs<R, REV, IDF>(c, w, j, q, qd, &jm, &jtab);
        for (int kk = 0; kk < n; ++kk) {
            w.at(idf(d, jdof + kk, DQ0)) = q[kk];
            w.at(idf(d, jdof + kk, DIMP)) = R(0);
        }
        if (n == 1) q0 = q[0];
    }
    // ---- geometry.  perr / rerr are small differences of O(1) poses and the
    // biased rows divide them by h, so plain fp32 sums put fresh velocity
    // noise of ulp(pose) / h ~ 1e-4 into every pass: perr is
    // summed error-free (cancel_sum); GeomT / GeomPT select the measurement
    // variants in double
    using Gt = typename GeomT<R>::type;      // orientations, rerr
    using Gp = typename GeomPT<R>::type;     // positions, perr
    Q4<Gt> qp, qc;
    if (!deltas) {
        qp = cq4<Gt>(w.l4(ib(d, p, BQ)));
        qc = cq4<Gt>(w.l4(ib(d, ch, BQ)));
    } else if constexpr (sizeof(Gt) > sizeof(R)) {   // refresh 718-756: normalize(exp(dang) q), recomputed in Gt
        qp = qnormalize_near(qmul(qexp_small(cv3<Gt>(w.l3(ib(d, p, BDA)))), cq4<Gt>(w.l4(ib(d, p, BQ)))));
        qc = qnormalize_near(qmul(qexp_small(cv3<Gt>(w.l3(ib(d, ch, BDA)))), cq4<Gt>(w.l4(ib(d, ch, BQ)))));
    } else {
        qp = cq4<Gt>(w.l4(ib(d, p, BQE)));
        qc = cq4<Gt>(w.l4(ib(d, ch, BQE)));
    }
    Q4<Gt> jqp = IDF ? qp : qmul(qp, cq4<Gt>(jq4(jt.origin_quat))), jqc = IDF ? qc : qmul(qc, cq4<Gt>(jq4(jt.child_quat)));
    V3<Gp> grp = cv3<Gp>(qrot(qp, cv3<Gt>(jv3(jt.origin_pos)))), grc = cv3<Gp>(qrot(qc, cv3<Gt>(jv3(jt.child_pos))));
    // ac - ap with the body-origin difference taken first (env-local), then the deltas'
#if BSIM_PERR_TWOSUM
    V3<Gp> gperr;
    {
        const V3<R> pc = w.l3(ib(d, ch, BP)), pp = w.l3(ib(d, p, BP));
        const V3<R> dc = deltas ? w.l3(ib(d, ch, BDP)) : zero3<R>(), dp = deltas ? w.l3(ib(d, p, BDP)) : zero3<R>();
        const V3<R> rc_ = cv3<R>(grc), rp_ = cv3<R>(grp);
        gperr = V3<Gp>{(Gp)cancel_sum(pc.x, pp.x, rc_.x, rp_.x, dc.x, dp.x),
                       (Gp)cancel_sum(pc.y, pp.y, rc_.y, rp_.y, dc.y, dp.y),
                       (Gp)cancel_sum(pc.z, pp.z, rc_.z, rp_.z, dc.z, dp.z)};
    }
#else
    V3<Gp> sep = cv3<Gp>(w.l3(ib(d, ch, BP))) - cv3<Gp>(w.l3(ib(d, p, BP)));
    if (deltas) sep = sep + (cv3<Gp>(w.l3(ib(d, ch, BDP))) - cv3<Gp>(w.l3(ib(d, p, BDP))));
    const V3<Gp> gperr = sep + (grc - grp);
#endif
    const Q4<Gt> qe = qmul(jqc, qconj(jqp));
    V3<Gt> grerr = qvec(qe) * (Gt(2) * signr(qe.w));
    const V3<Gt> ga = qrot(jqp, cv3<Gt>(jv3(jt.axis)));
#if BSIM_RERR_PROJ
    // revolute: only rerr's components normal to the axis reach the rows
    // (G a = 0), so drop the axial one before rounding to R
    if (kind == BSIM_REVOLUTE) grerr = grerr - ga * dot(ga, grerr);
#endif
    const V3<R> perr = cv3<R>(gperr), rerr = cv3<R>(grerr);
    const V3<R> rp = cv3<R>(grp), rc = cv3<R>(grc);
    V3<R> a = cv3<R>(ga);
    if (!freeze && jdof >= 0) {
        if (kind == BSIM_REVOLUTE) {
            Q4<R> qr = cq4<R>(qmul(qconj(jqp), jqc));
            q0 = wrap_pi(R(2) * r_atan2(dot(qvec(qr), jv3(jt.axis)), qr.w));
        } else if (kind == BSIM_PRISMATIC) {
            q0 = (R)dot(cv3<Gp>(a), gperr);
        }
    }
    // ---- row constants from the current world inverse inertias
    R mp = w.at(ib(d, p, BM)), mc = w.at(ib(d, ch, BM));
    S3<R> Ip = w.lS(ib(d, p, BI)), Ic = w.lS(ib(d, ch, BI));
    V3<R> t1{R(0), R(0), R(0)}, t2{R(0), R(0), R(0)};
    if (kind != BSIM_REVOLUTE) tangents(a, t1, t2);
    S3<R> KI, G{R(0), R(0), R(0), R(0), R(0), R(0)};
    if (kind != BSIM_PRISMATIC) {   // point-3 K^-1 (872-890)
#if BSIM_EXP_K64   // experiment: the point block in double
        double m = (double)mp + (double)mc;
        S3<double> K{m, 0.0, 0.0, m, 0.0, m};
        add_rIr(K, cv3<double>(rp), cs3<double>(Ip));
        add_rIr(K, cv3<double>(rc), cs3<double>(Ic));
        KI = cs3<R>(sinv(K));
#else
        R m = mp + mc;
        S3<R> K{m, R(0), R(0), m, R(0), m};
        add_rIr(K, rp, Ip);
        add_rIr(K, rc, Ic);
        KI = sinv(K);
#endif
    } else {                        // prismatic perpendicular pair (908-928)
        R m = mp + mc;
        V3<R> p1 = cross(rp, t1), p2 = cross(rp, t2), c1 = cross(rc, t1), c2 = cross(rc, t2);
        V3<R> Ip1 = smul(Ip, p1), Ip2 = smul(Ip, p2), Ic1 = smul(Ic, c1), Ic2 = smul(Ic, c2);
        R k00 = dot(t1, t1) * m + dot(p1, Ip1) + dot(c1, Ic1);
        R k01 = dot(t1, t2) * m + dot(p1, Ip2) + dot(c1, Ic2);
        R k11 = dot(t2, t2) * m + dot(p2, Ip2) + dot(c2, Ic2);
        KI = proj2(t1, t2, k00, k01, k11);
    }
    if (kind != BSIM_SPHERICAL) {   // angular block (892-906): G = T^T (T Isum T^T)^-1 T
        S3<R> Isum = sadd(Ip, Ic);
        if (kind == BSIM_REVOLUTE) {
            // T^T (T Isum T^T)^-1 T over the two tangents normal to the axis
            // a: the reference's 2x2 solve.  Round 1 used the algebraically
            // equal projected inverse M^-1 - (M^-1 a)(M^-1 a)^T / (a . M^-1 a),
            // M = Isum, which cancels catastrophically in fp32 when M is
            // near-singular along a (humanoid limbs: 0.11 rad/s per substep
            // on 1-4 of 4096 envs per control step).
            tangents(a, t1, t2);
            V3<R> s1 = smul(Isum, t1), s2 = smul(Isum, t2);
            G = proj2(t1, t2, dot(t1, s1), dot(t1, s2), dot(t2, s2));
        } else {
            G = proj3(t1, t2, a, Isum);
        }
    }
    // axis rows: drive (812-848) and limit (850-870), meff (777-788)
    V3<R> y1 = zero3<R>(), y2 = zero3<R>();
    R meff = R(0), DA = R(0), DB = R(0), LF = R(0), FRH = R(0), LV = R(0), LB = R(0);
    if (axis) {
        R k;
        V3<R> x1, x2;
        if (kind == BSIM_REVOLUTE) {
            x1 = a;
            x2 = a;
            k = dot(a, smul(sadd(Ip, Ic), a));
        } else {
            x1 = cross(rc, a);
            x2 = cross(rp, a);
            k = mp + mc + dot(x2, smul(Ip, x2)) + dot(x1, smul(Ic, x1));
        }
        y1 = smul(Ic, x1);
        y2 = smul(Ip, x2);
        meff = r_rcp(r_max(k, R(1e-12)));
        if (biased) {  // drive: lam = LF + clip(DA - DB qd, +-mf h) [+ friction]
            const int mode = g_mode;
            const R ia = meff + g_arm;
            const R mf = c.p.max_force;
            R tau = clampr(g_tau, -mf, mf);
            R kk = mode == BSIM_MODE_POSITION ? g_kp : R(0);
            R cc = mode == BSIM_MODE_FORCE ? R(0) : g_kd;
            const R iia = r_rcp(ia);
            const R hden = h * r_rcp(R(1) + h * (h * kk + cc) * iia);
            R err = g_tgt - q0;
            DA = (kk * err + cc * g_vt) * hden;
            DB = (kk * h + cc) * hden;
            LF = mode == BSIM_MODE_FORCE ? tau * h * meff * iia : R(0);
            FRH = g_fr > R(0) ? g_fr * h : R(0);
        }
        if (lim) {  // limit: q0 in biased passes, start-of-step q otherwise
            R lo = g_lo, hi = g_hi;
            R q = biased ? q0 : w.at(idf(d, jdof, DQ0));
            if (q < lo) {
                LV = R(1);
                LB = biased ? r_max(lo - q, R(0)) * r_rcp(h) : R(0);
            }
            if (q > hi) {
                LV = R(2);
                LB = biased ? r_max(q - hi, R(0)) * r_rcp(h) : R(0);
            }
        }
    }
    const R nih = -r_rcp(h);
    V3<R> pt = biased ? perr * nih : zero3<R>(), rt = biased ? rerr * nih : zero3<R>();   // 881, 898
    w.s4(ij(d, j, JRP), Q4<R>{rp.x, rp.y, rp.z, R(0)});
    w.s4(ij(d, j, JRC), Q4<R>{rc.x, rc.y, rc.z, meff});
    w.s4(ij(d, j, JPE), Q4<R>{pt.x, pt.y, pt.z, DA});
    w.s4(ij(d, j, JRE), Q4<R>{rt.x, rt.y, rt.z, DB});
    w.s4(ij(d, j, JAX), Q4<R>{a.x, a.y, a.z, LF});
    w.s4(ij(d, j, JKI), Q4<R>{KI.xx, KI.xy, KI.xz, KI.yy});
    w.s4(ij(d, j, JKI) + 4, Q4<R>{KI.yz, KI.zz, FRH, LV});
    w.s4(ij(d, j, JG), Q4<R>{G.xx, G.xy, G.xz, G.yy});
    w.s4(ij(d, j, JG) + 4, Q4<R>{G.yz, G.zz, LB, R(0)});
    w.s4(ij(d, j, JY1), Q4<R>{y1.x, y1.y, y1.z, R(0)});
    w.s4(ij(d, j, JY2), Q4<R>{y2.x, y2.y, y2.z, R(0)});
}

// plane-contact jacobians: xn = r x z, x1 = r x (0,-1,0), x2 = r x (1,0,0)
template <class R> BS_HD V3<R> plane_xn(V3<R> r) { return v3(r.y, -r.x, R(0)); }
template <class R> BS_HD V3<R> plane_x1(V3<R> r) { return v3(r.z, R(0), -r.x); }
template <class R> BS_HD V3<R> plane_x2(V3<R> r) { return v3(R(0), r.z, -r.y); }

// Plane contact slot i at freeze (physics.py:467-479, 683-697).  The
// friction anchor of this slot is consumed here (terr0) and immediately
// replaced by its end-of-step value (physics.py:1021-1033 depends only on
// frozen quantities).
template <class R> BS_HD void plane_freeze(const Ctx<R> &c, const Ws<R> &w, int e, int i, int b = -1) {
    const Dims &d = c.d;
    const auto &p = c.p;
    if (b < 0) b = c.L.plane_body[i];
    const R *off = c.s.plane_off + 3 * ((size_t)i * d.E + e);
    R rad = c.s.plane_rad[(size_t)i * d.E + e];
    V3<R> arm = qrot(w.l4(ib(d, b, BQ)), jv3(off));
    V3<R> pos = w.l3(ib(d, b, BP));
    R gap = (pos.z + arm.z) - rad;
    R depth = p.rest_offset - gap;
    V3<R> r = v3(arm.x, arm.y, arm.z - rad);
    V3<R> point = pos + r;
    const int an = d.o_anchor + ANCHOR_ITEMS * i;
    R ax = w.at(an), ay = w.at(an + 1);
    bool has = !(ax != ax);
    w.at(ipl(d, i, CTE)) = has ? point.x - ax : R(0);
    w.at(ipl(d, i, CTE + 1)) = has ? point.y - ay : R(0);
    bool near_ = depth > -p.friction_offset_threshold;
    if (near_ && !has) w.s3(an, point);
    if (!near_) {
        const R nanv = r_nan(R(0));
        w.s3(an, v3(nanv, nanv, nanv));
    }
    V3<R> v = w.l3(ib(d, b, BV_)) + cross(w.l3(ib(d, b, BW)), r);
    R vn = v.z;
    w.s3(ipl(d, i, CR), r);
    w.at(ipl(d, i, CD0)) = depth;
    w.at(ipl(d, i, CREST)) = vn < -p.bounce_threshold ? -p.restitution * vn : R(0);
    w.at(ipl(d, i, CACT)) = depth > -p.solver_offset_slop ? R(1) : R(0);
    w.at(ipl(d, i, CLN)) = R(0);
    w.at(ipl(d, i, CLT)) = R(0);
    w.at(ipl(d, i, CLT + 1)) = R(0);
}

// Narrow phase of one pair slot (contact normal a->b, surface gap, and the
// arm from body a's origin to the mid-gap contact point).  pab = pos_b - pos_a.
//   SS sphere-sphere: the reference pair (physics.py:481-497), same arithmetic;
//   PB sphere (or capsule end sphere / box corner, radius 0) vs box b;
//   PC sphere vs capsule b (the segment along b's local z, half height ext[1]);
//   CC capsule vs capsule (clamped segment-segment closest points).
// The reference has only SS: PB / PC / CC are this build's extension for the
// box and capsule pair types (parity unpinned -- checked
// against the C oracle's independent implementation and physics properties).
template <class R>
BS_HD void pair_shape_contact(int kind, Q4<R> qa, Q4<R> qb, V3<R> pab, const R *off, const R *rr, const R *ext,
                              V3<R> &n, R &gap, V3<R> &ra) {
    V3<R> arma = qrot(qa, jv3(off));
    if (kind == BSIM_PAIR_SS) {
        V3<R> armb = qrot(qb, jv3(off + 3));
        V3<R> dd = pab + (armb - arma);
        R dist = norm(dd);
        R dn = dist > R(1e-12) ? dist : R(1);
        n = v3(dd.x / dn, dd.y / dn, dd.z / dn);
        gap = dist - (rr[0] + rr[1]);
        ra = arma + n * (rr[0] + R(0.5) * gap);
        return;
    }
    V3<R> cb = pab + qrot(qb, jv3(off + 3));     // centre of b's box / segment, relative to pos_a
    V3<R> ca = arma;                             // sphere centre on a
    R rad = rr[0];
    if (kind == BSIM_PAIR_PB) {
        V3<R> pl = qrot(qconj(qb), ca - cb);      // sphere centre in the box frame
        V3<R> h = v3(ext[0], ext[1], ext[2]);
        V3<R> cl = v3(clampr(pl.x, -h.x, h.x), clampr(pl.y, -h.y, h.y), clampr(pl.z, -h.z, h.z));
        V3<R> dl = pl - cl;
        R dist = norm(dl);
        V3<R> nl;
        if (dist > R(1e-12)) {                    // outside: nearest surface point
            nl = v3(dl.x / dist, dl.y / dist, dl.z / dist);
            gap = dist - rad;
        } else {                                  // inside: nearest face
            R fx = h.x - r_abs(pl.x), fy = h.y - r_abs(pl.y), fz = h.z - r_abs(pl.z);
            R sx = pl.x < R(0) ? R(-1) : R(1), sy = pl.y < R(0) ? R(-1) : R(1), sz = pl.z < R(0) ? R(-1) : R(1);
            if (fx <= fy && fx <= fz) { nl = v3(sx, R(0), R(0)); gap = -fx - rad; }
            else if (fy <= fz) { nl = v3(R(0), sy, R(0)); gap = -fy - rad; }
            else { nl = v3(R(0), R(0), sz); gap = -fz - rad; }
        }
        n = -qrot(qb, nl);                        // from the sphere towards the box
        ra = ca + n * (rad + R(0.5) * gap);
        return;
    }
    V3<R> ub = qrot(qb, v3(R(0), R(0), R(1)));
    const R hb = ext[1];
    if (kind == BSIM_PAIR_CC) {                   // closest points of two clamped segments
        V3<R> ua = qrot(qa, v3(R(0), R(0), R(1)));
        const R ha = ext[0];
        V3<R> d0 = ca - cb;
        R b_ = dot(ua, ub), dA = dot(ua, d0), dB = dot(ub, d0);
        R den = R(1) - b_ * b_;
        R sa = den > R(1e-9) ? clampr((b_ * dB - dA) / den, -ha, ha) : R(0);
        R tb = clampr(dB + b_ * sa, -hb, hb);
        sa = clampr(b_ * tb - dA, -ha, ha);
        ca = ca + ua * sa;
        cb = cb + ub * tb;
    } else {                                      // PC: sphere centre vs segment
        R tb = clampr(dot(ca - cb, ub), -hb, hb);
        cb = cb + ub * tb;
    }
    V3<R> dd = cb - ca;
    R dist = norm(dd);
    R dn = dist > R(1e-12) ? dist : R(1);
    n = v3(dd.x / dn, dd.y / dn, dd.z / dn);
    gap = dist - (rr[0] + rr[1]);
    ra = ca + n * (rad + R(0.5) * gap);
}

// Pair slot i at freeze (physics.py:481-497, 698-712).
template <class R> BS_HD void pair_freeze(const Ctx<R> &c, const Ws<R> &w, int e, int i) {
    const Dims &d = c.d;
    const auto &p = c.p;
    int pa = c.L.pair_body[2 * i], pb = c.L.pair_body[2 * i + 1];
    const R *off = c.s.pair_off + 6 * ((size_t)i * d.E + e);
    const R *rr = c.s.pair_rad + 2 * ((size_t)i * d.E + e);
    V3<R> pa0 = w.l3(ib(d, pa, BP));
    V3<R> n, ra;
    R gap;
    pair_shape_contact(c.L.pair_kind[i], w.l4(ib(d, pa, BQ)), w.l4(ib(d, pb, BQ)), w.l3(ib(d, pb, BP)) - pa0, off,
                       rr, c.pair_ext() + 4 * i, n, gap, ra);
    R depth = p.rest_offset - gap;
    V3<R> r = (pa0 - w.l3(ib(d, pb, BP))) + ra;
    V3<R> va = w.l3(ib(d, pa, BV_)) + cross(w.l3(ib(d, pa, BW)), ra);
    V3<R> vb = w.l3(ib(d, pb, BV_)) + cross(w.l3(ib(d, pb, BW)), r);
    R vn = dot(n, vb - va);
    V3<R> t1, t2;
    tangents(n, t1, t2);
    w.s3(ipr(d, i, QR), r);
    w.s3(ipr(d, i, QRA), ra);
    w.s3(ipr(d, i, QN), n);
    w.s3(ipr(d, i, QT1), t1);
    w.s3(ipr(d, i, QT2), t2);
    w.s3(ipr(d, i, QPT), pa0 + ra);
    w.at(ipr(d, i, QD0)) = depth;
    w.at(ipr(d, i, QREST)) = vn < -p.bounce_threshold ? -p.restitution * vn : R(0);
    w.at(ipr(d, i, QACT)) = depth > -p.solver_offset_slop ? R(1) : R(0);
    w.at(ipr(d, i, QLN)) = R(0);
    w.at(ipr(d, i, QLT)) = R(0);
    w.at(ipr(d, i, QLT + 1)) = R(0);
    w.s3(ipr(d, i, QXN), cross(r, n));
    w.s3(ipr(d, i, QX1), cross(r, t1));
    w.s3(ipr(d, i, QX2), cross(r, t2));
    w.s3(ipr(d, i, QYN), cross(ra, n));
    w.s3(ipr(d, i, QY1), cross(ra, t1));
    w.s3(ipr(d, i, QY2), cross(ra, t2));
}

// contact row constants from the current inertia (physics.py:993-1006)
template <class R> BS_HD void plane_constants(const Ctx<R> &c, const Ws<R> &w, int i, int b = -1) {
    const Dims &d = c.d;
    if (b < 0) b = c.L.plane_body[i];
    R im = w.at(ib(d, b, BM));
    S3<R> I = w.lS(ib(d, b, BI));
    V3<R> r = w.l3(ipl(d, i, CR));
    V3<R> xn = plane_xn(r), x1 = plane_x1(r), x2 = plane_x2(r);
    V3<R> in = smul(I, xn), i1 = smul(I, x1), i2 = smul(I, x2);
    // whole 16-byte groups: [I xn | m_n], [I x1 | m_1], [I x2 | m_2]
    w.s4(ipl(d, i, CIXN), Q4<R>{in.x, in.y, in.z, r_rcp(r_max(im + dot(xn, in), R(1e-12)))});
    w.s4(ipl(d, i, CIX1), Q4<R>{i1.x, i1.y, i1.z, r_rcp(r_max(im + dot(x1, i1), R(1e-12)))});
    w.s4(ipl(d, i, CIX2), Q4<R>{i2.x, i2.y, i2.z, r_rcp(r_max(im + dot(x2, i2), R(1e-12)))});
}
template <class R> BS_HD void pair_constants(const Ctx<R> &c, const Ws<R> &w, int i) {
    const Dims &d = c.d;
    int pa = c.L.pair_body[2 * i], pb = c.L.pair_body[2 * i + 1];
    R ma = w.at(ib(d, pa, BM)), mb = w.at(ib(d, pb, BM));
    S3<R> Ia = w.lS(ib(d, pa, BI)), Ib = w.lS(ib(d, pb, BI));
    V3<R> xs[3] = {w.l3(ipr(d, i, QXN)), w.l3(ipr(d, i, QX1)), w.l3(ipr(d, i, QX2))};
    V3<R> ys[3] = {w.l3(ipr(d, i, QYN)), w.l3(ipr(d, i, QY1)), w.l3(ipr(d, i, QY2))};
    const int IX[3] = {QIXN, QIX1, QIX2}, IY[3] = {QIYN, QIY1, QIY2}, MM[3] = {QMN, QM1, QM2};
    for (int k = 0; k < 3; ++k) {
        V3<R> ix = smul(Ib, xs[k]), iy = smul(Ia, ys[k]);
        w.s3(ipr(d, i, IX[k]), ix);
        w.s3(ipr(d, i, IY[k]), iy);
        w.at(ipr(d, i, MM[k])) = r_rcp(r_max(ma + mb + dot(ys[k], iy) + dot(xs[k], ix), R(1e-12)));
    }
}

// per-pass contact constants: normal target and stiction (942-973; dpos is
// fixed during a pass)
template <class R> BS_HD void plane_pass_constants(const Ctx<R> &c, const Ws<R> &w, int i, bool biased, int b = -1) {
    const Dims &d = c.d;
    if (b < 0) b = c.L.plane_body[i];
    const R idt = r_rcp(c.p.dt);
    R depth = w.at(ipl(d, i, CD0));
    R bias = R(0), st1 = R(0), st2 = R(0);
    if (biased) {
        V3<R> dp = w.l3(ib(d, b, BDP));
        depth = depth + dp.z * R(-1);                       // 942
        bias = c.p.max_bias * r_max(depth, R(0)) * idt;     // 953
        R tex = w.at(ipl(d, i, CTE)) + dp.x, tey = w.at(ipl(d, i, CTE + 1)) + dp.y;
        st1 = (-tey) * idt;                                 // 971-973, t1 = (0,-1,0)
        st2 = tex * idt;                                    //           t2 = (1,0,0)
    }
    const R rest = w.at(ipl(d, i, CREST));
    w.at(ipl(d, i, CTGT)) = r_max(rest, bias);
    w.s4(ipl(d, i, CST1), Q4<R>{st1, st2, w.at(ipl(d, i, CD0)), rest});   // [st1 st2 | d0 rest]
}
template <class R> BS_HD void pair_pass_constants(const Ctx<R> &c, const Ws<R> &w, int i, bool biased) {
    const Dims &d = c.d;
    R depth = w.at(ipr(d, i, QD0));
    R bias = R(0);
    if (biased) {
        int pa = c.L.pair_body[2 * i], pb = c.L.pair_body[2 * i + 1];
        depth = depth + dot(w.l3(ipr(d, i, QN)), w.l3(ib(d, pb, BDP)) - w.l3(ib(d, pa, BDP))) * R(-1);  // 949
        bias = c.p.max_bias * r_max(depth, R(0)) * r_rcp(c.p.dt);
    }
    w.at(ipr(d, i, QTGT)) = r_max(w.at(ipr(d, i, QREST)), bias);
}

// ====================================================== phase B: the sweep
// Rows act on body velocities held in registers (BV); the generic sweep
// loads/stores them around each row, the topology-specialised sweep keeps
// every body of the env in registers for the whole pass.
template <class R> struct BV {
    V3<R> v, w;
    R m;   // inverse mass
};
template <class R> BS_HD BV<R> load_bv(const Dims &d, const Ws<R> &w, int b) {
    return BV<R>{w.l3(ib(d, b, BV_)), w.l3(ib(d, b, BW)), w.at(ib(d, b, BM))};
}
template <class R> BS_HD void store_bv(const Dims &d, const Ws<R> &w, int b, const BV<R> &x) {
    w.s3(ib(d, b, BV_), x.v);
    w.s3(ib(d, b, BW), x.w);
}

// Row operands shared by several rows of one joint, loaded once per joint
// (the axis rows' jacobians, both bodies' world inverse inertias) and the
// joint's DOF impulse accumulator kept in a register across its rows.
template <class R> struct JointOps {
    V3<R> a, y1, y2;   // world axis, I_c x1, I_p x2
    S3<R> Ic, Ip;
    R imp;             // dof_impulse (drive + limit, same addition order)
    // row scalars carried in the .w slots of the joint's record groups
    R lf, meff, da, db, frh, lv, lb;
};

// rate along a 1-DOF joint axis (physics.py:804-810)
template <class R>
BS_HD R axis_rate(const Dims &d, const Ws<R> &w, int j, bool lin, const JointOps<R> &o, const BV<R> &C,
                  const BV<R> &P) {
    if (!lin) return dot(o.a, C.w - P.w);
    return dot(cross(w.l3(ij(d, j, JRC)), o.a), C.w) - dot(cross(w.l3(ij(d, j, JRP)), o.a), P.w) +
           dot(o.a, C.v - P.v);
}
template <class R> BS_HD void axis_apply(bool lin, const JointOps<R> &o, R lam, BV<R> &C, BV<R> &P) {
    C.w = C.w + o.y1 * lam;
    P.w = P.w - o.y2 * lam;
    if (lin) {
        C.v = C.v + o.a * (lam * C.m);
        P.v = P.v - o.a * (lam * P.m);
    }
}

// PD drive / direct actuation / joint friction (physics.py:812-848)
template <class R>
BS_HD R row_drive(const Ctx<R> &c, const Ws<R> &w, int j, bool lin, R h, JointOps<R> &o, BV<R> &C, BV<R> &P) {
    R qd = axis_rate(c.d, w, j, lin, o, C, P);
    const R mfh = c.p.max_force * h;
    R lam = o.lf + clampr(o.da - o.db * qd, -mfh, mfh);
    if (o.frh > R(0)) lam = lam + clampr(-qd * o.meff, -o.frh, o.frh);
    axis_apply(lin, o, lam, C, P);
    o.imp += lam;
    return lam;
}

// one-sided limit (physics.py:850-870)
template <class R>
BS_HD void row_limit(const Ws<R> &w, const Dims &d, int j, bool lin, JointOps<R> &o, BV<R> &C, BV<R> &P) {
    // branch-free (an inactive limit applies lam = 0, which leaves the
    // velocities bit-identical) so the scheduler can overlap independent rows
    R qd = axis_rate(d, w, j, lin, o, C, P);
    R lam = o.lv == R(1) ? r_max(o.meff * (o.lb - qd), R(0)) : -r_max(o.meff * (o.lb + qd), R(0));
    lam = o.lv == R(0) ? R(0) : lam;
    axis_apply(lin, o, lam, C, P);
    o.imp += lam;
}

// point-3 (872-890) or prismatic perpendicular pair (908-928): P = G (tgt - rel)
template <class R>
BS_HD void row_linear(const Dims &d, const Ws<R> &w, int j, const JointOps<R> &o, BV<R> &C, BV<R> &P) {
    V3<R> rc = w.l3(ij(d, j, JRC)), rp = w.l3(ij(d, j, JRP));
    V3<R> rel = (C.v + cross(C.w, rc)) - (P.v + cross(P.w, rp));
    V3<R> imp = smul(w.lS(ij(d, j, JKI)), w.l3(ij(d, j, JPE)) - rel);
    C.v = C.v + imp * C.m;
    C.w = C.w + smul(o.Ic, cross(rc, imp));
    P.v = P.v - imp * P.m;
    P.w = P.w - smul(o.Ip, cross(rp, imp));
}

// angular rows (892-906): L = G (tgt - (w_c - w_p)); w_c += Ic L, w_p -= Ip L
template <class R>
BS_HD void row_angular(const Dims &d, const Ws<R> &w, int j, const JointOps<R> &o, BV<R> &C, BV<R> &P) {
    V3<R> L = smul(w.lS(ij(d, j, JG)), w.l3(ij(d, j, JRE)) - (C.w - P.w));
    C.w = C.w + smul(o.Ic, L);
    P.w = P.w - smul(o.Ip, L);
}

// all rows of joint j in reference order (physics.py:761-773)
template <class R>
BS_HD void joint_rows(const Ctx<R> &c, const Ws<R> &w, int j, int kind, int dof, bool limits, int pb, int cb,
                      R h, bool biased, BV<R> &C, BV<R> &P) {
    const Dims &d = c.d;
    const bool axis = dof >= 0 && kind != BSIM_SPHERICAL;
    const bool lin = kind == BSIM_PRISMATIC;
    JointOps<R> o;
    o.Ic = w.lS(ib(d, cb, BI));
    o.Ip = w.lS(ib(d, pb, BI));
    if (axis) {
        // whole record groups: [axis | LF], [Y1], [Y2], [RC | MEFF], [PE | DA],
        // [RE | DB], [KI4 KI5 FRH LV], [G4 G5 LB -]
        Q4<R> ax = w.l4(ij(d, j, JAX));
        o.a = qvec(ax);
        o.lf = ax.w;
        o.y1 = w.l3(ij(d, j, JY1));
        o.y2 = w.l3(ij(d, j, JY2));
        o.meff = w.l4(ij(d, j, JRC)).w;
        o.da = w.l4(ij(d, j, JPE)).w;
        o.db = w.l4(ij(d, j, JRE)).w;
        Q4<R> k4 = w.l4(ij(d, j, JKI) + 4);
        o.frh = k4.z;
        o.lv = k4.w;
        o.lb = w.l4(ij(d, j, JG) + 4).z;
        o.imp = w.at(idf(d, dof, DIMP));
    }
#if BSIM_DRIVE_POINT_OVERLAP
    if (biased && axis && kind == BSIM_REVOLUTE) {
        // the drive row moves only the angular velocities (w_c += y1 lam,
        // w_p -= y2 lam), so the point row's input after it is
        // rel0 + lam (y1 x rc + y2 x rp) and its impulse
        // K^-1 (pe - rel0) - lam K^-1 (y1 x rc + y2 x rp): both parts are
        // computed from the pre-drive velocities beside the drive row and
        // joined by one FMA, instead of the point row waiting for the drive
        // row's velocity update (the same values in exact arithmetic;
        // DESIGN.md 8)
        const V3<R> rc = w.l3(ij(d, j, JRC)), rp = w.l3(ij(d, j, JRP));
        const S3<R> KI = w.lS(ij(d, j, JKI));
        const V3<R> rel0 = (C.v + cross(C.w, rc)) - (P.v + cross(P.w, rp));
        const V3<R> imp0 = smul(KI, w.l3(ij(d, j, JPE)) - rel0);
        const V3<R> q = smul(KI, cross(o.y1, rc) + cross(o.y2, rp));
        const R lam = row_drive(c, w, j, false, h, o, C, P);
        const V3<R> imp = imp0 - q * lam;
        C.v = C.v + imp * C.m;
        C.w = C.w + smul(o.Ic, cross(rc, imp));
        P.v = P.v - imp * P.m;
        P.w = P.w - smul(o.Ip, cross(rp, imp));
    } else
#endif
    {
        if (biased && axis) row_drive(c, w, j, lin, h, o, C, P);
        if (kind != BSIM_PRISMATIC) row_linear(d, w, j, o, C, P);
    }
    if (kind != BSIM_SPHERICAL) row_angular(d, w, j, o, C, P);
    if (kind == BSIM_PRISMATIC) row_linear(d, w, j, o, C, P);
#if defined(__CUDA_ARCH__) && BSIM_LIMIT_VOTE
    // an inactive limit row applies exactly zero: skip it when no lane of the
    // warp has its limit active (each lane's own outcome is unchanged either
    // way; this only shortens the dependent chain of the common case)
    if (axis && limits && __any_sync(__activemask(), o.lv != R(0))) row_limit(w, d, j, lin, o, C, P);
#else
    if (axis && limits) row_limit(w, d, j, lin, o, C, P);
#endif
    if (axis && (biased || limits)) w.at(idf(d, dof, DIMP)) = o.imp;
}

// plane contact row (930-983) with the plane's fixed normal / tangents
// Branch-free: an inactive slot (CACT = 0) applies zero impulses, leaving
// velocities and accumulators bit-identical, so independent rows overlap.
template <class R> BS_HD void row_plane(const Ctx<R> &c, const Ws<R> &w, int i, BV<R> &X) {
    const Dims &d = c.d;
    // whole record groups: [r | act], [I xn | m_n], [I x1 | m_1], [I x2 | m_2],
    // [lam_n lt0 lt1 | tgt], [st1 st2 | d0 rest]
    const Q4<R> ra = w.l4(ipl(d, i, CR)), gn = w.l4(ipl(d, i, CIXN));
    const bool act = ra.w != R(0);
#if BSIM_SKIP_INACTIVE
    if (!act) return;   // an inactive slot applies no impulse (bitwise the branch-free result)
#endif
    const Q4<R> acc = w.l4(ipl(d, i, CLN)), stc = w.l4(ipl(d, i, CST1));
    V3<R> r = qvec(ra);
    R vn = X.v.z + dot(plane_xn(r), X.w);
    R lam_n = acc.x;
    R dl = gn.w * (acc.w - vn);
    R nl = r_max(lam_n + dl, R(0));
    dl = act ? nl - lam_n : R(0);
    lam_n = lam_n + dl;
    X.v.z = X.v.z + dl * X.m;
    X.w = X.w + qvec(gn) * dl;
    // friction with t1 = (0,-1,0), t2 = (1,0,0)
    R vt1 = -X.v.y + dot(plane_x1(r), X.w);
    R vt2 = X.v.x + dot(plane_x2(r), X.w);
    R mu = r_sqrt(vt1 * vt1 + vt2 * vt2) > R(1e-3) ? w.at(d.o_env + EMUD) : w.at(d.o_env + EMUS);
    vt1 = vt1 + stc.x;
    vt2 = vt2 + stc.y;
    const Q4<R> g1 = w.l4(ipl(d, i, CIX1)), g2 = w.l4(ipl(d, i, CIX2));
    R lt0 = acc.y, lt1 = acc.z;
    R c0 = lt0 + (-g1.w * vt1), c1 = lt1 + (-g2.w * vt2);
    R lim = mu * lam_n;
    R nrm = r_sqrt(c0 * c0 + c1 * c1);   // circular cone clamp
    R sc = nrm > lim ? lim * r_rcp(r_max(nrm, R(1e-12))) : R(1);
    c0 = c0 * sc;
    c1 = c1 * sc;
    R d0 = act ? c0 - lt0 : R(0), d1 = act ? c1 - lt1 : R(0);
    w.s4(ipl(d, i, CLN), Q4<R>{lam_n, lt0 + d0, lt1 + d1, acc.w});
    X.v.x = X.v.x + d1 * X.m;
    X.v.y = X.v.y + (-d0) * X.m;
    X.w = X.w + qvec(g1) * d0 + qvec(g2) * d1;
}

// sphere-sphere pair row (930-983, pair branches); A = body a, X = body b
template <class R> BS_HD void row_pair(const Ctx<R> &c, const Ws<R> &w, int i, BV<R> &A, BV<R> &X) {
    const Dims &d = c.d;
    if (w.at(ipr(d, i, QACT)) == R(0)) return;
    V3<R> n = w.l3(ipr(d, i, QN)), t1 = w.l3(ipr(d, i, QT1)), t2 = w.l3(ipr(d, i, QT2));
    V3<R> xn = w.l3(ipr(d, i, QXN)), yn = w.l3(ipr(d, i, QYN));
    R vn = dot(n, X.v - A.v) + dot(xn, X.w) - dot(yn, A.w);
    R lam_n = w.at(ipr(d, i, QLN));
    R dl = w.at(ipr(d, i, QMN)) * (w.at(ipr(d, i, QTGT)) - vn);
    R nl = r_max(lam_n + dl, R(0));
    dl = nl - lam_n;
    lam_n = lam_n + dl;
    w.at(ipr(d, i, QLN)) = lam_n;
    X.v = X.v + n * (dl * X.m);
    X.w = X.w + w.l3(ipr(d, i, QIXN)) * dl;
    A.v = A.v - n * (dl * A.m);
    A.w = A.w - w.l3(ipr(d, i, QIYN)) * dl;
    V3<R> dv = X.v - A.v;
    R vt1 = dot(t1, dv) + dot(w.l3(ipr(d, i, QX1)), X.w) - dot(w.l3(ipr(d, i, QY1)), A.w);
    R vt2 = dot(t2, dv) + dot(w.l3(ipr(d, i, QX2)), X.w) - dot(w.l3(ipr(d, i, QY2)), A.w);
    R mu = r_sqrt(vt1 * vt1 + vt2 * vt2) > R(1e-3) ? w.at(d.o_env + EMUD) : w.at(d.o_env + EMUS);
    R lt0 = w.at(ipr(d, i, QLT)), lt1 = w.at(ipr(d, i, QLT + 1));
    R c0 = lt0 + (-w.at(ipr(d, i, QM1)) * vt1), c1 = lt1 + (-w.at(ipr(d, i, QM2)) * vt2);
    R lim = mu * lam_n;
    R nrm2 = c0 * c0 + c1 * c1;
    if (nrm2 > lim * lim) {
        R nrm = r_sqrt(nrm2);
        if (nrm > lim) {
            R sc = lim / r_max(nrm, R(1e-12));
            c0 = c0 * sc;
            c1 = c1 * sc;
        }
    }
    R d0 = c0 - lt0, d1 = c1 - lt1;
    w.at(ipr(d, i, QLT)) = lt0 + d0;
    w.at(ipr(d, i, QLT + 1)) = lt1 + d1;
    V3<R> Q = t1 * d0 + t2 * d1;
    X.v = X.v + Q * X.m;
    X.w = X.w + w.l3(ipr(d, i, QIX1)) * d0 + w.l3(ipr(d, i, QIX2)) * d1;
    A.v = A.v - Q * A.m;
    A.w = A.w - (w.l3(ipr(d, i, QIY1)) * d0 + w.l3(ipr(d, i, QIY2)) * d1);
}

// after a biased pass: dpos += v h, dang += w h (physics.py:571-572)
template <class R> BS_HD void accumulate_deltas(const Dims &d, const Ws<R> &w, int b, const BV<R> &x, R h) {
    w.s3(ib(d, b, BDP), w.l3(ib(d, b, BDP)) + x.v * h);
    w.s3(ib(d, b, BDA), w.l3(ib(d, b, BDA)) + x.w * h);
}

// one Gauss-Seidel pass for one env, any topology (physics.py:760-775)
struct TopoGeneric;
template <class T> constexpr bool topo_rev();
template <class T> constexpr bool topo_pairs();
// (T: the compile-time topology, as in sched_row -- an all-revolute one
// compiles the revolute rows only, one without pair slots no pair rows)
template <class R, class T = TopoGeneric> BS_HD void sweep(const Ctx<R> &c, const Ws<R> &w, R h, bool biased) {
    const Dims &d = c.d;
    for (int j = 0; j < d.J; ++j) {
        const auto &jt = c.joints[j];
        BV<R> C = load_bv(d, w, jt.child), P = load_bv(d, w, jt.parent);
        const int kind = fold_kind<T>(jt.kind);
        joint_rows(c, w, j, kind, jt.dof, jt.has_limits != 0, jt.parent, jt.child, h, biased, C, P);
        store_bv(d, w, jt.child, C);
        store_bv(d, w, jt.parent, P);
    }
#if BSIM_SKIP_INACTIVE && BSIM_SEQ_ACT_MASK
    // the contact slots' activity first (independent loads, 64 slots per
    // mask), then only the active rows, in reference order (planes, pairs):
    // Franka cube-stack 865 -> 824 us per 8192-env control step (v34),
    // against testing each slot before its row (a dependent load + branch)
    const int nc = d.P + ((!T::is_static || topo_pairs<T>()) ? d.Q : 0);
    for (int base = 0; base < nc; base += 64) {
        unsigned long long am = 0;
        const int n = nc - base < 64 ? nc - base : 64;
        for (int k = 0; k < n; ++k) {
            const int i = base + k;
            const R a = i < d.P ? w.at(ipl(d, i, CACT)) : w.at(ipr(d, i - d.P, QACT));
            am |= (unsigned long long)(a != R(0)) << k;
        }
        while (am) {
#ifdef __CUDA_ARCH__
            const int k = __ffsll((long long)am) - 1;
#else
            const int k = __builtin_ctzll(am);
#endif
            am &= am - 1;
            const int i = base + k;
            if (i < d.P) {
                int b = c.L.plane_body[i];
                BV<R> X = load_bv(d, w, b);
                row_plane(c, w, i, X);
                store_bv(d, w, b, X);
            } else {
                const int q = i - d.P, pa = c.L.pair_body[2 * q], pb = c.L.pair_body[2 * q + 1];
                BV<R> A = load_bv(d, w, pa), X = load_bv(d, w, pb);
                row_pair(c, w, q, A, X);
                store_bv(d, w, pa, A);
                store_bv(d, w, pb, X);
            }
        }
    }
#else
    for (int i = 0; i < d.P; ++i) {
#if BSIM_SKIP_INACTIVE
        if (w.at(ipl(d, i, CACT)) == R(0)) continue;
#endif
        int b = c.L.plane_body[i];
        BV<R> X = load_bv(d, w, b);
        row_plane(c, w, i, X);
        store_bv(d, w, b, X);
    }
    for (int i = 0; i < ((!T::is_static || topo_pairs<T>()) ? d.Q : 0); ++i) {
#if BSIM_SKIP_INACTIVE
        if (w.at(ipr(d, i, QACT)) == R(0)) continue;
#endif
        int pa = c.L.pair_body[2 * i], pb = c.L.pair_body[2 * i + 1];
        BV<R> A = load_bv(d, w, pa), X = load_bv(d, w, pb);
        row_pair(c, w, i, A, X);
        store_bv(d, w, pa, A);
        store_bv(d, w, pb, X);
    }
#endif
    if (biased)
        for (int b = 0; b < d.B; ++b) accumulate_deltas(d, w, b, load_bv(d, w, b), h);
}

// One pass on the layout's row schedule (SceneLayout.sweep_schedule): stage
// by stage, lane l of the env runs row sched[s][l] on the body velocities in
// shared memory.  Rows of a stage touch disjoint bodies and every row follows
// each earlier row it shares a body with, so the result is the sequential
// sweep's (rows on disjoint bodies commute: same arithmetic, same values).
// `lane` in [0, lanes) indexes the env's threads; the stage loop runs on
// every thread of the CTA (uniform trip count) and __syncwarp(mask) orders a
// stage's shared-memory writes before the next stage's reads.
// contact row r >= J of the schedule: plane slot r - J or pair slot r - J - P
template <class R, class T = TopoGeneric> BS_HD void sched_contact_row(const Ctx<R> &c, const Ws<R> &w, int r) {
    const Dims &d = c.d;
    if (r < d.J + d.P) {
        const int i = r - d.J, b = c.L.plane_body[i];
#if BSIM_SKIP_INACTIVE
        if (w.at(ipl(d, i, CACT)) == R(0)) return;
#endif
        BV<R> X = load_bv(d, w, b);
        row_plane(c, w, i, X);
        store_bv(d, w, b, X);
    } else if (!T::is_static || topo_pairs<T>()) {
        const int i = r - d.J - d.P, pa = c.L.pair_body[2 * i], pb = c.L.pair_body[2 * i + 1];
#if BSIM_SKIP_INACTIVE
        if (w.at(ipr(d, i, QACT)) == R(0)) return;
#endif
        BV<R> A = load_bv(d, w, pa), X = load_bv(d, w, pb);
        row_pair(c, w, i, A, X);
        store_bv(d, w, pa, A);
        store_bv(d, w, pb, X);
    }
}
template <class R, class T = TopoGeneric>
BS_HD void sched_row(const Ctx<R> &c, const Ws<R> &w, int r, R h, bool biased) {
    const Dims &d = c.d;
    if (r < d.J) {
        const auto &jt = c.joints[r];
        BV<R> C = load_bv(d, w, jt.child), P = load_bv(d, w, jt.parent);
        // an all-revolute compile-time topology (the humanoid) compiles the
        // revolute rows only: one copy of the rows, no other kinds' code
        const int kind = fold_kind<T>(jt.kind);
        joint_rows(c, w, r, kind, jt.dof, jt.has_limits != 0, jt.parent, jt.child, h, biased, C, P);
        store_bv(d, w, jt.child, C);
        store_bv(d, w, jt.parent, P);
    } else {
        sched_contact_row<R, T>(c, w, r);
    }
}
#if defined(__CUDA_ARCH__)
template <class R, class T>
__device__ void sweep_sched(const Ctx<R> &c, const Ws<R> *w, R h, bool biased, int lane, int lanes, unsigned mask) {
    const Dims &d = c.d;
    const int S = c.L.sched_stages, W = c.L.sched_width;
    for (int s = 0; s < S; ++s) {
        if (w)
            for (int i = lane; i < W; i += lanes) {   // a stage's rows are independent: any lane may take any
                const int r = __ldg(c.L.sweep_sched + s * W + i);
                if (r >= 0) sched_row<R, T>(c, *w, r, h, biased);
            }
        __syncwarp(mask);
    }
    if (c.L.sched_flags & 1) {   // joint-only schedule: the contact rows in order
        // the env's lanes read the slots' activity side by side (one ballot per
        // `lanes` rows) and lane 0 runs the active rows in reference order,
        // instead of testing every slot one dependent load after another
        // (Shadow Hand 3026 -> 2671 us per 16384-env control step; v33)
        const int nc = d.P + d.Q, wl = (int)(threadIdx.x & 31) - lane;
        const unsigned sel = lanes >= 32 ? 0xffffffffu : ((1u << lanes) - 1u);
        for (int base = 0; base < nc; base += lanes) {
            const int i = base + lane;
            bool act = false;
            if (w && i < nc) act = (i < d.P ? w->at(ipl(d, i, CACT)) : w->at(ipr(d, i - d.P, QACT))) != R(0);
            unsigned bits = (__ballot_sync(mask, act) >> wl) & sel;
            if (w && lane == 0)
                while (bits) {
                    const int b = __ffs(bits) - 1;
                    bits &= bits - 1;
                    sched_contact_row<R, T>(c, *w, d.J + base + b);
                }
        }
        __syncwarp(mask);
    }
    if (biased && w)
        for (int b = lane; b < d.B; b += lanes) accumulate_deltas(d, *w, b, load_bv(d, *w, b), h);
}
#else
template <class R> void sweep_sched_host(const Ctx<R> &c, const Ws<R> &w, R h, bool biased) {
    const Dims &d = c.d;
    const int S = c.L.sched_stages, W = c.L.sched_width;
    for (int s = 0; s < S; ++s)
        for (int l = 0; l < W; ++l) {
            const int r = c.L.sweep_sched[s * W + l];
            if (r >= 0) sched_row(c, w, r, h, biased);
        }
    if (c.L.sched_flags & 1)
        for (int r = d.J; r < d.J + d.P + d.Q; ++r) sched_row(c, w, r, h, biased);
    if (biased)
        for (int b = 0; b < d.B; ++b) accumulate_deltas(d, w, b, load_bv(d, w, b), h);
}
#endif

// The same pass with the topology known at compile time (T = a generated
// bsim_topologies.cuh entry): every body velocity of the env stays in
// registers for the whole pass and rows on disjoint bodies can overlap.
template <class R, class T, bool BIASED, int j>
BS_HD void static_joints(const Ctx<R> &c, const Ws<R> &w, R h, BV<R> *bv) {
    if constexpr (j < T::J) {
        constexpr int kind = T::kind[j], dof = T::dof[j], ch = T::child[j], pa = T::parent[j];
        constexpr bool lim = T::limits[j] != 0;
        joint_rows(c, w, j, kind, dof, lim, pa, ch, h, BIASED, bv[ch], bv[pa]);
        static_joints<R, T, BIASED, j + 1>(c, w, h, bv);
    }
}
template <class R, class T, int i>
BS_HD void static_planes(const Ctx<R> &c, const Ws<R> &w, BV<R> *bv) {
    if constexpr (i < T::P) {
        constexpr int b = T::plane_body[i];
        row_plane(c, w, i, bv[b]);
        static_planes<R, T, i + 1>(c, w, bv);
    }
}
template <class R, class T, int i>
BS_HD void static_pairs(const Ctx<R> &c, const Ws<R> &w, BV<R> *bv) {
    if constexpr (i < T::Q) {
        constexpr int pa = T::pair_a[i], pb = T::pair_b[i];
        row_pair(c, w, i, bv[pa], bv[pb]);
        static_pairs<R, T, i + 1>(c, w, bv);
    }
}
// BIASED is a template parameter so each pass type is one straight-line
// block (no per-joint uniform branch): the scheduler interleaves rows on
// disjoint bodies (e.g. a knee row with the next hip row).
template <class R, class T, bool BIASED> BS_HD void sweep_static(const Ctx<R> &c, const Ws<R> &w, R h) {
    const Dims &d = c.d;
    BV<R> bv[T::B];
#pragma unroll
    for (int b = 0; b < T::B; ++b) bv[b] = load_bv(d, w, b);
    static_joints<R, T, BIASED, 0>(c, w, h, bv);
    static_planes<R, T, 0>(c, w, bv);
    static_pairs<R, T, 0>(c, w, bv);
#pragma unroll
    for (int b = 0; b < T::B; ++b) {
        store_bv(d, w, b, bv[b]);
        if (BIASED) accumulate_deltas(d, w, b, bv[b], h);
    }
}

#if defined(__CUDA_ARCH__)
// Two-lane pipelined sweep for a root with L legs that are 2-joint chains
// (codegen's `star_chain` = 2 trait, the Ant analog: joint 2l = root ->
// hip_l = link 2l+1, joint 2l+1 = hip_l -> knee_l = link 2l+2, all revolute
// with limits, dof = joint index, plane slots on the root then on each knee,
// no pairs).  Each env gets two lanes of the sweep warp: lane 0 runs the root
// chain j_0, j_2, ..., lane 1 the knee rows j_1, j_3, ... one step behind,
// receiving each hip's velocity from lane 0 by a shuffle.  Only rows on
// disjoint bodies run side by side and every row's arithmetic is unchanged,
// so the result is the reference's Gauss-Seidel order (physics.py:761-775):
// j_2s+1 and j_2s+2 share no body, and a plane row may run as soon as its
// body's last joint row is done because no later joint row touches it.
// 8 joint row times become 5; the plane rows and the delta accumulation run
// after a CTA barrier on every lane (star_body_tail).  (The same pipeline for 3-joint
// legs -- the ANYmal analog -- measured slower than the register-resident
// sequential sweep, so codegen only marks 2-joint stars.)
#ifndef BSIM_PLANE_OVERLAP
#define BSIM_PLANE_OVERLAP 1   // plane row constants built beside the chain sweep
#endif
template <class T> BS_HD constexpr int star_lanes() { return T::star_chain <= 2 ? 2 : 4; }
template <class R, class T>
__device__ void sweep_star(const Ctx<R> &c, const Ws<R> &w, R h, bool biased, int p, unsigned mask) {
    const Dims &d = c.d;
    constexpr int K = T::star_chain, G = star_lanes<T>(), L = T::J / K;
    static_assert(K >= 2 && K <= G && T::J % K == 0, "star chains of 2..4 joints");
    BV<R> P = load_bv(d, w, 0), C = P;          // lane 0 keeps the root in P
    for (int s = 0; s < L + K - 1; ++s) {
        // lane p: joint K (s - p) + p, stage p of leg s - p (link j -> link j + 1; the root for p = 0)
        const int leg = s - p;
        const bool active = p < K && leg >= 0 && leg < L;
        const int j = K * leg + p;
        const int cb = j + 1, pb = p == 0 ? 0 : j;
        if (active) {
            C = load_bv(d, w, cb);
            // 2-joint legs (the Ant analog): one copy of the rows with the pass
            // type at run time -- the smaller kernel measured 256 -> 254 us per
            // 16384-env step (bench value +1.1 %); the ANYmal analog's 3-joint
            // chains keep a copy per pass type (one copy: 449 -> 454 us)
            if constexpr (K == 2) {
                joint_rows(c, w, j, BSIM_REVOLUTE, j, true, pb, cb, h, biased, C, P);
            } else {
                if (biased)
                    joint_rows(c, w, j, BSIM_REVOLUTE, j, true, pb, cb, h, true, C, P);
                else
                    joint_rows(c, w, j, BSIM_REVOLUTE, j, true, pb, cb, h, false, C, P);
            }
        }
        // link j is final after its outgoing joint; the leg's last link after its own
        if (active && p >= 1) store_bv(d, w, pb, P);
        if (active && p == K - 1) store_bv(d, w, cb, C);
        // hand link j + 1 (C) to the next stage for joint j + 1
        BV<R> nx;
        nx.v.x = __shfl_up_sync(mask, C.v.x, 1, G);
        nx.v.y = __shfl_up_sync(mask, C.v.y, 1, G);
        nx.v.z = __shfl_up_sync(mask, C.v.z, 1, G);
        nx.w.x = __shfl_up_sync(mask, C.w.x, 1, G);
        nx.w.y = __shfl_up_sync(mask, C.w.y, 1, G);
        nx.w.z = __shfl_up_sync(mask, C.w.z, 1, G);
        nx.m = __shfl_up_sync(mask, C.m, 1, G);
        if (p >= 1) P = nx;
        // memory order between the stages: lane p + 1 stores link j + 1 at the
        // next step, after lane p loaded it at this one (a WAR through shared
        // memory that the shuffle's value dependency orders in practice;
        // __syncwarp makes it an ordering guarantee -- racecheck clean)
        __syncwarp(mask);
    }
    if (p == 0) store_bv(d, w, 0, P);
}

// The rest of the star pass, one item per (env, body) over the whole CTA
// after a barrier: the body's plane row (slot q with plane_body[q] == b; the
// star topologies carry at most one slot per body, so rows on distinct
// bodies commute and the reference's slot order is kept) and, after a
// biased pass, dpos += v h, dang += w h (physics.py:571-572).  One SIMT
// path for every lane, so the 5 plane rows of an env cost one row time
// instead of three on the two sweep lanes.
template <class T> BS_HD constexpr int star_plane_of(int b) {
    for (int q = 0; q < T::P; ++q)
        if (T::plane_body[q] == b) return q;
    return -1;
}
template <class T> BS_HD constexpr bool star_planes_unique() {
    for (int q = 0; q < T::P; ++q)
        for (int r = q + 1; r < T::P; ++r)
            if (T::plane_body[q] == T::plane_body[r]) return false;
    return true;
}
// body -> slot, folded at compile time (the tables are host constexpr arrays:
// device code must not index them at run time)
template <class T, int k = 0> __device__ __forceinline__ int star_plane_index(int b) {
    if constexpr (k < T::B) {
        constexpr int q = star_plane_of<T>(k);
        return b == k ? q : star_plane_index<T, k + 1>(b);
    } else {
        return -1;
    }
}
template <class R> BS_HD void body_phase_item(const Ctx<R> &c, const Ws<R> &w, int e, int b, int k, int N);
template <class R, class T>
__device__ void star_body_tail(const Ctx<R> &c, const Ws<R> &w, int e, int b, R h, int k, int N) {
    static_assert(star_planes_unique<T>(), "star tail assumes one plane slot per body");
    const Dims &d = c.d;
    const bool biased = k < N;
    const int q = star_plane_index<T>(b);
    BV<R> X = load_bv(d, w, b);
    if (q >= 0) {
        row_plane(c, w, q, X);
        store_bv(d, w, b, X);
    }
    if (biased) {
        accumulate_deltas(d, w, b, X, h);
        // pass k + 1's body phase needs only this body's own deltas: its
        // effective pose and world inverse inertia, in the same item
        body_phase_item(c, w, e, b, k + 1, N);
    }
}
#endif

// no compile-time topology: use the generic sweep
struct TopoGeneric {
    static constexpr bool is_static = false;
};
template <class T> constexpr bool topo_register_sweep() {
    if constexpr (T::is_static) return T::register_sweep; else return false;
}
template <class T> constexpr bool topo_star() {
    if constexpr (T::is_static) return T::star_chain > 0; else return false;
}
template <class R, class T> BS_HD void sweep_any(const Ctx<R> &c, const Ws<R> &w, R h, bool biased) {
    if constexpr (topo_register_sweep<T>()) {
        if (biased)
            sweep_static<R, T, true>(c, w, h);
        else
            sweep_static<R, T, false>(c, w, h);
    } else
        sweep<R, T>(c, w, h, biased);
}

// ------------------------------------------------------------ tendons
template <class T, class R> BS_HD R tendon_spring(const T &t, R L, R Ld) {  // tendons.py:52-62
    R f = -t.stiffness * (L - t.rest_length) - t.damping * Ld;
    if (t.has_limits) {
        R below = r_max(t.limit_lo - L, R(0)), above = r_max(L - t.limit_hi, R(0));
        f = f + t.limit_stiffness * below - t.limit_stiffness * above;
        if (below > R(0) || above > R(0)) f = f - t.damping * Ld;
    }
    return f;
}

template <class R> BS_HD void add_w(const Dims &d, const Ws<R> &w, int b, V3<R> dw) {
    w.s3(ib(d, b, BW), w.l3(ib(d, b, BW)) + dw);
}
template <class R> BS_HD void add_v(const Dims &d, const Ws<R> &w, int b, V3<R> dv) {
    w.s3(ib(d, b, BV_), w.l3(ib(d, b, BV_)) + dv);
}

// physics.py:598-653; fixed tendons read the dof_state buffer of the previous
// readout (physics.py:605-606), spatial tendons the current body state.
template <class R> BS_HD void apply_tendons(const Ctx<R> &c, const Ws<R> &w, int e) {
    const Dims &d = c.d;
    const R dt = c.p.dt;
    for (int ti = 0; ti < d.T; ++ti) {
        const auto &t = c.tendon(ti);
        const auto *el = c.elems() + t.first;
        if (t.kind == 0) {
            const int MAXE = 16;
            R len[MAXE], rate[MAXE];
            int n = t.count < MAXE ? t.count : MAXE;
            for (int i = 0; i < n; ++i) {
                const R *dq = c.s.dof_state + 2 * ((size_t)e * d.D + el[i].index);
                R pl = el[i].parent >= 0 ? len[el[i].parent] : R(0);
                R pr = el[i].parent >= 0 ? rate[el[i].parent] : R(0);
                len[i] = pl + el[i].v[0] * dq[0];
                rate[i] = pr + el[i].v[0] * dq[1];
            }
            int last = -1;   // ascending dof order (physics.py:614-620)
            for (int pass = 0; pass < n; ++pass) {
                int dof = 0x7fffffff;
                for (int i = 0; i < n; ++i)
                    if (el[i].index > last && el[i].index < dof) dof = el[i].index;
                if (dof == 0x7fffffff) break;
                last = dof;
                R qf = R(0);
                int jslot = -1;
                for (int i = 0; i < n; ++i)
                    if (el[i].index == dof) {
                        qf = qf + el[i].v[0] * tendon_spring(t, len[i], rate[i]);
                        jslot = el[i].joint;
                    }
                if (qf == R(0)) continue;
                const auto &jt = c.joints[jslot];
                int ci = jt.child, ri = t.reaction_body;
                V3<R> aw = qrot(qmul(w.l4(ib(d, jt.parent, BQ)), jq4(jt.origin_quat)), jv3(jt.axis));
                V3<R> P = aw * qf * dt;
                if (jt.kind == BSIM_REVOLUTE) {
                    add_w(d, w, ci, smul(w.lS(ib(d, ci, BI)), P));
                    add_w(d, w, ri, -smul(w.lS(ib(d, ri, BI)), P));
                } else {
                    add_v(d, w, ci, P * w.at(ib(d, ci, BM)));
                    add_v(d, w, ri, -(P * w.at(ib(d, ri, BM))));
                }
            }
        } else {
            const int MAXA = 16;
            V3<R> pts[MAXA], vel[MAXA];
            int n = t.count < MAXA ? t.count : MAXA;
            for (int i = 0; i < n; ++i) {
                int b = el[i].index;
                V3<R> r = qrot(w.l4(ib(d, b, BQ)), v3(el[i].v[0], el[i].v[1], el[i].v[2]));
                pts[i] = w.l3(ib(d, b, BP)) + r;
                V3<R> rr = pts[i] - w.l3(ib(d, b, BP));
                vel[i] = w.l3(ib(d, b, BV_)) + cross(w.l3(ib(d, b, BW)), rr);
            }
            const int32_t *pth = c.L.spatial_paths + t.path_offset;
            int npaths = pth[0];
            const int MAXENT = 32;   // all entries from the pre-application state
            V3<R> ef[MAXENT];
            int ei[MAXENT];
            int nent = 0;
            const int32_t *cur = pth + 1;
            for (int pi = 0; pi < npaths && nent + 2 <= MAXENT; ++pi) {
                int len = cur[0];
                const int32_t *ix = cur + 1;
                R L = R(0), Ld = R(0);
                for (int k = 1; k < len; ++k) {
                    V3<R> dd = pts[ix[k]] - pts[ix[k - 1]];
                    R dist = norm(dd);
                    R sf = dist > R(1e-12) ? dist : R(1);
                    L = L + el[ix[k]].v[3] * dist;
                    Ld = Ld + el[ix[k]].v[3] * dot(vel[ix[k]] - vel[ix[k - 1]], v3(dd.x / sf, dd.y / sf, dd.z / sf));
                }
                R f = tendon_spring(t, L, Ld);
                int leaf = ix[len - 1], root = ix[0];
                V3<R> dl = pts[ix[len - 2]] - pts[leaf], dr = pts[ix[1]] - pts[root];
                R nl = norm(dl), nr = norm(dr);
                nl = nl > R(1e-12) ? nl : R(1);
                nr = nr > R(1e-12) ? nr : R(1);
                ef[nent] = v3(dl.x / nl, dl.y / nl, dl.z / nl) * -f;
                ei[nent++] = leaf;
                ef[nent] = v3(dr.x / nr, dr.y / nr, dr.z / nr) * -f;
                ei[nent++] = root;
                cur += 1 + len;
            }
            for (int k = 0; k < nent; ++k) {
                int b = el[ei[k]].index;
                V3<R> r = pts[ei[k]] - w.l3(ib(d, b, BP));
                add_v(d, w, b, ef[k] * dt * w.at(ib(d, b, BM)));
                add_w(d, w, b, smul(w.lS(ib(d, b, BI)), cross(r, ef[k])) * dt);
            }
        }
    }
}

// compile-time properties of an AOT topology (the generic kernel: none)
template <class T> constexpr bool topo_rev() {
    if constexpr (T::is_static) return T::all_revolute; else return false;
}
template <class T> constexpr bool topo_idf() {
    if constexpr (T::is_static) return T::identity_frames; else return false;
}
template <class T> constexpr bool topo_pairs() {
    if constexpr (T::is_static) return T::Q > 0; else return true;
}
template <class T> constexpr bool topo_tendons() {
    if constexpr (T::is_static) return T::has_tendons; else return true;
}

// Per body, before the rows of pass k > 0 (refresh 718-756): [integrate
// (574-575) at k = N,] effective orientation, world inverse inertia.
template <class R> BS_HD void body_phase_item(const Ctx<R> &c, const Ws<R> &w, int e, int b, int k, int N) {
    const Dims &d = c.d;
    const bool deltas = k > 0 && k < N;
    if (k == N) {
        w.s3(ib(d, b, BP), w.l3(ib(d, b, BP)) + w.l3(ib(d, b, BDP)));
        w.s4(ib(d, b, BQ), qnormalize(qmul(qexp(w.l3(ib(d, b, BDA))), w.l4(ib(d, b, BQ)))));
    }
    if (deltas) w.s4(ib(d, b, BQE), qnormalize(qmul(qexp(w.l3(ib(d, b, BDA))), w.l4(ib(d, b, BQ)))));
    body_inertia(c, w, e, b, deltas ? BQE : BQ);
}

// ====================================================== the group step
// Loops over (env, item) pairs distributed over the CTA's threads; on the
// host (tid 0 of 1) they degenerate to plain sequential loops.
#define BS_ITEMS(g, count, el, k)                                                   \
    for (int it_ = (g).tid, n_ = (g).ne * (count); it_ < n_; it_ += (g).nth)       \
        for (int el = it_ % (g).ne, k = it_ / (g).ne, once_ = 1; once_; once_ = 0)
#define BS_ENVS(g, el) for (int el = (g).tid - (g).lane0; el >= 0 && el < (g).ne; el += (g).nth)

// Scene.step() for the CTA's envs on the resident workspace
// (physics.py:538-592).  `write_outputs`: contact-derived outputs of this
// step go to global memory (the last substep of a fused launch).
//
// The N biased passes and the final velocity stage share one phase-A body
// (freeze at k = 0, refresh-with-deltas at 0 < k < N, integrate + refresh at
// k = N), so every piece of the step appears once in the binary.
// SCHED: the instantiation's sweep for non-star / non-register topologies --
// the row schedule (true) or the one-lane sequential sweep (false).  Each
// kernel carries one of the two: with both compiled in, either ran 6-9 %
// slower (register allocation / code size), so the launcher
// picks the instantiation from the layout's schedule.  The host build keeps
// the run-time choice.
template <class R, class T, bool SCHED = false>
BS_HD void group_step(const Ctx<R> &c, const Grp<R> &g, bool write_outputs, int sub) {
    const Dims &d = c.d;
    const int ebad = d.o_env + EBAD + (sub & 1);
    const auto &p = c.p;
    const R dt = p.dt;
    const int N = p.position_iterations;
    const R h = dt / (R)N;

    // external forces, start-of-step inertia (545-555), zeroed TGS deltas (564-566)
    BS_ITEMS(g, d.B, el, b) {
        Ws<R> w = g.env(el);
        body_inertia(c, w, g.e0 + el, b, BQ);
        body_external(c, w, g.e0 + el, b);
        w.s3(ib(d, b, BDP), zero3<R>());
        w.s3(ib(d, b, BDA), zero3<R>());
        if (b == 0) w.at(d.o_env + EBAD + ((sub + 1) & 1)) = R(0);   // the previous substep's flag
    }
    BS_SYNC();
    if (topo_tendons<T>() && d.T) {
        BS_ENVS(g, el) { apply_tendons(c, g.env(el), g.e0 + el); }
        BS_SYNC();
    }
    const R ld = r_max(R(0), R(1) - p.linear_damping * dt), ad = r_max(R(0), R(1) - p.angular_damping * dt);
    if (ld != R(1) || ad != R(1)) {
        BS_ITEMS(g, d.B, el, b) {
            Ws<R> w = g.env(el);
            w.s3(ib(d, b, BV_), w.l3(ib(d, b, BV_)) * ld);
            w.s3(ib(d, b, BW), w.l3(ib(d, b, BW)) * ad);
        }
        BS_SYNC();
    }

#if defined(__CUDA_ARCH__)
    constexpr bool tail_body = topo_star<T>();   // body phase fused into the star tail
    // plane constants built beside the chain sweep by the warps without sweep lanes
    constexpr bool plane_overlap = BSIM_PLANE_OVERLAP && topo_star<T>();
#else
    constexpr bool tail_body = false, plane_overlap = false;
#endif
    for (int k = 0; k <= N; ++k) {
        const bool biased = k < N, freeze = k == 0, deltas = k > 0 && k < N;
#if defined(BSIM_EXP_PASS_CLOCKS) && defined(__CUDA_ARCH__)
        unsigned long long pass_t0_ = clock64();
        if (g.tid == 0) atomicAdd(&bsim_pass_clk[7], 1ull);
#endif
        // phase A: orientations -> inertias -> joint/contact geometry and row
        // constants (freeze 657-716, refresh 718-756)
#ifdef BSIM_EXP_SKIP_A   // timing experiment only: reuse the freeze-time constants
        if (!freeze && k < N) goto phase_b;
#endif
        if (!freeze && !(tail_body && k > 0)) {   // (tail_body: the previous pass's tail ran it)
            BS_ITEMS(g, d.B, el, b) { body_phase_item(c, g.env(el), g.e0 + el, b, k, N); }
            BS_SYNC();
        }
        BS_ITEMS(g, d.J, el, j) {
            joint_item<R, T, topo_rev<T>(), topo_idf<T>()>(c, g.env(el), g.e0 + el, j, h, biased, freeze, deltas,
                                                           g.jt);
        }
        auto plane_item = [&](int el, int i) {
            Ws<R> w = g.env(el);
            const int pb = plane_body_of<T>(c, i);
            if (freeze) plane_freeze(c, w, g.e0 + el, i, pb);
#if BSIM_SKIP_INACTIVE
            // an inactive slot's rows apply nothing (row_plane returns before
            // reading them), so its row constants are not built
            if (w.at(ipl(d, i, CACT)) == R(0)) return;
#endif
            plane_constants(c, w, i, pb);
            plane_pass_constants(c, w, i, biased, pb);
        };
        // the freeze reads the bodies' start-of-pass velocities (restitution
        // target, 687-688), so at k = 0 it runs here, before the sweep writes them
        if (!plane_overlap || freeze) {
            BS_ITEMS(g, d.P, el, i) { plane_item(el, i); }
        }
        if (topo_pairs<T>()) {
            BS_ITEMS(g, d.Q, el, i) {
                Ws<R> w = g.env(el);
                if (freeze) pair_freeze(c, w, g.e0 + el, i);
#if BSIM_SKIP_INACTIVE
                if (w.at(ipr(d, i, QACT)) == R(0)) continue;   // row_pair returns before using them
#endif
                pair_constants(c, w, i);
                pair_pass_constants(c, w, i, biased);
            }
        }
        BS_SYNC();
        BSIM_PASSCLK(0);
#ifdef BSIM_EXP_SKIP_A
    phase_b:
#endif
        // phase B: one biased pass (567-572) or the velocity passes (580-581)
#ifdef BSIM_EXP_SKIP_B   // timing experiment only
        const int reps = 0;
#else
        const int reps = biased ? 1 : p.velocity_iterations;
#endif
        for (int r = 0; r < reps; ++r) {
#if defined(__CUDA_ARCH__)
            if constexpr (topo_star<T>()) {   // two lanes per env (sweep_star)
                // star_lanes lanes per env from the claimed sweep warp on (wrapping
                // into the next warp when the CTA's envs need more than 32 lanes)
                constexpr int G = star_lanes<T>();
                const int t = (g.tid - g.lane0 + g.nth) % g.nth;
                const bool on = t < G * g.ne;
                const unsigned mask = __ballot_sync(0xffffffffu, on);
                if (on) {
                    sweep_star<R, T>(c, g.env(t / G), h, biased, t % G, mask);
                } else if (plane_overlap && r == 0 && !freeze) {
                    // the plane slots' row constants need only the bodies' pass
                    // poses: the warps without sweep lanes build them while the
                    // sweep runs (the plane rows use them in the tail below)
                    const int w0 = 32 * ((G * g.ne + 31) / 32);
                    for (int it = t - w0; it >= 0 && it < g.ne * d.P; it += g.nth - w0)
                        plane_item(it % g.ne, it / g.ne);
                }
                BS_SYNC();
                BSIM_PASSCLK(1);
                BS_ITEMS(g, T::B, el, b) { star_body_tail<R, T>(c, g.env(el), g.e0 + el, b, h, k, N); }
            } else
#endif
            {
#if defined(__CUDA_ARCH__)
                if constexpr (SCHED && !topo_register_sweep<T>()) {   // launcher: sched_stages > 0
                    // the row schedule on BSIM_SCHED_WARPS warps from the claimed sweep
                    // warp on: 32 SW / NE lanes per env, each env's lanes inside one warp
                    // (a stage's rows run side by side; a stage ends at a __syncwarp)
                    constexpr int NE = Shape<R>::NE, NW = Shape<R>::NTH / 32;
                    constexpr int SW = BSIM_SCHED_WARPS < NW ? BSIM_SCHED_WARPS : NW;
                    constexpr int LPE = NE >= 32 * SW ? 1 : (32 * SW / NE > 32 ? 32 : 32 * SW / NE);
                    static_assert(32 % LPE == 0, "an env's sweep lanes must share a warp");
                    const int t = (g.tid - g.lane0 + g.nth) % g.nth;
                    if (t < 32 * SW) {
                        const int el = t / LPE, lane = t % LPE;
                        const Ws<R> w = g.env(el);
                        sweep_sched<R, T>(c, el < g.ne ? &w : nullptr, h, biased, lane, LPE, 0xffffffffu);
                    }
                } else
#else
                if (!topo_register_sweep<T>() && c.L.sched_stages > 0) {
                    BS_ENVS(g, el) { sweep_sched_host<R>(c, g.env(el), h, biased); }
                } else
#endif
                {
                    BS_ENVS(g, el) { sweep_any<R, T>(c, g.env(el), h, biased); }
                }
            }
            BS_SYNC();
            BSIM_PASSCLK(2);
        }
    }
    // velocity clamps (584-587)
    BS_ITEMS(g, d.B, el, b) {
        Ws<R> w = g.env(el);
        V3<R> lv = w.l3(ib(d, b, BV_)), av = w.l3(ib(d, b, BW));
        R sl = r_min(R(1), p.max_linear_velocity / r_max(norm(lv), R(1e-12)));
        R sa = r_min(R(1), p.max_angular_velocity / r_max(norm(av), R(1e-12)));
        w.s3(ib(d, b, BV_), lv * sl);
        w.s3(ib(d, b, BW), av * sa);
        // _flag_nonfinite (1073-1088) check on the final state of this body
        bool ok = true;
        for (int kk = 0; kk < 13; ++kk) ok = ok && finite_r(w.at(ib(d, b, body_item13(kk))));
        if (!ok) w.at(ebad) = R(1);
    }
    BS_SYNC();

    // refresh_buffers(ctx) (1037-1071): contact wrench per body (BDP/BDA reused)
    if (write_outputs) {
        BS_ITEMS(g, d.B, el, b) {
            Ws<R> w = g.env(el);
            V3<R> F = zero3<R>(), Tq = zero3<R>();
            for (int i = 0; i < d.P; ++i) {
                if (c.L.plane_body[i] != b) continue;
                V3<R> P = v3(R(0), R(0), R(1)) * w.at(ipl(d, i, CLN)) + v3(R(0), R(-1), R(0)) * w.at(ipl(d, i, CLT)) +
                          v3(R(1), R(0), R(0)) * w.at(ipl(d, i, CLT + 1));
                V3<R> f = v3(P.x / dt, P.y / dt, P.z / dt);
                F = F + f;
                Tq = Tq + cross(w.l3(ipl(d, i, CR)), f);
            }
            for (int i = 0; i < d.Q; ++i) {
                int pa = c.L.pair_body[2 * i], pb = c.L.pair_body[2 * i + 1];
                if (pa != b && pb != b) continue;
                V3<R> P = w.l3(ipr(d, i, QN)) * w.at(ipr(d, i, QLN)) + w.l3(ipr(d, i, QT1)) * w.at(ipr(d, i, QLT)) +
                          w.l3(ipr(d, i, QT2)) * w.at(ipr(d, i, QLT + 1));
                V3<R> f = v3(P.x / dt, P.y / dt, P.z / dt);
                if (pb == b) {
                    F = F + f;
                    Tq = Tq + cross(w.l3(ipr(d, i, QR)), f);
                }
                if (pa == b) {
                    F = F + (-f);
                    Tq = Tq + cross(w.l3(ipr(d, i, QRA)), -f);
                }
            }
            w.s3(ib(d, b, BDP), F);
            w.s3(ib(d, b, BDA), Tq);
            R *o = c.s.net_contact + 3 * ((size_t)(g.e0 + el) * d.B + b);
            o[0] = F.x; o[1] = F.y; o[2] = F.z;
        }
        BS_ITEMS(g, d.D, el, k) {
            c.s.dof_force[(size_t)(g.e0 + el) * d.D + k] = g.env(el).at(idf(d, k, DIMP)) / dt;
        }
        BS_SYNC();
        BS_ITEMS(g, d.S, el, k) {
            Ws<R> w = g.env(el);
            int b = c.L.sensor_body[k];
            Q4<R> qi = qconj(w.l4(ib(d, b, BQ)));
            V3<R> f = qrot(qi, w.l3(ib(d, b, BDP))), t = qrot(qi, w.l3(ib(d, b, BDA)));
            R *o = c.s.sensor_forces + 6 * ((size_t)(g.e0 + el) * d.S + k);
            o[0] = f.x; o[1] = f.y; o[2] = f.z; o[3] = t.x; o[4] = t.y; o[5] = t.z;
        }
    }

    // _flag_nonfinite (1073-1088): sanitize poisoned envs (sticky flag; the
    // check ran with the velocity clamps)
    if (write_outputs) BS_SYNC();   // the output stage above reads the pre-sanitize state
    BS_ITEMS(g, d.B, el, b) {
        Ws<R> w = g.env(el);
        if (w.at(ebad) != R(0)) {
            int e = g.e0 + el;
            if (b == 0) c.s.nonfinite[e] = 1;
            for (int k = 0; k < 13; ++k) {
                R &x = w.at(ib(d, b, body_item13(k)));
                // the reference zeroes the WORLD position (physics.py:1081)
                if (!finite_r(x)) x = k < 3 ? -c.s.env_origins[3 * (size_t)e + k] : R(0);
            }
            Q4<R> q = w.l4(ib(d, b, BQ));
            if (r_sqrt(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w) < R(1e-9)) q = Q4<R>{0, 0, 0, 1};
            w.s4(ib(d, b, BQ), qnormalize(q));
        }
    }
    BS_SYNC();
}

// dof_state readout from the workspace (physics.py:427-459, 1038)
template <class R> BS_HD void readout_group(const Ctx<R> &c, const Grp<R> &g) {
    const Dims &d = c.d;
    BS_ITEMS(g, d.J, el, j) {
        Ws<R> w = g.env(el);
        R q[3], qd[3];
        int n = joint_dofs(c, w, j, q, qd);
        for (int k = 0; k < n; ++k) {
            R *o = c.s.dof_state + 2 * ((size_t)(g.e0 + el) * d.D + c.joints[j].dof + k);
            o[0] = q[k];
            o[1] = qd[k];
        }
    }
}

// staging of the per-env inputs the rows reuse (once per launch)
template <class R> BS_HD void stage_group(const Ctx<R> &c, const Grp<R> &g) {
    const Dims &d = c.d;
    BS_ENVS(g, el) { stage_env(c, g.env(el), g.e0 + el); }
    BS_ITEMS(g, d.B, el, b) {
        Ws<R> w = g.env(el);
        const size_t gb = (size_t)(g.e0 + el) * d.B + b;
        w.at(ib(d, b, BM)) = c.s.inv_mass[gb];
        w.at(ib(d, b, BI) + 6) = c.s.inv_inertia_local[3 * gb];
        w.at(ib(d, b, BI) + 7) = c.s.inv_inertia_local[3 * gb + 1];
        w.at(ib(d, b, BW) + 3) = c.s.inv_inertia_local[3 * gb + 2];
    }
    BS_ITEMS(g, d.P, el, i) {
        for (int k = 0; k < 3; ++k)
            g.env(el).at(d.o_anchor + ANCHOR_ITEMS * i + k) = c.s.friction_anchor[3 * ((size_t)i * d.E + g.e0 + el) + k];
    }
}

}  // namespace bsim
