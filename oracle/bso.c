/*
 * bso.c -- CPU ORACLE (test infrastructure only; see bso.h).
 *
 * float64 restatement of the reference step, one environment at a time.
 * Environments are disjoint constraint islands (physics.py:5-9), so solving
 * the reference's env-vectorized rows env by env is the same arithmetic.
 * Every function cites the reference lines it restates.
 */
#include "bso.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { K_FIXED = 0, K_REV = 1, K_PRISM = 2, K_SPH = 3 };
enum { M_FORCE = 0, M_POS = 1, M_VEL = 2 };

/* ------------------------------------------------------------------ math */
/* spatial.py:18-162; quaternions are (x, y, z, w). */
static double dot3(const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static void cross3(double *o, const double *a, const double *b) {
    double x = a[1] * b[2] - a[2] * b[1], y = a[2] * b[0] - a[0] * b[2], z = a[0] * b[1] - a[1] * b[0];
    o[0] = x; o[1] = y; o[2] = z;
}
static void qmul(double *o, const double *a, const double *b) {
    double x = a[3] * b[0] + a[0] * b[3] + a[1] * b[2] - a[2] * b[1];
    double y = a[3] * b[1] - a[0] * b[2] + a[1] * b[3] + a[2] * b[0];
    double z = a[3] * b[2] + a[0] * b[1] - a[1] * b[0] + a[2] * b[3];
    double w = a[3] * b[3] - a[0] * b[0] - a[1] * b[1] - a[2] * b[2];
    o[0] = x; o[1] = y; o[2] = z; o[3] = w;
}
static void qconj(double *o, const double *q) { o[0] = -q[0]; o[1] = -q[1]; o[2] = -q[2]; o[3] = q[3]; }
static void qnormalize(double *q) {
    double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (n > 0) { q[0] /= n; q[1] /= n; q[2] /= n; q[3] /= n; }
}
/* v + w t + u x t, t = 2 u x v  (spatial.py:57-64) */
static void qrot(double *o, const double *q, const double *v) {
    double t[3], ut[3];
    double u[3] = {q[0], q[1], q[2]};
    cross3(t, u, v);
    t[0] *= 2.0; t[1] *= 2.0; t[2] *= 2.0;
    cross3(ut, u, t);
    double x = v[0] + q[3] * t[0] + ut[0], y = v[1] + q[3] * t[1] + ut[1], z = v[2] + q[3] * t[2] + ut[2];
    o[0] = x; o[1] = y; o[2] = z;
}
static void qexp(double *o, const double *v) { /* spatial.py:143-152 */
    double ang = sqrt(dot3(v, v));
    double ax[3] = {1.0, 0.0, 0.0};
    if (!(ang < 1e-12)) {
        double d = ang > 0 ? ang : 1.0;
        ax[0] = v[0] / d; ax[1] = v[1] / d; ax[2] = v[2] / d;
    }
    double s = sin(0.5 * ang), c = cos(0.5 * ang);
    o[0] = ax[0] * s; o[1] = ax[1] * s; o[2] = ax[2] * s; o[3] = c;
}
static void qlog(double *o, const double *qin) { /* spatial.py:155-162 */
    double q[4] = {qin[0], qin[1], qin[2], qin[3]};
    if (q[3] < 0) { q[0] = -q[0]; q[1] = -q[1]; q[2] = -q[2]; q[3] = -q[3]; }
    double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2]);
    double ang = 2.0 * atan2(n, q[3]);
    double sc = n > 1e-12 ? ang / (n > 0 ? n : 1.0) : 2.0;
    o[0] = q[0] * sc; o[1] = q[1] * sc; o[2] = q[2] * sc;
}
static void qmat(double R[9], const double *q) { /* spatial.py:80-95 */
    double x = q[0], y = q[1], z = q[2], w = q[3];
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - z * w); R[2] = 2 * (x * z + y * w);
    R[3] = 2 * (x * y + z * w); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - x * w);
    R[6] = 2 * (x * z - y * w); R[7] = 2 * (y * z + x * w); R[8] = 1 - 2 * (x * x + y * y);
}
static void mv3(double *o, const double M[9], const double *v) {
    double x = M[0] * v[0] + M[1] * v[1] + M[2] * v[2];
    double y = M[3] * v[0] + M[4] * v[1] + M[5] * v[2];
    double z = M[6] * v[0] + M[7] * v[1] + M[8] * v[2];
    o[0] = x; o[1] = y; o[2] = z;
}
static double vMv(const double *a, const double M[9], const double *b) {
    double t[3];
    mv3(t, M, b);
    return dot3(a, t);
}
static void tangents(double *t1, double *t2, const double *n) { /* physics.py:131-137 */
    double ref[3] = {0, 0, 1};
    if (!(fabs(n[2]) < 0.9)) { ref[0] = 1; ref[2] = 0; }
    cross3(t1, ref, n);
    double l = sqrt(dot3(t1, t1));
    t1[0] /= l; t1[1] /= l; t1[2] /= l;
    cross3(t2, n, t1);
}
static double clampd(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }
static double signd(double x) { return x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0); }
static double wrap_pi(double a) { /* (a + pi) % (2 pi) - pi with Python's floor-mod */
    double m = 2.0 * M_PI;
    double r = fmod(a + M_PI, m);
    if (r < 0) r += m;
    return r - M_PI;
}

/* Gaussian elimination with partial pivoting (stands in for LAPACK gesv,
   physics.py:886,903,923). */
static void solve_n(int n, double *K, double *x) {
    for (int c = 0; c < n; ++c) {
        int p = c;
        for (int r = c + 1; r < n; ++r) if (fabs(K[r * n + c]) > fabs(K[p * n + c])) p = r;
        if (p != c) {
            for (int k = 0; k < n; ++k) { double t = K[c * n + k]; K[c * n + k] = K[p * n + k]; K[p * n + k] = t; }
            double t = x[c]; x[c] = x[p]; x[p] = t;
        }
        for (int r = c + 1; r < n; ++r) {
            double f = K[r * n + c] / K[c * n + c];
            for (int k = c; k < n; ++k) K[r * n + k] -= f * K[c * n + k];
            x[r] -= f * x[c];
        }
    }
    for (int c = n - 1; c >= 0; --c) {
        double s = x[c];
        for (int k = c + 1; k < n; ++k) s -= K[c * n + k] * x[k];
        x[c] = s / K[c * n + c];
    }
}

/* ----------------------------------------------------------- per-env ctx */
typedef struct {
    double rp[3], rc[3], perr0[3], rerr0[3], axis[3], t1[3], t2[3], q0;
    int has_q0;
} jctx;

typedef struct {
    int body, body_a; /* body_a = -1 for plane */
    double r[3], ra[3], n[3], depth0, rest, lam_n, lam_t[2], point[3], terr0[3];
    int active;
} cctx;

typedef struct {
    const bso_scene *s;
    int e;
    double *pos, *quat, *v, *w;      /* env slices of canonical state */
    double *invI;                    /* [B][9] current world inverse inertia */
    double *dpos, *dang;             /* [B][3] */
    double *pos_eff, *quat_eff;      /* [B][3], [B][4] */
    jctx *jc;
    cctx *cc;
    double *dof_impulse;             /* [D] */
    uint64_t ncall;                  /* limit evaluations so far (limit_jitter hash) */
} envw;

static double jparam(const double *arr, const bso_scene *s, int j, int e) { return arr[(size_t)j * s->E + e]; }

/* decision-margin instrumentation (bso.h: margin) */
static void note_margin(const bso_scene *s, int e, int k, double m) {
    if (!s->margin) return;
    double *p = s->margin + 4 * (size_t)e + k;
    m = fabs(m);
    if (m < *p) *p = m;
}

static void inv_inertia_world(envw *w, const double *quat) { /* physics.py:594-596 */
    const bso_scene *s = w->s;
    for (int b = 0; b < s->B; ++b) {
        double R[9];
        qmat(R, quat + 4 * b);
        const double *d = s->inv_inertia_local + 3 * ((size_t)w->e * s->B + b);
        double *I = w->invI + 9 * b;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j)
                I[3 * i + j] = R[3 * i + 0] * d[0] * R[3 * j + 0] + R[3 * i + 1] * d[1] * R[3 * j + 1] +
                               R[3 * i + 2] * d[2] * R[3 * j + 2];
    }
}

static double imass(const envw *w, int b) { return w->s->inv_mass[(size_t)w->e * w->s->B + b]; }

/* physics.py:427-459 for one env */
static void read_dofs_env(const bso_scene *s, int e) {
    const double *pos = s->pos + 3 * (size_t)e * s->B, *quat = s->quat + 4 * (size_t)e * s->B;
    const double *av = s->angvel + 3 * (size_t)e * s->B, *lv = s->linvel + 3 * (size_t)e * s->B;
    double *dof = s->dof_state + 2 * (size_t)e * s->D;
    for (int j = 0; j < s->J; ++j) {
        const bso_joint *jt = &s->joints[j];
        if (jt->dof < 0) continue;
        int p = jt->parent, c = jt->child;
        double jqp[4], jqc[4];
        qmul(jqp, quat + 4 * p, jt->origin_quat);
        qmul(jqc, quat + 4 * c, jt->child_quat);
        if (jt->kind == K_REV) {
            double cj[4], qr[4], aw[3], dw[3];
            qconj(cj, jqp);
            qmul(qr, cj, jqc);
            double sn = dot3(qr, jt->axis);
            double ang = wrap_pi(2.0 * atan2(sn, qr[3]));
            qrot(aw, jqp, jt->axis);
            for (int k = 0; k < 3; ++k) dw[k] = av[3 * c + k] - av[3 * p + k];
            dof[2 * jt->dof] = ang;
            dof[2 * jt->dof + 1] = dot3(aw, dw);
        } else if (jt->kind == K_PRISM) {
            double ap[3], ac[3], aw[3], d[3], vap[3], vac[3], rpp[3], rcc[3];
            qrot(ap, quat + 4 * p, jt->origin_pos);
            qrot(ac, quat + 4 * c, jt->child_pos);
            for (int k = 0; k < 3; ++k) { ap[k] += pos[3 * p + k]; ac[k] += pos[3 * c + k]; }
            qrot(aw, jqp, jt->axis);
            for (int k = 0; k < 3; ++k) d[k] = ac[k] - ap[k];
            dof[2 * jt->dof] = dot3(aw, d);
            for (int k = 0; k < 3; ++k) { rpp[k] = ap[k] - pos[3 * p + k]; rcc[k] = ac[k] - pos[3 * c + k]; }
            cross3(vap, av + 3 * p, rpp);
            cross3(vac, av + 3 * c, rcc);
            for (int k = 0; k < 3; ++k) d[k] = (lv[3 * c + k] + vac[k]) - (lv[3 * p + k] + vap[k]);
            dof[2 * jt->dof + 1] = dot3(aw, d);
        } else if (jt->kind == K_SPH) {
            double cj[4], qr[4], rv[3], dw[3], wr[3];
            qconj(cj, jqp);
            qmul(qr, cj, jqc);
            qlog(rv, qr);
            for (int k = 0; k < 3; ++k) dw[k] = av[3 * c + k] - av[3 * p + k];
            qrot(wr, cj, dw);
            for (int k = 0; k < 3; ++k) { dof[2 * (jt->dof + k)] = rv[k]; dof[2 * (jt->dof + k) + 1] = wr[k]; }
        }
    }
}

/* physics.py:366-425 for one env, restricted to actor_mask */
static void fk_env(const bso_scene *s, int e, uint32_t actor_mask) {
    double *pos = s->pos + 3 * (size_t)e * s->B, *quat = s->quat + 4 * (size_t)e * s->B;
    double *av = s->angvel + 3 * (size_t)e * s->B, *lv = s->linvel + 3 * (size_t)e * s->B;
    const double *dof = s->dof_state + 2 * (size_t)e * s->D;
    static const double QI[4] = {0, 0, 0, 1};
    for (int j = 0; j < s->J; ++j) {
        const bso_joint *jt = &s->joints[j];
        if (!((actor_mask >> jt->actor) & 1u)) continue;
        int p = jt->parent, c = jt->child;
        double jq[4], jp[3], mq[4] = {0, 0, 0, 1}, mp[3] = {0, 0, 0}, qda[3] = {0, 0, 0}, qdl[3] = {0, 0, 0};
        qmul(jq, quat + 4 * p, jt->origin_quat);
        qrot(jp, quat + 4 * p, jt->origin_pos);
        for (int k = 0; k < 3; ++k) jp[k] += pos[3 * p + k];
        if (jt->kind == K_REV) {
            double q = dof[2 * jt->dof], qd = dof[2 * jt->dof + 1];
            double sh = sin(0.5 * q), ch = cos(0.5 * q);
            mq[0] = jt->axis[0] * sh; mq[1] = jt->axis[1] * sh; mq[2] = jt->axis[2] * sh; mq[3] = ch;
            qrot(qda, jq, jt->axis);
            for (int k = 0; k < 3; ++k) qda[k] *= qd;
        } else if (jt->kind == K_PRISM) {
            double q = dof[2 * jt->dof], qd = dof[2 * jt->dof + 1];
            for (int k = 0; k < 3; ++k) mp[k] = jt->axis[k] * q;
            qrot(qdl, jq, jt->axis);
            for (int k = 0; k < 3; ++k) qdl[k] *= qd;
        } else if (jt->kind == K_SPH) {
            double q3[3], qd3[3];
            for (int k = 0; k < 3; ++k) { q3[k] = dof[2 * (jt->dof + k)]; qd3[k] = dof[2 * (jt->dof + k) + 1]; }
            qexp(mq, q3);
            qrot(qda, jq, qd3);
        }
        (void)QI;
        double qcf[4], anchor[3], cc[4], qc[4], pc[3], t[3];
        qmul(qcf, jq, mq);
        qrot(anchor, jq, mp);
        for (int k = 0; k < 3; ++k) anchor[k] += jp[k];
        qconj(cc, jt->child_quat);
        qmul(qc, qcf, cc);
        qnormalize(qc);
        qrot(t, qc, jt->child_pos);
        for (int k = 0; k < 3; ++k) pc[k] = anchor[k] - t[k];
        memcpy(quat + 4 * c, qc, sizeof qc);
        memcpy(pos + 3 * c, pc, sizeof pc);
        double ra[3], va[3], wc[3], rr[3], wxr[3];
        for (int k = 0; k < 3; ++k) ra[k] = anchor[k] - pos[3 * p + k];
        cross3(va, av + 3 * p, ra);
        for (int k = 0; k < 3; ++k) { va[k] += lv[3 * p + k]; wc[k] = av[3 * p + k] + qda[k]; }
        for (int k = 0; k < 3; ++k) rr[k] = pc[k] - anchor[k];
        cross3(wxr, wc, rr);
        for (int k = 0; k < 3; ++k) { av[3 * c + k] = wc[k]; lv[3 * c + k] = va[k] + qdl[k] + wxr[k]; }
    }
}

/* joint geometry from an effective pose (physics.py:660-680, 733-756) */
static void joint_geometry(envw *w, const double *pos, const double *quat, int with_q0_refresh) {
    const bso_scene *s = w->s;
    for (int j = 0; j < s->J; ++j) {
        const bso_joint *jt = &s->joints[j];
        jctx *c = &w->jc[j];
        int p = jt->parent, ch = jt->child;
        double jqp[4], jqc[4], ap[3], ac[3], cj[4], qe[4];
        qmul(jqp, quat + 4 * p, jt->origin_quat);
        qmul(jqc, quat + 4 * ch, jt->child_quat);
        qrot(ap, quat + 4 * p, jt->origin_pos);
        qrot(ac, quat + 4 * ch, jt->child_pos);
        for (int k = 0; k < 3; ++k) { ap[k] += pos[3 * p + k]; ac[k] += pos[3 * ch + k]; }
        for (int k = 0; k < 3; ++k) {
            c->rp[k] = ap[k] - pos[3 * p + k];
            c->rc[k] = ac[k] - pos[3 * ch + k];
            c->perr0[k] = ac[k] - ap[k];
        }
        qconj(cj, jqp);
        qmul(qe, jqc, cj);
        double sg = signd(qe[3]);
        for (int k = 0; k < 3; ++k) c->rerr0[k] = 2.0 * qe[k] * sg;
        qrot(c->axis, jqp, jt->axis);
        tangents(c->t1, c->t2, c->axis);
        if (with_q0_refresh && c->has_q0) {
            if (jt->kind == K_REV) {
                double qr[4];
                qmul(qr, cj, jqc);
                c->q0 = wrap_pi(2.0 * atan2(dot3(qr, jt->axis), qr[3]));
            } else {
                double d[3] = {ac[0] - ap[0], ac[1] - ap[1], ac[2] - ap[2]};
                c->q0 = dot3(c->axis, d);
            }
        }
    }
}

/* _refresh_joint_geometry (physics.py:718-756) */
static void refresh(envw *w, int with_deltas) {
    const bso_scene *s = w->s;
    const double *pe = w->pos, *qe = w->quat;
    if (with_deltas) {
        for (int b = 0; b < s->B; ++b) {
            double dq[4];
            for (int k = 0; k < 3; ++k) w->pos_eff[3 * b + k] = w->pos[3 * b + k] + w->dpos[3 * b + k];
            qexp(dq, w->dang + 3 * b);
            qmul(w->quat_eff + 4 * b, dq, w->quat + 4 * b);
            qnormalize(w->quat_eff + 4 * b);
        }
        pe = w->pos_eff;
        qe = w->quat_eff;
    }
    inv_inertia_world(w, qe);
    joint_geometry(w, pe, qe, 1);
}

/* ----------------------------------------------------------- row helpers */
static void vel_at(const envw *w, int b, const double *r, double *out) {
    double t[3];
    cross3(t, w->w + 3 * b, r);
    for (int k = 0; k < 3; ++k) out[k] = w->v[3 * b + k] + t[k];
}
static double axis_rel_vel(const envw *w, const bso_joint *jt, const jctx *c, int angular) { /* 804-810 */
    int p = jt->parent, ch = jt->child;
    if (angular) {
        double d[3];
        for (int k = 0; k < 3; ++k) d[k] = w->w[3 * ch + k] - w->w[3 * p + k];
        return dot3(c->axis, d);
    }
    double vp[3], vc[3], d[3];
    vel_at(w, p, c->rp, vp);
    vel_at(w, ch, c->rc, vc);
    for (int k = 0; k < 3; ++k) d[k] = vc[k] - vp[k];
    return dot3(c->axis, d);
}
static double axis_meff(const envw *w, const bso_joint *jt, const jctx *c, int angular) { /* 777-788 */
    int p = jt->parent, ch = jt->child;
    double k;
    if (angular) {
        double I[9];
        for (int i = 0; i < 9; ++i) I[i] = w->invI[9 * p + i] + w->invI[9 * ch + i];
        k = vMv(c->axis, I, c->axis);
    } else {
        double a[3], b[3];
        cross3(a, c->rp, c->axis);
        cross3(b, c->rc, c->axis);
        k = imass(w, p) + imass(w, ch) + vMv(a, w->invI + 9 * p, a) + vMv(b, w->invI + 9 * ch, b);
    }
    return 1.0 / (k > 1e-12 ? k : 1e-12);
}
static void apply_linear(envw *w, int b, const double *r, const double *P, double sgn) {
    double t[3], u[3];
    double m = imass(w, b);
    for (int k = 0; k < 3; ++k) w->v[3 * b + k] += sgn * (P[k] * m);
    cross3(t, r, P);
    mv3(u, w->invI + 9 * b, t);
    for (int k = 0; k < 3; ++k) w->w[3 * b + k] += sgn * u[k];
}
static void apply_angular(envw *w, int b, const double *L, double sgn) {
    double u[3];
    mv3(u, w->invI + 9 * b, L);
    for (int k = 0; k < 3; ++k) w->w[3 * b + k] += sgn * u[k];
}
static void apply_axis_impulse(envw *w, const bso_joint *jt, const jctx *c, double lam, int angular) { /* 790-802 */
    double P[3] = {c->axis[0] * lam, c->axis[1] * lam, c->axis[2] * lam};
    if (angular) {
        apply_angular(w, jt->child, P, 1.0);
        apply_angular(w, jt->parent, P, -1.0);
    } else {
        apply_linear(w, jt->child, c->rc, P, 1.0);
        apply_linear(w, jt->parent, c->rp, P, -1.0);
    }
}

static void solve_drive(envw *w, int j, double h, int biased) { /* 812-848 */
    const bso_scene *s = w->s;
    const bso_joint *jt = &s->joints[j];
    const jctx *c = &w->jc[j];
    if (jt->dof < 0 || jt->kind == K_SPH || !biased) return;
    const bso_params *pp = &s->params;
    size_t off = (size_t)w->e * s->D + jt->dof;
    int angular = jt->kind == K_REV;
    double qd = axis_rel_vel(w, jt, c, angular);
    int mode = s->dof_mode[off];
    double q = c->q0;
    double meff = axis_meff(w, jt, c, angular);
    double ia = meff + jparam(s->joint_armature, s, j, w->e);
    double tau = clampd(s->ctrl_dof_force[off], -pp->max_force, pp->max_force);
    double lam = mode == M_FORCE ? tau * h * meff / ia : 0.0;
    double kk = mode == M_POS ? jparam(s->joint_stiffness, s, j, w->e) : 0.0;
    double cc = mode == M_FORCE ? 0.0 : jparam(s->joint_damping, s, j, w->e);
    double err = s->ctrl_dof_pos_target[off] - q;
    double dv = s->ctrl_dof_vel_target[off] - qd;
    double lpd = h * (kk * (err - h * qd) + cc * dv) / (1.0 + h * (h * kk + cc) / ia);
    lpd = clampd(lpd, -pp->max_force * h, pp->max_force * h);
    lam = lam + lpd;
    double fr = jparam(s->joint_friction, s, j, w->e);
    if (fr > 0.0) lam = lam + clampd(-qd * meff, -fr * h, fr * h);
    apply_axis_impulse(w, jt, c, lam, angular);
    w->dof_impulse[jt->dof] += lam;
}

static void solve_limit(envw *w, int j, double h, int biased) { /* 850-870 */
    const bso_scene *s = w->s;
    const bso_joint *jt = &s->joints[j];
    const jctx *c = &w->jc[j];
    if (!jt->has_limits || jt->dof < 0 || jt->kind == K_SPH) return;
    double lo = jparam(s->joint_limit_lo, s, j, w->e), hi = jparam(s->joint_limit_hi, s, j, w->e);
    int angular = jt->kind == K_REV;
    double q = biased ? c->q0 : s->dof_state[2 * ((size_t)w->e * s->D + jt->dof)];
    if (s->limit_jitter_seed) {   /* bso.h: re-decide knife-edge limits at random */
        double tlo = s->limit_jitter * fmax(1.0, fabs(lo)), thi = s->limit_jitter * fmax(1.0, fabs(hi));
        double tol = fabs(q - lo) <= tlo ? tlo : (fabs(q - hi) <= thi ? thi : 0.0);
        if (tol > 0.0) {
            uint64_t z = s->limit_jitter_seed * 0x9E3779B97F4A7C15ull ^ ((uint64_t)w->e << 32) ^
                         ((uint64_t)j << 20) ^ w->ncall;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;   /* splitmix64 finaliser */
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            z ^= z >> 31;
            q += tol * (2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0);
        }
        w->ncall++;
    }
    double qd = axis_rel_vel(w, jt, c, angular);
    double meff = axis_meff(w, jt, c, angular);
    double blo = biased ? fmax(lo - q, 0.0) / h : 0.0;
    double bhi = biased ? fmax(q - hi, 0.0) / h : 0.0;
    note_margin(s, w->e, 0, fmin(fabs(q - lo) / fmax(1.0, fabs(lo)), fabs(q - hi) / fmax(1.0, fabs(hi))));
    double lam = 0.0;
    int viol = 0;
    if (q < lo) { lam = fmax(meff * (blo - qd), 0.0); viol = 1; }
    if (q > hi) { lam = -fmax(meff * (bhi + qd), 0.0); viol = 1; }
    if (!viol) return;
    apply_axis_impulse(w, jt, c, lam, angular);
    w->dof_impulse[jt->dof] += lam;
}

static void skew_sym_term(double *K, const double *r, const double *I) {
    /* K -= [r]x I [r]x */
    double S[9] = {0, -r[2], r[1], r[2], 0, -r[0], -r[1], r[0], 0};
    double T[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            T[3 * i + j] = S[3 * i] * I[j] + S[3 * i + 1] * I[3 + j] + S[3 * i + 2] * I[6 + j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            K[3 * i + j] -= T[3 * i] * S[j] + T[3 * i + 1] * S[3 + j] + T[3 * i + 2] * S[6 + j];
}

static void solve_point3(envw *w, int j, double h, int biased) { /* 872-890 */
    const bso_joint *jt = &w->s->joints[j];
    const jctx *c = &w->jc[j];
    int p = jt->parent, ch = jt->child;
    double vp[3], vc[3], rhs[3], K[9] = {0};
    vel_at(w, p, c->rp, vp);
    vel_at(w, ch, c->rc, vc);
    for (int k = 0; k < 3; ++k) {
        double target = biased ? -c->perr0[k] / h : 0.0;
        rhs[k] = target - (vc[k] - vp[k]);
    }
    double m = imass(w, p) + imass(w, ch);
    K[0] = K[4] = K[8] = m;
    skew_sym_term(K, c->rp, w->invI + 9 * p);
    skew_sym_term(K, c->rc, w->invI + 9 * ch);
    solve_n(3, K, rhs);
    apply_linear(w, ch, c->rc, rhs, 1.0);
    apply_linear(w, p, c->rp, rhs, -1.0);
}

static void solve_angular(envw *w, int j, double h, int biased, int lock) { /* 892-906 */
    const bso_joint *jt = &w->s->joints[j];
    const jctx *c = &w->jc[j];
    int p = jt->parent, ch = jt->child;
    const double *A[3] = {c->t1, c->t2, c->axis};
    int n = lock ? 3 : 2;
    double I[9], rel[3], d[3], K[9], rhs[3], L[3] = {0, 0, 0};
    for (int i = 0; i < 9; ++i) I[i] = w->invI[9 * p + i] + w->invI[9 * ch + i];
    for (int k = 0; k < 3; ++k) {
        rel[k] = w->w[3 * ch + k] - w->w[3 * p + k];
        d[k] = (biased ? -c->rerr0[k] / h : 0.0) - rel[k];
    }
    for (int a = 0; a < n; ++a) {
        for (int b = 0; b < n; ++b) K[a * n + b] = vMv(A[a], I, A[b]);
        rhs[a] = dot3(A[a], d);
    }
    solve_n(n, K, rhs);
    for (int a = 0; a < n; ++a)
        for (int k = 0; k < 3; ++k) L[k] += rhs[a] * A[a][k];
    apply_angular(w, ch, L, 1.0);
    apply_angular(w, p, L, -1.0);
}

static void solve_prismatic_perp(envw *w, int j, double h, int biased) { /* 908-928 */
    const bso_joint *jt = &w->s->joints[j];
    const jctx *c = &w->jc[j];
    int p = jt->parent, ch = jt->child;
    const double *T[2] = {c->t1, c->t2};
    double vp[3], vc[3], d[3], K[4], rhs[2], P[3] = {0, 0, 0};
    vel_at(w, p, c->rp, vp);
    vel_at(w, ch, c->rc, vc);
    for (int k = 0; k < 3; ++k) d[k] = (biased ? -c->perr0[k] / h : 0.0) - (vc[k] - vp[k]);
    double m = imass(w, p) + imass(w, ch);
    double rpt[2][3], rct[2][3];
    for (int a = 0; a < 2; ++a) { cross3(rpt[a], c->rp, T[a]); cross3(rct[a], c->rc, T[a]); }
    for (int a = 0; a < 2; ++a) {
        for (int b = 0; b < 2; ++b)
            K[2 * a + b] = dot3(T[a], T[b]) * m + vMv(rpt[a], w->invI + 9 * p, rpt[b]) +
                           vMv(rct[a], w->invI + 9 * ch, rct[b]);
        rhs[a] = dot3(T[a], d);
    }
    solve_n(2, K, rhs);
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 3; ++k) P[k] += rhs[a] * T[a][k];
    apply_linear(w, ch, c->rc, P, 1.0);
    apply_linear(w, p, c->rp, P, -1.0);
}

static void contact_rel_vel(const envw *w, const cctx *c, double *out) { /* 985-991 */
    vel_at(w, c->body, c->r, out);
    if (c->body_a >= 0) {
        double va[3];
        vel_at(w, c->body_a, c->ra, va);
        for (int k = 0; k < 3; ++k) out[k] -= va[k];
    }
}
static double contact_meff(const envw *w, const cctx *c, const double *d) { /* 993-1006 */
    double a[3];
    cross3(a, c->r, d);
    double k = imass(w, c->body) + vMv(a, w->invI + 9 * c->body, a);
    if (c->body_a >= 0) {
        double b[3];
        cross3(b, c->ra, d);
        k = imass(w, c->body_a) + imass(w, c->body) + vMv(b, w->invI + 9 * c->body_a, b) +
            vMv(a, w->invI + 9 * c->body, a);
    }
    return 1.0 / (k > 1e-12 ? k : 1e-12);
}
static void contact_apply(envw *w, const cctx *c, const double *P) { /* 1008-1019 */
    apply_linear(w, c->body, c->r, P, 1.0);
    if (c->body_a >= 0) apply_linear(w, c->body_a, c->ra, P, -1.0);
}

static void solve_contact(envw *w, cctx *c, int biased) { /* 930-983 */
    const bso_params *pp = &w->s->params;
    if (!c->active) return;
    double v[3];
    contact_rel_vel(w, c, v);
    double vn = dot3(c->n, v);
    double depth = c->depth0;
    if (biased) {
        double d[3];
        for (int k = 0; k < 3; ++k) d[k] = w->dpos[3 * c->body + k] - (c->body_a >= 0 ? w->dpos[3 * c->body_a + k] : 0.0);
        depth = c->depth0 + dot3(c->n, d) * -1.0;
    }
    double bias = biased ? pp->max_bias * fmax(depth, 0.0) / pp->dt : 0.0;
    double target = fmax(c->rest, bias);
    double mn = contact_meff(w, c, c->n);
    double dl = mn * (target - vn);
    double nl = fmax(c->lam_n + dl, 0.0);
    dl = nl - c->lam_n;
    c->lam_n = c->lam_n + dl;
    double P[3] = {c->n[0] * dl, c->n[1] * dl, c->n[2] * dl};
    contact_apply(w, c, P);

    double t1[3], t2[3], rt[3];
    tangents(t1, t2, c->n);
    contact_rel_vel(w, c, rt);
    double vt1 = dot3(t1, rt), vt2 = dot3(t2, rt);
    double mu = hypot(vt1, vt2) > 1e-3 ? w->s->mu_dynamic[w->e] : w->s->mu_static[w->e];
    note_margin(w->s, w->e, 2, hypot(vt1, vt2) - 1e-3);
    if (biased && c->body_a < 0) {
        double te[3];
        for (int k = 0; k < 3; ++k) te[k] = c->terr0[k] + w->dpos[3 * c->body + k];
        vt1 = vt1 + dot3(t1, te) / pp->dt;
        vt2 = vt2 + dot3(t2, te) / pp->dt;
    }
    double m1 = contact_meff(w, c, t1), m2 = contact_meff(w, c, t2);
    double c0 = c->lam_t[0] + (-m1 * vt1), c1 = c->lam_t[1] + (-m2 * vt2);
    double lim = mu * c->lam_n;
    double nrm = sqrt(c0 * c0 + c1 * c1);
    double sc = nrm > lim ? lim / fmax(nrm, 1e-12) : 1.0;
    c0 *= sc;
    c1 *= sc;
    double d0 = c0 - c->lam_t[0], d1 = c1 - c->lam_t[1];
    c->lam_t[0] += d0;
    c->lam_t[1] += d1;
    double Q[3];
    for (int k = 0; k < 3; ++k) Q[k] = t1[k] * d0 + t2[k] * d1;
    contact_apply(w, c, Q);
}

static void solve_pass(envw *w, double h, int biased) { /* 760-775 */
    const bso_scene *s = w->s;
    for (int j = 0; j < s->J; ++j) {
        int kind = s->joints[j].kind;
        solve_drive(w, j, h, biased);
        if (kind == K_REV || kind == K_SPH || kind == K_FIXED) solve_point3(w, j, h, biased);
        if (kind == K_REV) solve_angular(w, j, h, biased, 0);
        else if (kind == K_FIXED) solve_angular(w, j, h, biased, 1);
        else if (kind == K_PRISM) { solve_angular(w, j, h, biased, 1); solve_prismatic_perp(w, j, h, biased); }
        solve_limit(w, j, h, biased);
    }
    for (int i = 0; i < s->P + s->Q; ++i) solve_contact(w, &w->cc[i], biased);
}

/* ------------------------------------------------------------- contacts */
static void plane_geometry(const bso_scene *s, int e, int i, const double *pos, const double *quat,
                           double *point, double *depth, int *active) { /* 467-479 */
    int b = s->plane_body[i];
    double c[3];
    qrot(c, quat + 4 * b, s->plane_off + 3 * ((size_t)i * s->E + e));
    for (int k = 0; k < 3; ++k) c[k] += pos[3 * b + k];
    double rad = s->plane_rad[(size_t)i * s->E + e];
    double gap = c[2] - rad;
    *depth = s->params.rest_offset - gap;
    point[0] = c[0]; point[1] = c[1]; point[2] = c[2] - rad;
    *active = *depth > -s->params.solver_offset_slop;
    note_margin(s, e, 1, *depth + s->params.solver_offset_slop);
    note_margin(s, e, 1, *depth + s->params.friction_offset_threshold);
}
/* Pair slot narrow phase.  Kind 0 (SS) is the reference's sphere-sphere pair
   (physics.py:481-497).  Kinds 1-3 are NOT in the reference: box / capsule
   pairs of this build (sphere|corner vs box, sphere|corner vs capsule
   segment, capsule vs capsule), restated here independently of the CUDA code
   so the GPU path has a float64 checker (parity unpinned to the reference). */
static void pair_geometry(const bso_scene *s, int e, int i, const double *pos, const double *quat,
                          double *point, double *n, double *depth, int *active) { /* 481-497 */
    int a = s->pair_body[2 * i], b = s->pair_body[2 * i + 1];
    int kind = s->pair_kind[i];
    const double *ext = s->pair_ext + 4 * i;
    const double *off = s->pair_off + 6 * ((size_t)i * s->E + e);
    double ra = s->pair_rad[2 * ((size_t)i * s->E + e)], rb = s->pair_rad[2 * ((size_t)i * s->E + e) + 1];
    double ca[3], cb[3], d[3], gap;
    qrot(ca, quat + 4 * a, off);
    qrot(cb, quat + 4 * b, off + 3);
    for (int k = 0; k < 3; ++k) { ca[k] += pos[3 * a + k]; cb[k] += pos[3 * b + k]; }
    if (kind == 1) { /* sphere centre ca vs box centred at cb, axes of body b */
        double rel[3], pl[3], cl[3], dl[3], nl[3] = {0, 0, 0}, qi[4];
        for (int k = 0; k < 3; ++k) rel[k] = ca[k] - cb[k];
        qconj(qi, quat + 4 * b);
        qrot(pl, qi, rel);
        for (int k = 0; k < 3; ++k) { cl[k] = clampd(pl[k], -ext[k], ext[k]); dl[k] = pl[k] - cl[k]; }
        double dist = sqrt(dot3(dl, dl));
        if (dist > 1e-12) {
            for (int k = 0; k < 3; ++k) nl[k] = dl[k] / dist;
            gap = dist - ra;
        } else {
            int best = 0;
            double f[3];
            for (int k = 0; k < 3; ++k) f[k] = ext[k] - fabs(pl[k]);
            if (f[1] < f[best]) best = 1;
            if (f[2] < f[best]) best = 2;
            nl[best] = pl[best] < 0 ? -1.0 : 1.0;
            gap = -f[best] - ra;
        }
        double nw[3];
        qrot(nw, quat + 4 * b, nl);
        for (int k = 0; k < 3; ++k) n[k] = -nw[k];
    } else {
        if (kind == 2 || kind == 3) { /* segment(s) along the bodies' local z */
            double ez[3] = {0, 0, 1}, ub[3], ua[3], d0[3];
            qrot(ub, quat + 4 * b, ez);
            double hb = ext[1], t;
            if (kind == 3) {
                qrot(ua, quat + 4 * a, ez);
                double ha = ext[0];
                for (int k = 0; k < 3; ++k) d0[k] = ca[k] - cb[k];
                double bb = dot3(ua, ub), dA = dot3(ua, d0), dB = dot3(ub, d0);
                double den = 1.0 - bb * bb;
                double sa = den > 1e-9 ? clampd((bb * dB - dA) / den, -ha, ha) : 0.0;
                t = clampd(dB + bb * sa, -hb, hb);
                sa = clampd(bb * t - dA, -ha, ha);
                for (int k = 0; k < 3; ++k) ca[k] += ua[k] * sa;
            } else {
                for (int k = 0; k < 3; ++k) d0[k] = ca[k] - cb[k];
                t = clampd(dot3(d0, ub), -hb, hb);
            }
            for (int k = 0; k < 3; ++k) cb[k] += ub[k] * t;
        }
        for (int k = 0; k < 3; ++k) d[k] = cb[k] - ca[k];
        double dist = sqrt(dot3(d, d));
        double dd = dist > 1e-12 ? dist : 1.0;
        for (int k = 0; k < 3; ++k) n[k] = d[k] / dd;
        gap = dist - (ra + rb);
    }
    *depth = s->params.rest_offset - gap;
    for (int k = 0; k < 3; ++k) point[k] = ca[k] + n[k] * (ra + 0.5 * gap);
    *active = *depth > -s->params.solver_offset_slop;
    note_margin(s, e, 1, *depth + s->params.solver_offset_slop);
}

/* ------------------------------------------------------------- tendons */
static double spring_force(const bso_tendon *t, double L, double Ld) { /* tendons.py:52-62 */
    double f = -t->stiffness * (L - t->rest_length) - t->damping * Ld;
    if (t->has_limits) {
        double below = fmax(t->limit_lo - L, 0.0), above = fmax(L - t->limit_hi, 0.0);
        f = f + t->limit_stiffness * below - t->limit_stiffness * above;
        if (below > 0 || above > 0) f = f - t->damping * Ld;
    }
    return f;
}

static void apply_tendons(envw *w) { /* physics.py:598-653 */
    const bso_scene *s = w->s;
    double dt = s->params.dt;
    const double *dof = s->dof_state + 2 * (size_t)w->e * s->D;
    for (int ti = 0; ti < s->T; ++ti) {
        const bso_tendon *t = &s->tendons[ti];
        const bso_telem *el = s->telems + t->first;
        if (t->kind == 0) {
            /* lengths and rates along the tendon tree (tendons.py:40-49, 65-95) */
            double len[64], rate[64], qf_by_dof[64];
            int ndof = 0;
            int dofs[64];
            for (int i = 0; i < t->count; ++i) {
                double pl = el[i].parent >= 0 ? len[el[i].parent] : 0.0;
                double pr = el[i].parent >= 0 ? rate[el[i].parent] : 0.0;
                len[i] = pl + el[i].v[0] * dof[2 * el[i].index];
                rate[i] = pr + el[i].v[0] * dof[2 * el[i].index + 1];
            }
            /* generalized force per local dof (accumulated), in DOF order */
            for (int i = 0; i < t->count; ++i) {
                double q = el[i].v[0] * spring_force(t, len[i], rate[i]);
                int found = -1;
                for (int k = 0; k < ndof; ++k) if (dofs[k] == el[i].index) found = k;
                if (found < 0) { found = ndof++; dofs[found] = el[i].index; qf_by_dof[found] = 0.0; }
                qf_by_dof[found] += q;
            }
            /* apply in ascending dof order (physics.py:614-620) */
            for (int pass = 0; pass < ndof; ++pass) {
                int best = -1;
                for (int k = 0; k < ndof; ++k)
                    if (dofs[k] >= 0 && (best < 0 || dofs[k] < dofs[best])) best = k;
                double qf = qf_by_dof[best];
                int jslot = -1;
                for (int i = 0; i < t->count; ++i) if (el[i].index == dofs[best]) jslot = el[i].joint;
                dofs[best] = -1 - dofs[best];
                if (qf == 0.0) continue;
                const bso_joint *jt = &s->joints[jslot];
                int ci = jt->child, ri = t->reaction_body;
                double jq[4], aw[3], P[3];
                qmul(jq, w->quat + 4 * jt->parent, jt->origin_quat);
                qrot(aw, jq, jt->axis);
                for (int k = 0; k < 3; ++k) P[k] = aw[k] * qf * dt;
                if (jt->kind == K_REV) {
                    apply_angular(w, ci, P, 1.0);
                    apply_angular(w, ri, P, -1.0);
                } else {
                    for (int k = 0; k < 3; ++k) {
                        w->v[3 * ci + k] += P[k] * imass(w, ci);
                        w->v[3 * ri + k] -= P[k] * imass(w, ri);
                    }
                }
            }
        } else {
            /* spatial: all entries from the pre-application state (tendons.py:148-188) */
            double pts[64][3], vel[64][3];
            for (int i = 0; i < t->count; ++i) {
                int b = el[i].index;
                double r[3];
                qrot(pts[i], w->quat + 4 * b, el[i].v);
                for (int k = 0; k < 3; ++k) pts[i][k] += w->pos[3 * b + k];
                for (int k = 0; k < 3; ++k) r[k] = pts[i][k] - w->pos[3 * b + k];
                vel_at(w, b, r, vel[i]);
            }
            const int32_t *pth = s->spatial_paths + s->spatial_path_off[ti];
            int npaths = pth[0];
            const int32_t *cur = pth + 1;
            double ent_f[128][3];
            int ent_i[128], nent = 0;
            for (int pi = 0; pi < npaths; ++pi) {
                int len = cur[0];
                const int32_t *ix = cur + 1;
                double L = 0.0, Ld = 0.0;
                for (int k = 1; k < len; ++k) {
                    int pa = ix[k - 1], ch = ix[k];
                    double d[3], dv[3];
                    for (int m = 0; m < 3; ++m) { d[m] = pts[ch][m] - pts[pa][m]; dv[m] = vel[ch][m] - vel[pa][m]; }
                    double dist = sqrt(dot3(d, d));
                    double sf = dist > 1e-12 ? dist : 1.0;
                    double u[3] = {d[0] / sf, d[1] / sf, d[2] / sf};
                    L = L + el[ch].v[3] * dist;
                    Ld = Ld + el[ch].v[3] * dot3(dv, u);
                }
                double f = spring_force(t, L, Ld);
                int leaf = ix[len - 1], root = ix[0];
                double dl[3], dr[3];
                for (int m = 0; m < 3; ++m) { dl[m] = pts[ix[len - 2]][m] - pts[leaf][m]; dr[m] = pts[ix[1]][m] - pts[root][m]; }
                double nl = sqrt(dot3(dl, dl)), nr = sqrt(dot3(dr, dr));
                nl = nl > 1e-12 ? nl : 1.0;
                nr = nr > 1e-12 ? nr : 1.0;
                for (int m = 0; m < 3; ++m) { ent_f[nent][m] = -f * (dl[m] / nl); }
                ent_i[nent++] = leaf;
                for (int m = 0; m < 3; ++m) { ent_f[nent][m] = -f * (dr[m] / nr); }
                ent_i[nent++] = root;
                cur += 1 + len;
            }
            for (int k = 0; k < nent; ++k) {
                int ai = ent_i[k], b = el[ai].index;
                double r[3], F[3], tq[3];
                for (int m = 0; m < 3; ++m) { r[m] = pts[ai][m] - w->pos[3 * b + m]; F[m] = dt * ent_f[k][m]; }
                double im = imass(w, b);
                for (int m = 0; m < 3; ++m) w->v[3 * b + m] += dt * ent_f[k][m] * im;
                cross3(tq, r, ent_f[k]);
                double u[3];
                mv3(u, w->invI + 9 * b, tq);
                for (int m = 0; m < 3; ++m) w->w[3 * b + m] += dt * u[m];
                (void)F;
            }
        }
    }
}

/* ----------------------------------------------------------- packing */
static void pack_env(const bso_scene *s, int e) { /* 1039-1046 */
    for (int b = 0; b < s->B; ++b) {
        size_t g = (size_t)e * s->B + b;
        double *row = s->body_state + 13 * g;
        memcpy(row, s->pos + 3 * g, 3 * sizeof(double));
        memcpy(row + 3, s->quat + 4 * g, 4 * sizeof(double));
        memcpy(row + 7, s->linvel + 3 * g, 3 * sizeof(double));
        memcpy(row + 10, s->angvel + 3 * g, 3 * sizeof(double));
    }
    for (int a = 0; a < s->A; ++a)
        memcpy(s->root_state + 13 * ((size_t)e * s->A + a),
               s->body_state + 13 * ((size_t)e * s->B + s->actor_body_offset[a]), 13 * sizeof(double));
}

static int env_finite(const bso_scene *s, int e) {
    for (int i = 0; i < 13 * s->B; ++i)
        if (!isfinite(s->body_state[13 * (size_t)e * s->B + i])) return 0;
    return 1;
}

static void sanitize_env(const bso_scene *s, int e) { /* 1080-1087 */
    for (int b = 0; b < s->B; ++b) {
        size_t g = (size_t)e * s->B + b;
        double *p = s->pos + 3 * g, *q = s->quat + 4 * g, *lv = s->linvel + 3 * g, *av = s->angvel + 3 * g;
        for (int k = 0; k < 3; ++k) {
            if (!isfinite(p[k])) p[k] = 0.0;
            if (!isfinite(lv[k])) lv[k] = 0.0;
            if (!isfinite(av[k])) av[k] = 0.0;
        }
        for (int k = 0; k < 4; ++k) if (!isfinite(q[k])) q[k] = 0.0;
        double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
        if (n < 1e-9) { q[0] = q[1] = q[2] = 0.0; q[3] = 1.0; }
        qnormalize(q);
    }
}

/* ------------------------------------------------------------- the step */
static void step_env(const bso_scene *s, int e, envw *w) { /* physics.py:538-592 */
    const bso_params *pp = &s->params;
    const int B = s->B;
    double dt = pp->dt;
    int N = pp->position_iterations;
    double h = dt / N;
    w->e = e;
    w->ncall = 0;
    w->pos = s->pos + 3 * (size_t)e * B;
    w->quat = s->quat + 4 * (size_t)e * B;
    w->v = s->linvel + 3 * (size_t)e * B;
    w->w = s->angvel + 3 * (size_t)e * B;
    const double *g = s->gravity + 3 * (size_t)e;

    for (int b = 0; b < B; ++b) {
        double im = imass(w, b);
        if (im > 0) for (int k = 0; k < 3; ++k) w->v[3 * b + k] += dt * g[k];
    }
    for (int b = 0; b < B; ++b) {
        double im = imass(w, b);
        const double *f = s->ctrl_body_force + 3 * ((size_t)e * B + b);
        for (int k = 0; k < 3; ++k) w->v[3 * b + k] += dt * clampd(f[k], -pp->max_force, pp->max_force) * im;
    }
    inv_inertia_world(w, w->quat);
    for (int b = 0; b < B; ++b) {
        const double *tq = s->ctrl_body_torque + 3 * ((size_t)e * B + b);
        double t[3] = {clampd(tq[0], -pp->max_force, pp->max_force), clampd(tq[1], -pp->max_force, pp->max_force),
                       clampd(tq[2], -pp->max_force, pp->max_force)};
        double u[3];
        mv3(u, w->invI + 9 * b, t);
        for (int k = 0; k < 3; ++k) w->w[3 * b + k] += dt * u[k];
    }
    if (s->T) apply_tendons(w);
    double ld = fmax(0.0, 1.0 - pp->linear_damping * dt), ad = fmax(0.0, 1.0 - pp->angular_damping * dt);
    for (int i = 0; i < 3 * B; ++i) { w->v[i] *= ld; w->w[i] *= ad; }

    read_dofs_env(s, e);

    /* freeze (657-716) */
    for (int j = 0; j < s->J; ++j) {
        const bso_joint *jt = &s->joints[j];
        w->jc[j].has_q0 = jt->dof >= 0 && (jt->kind == K_REV || jt->kind == K_PRISM);
        if (w->jc[j].has_q0) w->jc[j].q0 = s->dof_state[2 * ((size_t)e * s->D + jt->dof)];
    }
    joint_geometry(w, w->pos, w->quat, 0);
    for (int i = 0; i < s->P; ++i) {
        cctx *c = &w->cc[i];
        c->body = s->plane_body[i];
        c->body_a = -1;
        plane_geometry(s, e, i, w->pos, w->quat, c->point, &c->depth0, &c->active);
        c->n[0] = 0; c->n[1] = 0; c->n[2] = 1;
        for (int k = 0; k < 3; ++k) c->r[k] = c->point[k] - w->pos[3 * c->body + k];
        double v[3];
        vel_at(w, c->body, c->r, v);
        double vn = dot3(c->n, v);
        c->rest = vn < -pp->bounce_threshold ? -pp->restitution * vn : 0.0;
        note_margin(s, e, 3, vn + pp->bounce_threshold);
        const double *an = s->friction_anchor + 3 * ((size_t)i * s->E + e);
        if (isnan(an[0])) { c->terr0[0] = c->terr0[1] = c->terr0[2] = 0.0; }
        else for (int k = 0; k < 3; ++k) c->terr0[k] = c->point[k] - an[k];
        c->terr0[2] = 0.0;
        c->lam_n = 0; c->lam_t[0] = c->lam_t[1] = 0;
    }
    for (int i = 0; i < s->Q; ++i) {
        cctx *c = &w->cc[s->P + i];
        c->body_a = s->pair_body[2 * i];
        c->body = s->pair_body[2 * i + 1];
        pair_geometry(s, e, i, w->pos, w->quat, c->point, c->n, &c->depth0, &c->active);
        double va[3], vb[3], d[3];
        for (int k = 0; k < 3; ++k) { c->ra[k] = c->point[k] - w->pos[3 * c->body_a + k]; c->r[k] = c->point[k] - w->pos[3 * c->body + k]; }
        vel_at(w, c->body_a, c->ra, va);
        vel_at(w, c->body, c->r, vb);
        for (int k = 0; k < 3; ++k) d[k] = vb[k] - va[k];
        double vn = dot3(c->n, d);
        c->rest = vn < -pp->bounce_threshold ? -pp->restitution * vn : 0.0;
        note_margin(s, e, 3, vn + pp->bounce_threshold);
        c->lam_n = 0; c->lam_t[0] = c->lam_t[1] = 0;
        c->terr0[0] = c->terr0[1] = c->terr0[2] = 0;
    }
    memset(w->dof_impulse, 0, sizeof(double) * s->D);
    memset(w->dpos, 0, sizeof(double) * 3 * B);
    memset(w->dang, 0, sizeof(double) * 3 * B);

    for (int k = 0; k < N; ++k) { /* 567-572 */
        if (k) refresh(w, 1);
        solve_pass(w, h, 1);
        for (int i = 0; i < 3 * B; ++i) { w->dpos[i] += w->v[i] * h; w->dang[i] += w->w[i] * h; }
    }
    for (int b = 0; b < B; ++b) { /* 574-575 */
        double dq[4];
        for (int k = 0; k < 3; ++k) w->pos[3 * b + k] += w->dpos[3 * b + k];
        qexp(dq, w->dang + 3 * b);
        qmul(w->quat + 4 * b, dq, w->quat + 4 * b);
        qnormalize(w->quat + 4 * b);
    }
    refresh(w, 0);
    for (int k = 0; k < pp->velocity_iterations; ++k) solve_pass(w, h, 0);

    for (int b = 0; b < B; ++b) { /* 584-587 */
        double *lv = w->v + 3 * b, *av = w->w + 3 * b;
        double ln = sqrt(dot3(lv, lv)), an = sqrt(dot3(av, av));
        double sl = fmin(1.0, pp->max_linear_velocity / fmax(ln, 1e-12));
        double sa = fmin(1.0, pp->max_angular_velocity / fmax(an, 1e-12));
        for (int k = 0; k < 3; ++k) { lv[k] *= sl; av[k] *= sa; }
    }
    for (int i = 0; i < s->P; ++i) { /* 1021-1033 */
        const cctx *c = &w->cc[i];
        double *an = s->friction_anchor + 3 * ((size_t)i * s->E + e);
        int near = c->depth0 > -pp->friction_offset_threshold;
        if (near && isnan(an[0])) memcpy(an, c->point, 3 * sizeof(double));
        if (!near) an[0] = an[1] = an[2] = NAN;
    }

    /* refresh_buffers(ctx) (1037-1071) */
    read_dofs_env(s, e);
    pack_env(s, e);
    double *net = s->net_contact + 3 * (size_t)e * B;
    double tq[64][3];
    for (int b = 0; b < B; ++b) for (int k = 0; k < 3; ++k) { net[3 * b + k] = 0.0; tq[b][k] = 0.0; }
    for (int i = 0; i < s->P + s->Q; ++i) {
        const cctx *c = &w->cc[i];
        double t1[3], t2[3], P[3], F[3], x[3];
        tangents(t1, t2, c->n);
        for (int k = 0; k < 3; ++k) {
            P[k] = c->n[k] * c->lam_n + t1[k] * c->lam_t[0] + t2[k] * c->lam_t[1];
            F[k] = P[k] / dt;
        }
        for (int k = 0; k < 3; ++k) net[3 * c->body + k] += F[k];
        cross3(x, c->r, F);
        for (int k = 0; k < 3; ++k) tq[c->body][k] += x[k];
        if (c->body_a >= 0) {
            double nF[3] = {-F[0], -F[1], -F[2]};
            for (int k = 0; k < 3; ++k) net[3 * c->body_a + k] += nF[k];
            cross3(x, c->ra, nF);
            for (int k = 0; k < 3; ++k) tq[c->body_a][k] += x[k];
        }
    }
    for (int d = 0; d < s->D; ++d) s->dof_force[(size_t)e * s->D + d] = w->dof_impulse[d] / dt;
    for (int k = 0; k < s->S; ++k) {
        int b = s->sensor_body[k];
        double qi[4];
        qconj(qi, w->quat + 4 * b);
        double *row = s->sensor_forces + 6 * ((size_t)e * s->S + k);
        qrot(row, qi, net + 3 * b);
        qrot(row + 3, qi, tq[b]);
    }
    /* _flag_nonfinite (1073-1088) */
    if (!env_finite(s, e)) {
        s->nonfinite[e] = 1;
        sanitize_env(s, e);
        read_dofs_env(s, e);
        pack_env(s, e);
    }
}

void bso_step(const bso_scene *s, int threads) {
    int B = s->B, J = s->J, C = s->P + s->Q, D = s->D;
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel num_threads(threads)
#endif
    {
        envw w;
        memset(&w, 0, sizeof w);
        w.s = s;
        w.invI = malloc(sizeof(double) * 9 * B);
        w.dpos = malloc(sizeof(double) * 3 * B);
        w.dang = malloc(sizeof(double) * 3 * B);
        w.pos_eff = malloc(sizeof(double) * 3 * B);
        w.quat_eff = malloc(sizeof(double) * 4 * B);
        w.jc = malloc(sizeof(jctx) * (J ? J : 1));
        w.cc = malloc(sizeof(cctx) * (C ? C : 1));
        w.dof_impulse = malloc(sizeof(double) * (D ? D : 1));
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int e = 0; e < s->E; ++e) step_env(s, e, &w);
        free(w.invI); free(w.dpos); free(w.dang); free(w.pos_eff); free(w.quat_eff);
        free(w.jc); free(w.cc); free(w.dof_impulse);
    }
    (void)threads;
}

void bso_forward_kinematics(const bso_scene *s, const uint8_t *env_mask, uint32_t actor_mask) {
    for (int e = 0; e < s->E; ++e)
        if (!env_mask || env_mask[e]) fk_env(s, e, actor_mask);
}

void bso_read_dof_states(const bso_scene *s) {
    for (int e = 0; e < s->E; ++e) read_dofs_env(s, e);
}

void bso_refresh_buffers(const bso_scene *s) {
    for (int e = 0; e < s->E; ++e) { read_dofs_env(s, e); pack_env(s, e); }
}

void bso_contact_geometry(const bso_scene *s, uint8_t *active, double *depth, double *point, double *normal) {
    for (int i = 0; i < s->P + s->Q; ++i)
        for (int e = 0; e < s->E; ++e) {
            size_t o = (size_t)i * s->E + e;
            const double *pos = s->pos + 3 * (size_t)e * s->B, *quat = s->quat + 4 * (size_t)e * s->B;
            int act;
            if (i < s->P) {
                plane_geometry(s, e, i, pos, quat, point + 3 * o, depth + o, &act);
                normal[3 * o] = 0; normal[3 * o + 1] = 0; normal[3 * o + 2] = 1;
            } else {
                pair_geometry(s, e, i - s->P, pos, quat, point + 3 * o, normal + 3 * o, depth + o, &act);
            }
            active[o] = (uint8_t)act;
        }
}

int bso_version(void) { return 1; }
