// bsim_math.cuh -- vector / quaternion helpers (host+device), templated on
// the scalar type R (float: the fast path; double: the exact-parity path on
// B200's FP64 units).
//
// Conventions follow the reference spatial module
// (/root/reference/pkg/src/batchsim/spatial.py:18-162): quaternions are
// (x, y, z, w), Hamilton product, rotation v' = v + w t + u x t with t = 2 u x v.
#pragma once

#include <cmath>
#include <cstdint>

#ifndef __CUDACC__
#define __host__
#define __device__
#define __forceinline__ inline
#endif

#define BS_HD __host__ __device__ __forceinline__
// large per-item phase functions: one copy in the binary (instruction-cache footprint)
#define BS_NI __host__ __device__ __noinline__

namespace bsim {

// scalar helpers resolving to the float or double libm entry points
BS_HD float r_sqrt(float x) { return sqrtf(x); }
BS_HD double r_sqrt(double x) { return sqrt(x); }
BS_HD float r_sin(float x) { return sinf(x); }
BS_HD double r_sin(double x) { return sin(x); }
BS_HD float r_cos(float x) { return cosf(x); }
BS_HD double r_cos(double x) { return cos(x); }
// fp32 sin / cos of a half rotation angle.  TGS deltas rotate a body by far
// less than pi/4 per pass, where degree-9/8 Taylor polynomials are exact to
// fp32 rounding (truncation < 3e-10) and cost a handful of FMAs instead of
// sincosf's range reduction; larger angles take the libm path.
BS_HD void r_sincos(float x, float &s, float &c) {
#if defined(__CUDA_ARCH__) && !defined(BSIM_IEEE_FP32)
    if (fabsf(x) < 0.78539816f) {
        const float x2 = x * x;
        s = x * (1.0f + x2 * (-1.0f / 6.0f + x2 * (1.0f / 120.0f + x2 * (-1.0f / 5040.0f + x2 * (1.0f / 362880.0f)))));
        c = 1.0f + x2 * (-0.5f + x2 * (1.0f / 24.0f + x2 * (-1.0f / 720.0f + x2 * (1.0f / 40320.0f))));
    } else {
        sincosf(x, &s, &c);
    }
#else
    s = sinf(x); c = cosf(x);
#endif
}
BS_HD void r_sincos(double x, double &s, double &c) {
#if defined(__CUDA_ARCH__)
    sincos(x, &s, &c);
#else
    s = sin(x); c = cos(x);
#endif
}
BS_HD float r_atan2(float y, float x) { return atan2f(y, x); }
BS_HD double r_atan2(double y, double x) { return atan2(y, x); }
BS_HD float r_floor(float x) { return floorf(x); }
BS_HD double r_floor(double x) { return floor(x); }
BS_HD float r_abs(float x) { return fabsf(x); }
BS_HD double r_abs(double x) { return fabs(x); }
BS_HD float r_max(float a, float b) { return fmaxf(a, b); }
BS_HD double r_max(double a, double b) { return fmax(a, b); }
BS_HD float r_min(float a, float b) { return fminf(a, b); }
BS_HD double r_min(double a, double b) { return fmin(a, b); }
BS_HD float exp_r(float x) { return expf(x); }
BS_HD double exp_r(double x) { return exp(x); }
BS_HD float r_nan(float) { return nanf(""); }
// reciprocal / reciprocal square root: one MUFU op (+ multiply) on the fp32
// device path instead of an IEEE division sequence (<= 2 ulp; the fp32 parity
// budget is 1e-4); exact IEEE on the host and in the fp64 parity path.
#if defined(__CUDA_ARCH__) && !defined(BSIM_IEEE_FP32)   // BSIM_IEEE_FP32: build.py --ieee
BS_HD float r_rcp(float x) { return __fdividef(1.0f, x); }
BS_HD float r_rsqrt(float x) { return rsqrtf(x); }
#else
BS_HD float r_rcp(float x) { return 1.0f / x; }
BS_HD float r_rsqrt(float x) { return 1.0f / sqrtf(x); }
#endif
BS_HD double r_rcp(double x) { return 1.0 / x; }
BS_HD double r_rsqrt(double x) { return 1.0 / sqrt(x); }
BS_HD double r_nan(double) { return nan(""); }

template <class R> struct V3 {
    R x, y, z;
};
template <class R> struct Q4 {
    R x, y, z, w;
};
template <class R> struct S3 {  // symmetric 3x3: (xx, xy, xz, yy, yz, zz)
    R xx, xy, xz, yy, yz, zz;
};
template <class R> struct M3 {  // general 3x3, row-major
    R a00, a01, a02, a10, a11, a12, a20, a21, a22;
};

template <class R> BS_HD V3<R> v3(R x, R y, R z) { return V3<R>{x, y, z}; }
template <class G, class R> BS_HD S3<G> cs3(const S3<R> &m) {
    return S3<G>{(G)m.xx, (G)m.xy, (G)m.xz, (G)m.yy, (G)m.yz, (G)m.zz};
}
// error-free sum (Knuth TwoSum): a + b = s + e exactly, s = fl(a + b)
template <class R> BS_HD R two_sum(R a, R b, R &e) {
    const R s = a + b;
    const R bb = s - a;
    e = (a - (s - bb)) + (b - bb);
    return s;
}
// (a - b) + (c - d) + (f - g) for a ~ b, c ~ d O(1) and the result small:
// the two O(1) differences and their sum are carried with their rounding
// errors (TwoSum), so the result is accurate to ~1 ulp of ITSELF rather
// than of the O(1) operands (the TGS position error, bsim_step.cuh joint_item)
template <class R> BS_HD R cancel_sum(R a, R b, R c, R dd, R f, R g) {
    R e1, e2, e3;
    const R s1 = two_sum(a, -b, e1);
    const R s2 = two_sum(c, -dd, e2);
    const R h = two_sum(s1, s2, e3);
    return h + (((e1 + e2) + e3) + (f - g));
}
// precision conversions (the fp32 step's joint geometry is evaluated in double: bsim_step.cuh GeomT)
template <class G, class R> BS_HD V3<G> cv3(V3<R> a) { return V3<G>{(G)a.x, (G)a.y, (G)a.z}; }
template <class G, class R> BS_HD Q4<G> cq4(Q4<R> a) { return Q4<G>{(G)a.x, (G)a.y, (G)a.z, (G)a.w}; }

template <class R> BS_HD V3<R> zero3() { return V3<R>{R(0), R(0), R(0)}; }
template <class R> BS_HD V3<R> operator+(V3<R> a, V3<R> b) { return V3<R>{a.x + b.x, a.y + b.y, a.z + b.z}; }
template <class R> BS_HD V3<R> operator-(V3<R> a, V3<R> b) { return V3<R>{a.x - b.x, a.y - b.y, a.z - b.z}; }
template <class R> BS_HD V3<R> operator-(V3<R> a) { return V3<R>{-a.x, -a.y, -a.z}; }
template <class R> BS_HD V3<R> operator*(V3<R> a, R s) { return V3<R>{a.x * s, a.y * s, a.z * s}; }
template <class R> BS_HD R dot(V3<R> a, V3<R> b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
template <class R> BS_HD V3<R> cross(V3<R> a, V3<R> b) {
    return V3<R>{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <class R> BS_HD R norm(V3<R> a) { return r_sqrt(dot(a, a)); }

template <class R> BS_HD Q4<R> qmul(Q4<R> a, Q4<R> b) {
    return Q4<R>{a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y,
                 a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x,
                 a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w,
                 a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z};
}
template <class R> BS_HD Q4<R> qconj(Q4<R> q) { return Q4<R>{-q.x, -q.y, -q.z, q.w}; }
template <class R> BS_HD Q4<R> qnormalize(Q4<R> q) {
    R n2 = q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w;
    if (n2 > R(0)) {
        R in = r_rsqrt(n2);
        q.x = q.x * in; q.y = q.y * in; q.z = q.z * in; q.w = q.w * in;
    }
    return q;
}
template <class R> BS_HD V3<R> qvec(Q4<R> q) { return V3<R>{q.x, q.y, q.z}; }
template <class R> BS_HD V3<R> qrot(Q4<R> q, V3<R> v) {
    V3<R> u = qvec(q);
    V3<R> t = cross(u, v) * R(2);
    return v + t * q.w + cross(u, t);
}

// exp map of a rotation vector (spatial.py:143-152)
template <class R> BS_HD Q4<R> qexp(V3<R> v) {
    R ang = norm(v);
    V3<R> ax = v3(R(1), R(0), R(0));
    if (!(ang < R(1e-12))) ax = v * r_rcp(ang);
    R s, c;
    r_sincos(R(0.5) * ang, s, c);
    return Q4<R>{ax.x * s, ax.y * s, ax.z * s, c};
}
// exp map for |v| < 0.25 rad as even series in |v|^2 (no square root, no
// range reduction): sin(a/2)/a and cos(a/2) to degree 10 (truncation < 1e-13
// relative); larger rotations take qexp.
template <class R> BS_HD Q4<R> qexp_small(V3<R> v) {
    const R a2 = dot(v, v);
    if (!(a2 < R(0.0625))) return qexp(v);
    const R sa = R(0.5) + a2 * (R(-1.0 / 48) + a2 * (R(1.0 / 3840) + a2 * (R(-1.0 / 645120) + a2 * R(1.0 / 185794560))));
    const R c = R(1) + a2 * (R(-1.0 / 8) + a2 * (R(1.0 / 384) + a2 * (R(-1.0 / 46080) + a2 * R(1.0 / 10321920))));
    return Q4<R>{v.x * sa, v.y * sa, v.z * sa, c};
}
// normalisation of a quaternion whose norm is 1 to within ~1e-6 (one Newton
// step of 1/sqrt from 1: relative error 3/8 (n2 - 1)^2)
template <class R> BS_HD Q4<R> qnormalize_near(Q4<R> q) {
    const R n2 = q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w;
    const R e = n2 - R(1);
    const R in = R(1) - R(0.5) * e + R(0.375) * e * e;
    return Q4<R>{q.x * in, q.y * in, q.z * in, q.w * in};
}
// log map (spatial.py:155-162)
template <class R> BS_HD V3<R> qlog(Q4<R> q) {
    if (q.w < R(0)) q = Q4<R>{-q.x, -q.y, -q.z, -q.w};
    R n = r_sqrt(q.x * q.x + q.y * q.y + q.z * q.z);
    R ang = R(2) * r_atan2(n, q.w);
    R sc = n > R(1e-12) ? ang / n : R(2);
    return V3<R>{q.x * sc, q.y * sc, q.z * sc};
}

template <class R> BS_HD V3<R> smul(const S3<R> &m, V3<R> v) {
    return V3<R>{m.xx * v.x + m.xy * v.y + m.xz * v.z, m.xy * v.x + m.yy * v.y + m.yz * v.z,
                 m.xz * v.x + m.yz * v.y + m.zz * v.z};
}
template <class R> BS_HD S3<R> sadd(const S3<R> &a, const S3<R> &b) {
    return S3<R>{a.xx + b.xx, a.xy + b.xy, a.xz + b.xz, a.yy + b.yy, a.yz + b.yz, a.zz + b.zz};
}
// R diag(d) R^T from a unit quaternion (physics.py:594-596)
template <class R> BS_HD S3<R> world_inertia(Q4<R> q, V3<R> d) {
    R x = q.x, y = q.y, z = q.z, w = q.w;
    R r00 = 1 - 2 * (y * y + z * z), r01 = 2 * (x * y - z * w), r02 = 2 * (x * z + y * w);
    R r10 = 2 * (x * y + z * w), r11 = 1 - 2 * (x * x + z * z), r12 = 2 * (y * z - x * w);
    R r20 = 2 * (x * z - y * w), r21 = 2 * (y * z + x * w), r22 = 1 - 2 * (x * x + y * y);
    S3<R> m;
    m.xx = r00 * d.x * r00 + r01 * d.y * r01 + r02 * d.z * r02;
    m.xy = r00 * d.x * r10 + r01 * d.y * r11 + r02 * d.z * r12;
    m.xz = r00 * d.x * r20 + r01 * d.y * r21 + r02 * d.z * r22;
    m.yy = r10 * d.x * r10 + r11 * d.y * r11 + r12 * d.z * r12;
    m.yz = r10 * d.x * r20 + r11 * d.y * r21 + r12 * d.z * r22;
    m.zz = r20 * d.x * r20 + r21 * d.y * r21 + r22 * d.z * r22;
    return m;
}
// K += [r]x^T I [r]x  (== -[r]x I [r]x, physics.py:884-885)
template <class R> BS_HD void add_rIr(S3<R> &K, V3<R> r, const S3<R> &I) {
    // columns of [r]x: c0 = (0, r.z, -r.y), c1 = (-r.z, 0, r.x), c2 = (r.y, -r.x, 0)
    V3<R> c0 = v3(R(0), r.z, -r.y), c1 = v3(-r.z, R(0), r.x), c2 = v3(r.y, -r.x, R(0));
    V3<R> i0 = smul(I, c0), i1 = smul(I, c1), i2 = smul(I, c2);
    K.xx += dot(c0, i0);
    K.xy += dot(c0, i1);
    K.xz += dot(c0, i2);
    K.yy += dot(c1, i1);
    K.yz += dot(c1, i2);
    K.zz += dot(c2, i2);
}
// Solve K x = b for symmetric positive definite K by LDL^T (replaces LAPACK
// gesv at physics.py:886,903,923; same solution up to rounding).
template <class R> BS_HD V3<R> ssolve(const S3<R> &K, V3<R> b) {
    R d0 = K.xx;
    R l10 = K.xy / d0, l20 = K.xz / d0;
    R d1 = K.yy - l10 * K.xy;
    R k21 = K.yz - l20 * K.xy;
    R l21 = k21 / d1;
    R d2 = K.zz - l20 * K.xz - l21 * k21;
    R y0 = b.x, y1 = b.y - l10 * y0, y2 = b.z - l20 * y0 - l21 * y1;
    R z2 = y2 / d2, z1 = y1 / d1 - l21 * z2, z0 = y0 / d0 - l10 * z1 - l20 * z2;
    return V3<R>{z0, z1, z2};
}
// inverse of a symmetric positive definite 3x3 (adjugate / determinant)
template <class R> BS_HD S3<R> sinv(const S3<R> &K) {
    R c00 = K.yy * K.zz - K.yz * K.yz, c01 = K.xz * K.yz - K.xy * K.zz, c02 = K.xy * K.yz - K.xz * K.yy;
    R c11 = K.xx * K.zz - K.xz * K.xz, c12 = K.xy * K.xz - K.xx * K.yz, c22 = K.xx * K.yy - K.xy * K.xy;
    R id = r_rcp(K.xx * c00 + K.xy * c01 + K.xz * c02);
    return S3<R>{c00 * id, c01 * id, c02 * id, c11 * id, c12 * id, c22 * id};
}
// T^T K^-1 T for T = [t1; t2] and K = [[k00, k01], [k01, k11]]
template <class R> BS_HD S3<R> proj2(V3<R> t1, V3<R> t2, R k00, R k01, R k11) {
    R id = r_rcp(k00 * k11 - k01 * k01);
    R i00 = k11 * id, i01 = -k01 * id, i11 = k00 * id;
    auto el = [&](R a1, R b1, R a2, R b2) { return i00 * a1 * b1 + i01 * (a1 * b2 + a2 * b1) + i11 * a2 * b2; };
    return S3<R>{el(t1.x, t1.x, t2.x, t2.x), el(t1.x, t1.y, t2.x, t2.y), el(t1.x, t1.z, t2.x, t2.z),
                 el(t1.y, t1.y, t2.y, t2.y), el(t1.y, t1.z, t2.y, t2.z), el(t1.z, t1.z, t2.z, t2.z)};
}
// T^T (T I T^T)^-1 T for an orthonormal basis T = [t1; t2; a]  (= I^-1)
template <class R> BS_HD S3<R> proj3(V3<R>, V3<R>, V3<R>, const S3<R> &I) { return sinv(I); }
// I [r]x : the map P -> I (r x P)
template <class R> BS_HD M3<R> mskew(const S3<R> &I, V3<R> r) {
    V3<R> c0 = smul(I, v3(R(0), r.z, -r.y)), c1 = smul(I, v3(-r.z, R(0), r.x)), c2 = smul(I, v3(r.y, -r.x, R(0)));
    return M3<R>{c0.x, c1.x, c2.x, c0.y, c1.y, c2.y, c0.z, c1.z, c2.z};
}
// symmetric x symmetric
template <class R> BS_HD M3<R> smm(const S3<R> &A, const S3<R> &B) {
    V3<R> c0 = smul(A, v3(B.xx, B.xy, B.xz)), c1 = smul(A, v3(B.xy, B.yy, B.yz)), c2 = smul(A, v3(B.xz, B.yz, B.zz));
    return M3<R>{c0.x, c1.x, c2.x, c0.y, c1.y, c2.y, c0.z, c1.z, c2.z};
}
template <class R> BS_HD V3<R> mmul(const M3<R> &m, V3<R> v) {
    return V3<R>{m.a00 * v.x + m.a01 * v.y + m.a02 * v.z, m.a10 * v.x + m.a11 * v.y + m.a12 * v.z,
                 m.a20 * v.x + m.a21 * v.y + m.a22 * v.z};
}
// 2x2 symmetric solve
template <class R> BS_HD void ssolve2(R a, R b, R c, R r0, R r1, R &x0, R &x1) {
    R det = a * c - b * b;
    x0 = (c * r0 - b * r1) / det;
    x1 = (a * r1 - b * r0) / det;
}

// two unit tangents (physics.py:131-137)
template <class R> BS_HD void tangents(V3<R> n, V3<R> &t1, V3<R> &t2) {
    V3<R> ref = r_abs(n.z) < R(0.9) ? v3(R(0), R(0), R(1)) : v3(R(1), R(0), R(0));
    V3<R> t = cross(ref, n);
    R il = r_rsqrt(dot(t, t));
    t1 = v3(t.x * il, t.y * il, t.z * il);
    t2 = cross(n, t1);
}

template <class R> BS_HD R clampr(R x, R lo, R hi) { return x < lo ? lo : (x > hi ? hi : x); }
template <class R> BS_HD R signr(R x) { return x > R(0) ? R(1) : (x < R(0) ? R(-1) : R(0)); }
// (a + pi) mod 2 pi - pi with a floor-mod (physics.py:440)
template <class R> BS_HD R wrap_pi(R a) {
    const R TWO_PI = R(6.28318530717958647692), PI = R(3.14159265358979323846);
    R r = a + PI;
    r = r - TWO_PI * r_floor(r * R(0.15915494309189533577));
    return r - PI;
}
template <class R> BS_HD bool finite_r(R x) { return x - x == R(0); }

}  // namespace bsim
