/*
 * pswim_oracle.c — TEST INFRASTRUCTURE ONLY (see pswim_oracle.h).
 *
 * Plain-C restatement of the reference hot path, operation order preserved statement by
 * statement so that, compiled with -ffp-contract=off on x86-64, it reproduces the reference
 * library bitwise.  Citations are /root/reference/proj paths.
 */
#include "pswim_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define KPI 3.14159265358979323846 /* stokes.cpp:9 */

/* ------------------------------------------------------------------------------------ */
/* geom.hpp:9-118 value semantics                                                        */
/* ------------------------------------------------------------------------------------ */
typedef struct { double x, y, z; } v3;
typedef struct { double m[9]; } m3;

static inline v3 V(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static inline v3 ld3(const double* p) { return V(p[0], p[1], p[2]); }
static inline void st3(double* p, v3 a) { p[0] = a.x; p[1] = a.y; p[2] = a.z; }
static inline double vget(v3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }
static inline void vset(v3* a, int i, double v) { if (i == 0) a->x = v; else if (i == 1) a->y = v; else a->z = v; }
static inline v3 add(v3 a, v3 b) { return V(a.x + b.x, a.y + b.y, a.z + b.z); }   /* :15,20 */
static inline v3 sub(v3 a, v3 b) { return V(a.x - b.x, a.y - b.y, a.z - b.z); }   /* :16,21 */
static inline v3 scl(v3 v, double a) { return V(v.x * a, v.y * a, v.z * a); }      /* :17,22-23 */
static inline v3 dv(v3 v, double a) { return scl(v, 1.0 / a); }                    /* :24 */
static inline v3 neg(v3 v) { return V(-v.x, -v.y, -v.z); }                         /* :25 */
static inline double dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; } /* :27 */
static inline v3 cross(v3 a, v3 b) {                                                /* :28-30 */
    return V(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static inline double norm(v3 v) { return sqrt(dot(v, v)); }                         /* :31 */
static inline double norm2(v3 v) { return dot(v, v); }                              /* :32 */
static inline v3 normalized(v3 v) { return dv(v, norm(v)); }                        /* :33 */

static inline double M(const m3* a, int i, int j) { return a->m[3 * i + j]; }
static inline m3 m3_identity(void) { m3 r = {{1, 0, 0, 0, 1, 0, 0, 0, 1}}; return r; }
static inline m3 m3_zero(void) { m3 r; memset(&r, 0, sizeof r); return r; }
static inline m3 m3_add(m3 a, m3 b) { for (int i = 0; i < 9; ++i) a.m[i] += b.m[i]; return a; }
static inline m3 m3_sub(m3 a, m3 b) { for (int i = 0; i < 9; ++i) a.m[i] -= b.m[i]; return a; }
static inline m3 m3_scl(double s, m3 a) { for (int i = 0; i < 9; ++i) a.m[i] *= s; return a; }
static inline m3 m3_mul(m3 a, m3 b) {                                               /* :67-76 */
    m3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = 0.0;
            for (int k = 0; k < 3; ++k) s += M(&a, i, k) * M(&b, k, j);
            r.m[3 * i + j] = s;
        }
    return r;
}
static inline v3 m3_v(const m3* a, v3 v) {                                           /* :78-82 */
    return V(M(a, 0, 0) * v.x + M(a, 0, 1) * v.y + M(a, 0, 2) * v.z,
             M(a, 1, 0) * v.x + M(a, 1, 1) * v.y + M(a, 1, 2) * v.z,
             M(a, 2, 0) * v.x + M(a, 2, 1) * v.y + M(a, 2, 2) * v.z);
}
static inline m3 m3_t(m3 a) {
    m3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[3 * i + j] = M(&a, j, i);
    return r;
}
static inline m3 outer(v3 a, v3 b) {                                                 /* :92-97 */
    m3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.m[3 * i + j] = vget(a, i) * vget(b, j);
    return r;
}
static inline m3 skew(v3 n) {                                                        /* :100-104 */
    m3 r = {{0, -n.z, n.y, n.z, 0, -n.x, -n.y, n.x, 0}};
    return r;
}
static inline double m3_trace(const m3* a) { return M(a, 0, 0) + M(a, 1, 1) + M(a, 2, 2); }
static inline double m3_det(const m3* a) {
    return M(a, 0, 0) * (M(a, 1, 1) * M(a, 2, 2) - M(a, 1, 2) * M(a, 2, 1)) -
           M(a, 0, 1) * (M(a, 1, 0) * M(a, 2, 2) - M(a, 1, 2) * M(a, 2, 0)) +
           M(a, 0, 2) * (M(a, 1, 0) * M(a, 2, 1) - M(a, 1, 1) * M(a, 2, 0));
}
static inline double frob(const m3* a) {
    double s = 0.0;
    for (int i = 0; i < 9; ++i) s += a->m[i] * a->m[i];
    return sqrt(s);
}
static inline double dmin(double a, double b) { return (b < a) ? b : a; }  /* std::min */
static inline double dmax(double a, double b) { return (a < b) ? b : a; }  /* std::max */
static inline double dclamp(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* ------------------------------------------------------------------------------------ */
/* RNG: std::mt19937_64 and the helpers of scenario.cpp:33 / tests/oracles.hpp:41-54      */
/* ------------------------------------------------------------------------------------ */
void or_rng_seed(or_rng* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}
uint64_t or_rng_next(or_rng* g) {
    if (g->idx >= 312) {
        const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}
static double uniform01(or_rng* g) { return (double)(or_rng_next(g) >> 11) * 0x1.0p-53; }
double or_uniform(or_rng* g, double lo, double hi) { return lo + (hi - lo) * uniform01(g); }
void or_random_unit(or_rng* g, double* out) {
    const double z = or_uniform(g, -1.0, 1.0);
    const double phi = or_uniform(g, 0.0, 2.0 * M_PI);
    const double s = sqrt(dmax(0.0, 1.0 - z * z));
    out[0] = s * cos(phi);
    out[1] = s * sin(phi);
    out[2] = z;
}
void or_random_vec(or_rng* g, double scale, double* out) {
    out[0] = or_uniform(g, -scale, scale);
    out[1] = or_uniform(g, -scale, scale);
    out[2] = or_uniform(g, -scale, scale);
}

/* ------------------------------------------------------------------------------------ */
/* stokes.cpp                                                                            */
/* ------------------------------------------------------------------------------------ */
/* accumulate, stokes.cpp:29-55 */
static inline void accumulate(v3 r, v3 f, v3 n, double eps, v3* u, v3* w) {
    const double r2 = dot(r, r);
    const double e2 = eps * eps;
    const double big_r2 = r2 + e2;
    const double big_r = sqrt(big_r2);
    const double inv_r3 = 1.0 / (big_r2 * big_r);
    const double inv_r5 = inv_r3 / big_r2;
    const double inv_r7 = inv_r5 / big_r2;

    const double h1 = (r2 + 2.0 * e2) * (1.0 / (8.0 * KPI)) * inv_r3;
    const double h2 = (1.0 / (8.0 * KPI)) * inv_r3;
    const double h3 = (2.0 * r2 + 5.0 * e2) * (1.0 / (16.0 * KPI)) * inv_r5;
    const double h4 = (10.0 * e2 * e2 - 7.0 * e2 * r2 - 2.0 * r2 * r2) * (1.0 / (32.0 * KPI)) * inv_r7;
    const double h5 = (6.0 * r2 + 21.0 * e2) * (1.0 / (32.0 * KPI)) * inv_r7;

    const double fr = dot(f, r);
    const double nr = dot(n, r);
    const v3 nxr = cross(n, r);
    const v3 fxr = cross(f, r);

    u->x += f.x * h1 + fr * r.x * h2 + nxr.x * h3;
    u->y += f.y * h1 + fr * r.y * h2 + nxr.y * h3;
    u->z += f.z * h1 + fr * r.z * h2 + nxr.z * h3;
    w->x += fxr.x * h3 + n.x * h4 + nr * r.x * h5;
    w->y += fxr.y * h3 + n.y * h4 + nr * r.y * h5;
    w->z += fxr.z * h3 + n.z * h4 + nr * r.z * h5;
}

void or_h_functions(double r, double epsilon, double* h) { /* stokes.cpp:59-74 */
    const double r2 = r * r;
    const double e2 = epsilon * epsilon;
    const double big_r = sqrt(r2 + e2);
    const double r3 = big_r * big_r * big_r;
    const double r5 = r3 * big_r * big_r;
    const double r7 = r5 * big_r * big_r;
    h[0] = (r2 + 2.0 * e2) / (8.0 * KPI * r3);
    h[1] = 1.0 / (8.0 * KPI * r3);
    h[2] = (2.0 * r2 + 5.0 * e2) / (16.0 * KPI * r5);
    h[3] = (10.0 * e2 * e2 - 7.0 * e2 * r2 - 2.0 * r2 * r2) / (32.0 * KPI * r7);
    h[4] = (6.0 * r2 + 21.0 * e2) / (32.0 * KPI * r7);
}

/* check_inputs, stokes.cpp:11-26 */
static int check_inputs(const double* f, const double* n, int64_t ns, double eps, double mu, int wall) {
    if (eps <= 0.0 || mu <= 0.0) return PSWIM_EINVAL;
    if (wall == 1) return PSWIM_EUNSUPPORTED_WALL;
    for (int64_t i = 0; i < ns; ++i) {
        const v3 fi = ld3(f + 3 * i), ni = ld3(n + 3 * i);
        if (!isfinite(dot(fi, fi)) || !isfinite(dot(ni, ni))) return PSWIM_ENONFINITE;
    }
    return PSWIM_OK;
}

static void mrs_rows(const double* tgt, int64_t t0, int64_t t1, const double* src, const double* f,
                     const double* n, int64_t ns, double eps, double mu, double* u, double* w, int threads) {
    const double inv_mu = 1.0 / mu;
    (void)threads;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1) if (threads > 1)
#endif
    for (int64_t i = t0; i < t1; ++i) {
        v3 ui = V(0, 0, 0), wi = V(0, 0, 0);
        const v3 ti = ld3(tgt + 3 * i);
        for (int64_t j = 0; j < ns; ++j) {
            accumulate(sub(ti, ld3(src + 3 * j)), ld3(f + 3 * j), ld3(n + 3 * j), eps, &ui, &wi);
        }
        st3(u + 3 * i, scl(ui, inv_mu));
        st3(w + 3 * i, scl(wi, inv_mu));
    }
}

int or_evaluate_velocities(const double* tgt, int64_t nt, const double* src, const double* f,
                           const double* n, int64_t ns, double eps, double mu, int wall, double* u,
                           double* w) { /* stokes.cpp:97-113 (serial twin) */
    const int rc = check_inputs(f, n, ns, eps, mu, wall);
    if (rc) return rc;
    mrs_rows(tgt, 0, nt, src, f, n, ns, eps, mu, u, w, 1);
    return PSWIM_OK;
}

int or_evaluate_velocities_rows(const double* tgt, int64_t t_begin, int64_t t_end, const double* src,
                                const double* f, const double* n, int64_t ns, double eps, double mu,
                                double* u, double* w, int threads) {
    mrs_rows(tgt, t_begin, t_end, src, f, n, ns, eps, mu, u, w, threads);
    return PSWIM_OK;
}

int or_grand_mobility(const double* nodes, int64_t n, double eps, double mu, double* mat) {
    /* stokes.cpp:115-154 */
    if (eps <= 0.0 || mu <= 0.0) return PSWIM_EINVAL;
    const int64_t dim = 6 * n;
    memset(mat, 0, sizeof(double) * (size_t)(dim * dim));
    const double inv_mu = 1.0 / mu;
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = 0; j < n; ++j) {
            const v3 r = sub(ld3(nodes + 3 * i), ld3(nodes + 3 * j));
            double h[5];
            or_h_functions(norm(r), eps, h);
            const m3 rr = outer(r, r);
            const m3 rx = skew(r);
            const m3 uu = m3_add(m3_scl(h[0], m3_identity()), m3_scl(h[1], rr));
            const m3 un = m3_scl(-h[2], rx);
            const m3 wf = m3_scl(-h[2], rx);
            const m3 ww = m3_add(m3_scl(h[3], m3_identity()), m3_scl(h[4], rr));
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) {
                    mat[(6 * i + a) * dim + (6 * j + b)] = M(&uu, a, b) * inv_mu;
                    mat[(6 * i + a) * dim + (6 * j + 3 + b)] = M(&un, a, b) * inv_mu;
                    mat[(6 * i + 3 + a) * dim + (6 * j + b)] = M(&wf, a, b) * inv_mu;
                    mat[(6 * i + 3 + a) * dim + (6 * j + 3 + b)] = M(&ww, a, b) * inv_mu;
                }
        }
    }
    return PSWIM_OK;
}

/* ------------------------------------------------------------------------------------ */
/* rotation.cpp                                                                          */
/* ------------------------------------------------------------------------------------ */
static int from_axis_angle(v3 n, double angle, m3* out) { /* rotation.cpp:19-34 */
    const double len = norm(n);
    if (fabs(len - 1.0) > 1e-6) return PSWIM_EINVAL;
    if (len != 1.0) n = dv(n, len);
    const double c = cos(angle);
    const double s = sin(angle);
    *out = m3_add(m3_add(m3_scl(c, m3_identity()), m3_scl(1.0 - c, outer(n, n))), m3_scl(s, skew(n)));
    return PSWIM_OK;
}
int or_from_axis_angle(const double* axis3, double angle, double* r9) {
    m3 r;
    const int rc = from_axis_angle(ld3(axis3), angle, &r);
    if (rc == PSWIM_OK) memcpy(r9, r.m, sizeof r.m);
    return rc;
}

static v3 skew_vector(const m3* r) { /* rotation.cpp:39-41 */
    return V(0.5 * (M(r, 2, 1) - M(r, 1, 2)), 0.5 * (M(r, 0, 2) - M(r, 2, 0)), 0.5 * (M(r, 1, 0) - M(r, 0, 1)));
}

static v3 axis_from_diagonal(const m3* r, double cos_theta) { /* rotation.cpp:48-70 */
    const double omc = 1.0 - cos_theta;
    v3 n;
    for (int i = 0; i < 3; ++i) vset(&n, i, sqrt(dmax(0.0, (M(r, i, i) - cos_theta) / omc)));
    int k = 0;
    if (n.y > vget(n, k)) k = 1;
    if (n.z > vget(n, k)) k = 2;
    const double sym01 = 0.5 * (M(r, 0, 1) + M(r, 1, 0));
    const double sym02 = 0.5 * (M(r, 0, 2) + M(r, 2, 0));
    const double sym12 = 0.5 * (M(r, 1, 2) + M(r, 2, 1));
    for (int j = 0; j < 3; ++j) {
        if (j == k) continue;
        const int s = k + j;
        const double sy = (s == 1) ? sym01 : (s == 2 ? sym02 : sym12);
        if (sy < 0.0) vset(&n, j, -vget(n, j));
    }
    const double len = norm(n);
    if (len == 0.0) return V(0, 0, 1);
    n = dv(n, len);
    if (dot(n, skew_vector(r)) < 0.0) n = neg(n);
    return n;
}

void or_to_axis_angle(const double* r9, double* axis3, double* angle) { /* rotation.cpp:74-89 */
    m3 r;
    memcpy(r.m, r9, sizeof r.m);
    const double cos_theta = dclamp(0.5 * (m3_trace(&r) - 1.0), -1.0, 1.0);
    const v3 s = skew_vector(&r);
    const double sin_theta = dmin(norm(s), 1.0);
    const double theta = atan2(sin_theta, cos_theta);
    v3 axis;
    if (theta < 1e-7) {
        axis = sin_theta > 0.0 ? dv(s, norm(s)) : V(0, 0, 1);
    } else if (theta > M_PI - 1e-2) {
        axis = axis_from_diagonal(&r, cos_theta);
    } else {
        axis = dv(s, norm(s));
    }
    st3(axis3, axis);
    *angle = theta;
}

static m3 sqrt_rotation(const m3* r) { /* rotation.cpp:91-107 */
    const double cos_theta = dclamp(0.5 * (m3_trace(r) - 1.0), -1.0, 1.0);
    const v3 s = skew_vector(r);
    const double theta = atan2(dmin(norm(s), 1.0), cos_theta);
    m3 out;
    if (theta < 1e-7) {
        const m3 w = skew(s);
        return m3_add(m3_add(m3_identity(), m3_scl(0.5, w)), m3_scl(0.125, m3_mul(w, w)));
    }
    if (theta > M_PI - 1e-2) {
        const v3 n = axis_from_diagonal(r, cos_theta);
        from_axis_angle(n, 0.5 * theta, &out);
        return out;
    }
    from_axis_angle(dv(s, norm(s)), 0.5 * theta, &out);
    return out;
}
void or_sqrt_rotation(const double* r9, double* s9) {
    m3 r;
    memcpy(r.m, r9, sizeof r.m);
    const m3 s = sqrt_rotation(&r);
    memcpy(s9, s.m, sizeof s.m);
}

double or_rotation_residual(const double* r9) { /* rotation.cpp:10-15 */
    m3 r;
    memcpy(r.m, r9, sizeof r.m);
    const m3 g = m3_sub(m3_mul(m3_t(r), r), m3_identity());
    const double ortho = frob(&g);
    const double d = m3_det(&r) - 1.0;
    return sqrt(ortho * ortho + d * d);
}

/* ------------------------------------------------------------------------------------ */
/* rod.cpp                                                                               */
/* ------------------------------------------------------------------------------------ */
#define NX(p, k) ld3((p) + 12 * (k) + 0)
#define ND1(p, k) ld3((p) + 12 * (k) + 3)
#define ND2(p, k) ld3((p) + 12 * (k) + 6)
#define ND3(p, k) ld3((p) + 12 * (k) + 9)

void or_preferred_strain(double s, double t, const double* wave3, double* out) { /* rod.cpp:29-32 */
    const double k = 2.0 * M_PI / wave3[2]; /* WaveformParams::wavenumber, rod.cpp:27 */
    out[0] = 0.0;
    out[1] = -k * k * wave3[0] * sin(k * s + wave3[1] * t);
    out[2] = 0.0;
}

int or_internal_loads(const double* rod, int64_t m, double length, const double* mat6,
                      const double* wave3, double t, double* force, double* moment) { /* rod.cpp:36-82 */
    if (m < 2) return PSWIM_EINVAL;
    const double ds = length / (double)(m - 1); /* RodDiscretization::ds, rod.hpp:14 */
    const double inv_ds = 1.0 / ds;
    const double a_mod[3] = {mat6[0], mat6[1], mat6[2]};
    const double b_mod[3] = {mat6[3], mat6[4], mat6[5]};
    for (int64_t k = 0; k + 1 < m; ++k) {
        const v3 dx = sub(NX(rod, k + 1), NX(rod, k));
        if (norm2(dx) == 0.0) return PSWIM_EDEGENERATE;
        const v3 tangent = scl(dx, inv_ds);
        const v3 lo[3] = {ND1(rod, k), ND2(rod, k), ND3(rod, k)};
        const v3 hi[3] = {ND1(rod, k + 1), ND2(rod, k + 1), ND3(rod, k + 1)};
        m3 a = m3_zero();
        for (int j = 0; j < 3; ++j) a = m3_add(a, outer(hi[j], lo[j]));
        const m3 half = sqrt_rotation(&a);
        const v3 mid[3] = {m3_v(&half, lo[0]), m3_v(&half, lo[1]), m3_v(&half, lo[2])};
        double om[3];
        or_preferred_strain(((double)k + 0.5) * ds, t, wave3, om);
        v3 f = V(0, 0, 0), n = V(0, 0, 0);
        for (int i = 0; i < 3; ++i) {
            const int j = (i + 1) % 3;
            const int kk = (i + 2) % 3;
            const double stretch = dot(tangent, mid[i]) - (i == 2 ? 1.0 : 0.0);
            const double bend = dot(scl(sub(hi[j], lo[j]), inv_ds), mid[kk]) - om[i];
            f = add(f, scl(mid[i], b_mod[i] * stretch));
            n = add(n, scl(mid[i], a_mod[i] * bend));
        }
        st3(force + 3 * k, f);
        st3(moment + 3 * k, n);
    }
    return PSWIM_OK;
}

int or_nodal_loads(const double* rod, int64_t m, double length, const double* force,
                   const double* moment, double* fo, double* no) { /* rod.cpp:84-109 */
    const double inv_ds = 1.0 / (length / (double)(m - 1));
    const v3 zero = V(0, 0, 0);
    for (int64_t k = 0; k < m; ++k) {
        const v3 f_plus = (k < m - 1) ? ld3(force + 3 * k) : zero;
        const v3 f_minus = (k > 0) ? ld3(force + 3 * (k - 1)) : zero;
        const v3 n_plus = (k < m - 1) ? ld3(moment + 3 * k) : zero;
        const v3 n_minus = (k > 0) ? ld3(moment + 3 * (k - 1)) : zero;
        st3(fo + 3 * k, scl(sub(f_plus, f_minus), inv_ds));
        v3 torque = scl(sub(n_plus, n_minus), inv_ds);
        if (k < m - 1) torque = add(torque, scl(cross(scl(sub(NX(rod, k + 1), NX(rod, k)), inv_ds), f_plus), 0.5));
        if (k > 0) torque = add(torque, scl(cross(scl(sub(NX(rod, k), NX(rod, k - 1)), inv_ds), f_minus), 0.5));
        st3(no + 3 * k, torque);
    }
    return PSWIM_OK;
}

static double lj_force_over_r(double r, double well_depth, double sigma) { /* rod.cpp:116-120 */
    const double sr2 = (sigma * sigma) / (r * r);
    const double sr6 = sr2 * sr2 * sr2;
    return 24.0 * well_depth * (2.0 * sr6 * sr6 - sr6) / (r * r);
}

void or_lj_repulsion(const double* state, int64_t rods, int64_t m, double well_depth, double sigma,
                     int64_t self_exclusion, double* forces) { /* rod.cpp:124-174 */
    const int64_t total = rods * m;
    memset(forces, 0, sizeof(double) * (size_t)(3 * total));
    if (rods < 2) return;
    const int64_t excl = self_exclusion > 4 ? self_exclusion : 4;
    const double rc = pow(2.0, 1.0 / 6.0) * sigma;
    const double rc2 = rc * rc;
    const double r_min = 1e-3 * sigma;
    const double cap = lj_force_over_r(r_min, well_depth, sigma) * r_min;
    for (int64_t ra = 0; ra < rods; ++ra) {
        for (int64_t rb = ra; rb < rods; ++rb) {
            const double* a = state + 12 * m * ra;
            const double* b = state + 12 * m * rb;
            for (int64_t i = 0; i < m; ++i) {
                const int64_t j0 = (ra == rb) ? i + excl : 0;
                for (int64_t j = j0; j < m; ++j) {
                    const v3 d = sub(NX(a, i), NX(b, j));
                    const double r2 = norm2(d);
                    if (r2 >= rc2) continue;
                    const double r = sqrt(r2);
                    v3 force;
                    if (r < r_min) {
                        const v3 dir = (r > 0.0) ? dv(d, r) : V(1, 0, 0);
                        force = scl(dir, cap);
                    } else {
                        force = scl(d, lj_force_over_r(r, well_depth, sigma));
                    }
                    double* fa = forces + 3 * (m * ra + i);
                    double* fb = forces + 3 * (m * rb + j);
                    st3(fa, add(ld3(fa), force));
                    st3(fb, sub(ld3(fb), force));
                }
            }
        }
    }
}

int64_t or_reorthonormalize(double* rod, int64_t m, double tol) { /* rod.cpp:176-195 */
    int64_t touched = 0;
    for (int64_t k = 0; k < m; ++k) {
        m3 d;
        const v3 c1 = ND1(rod, k), c2 = ND2(rod, k), c3 = ND3(rod, k);
        for (int c = 0; c < 3; ++c) {
            d.m[3 * c + 0] = vget(c1, c);
            d.m[3 * c + 1] = vget(c2, c);
            d.m[3 * c + 2] = vget(c3, c);
        }
        const m3 g = m3_sub(m3_mul(m3_t(d), d), m3_identity());
        if (frob(&g) <= tol) continue;
        const v3 t3 = normalized(c3);
        v3 t1 = sub(c1, scl(t3, dot(c1, t3)));
        t1 = normalized(t1);
        st3(rod + 12 * k + 9, t3);
        st3(rod + 12 * k + 3, t1);
        st3(rod + 12 * k + 6, cross(t3, t1));
        ++touched;
    }
    return touched;
}

/* ------------------------------------------------------------------------------------ */
/* scenario.cpp                                                                          */
/* ------------------------------------------------------------------------------------ */
int or_resolve(const pswim_scenario* sc, pswim_resolved* out) { /* scenario.cpp:10-29 */
    if (sc->nodes_per_rod < 3 || sc->rod_count < 1) return PSWIM_EINVAL;
    if (sc->rod_length <= 0.0 || sc->mu <= 0.0) return PSWIM_EINVAL;
    const double ds = sc->rod_length / (double)(sc->nodes_per_rod - 1);
    out->ds = ds;
    out->epsilon = sc->epsilon > 0.0 ? sc->epsilon : 4.0 * ds;
    out->mu = sc->mu;
    out->lj_sigma = sc->lj_sigma > 0.0 ? sc->lj_sigma : 3.0 * out->epsilon;
    out->lj_cutoff = pow(2.0, 1.0 / 6.0) * out->lj_sigma;
    int64_t excl = (int64_t)ceil(out->lj_cutoff / ds) + 1;
    if (excl < 4) excl = 4;
    out->lj_self_exclusion = excl;
    out->total_nodes = sc->rod_count * sc->nodes_per_rod;
    return PSWIM_OK;
}

static void straight_rod(int64_t m, double ds, v3 start, v3 axis, v3 normal, double* rod) { /* scenario.cpp:42-53 */
    const v3 d2 = cross(axis, normal);
    for (int64_t k = 0; k < m; ++k) {
        st3(rod + 12 * k + 0, add(start, scl(axis, (double)k * ds)));
        st3(rod + 12 * k + 3, normal);
        st3(rod + 12 * k + 6, d2);
        st3(rod + 12 * k + 9, axis);
    }
}

static v3 any_normal(v3 a) { /* scenario.cpp:56-62 */
    const v3 pick = fabs(a.x) <= fabs(a.y) && fabs(a.x) <= fabs(a.z) ? V(1, 0, 0)
                    : fabs(a.y) <= fabs(a.z)                         ? V(0, 1, 0)
                                                                     : V(0, 0, 1);
    return normalized(sub(pick, scl(a, dot(pick, a))));
}

int or_build_initial_state(const pswim_scenario* sc, double* state) { /* scenario.cpp:71-120 */
    pswim_resolved rs;
    int rc = or_resolve(sc, &rs);
    if (rc) return rc;
    const int64_t m = sc->nodes_per_rod;
    const double L = sc->rod_length;
    if (sc->placement == 0) {
        const double gap = dmax(4.0 * rs.lj_sigma, 0.2 * L);
        const int64_t cols = (int64_t)ceil(sqrt((double)sc->rod_count));
        for (int64_t i = 0; i < sc->rod_count; ++i) {
            const double gx = (double)(i % cols) * (L + gap);
            const double gy = (double)(i / cols) * gap;
            straight_rod(m, rs.ds, V(gx, gy, sc->wall_clearance), V(1, 0, 0), V(0, 1, 0), state + 12 * m * i);
        }
        return PSWIM_OK;
    }
    or_rng g;
    or_rng_seed(&g, sc->seed);
    const double box_xy = 4.0 * L;
    const double dz = sc->wall_clearance;
    const double min_sep = 2.0 * rs.lj_sigma;
    for (int64_t i = 0; i < sc->rod_count; ++i) {
        int placed = 0;
        double* rod = state + 12 * m * i;
        for (int attempt = 0; attempt < 10000 && !placed; ++attempt) {
            const double cx = box_xy * uniform01(&g);
            const double cy = box_xy * uniform01(&g);
            const double cz = dz + 2.0 * L * uniform01(&g);
            const v3 centre = V(cx, cy, cz);
            /* random_unit, scenario.cpp:35-40 */
            const double z = 2.0 * uniform01(&g) - 1.0;
            const double phi = 2.0 * M_PI * uniform01(&g);
            const double s = sqrt(dmax(0.0, 1.0 - z * z));
            const v3 axis = V(s * cos(phi), s * sin(phi), z);
            const v3 start = sub(centre, scl(axis, 0.5 * L));
            straight_rod(m, rs.ds, start, axis, any_normal(axis), rod);
            int ok = 1;
            for (int64_t k = 0; k < m; ++k) {
                if (rod[12 * k + 2] < 0.5 * dz) { ok = 0; break; }
            }
            for (int64_t j = 0; ok && j < i; ++j) {
                const double* other = state + 12 * m * j;
                double best = INFINITY;
                for (int64_t a = 0; a < m; ++a)
                    for (int64_t b = 0; b < m; ++b) best = dmin(best, norm(sub(NX(rod, a), NX(other, b))));
                if (best < min_sep) ok = 0;
            }
            if (ok) placed = 1;
        }
        if (!placed) return PSWIM_EINVAL;
    }
    return PSWIM_OK;
}

/* ------------------------------------------------------------------------------------ */
/* propagators.cpp                                                                       */
/* ------------------------------------------------------------------------------------ */
static void scenario_arrays(const pswim_scenario* sc, double* mat6, double* wave3) {
    mat6[0] = sc->a1; mat6[1] = sc->a2; mat6[2] = sc->a3;
    mat6[3] = sc->b1; mat6[4] = sc->b2; mat6[5] = sc->b3;
    wave3[0] = sc->amplitude; wave3[1] = sc->frequency; wave3[2] = sc->wavelength;
}

int or_rhs(const pswim_scenario* sc, const double* state, double t, const double* extra_f,
           const double* extra_n, double* u, double* w, int threads) { /* propagators.cpp:38-91 */
    pswim_resolved rs;
    int rc = or_resolve(sc, &rs);
    if (rc) return rc;
    const int64_t rods = sc->rod_count, m = sc->nodes_per_rod, total = rods * m;
    double mat6[6], wave3[3];
    scenario_arrays(sc, mat6, wave3);
    double* pos = (double*)malloc(sizeof(double) * 3 * (size_t)total);
    double* lf = (double*)malloc(sizeof(double) * 3 * (size_t)total);
    double* ln = (double*)malloc(sizeof(double) * 3 * (size_t)total);
    double* force = (double*)malloc(sizeof(double) * 3 * (size_t)m);
    double* moment = (double*)malloc(sizeof(double) * 3 * (size_t)m);
    for (int64_t r = 0; r < rods && rc == PSWIM_OK; ++r) {
        const double* rod = state + 12 * m * r;
        rc = or_internal_loads(rod, m, sc->rod_length, mat6, wave3, t, force, moment);
        if (rc) break;
        or_nodal_loads(rod, m, sc->rod_length, force, moment, lf + 3 * m * r, ln + 3 * m * r);
        for (int64_t k = 0; k < m; ++k) st3(pos + 3 * (m * r + k), NX(rod, k));
    }
    if (rc == PSWIM_OK && rods >= 2 && sc->lj_well_depth > 0.0) {
        double* lj = (double*)malloc(sizeof(double) * 3 * (size_t)total);
        or_lj_repulsion(state, rods, m, sc->lj_well_depth, rs.lj_sigma, rs.lj_self_exclusion, lj);
        const double inv_ds = 1.0 / rs.ds;
        for (int64_t i = 0; i < total; ++i) st3(lf + 3 * i, add(ld3(lf + 3 * i), scl(ld3(lj + 3 * i), inv_ds)));
        free(lj);
    }
    if (rc == PSWIM_OK && extra_f && extra_n) {
        for (int64_t i = 0; i < total; ++i) {
            st3(lf + 3 * i, add(ld3(lf + 3 * i), ld3(extra_f + 3 * i)));
            st3(ln + 3 * i, add(ld3(ln + 3 * i), ld3(extra_n + 3 * i)));
        }
    }
    if (rc == PSWIM_OK) {
        rc = check_inputs(lf, ln, total, rs.epsilon, rs.mu, sc->wall_mode);
        if (rc == PSWIM_OK) mrs_rows(pos, 0, total, pos, lf, ln, total, rs.epsilon, rs.mu, u, w, threads);
    }
    free(pos); free(lf); free(ln); free(force); free(moment);
    return rc;
}

int or_advance_state(const pswim_scenario* sc, const double* state, const double* u, const double* w,
                     double dt, double* out) { /* propagators.cpp:93-124 */
    pswim_resolved rs;
    int rc = or_resolve(sc, &rs);
    if (rc) return rc;
    const int64_t rods = sc->rod_count, m = sc->nodes_per_rod;
    const double max_disp = 10.0 * rs.ds;
    memcpy(out, state, sizeof(double) * 12 * (size_t)(rods * m));
    int64_t idx = 0;
    for (int64_t r = 0; r < rods; ++r) {
        double* rod = out + 12 * m * r;
        for (int64_t k = 0; k < m; ++k, ++idx) {
            const v3 du = scl(ld3(u + 3 * idx), dt);
            if (norm(du) > max_disp) return PSWIM_ESTIFF;
            st3(rod + 12 * k, add(NX(rod, k), du));
            const v3 wv = ld3(w + 3 * idx);
            const double speed = norm(wv);
            if (speed > 0.0) {
                m3 q;
                rc = from_axis_angle(dv(wv, speed), speed * dt, &q);
                if (rc) return rc;
                const v3 d1 = m3_v(&q, ND1(rod, k)), d2 = m3_v(&q, ND2(rod, k)), d3 = m3_v(&q, ND3(rod, k));
                st3(rod + 12 * k + 3, d1);
                st3(rod + 12 * k + 6, d2);
                st3(rod + 12 * k + 9, d3);
            }
        }
        or_reorthonormalize(rod, m, 1e-9);
    }
    return PSWIM_OK;
}

int or_step(const pswim_scenario* sc, int scheme, const double* state, double t, double dt, double* out,
            int threads) { /* propagators.cpp:126-133 */
    const int64_t total = sc->rod_count * sc->nodes_per_rod;
    double* u = (double*)malloc(sizeof(double) * 3 * (size_t)total);
    double* w = (double*)malloc(sizeof(double) * 3 * (size_t)total);
    int rc = or_rhs(sc, state, t, NULL, NULL, u, w, threads);
    if (rc == PSWIM_OK) {
        if (scheme == PSWIM_EULER) {
            rc = or_advance_state(sc, state, u, w, dt, out);
        } else {
            double* mid = (double*)malloc(sizeof(double) * 12 * (size_t)total);
            rc = or_advance_state(sc, state, u, w, 0.5 * dt, mid);
            if (rc == PSWIM_OK) rc = or_rhs(sc, mid, t + 0.5 * dt, NULL, NULL, u, w, threads);
            if (rc == PSWIM_OK) rc = or_advance_state(sc, state, u, w, dt, out);
            free(mid);
        }
    }
    free(u);
    free(w);
    return rc;
}

int or_propagate(const pswim_scenario* sc, const double* in, double t0, double t1, int scheme,
                 int64_t steps_per_interval, double dtc, double* out, int threads) { /* :135-162 */
    const size_t bytes = sizeof(double) * 12 * (size_t)(sc->rod_count * sc->nodes_per_rod);
    if (t1 < t0) return PSWIM_EINVAL;
    if (t1 == t0) { memmove(out, in, bytes); return PSWIM_OK; }
    int64_t steps;
    double dt;
    if (steps_per_interval > 0) {
        steps = steps_per_interval;
        dt = (t1 - t0) / (double)steps;
    } else {
        if (dtc <= 0.0) return PSWIM_EINVAL;
        const double ratio = (t1 - t0) / dtc;
        steps = (int64_t)llround(ratio);
        if (steps == 0 || fabs(ratio - (double)steps) > 1e-9 * (double)steps) return PSWIM_EINVAL;
        dt = dtc;
    }
    double* cur = (double*)malloc(bytes);
    double* nxt = (double*)malloc(bytes);
    memcpy(cur, in, bytes);
    double t = t0;
    int rc = PSWIM_OK;
    for (int64_t i = 0; i < steps && rc == PSWIM_OK; ++i) {
        rc = or_step(sc, scheme, cur, t, dt, nxt, threads);
        double* tmp = cur; cur = nxt; nxt = tmp;
        t += dt;
    }
    if (rc == PSWIM_OK) memcpy(out, cur, bytes);
    free(cur);
    free(nxt);
    return rc;
}

/* ------------------------------------------------------------------------------------ */
/* io.cpp / parareal.cpp                                                                 */
/* ------------------------------------------------------------------------------------ */
double or_position_metric(const double* x, const double* y, int64_t len) { /* io.cpp:49-68 */
    double worst = 0.0;
    for (int64_t i = 0; i < len; i += 12) {
        double num = 0.0, den = 0.0;
        for (int c = 0; c < 3; ++c) {
            const double d = x[i + c] - y[i + c];
            num += d * d;
            den += x[i + c] * x[i + c];
        }
        num = sqrt(num);
        den = sqrt(den);
        worst = dmax(worst, den < 1e-14 ? num : num / den);
    }
    return worst;
}

double or_pointwise_metric(const double* x, const double* y, int64_t len, int64_t dim) { /* parareal.cpp:15-34 */
    double worst = 0.0;
    for (int64_t i = 0; i < len; i += dim) {
        double num = 0.0, den = 0.0;
        for (int64_t c = 0; c < dim; ++c) {
            const double d = x[i + c] - y[i + c];
            num += d * d;
            den += x[i + c] * x[i + c];
        }
        num = sqrt(num);
        den = sqrt(den);
        worst = dmax(worst, den < 1e-14 ? num : num / den);
    }
    return worst;
}

int or_parareal_rod(const pswim_scenario* sc, double t0, double horizon, int nI, int iterations,
                    int64_t fine_steps, int64_t coarse_steps, const double* x0, double* states,
                    double* eta_tilde, int threads) {
    /* tests/test_parareal.cpp:41-65 brute-force recurrence (== parareal.cpp:58-89) */
    const int64_t len = 12 * sc->rod_count * sc->nodes_per_rod;
    const size_t bytes = sizeof(double) * (size_t)len;
#define BT(i) (t0 + (horizon / nI) * (i)) /* ParallelPlan::boundary_time, parareal.hpp:44 */
    double* x = states;
    double* g_old = (double*)malloc(bytes * (size_t)(nI + 1));
    double* xp = (double*)malloc(bytes * (size_t)(nI + 1));
    double* xn = (double*)malloc(bytes * (size_t)(nI + 1));
    double* g_new = (double*)malloc(bytes);
    int rc = PSWIM_OK;
    memcpy(x, x0, bytes);
    for (int i = 1; i <= nI && rc == PSWIM_OK; ++i) {
        rc = or_propagate(sc, x + len * (i - 1), BT(i - 1), BT(i), PSWIM_EULER, coarse_steps, 0.0,
                          g_old + len * i, threads);
        memcpy(x + len * i, g_old + len * i, bytes);
    }
    for (int k = 1; k <= iterations && rc == PSWIM_OK; ++k) {
        for (int i = k; i <= nI && rc == PSWIM_OK; ++i)
            rc = or_propagate(sc, x + len * (i - 1), BT(i - 1), BT(i), PSWIM_RK2, fine_steps, 0.0, xp + len * i, threads);
        memcpy(xn, x, bytes * (size_t)(nI + 1));
        if (k <= nI) memcpy(xn + len * k, xp + len * k, bytes);
        for (int i = k + 1; i <= nI && rc == PSWIM_OK; ++i) {
            rc = or_propagate(sc, xn + len * (i - 1), BT(i - 1), BT(i), PSWIM_EULER, coarse_steps, 0.0, g_new, threads);
            for (int64_t c = 0; c < len; ++c) xn[len * i + c] = xp[len * i + c] + g_new[c] - g_old[len * i + c];
            memcpy(g_old + len * i, g_new, bytes);
        }
        if (eta_tilde) {
            double e = 0.0;
            for (int i = 1; i <= nI; ++i) e = dmax(e, or_position_metric(xn + len * i, x + len * i, len));
            eta_tilde[k - 1] = e;
        }
        memcpy(x, xn, bytes * (size_t)(nI + 1));
    }
#undef BT
    free(g_old); free(xp); free(xn); free(g_new);
    return rc;
}

/* ------------------------------------------------------------------------------------ */
/* tests/oracles.cpp — the reference's independent test oracles                          */
/* ------------------------------------------------------------------------------------ */
static double blob(double s, double eps) { /* oracles.cpp:14-17 */
    const double q = s * s + eps * eps;
    return 15.0 * eps * eps * eps * eps / (8.0 * KPI * q * q * q * sqrt(q));
}

void or_dense_mobility_apply(const double* nodes, int64_t n, const double* fl, const double* tl,
                             double eps, double mu, double* uo, double* wo) { /* oracles.cpp:87-140 */
    for (int64_t i = 0; i < n; ++i) {
        double u[3] = {0, 0, 0}, w[3] = {0, 0, 0};
        for (int64_t j = 0; j < n; ++j) {
            const double rv[3] = {nodes[3 * i] - nodes[3 * j], nodes[3 * i + 1] - nodes[3 * j + 1],
                                  nodes[3 * i + 2] - nodes[3 * j + 2]};
            const double r2 = rv[0] * rv[0] + rv[1] * rv[1] + rv[2] * rv[2];
            const double r = sqrt(r2);
            const double cap_r = sqrt(r2 + eps * eps);
            const double g = -(3.0 * eps * eps + 2.0 * r2) / (8.0 * KPI * pow(cap_r, 3));
            const double gp = r * (5.0 * eps * eps + 2.0 * r2) / (8.0 * KPI * pow(cap_r, 5));
            const double bp = -r / (8.0 * KPI * cap_r);
            const double bpp = -eps * eps / (8.0 * KPI * pow(cap_r, 3));
            const double phi = blob(r, eps);
            const double h1 = r == 0.0 ? bpp - g : bp / r - g;
            const double h2 = r == 0.0 ? 0.0 : (bpp - bp / r) / r2;
            const double h3 = r == 0.0 ? 0.0 : gp / (2.0 * r);
            const double h4 = r == 0.0 ? 0.25 * (phi - phi / 3.0) : 0.25 * (phi - gp / r);
            const double h5 = r == 0.0 ? 0.0 : (3.0 * gp - r * phi) / (4.0 * r2 * r);
            const double f[3] = {fl[3 * j], fl[3 * j + 1], fl[3 * j + 2]};
            const double t[3] = {tl[3 * j], tl[3 * j + 1], tl[3 * j + 2]};
            double fr = 0.0, tr = 0.0;
            for (int a = 0; a < 3; ++a) {
                fr += f[a] * rv[a];
                tr += t[a] * rv[a];
            }
            const double nxr[3] = {t[1] * rv[2] - t[2] * rv[1], t[2] * rv[0] - t[0] * rv[2], t[0] * rv[1] - t[1] * rv[0]};
            const double fxr[3] = {f[1] * rv[2] - f[2] * rv[1], f[2] * rv[0] - f[0] * rv[2], f[0] * rv[1] - f[1] * rv[0]};
            for (int a = 0; a < 3; ++a) {
                u[a] += f[a] * h1 + fr * rv[a] * h2 + nxr[a] * h3;
                w[a] += fxr[a] * h3 + t[a] * h4 + tr * rv[a] * h5;
            }
        }
        for (int a = 0; a < 3; ++a) {
            uo[3 * i + a] = u[a] / mu;
            wo[3 * i + a] = w[a] / mu;
        }
    }
}

double or_elastic_energy(const double* rod, int64_t m, double length, const double* mat6,
                         const double* wave3, double t) { /* oracles.cpp:142-167 */
    const double ds = length / (double)(m - 1);
    double energy = 0.0;
    for (int64_t k = 0; k + 1 < m; ++k) {
        const v3 tangent = dv(sub(NX(rod, k + 1), NX(rod, k)), ds);
        const v3 lo[3] = {ND1(rod, k), ND2(rod, k), ND3(rod, k)};
        const v3 hi[3] = {ND1(rod, k + 1), ND2(rod, k + 1), ND3(rod, k + 1)};
        m3 a = m3_zero();
        for (int j = 0; j < 3; ++j) a = m3_add(a, outer(hi[j], lo[j]));
        const m3 half = sqrt_rotation(&a);
        const v3 mid[3] = {m3_v(&half, lo[0]), m3_v(&half, lo[1]), m3_v(&half, lo[2])};
        double om[3];
        or_preferred_strain(((double)k + 0.5) * ds, t, wave3, om);
        for (int i = 0; i < 3; ++i) {
            const int j = (i + 1) % 3;
            const int kk = (i + 2) % 3;
            const double stretch = dot(tangent, mid[i]) - (i == 2 ? 1.0 : 0.0);
            const double bend = dot(dv(sub(hi[j], lo[j]), ds), mid[kk]) - om[i];
            energy += 0.5 * ds * (mat6[3 + i] * stretch * stretch + mat6[i] * bend * bend);
        }
    }
    return energy;
}

void or_perturbed_rod(int64_t m, double length, or_rng* g, double pj, double aj, double* rod) {
    /* oracles.cpp:204-222 */
    const double ds = length / (double)(m - 1);
    for (int64_t k = 0; k < m; ++k) {
        double jit[3], axis[3];
        or_random_vec(g, pj * ds, jit);
        st3(rod + 12 * k, add(V((double)k * ds, 0.0, 0.0), ld3(jit)));
        or_random_unit(g, axis);
        const double ang = or_uniform(g, 0.0, aj);
        m3 q;
        from_axis_angle(ld3(axis), ang, &q);
        st3(rod + 12 * k + 3, m3_v(&q, V(0, 1, 0)));
        st3(rod + 12 * k + 6, m3_v(&q, V(0, 0, 1)));
        st3(rod + 12 * k + 9, m3_v(&q, V(1, 0, 0)));
    }
}
