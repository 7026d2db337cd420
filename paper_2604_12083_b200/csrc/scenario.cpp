// scenario.cpp — host-side scenario resolution and initial-state construction.
//
// make_scenario (reference src/scenario.cpp:10-29) and build_initial_state (:71-120) in the
// packed 12-doubles-per-node layout of pack_state (src/io.cpp:10-25).  Uses std::mt19937_64
// and the same draw order as the reference so random placements are identical.
#include <algorithm>
#include <cmath>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "internal.h"

namespace pswim {
namespace {

struct V3 {
    double x, y, z;
};
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 scl(V3 v, double s) { return {v.x * s, v.y * s, v.z * s}; }
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline double norm(V3 v) { return std::sqrt(dot(v, v)); }
inline V3 normalized(V3 v) { return scl(v, 1.0 / norm(v)); }

double uniform01(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

void straight_rod(int64_t m, double ds, V3 start, V3 axis, V3 normal, double* rod) {
    const V3 d2 = cross(axis, normal);
    for (int64_t k = 0; k < m; ++k) {
        const V3 x = add(start, scl(axis, static_cast<double>(k) * ds));
        double* q = rod + 12 * k;
        q[0] = x.x; q[1] = x.y; q[2] = x.z;
        q[3] = normal.x; q[4] = normal.y; q[5] = normal.z;
        q[6] = d2.x; q[7] = d2.y; q[8] = d2.z;
        q[9] = axis.x; q[10] = axis.y; q[11] = axis.z;
    }
}

V3 any_normal(V3 a) {
    const V3 pick = std::abs(a.x) <= std::abs(a.y) && std::abs(a.x) <= std::abs(a.z) ? V3{1, 0, 0}
                    : std::abs(a.y) <= std::abs(a.z)                                 ? V3{0, 1, 0}
                                                                                     : V3{0, 0, 1};
    return normalized(sub(pick, scl(a, dot(pick, a))));
}

}  // namespace

int resolve_scenario(const pswim_scenario* sc, pswim_resolved* out, std::string* err) {
    if (!sc) {
        if (err) *err = "scenario: null";
        return PSWIM_EINVAL;
    }
    if (sc->nodes_per_rod < 3) {
        if (err) *err = "scenario: need at least 3 nodes per rod";
        return PSWIM_EINVAL;
    }
    if (sc->rod_count < 1) {
        if (err) *err = "scenario: need at least one rod";
        return PSWIM_EINVAL;
    }
    if (sc->rod_length <= 0.0 || sc->mu <= 0.0) {
        if (err) *err = "scenario: L and mu must be positive";
        return PSWIM_EINVAL;
    }
    const double ds = sc->rod_length / static_cast<double>(sc->nodes_per_rod - 1);
    out->ds = ds;
    out->epsilon = sc->epsilon > 0.0 ? sc->epsilon : 4.0 * ds;
    out->mu = sc->mu;
    out->lj_sigma = sc->lj_sigma > 0.0 ? sc->lj_sigma : 3.0 * out->epsilon;
    out->lj_cutoff = std::pow(2.0, 1.0 / 6.0) * out->lj_sigma;
    int64_t excl = static_cast<int64_t>(std::ceil(out->lj_cutoff / ds)) + 1;
    out->lj_self_exclusion = excl < 4 ? 4 : excl;
    out->total_nodes = sc->rod_count * sc->nodes_per_rod;
    return PSWIM_OK;
}

RodParams rod_params(const pswim_scenario* sc, const pswim_resolved& rs) {
    RodParams p;
    p.rods = sc->rod_count;
    p.m = sc->nodes_per_rod;
    p.length = sc->rod_length;
    p.ds = rs.ds;
    p.inv_ds = 1.0 / rs.ds;
    p.a[0] = sc->a1; p.a[1] = sc->a2; p.a[2] = sc->a3;
    p.b[0] = sc->b1; p.b[1] = sc->b2; p.b[2] = sc->b3;
    p.amplitude = sc->amplitude;
    p.frequency = sc->frequency;
    p.wavelength = sc->wavelength;
    p.epsilon = rs.epsilon;
    p.mu = rs.mu;
    p.lj_well = sc->lj_well_depth;
    p.lj_sigma = rs.lj_sigma;
    p.lj_cutoff = rs.lj_cutoff;
    p.lj_excl = rs.lj_self_exclusion;
    return p;
}

}  // namespace pswim

extern "C" {

void pswim_scenario_defaults(pswim_scenario* s) {
    // ScenarioConfig defaults, scenario.hpp:16-35
    s->rod_count = 1;
    s->nodes_per_rod = 51;
    s->rod_length = 1.0;
    s->a1 = s->a2 = s->a3 = 0.01;
    s->b1 = s->b2 = s->b3 = 2.0;
    s->amplitude = 0.05;
    s->frequency = 2.0 * M_PI;
    s->wavelength = 1.0;
    s->epsilon = 0.0;
    s->mu = 1.0;
    s->wall_mode = 0;
    s->placement = 0;
    s->lj_well_depth = 0.0;
    s->lj_sigma = 0.0;
    s->wall_clearance = 1.0;
    s->seed = 1;
    s->fine_dt = 1e-6;
    s->horizon = 1e-3;
}

int pswim_scenario_resolve(const pswim_scenario* sc, pswim_resolved* out) {
    return pswim::resolve_scenario(sc, out, nullptr);
}

int pswim_build_initial_state(const pswim_scenario* sc, double* state) {
    using namespace pswim;
    pswim_resolved rs;
    const int rc = resolve_scenario(sc, &rs, nullptr);
    if (rc) return rc;
    const int64_t m = sc->nodes_per_rod;
    const double L = sc->rod_length;
    if (sc->placement == 0) {
        // grid: rods parallel to x at height d_z (scenario.cpp:76-84)
        const double gap = std::max(4.0 * rs.lj_sigma, 0.2 * L);
        const auto cols = static_cast<int64_t>(std::ceil(std::sqrt(static_cast<double>(sc->rod_count))));
        for (int64_t i = 0; i < sc->rod_count; ++i) {
            const double gx = static_cast<double>(i % cols) * (L + gap);
            const double gy = static_cast<double>(i / cols) * gap;
            straight_rod(m, rs.ds, V3{gx, gy, sc->wall_clearance}, V3{1, 0, 0}, V3{0, 1, 0}, state + 12 * m * i);
        }
        return PSWIM_OK;
    }
    // random: seeded centre + orientation, rejection on wall clearance and 2 sigma
    // separation (scenario.cpp:86-119)
    std::mt19937_64 rng(sc->seed);
    const double box_xy = 4.0 * L;
    const double dz = sc->wall_clearance;
    const double min_sep = 2.0 * rs.lj_sigma;
    for (int64_t i = 0; i < sc->rod_count; ++i) {
        bool placed = false;
        double* rod = state + 12 * m * i;
        for (int attempt = 0; attempt < 10000 && !placed; ++attempt) {
            const double cx = box_xy * uniform01(rng);
            const double cy = box_xy * uniform01(rng);
            const double cz = dz + 2.0 * L * uniform01(rng);
            const double z = 2.0 * uniform01(rng) - 1.0;
            const double phi = 2.0 * M_PI * uniform01(rng);
            const double s = std::sqrt(std::max(0.0, 1.0 - z * z));
            const V3 axis{s * std::cos(phi), s * std::sin(phi), z};
            const V3 start = sub(V3{cx, cy, cz}, scl(axis, 0.5 * L));
            straight_rod(m, rs.ds, start, axis, any_normal(axis), rod);
            bool ok = true;
            for (int64_t k = 0; k < m && ok; ++k) ok = !(rod[12 * k + 2] < 0.5 * dz);
            for (int64_t j = 0; ok && j < i; ++j) {
                const double* other = state + 12 * m * j;
                double best = std::numeric_limits<double>::infinity();
                for (int64_t a = 0; a < m; ++a)
                    for (int64_t b = 0; b < m; ++b) {
                        const V3 d{rod[12 * a] - other[12 * b], rod[12 * a + 1] - other[12 * b + 1],
                                   rod[12 * a + 2] - other[12 * b + 2]};
                        best = std::min(best, norm(d));
                    }
                if (best < min_sep) ok = false;
            }
            placed = ok;
        }
        if (!placed) return PSWIM_EINVAL;
    }
    return PSWIM_OK;
}

}  // extern "C"
