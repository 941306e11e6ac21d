// oracle/kpo.hpp — CPU restatement of the reference Kino-PAX+ planner.
//
// TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2602_02846_b200/,
// include/) includes, links or calls this file.  Only tests/, the
// __graft_entry__.smoke() checker and bench.py's cpu_baseline / --impl
// reference leg load the shared library built from it (oracle/build/libkpo.so).
//
// What it restates (the reference's planner sources src/*.cpp are absent, see
// SURVEY.md §0; the behaviour is fixed by the shipped headers + SPEC.md):
//   core     proj/include/kinoplan/core/{types,rng,cost,errors}.hpp
//   dynamics proj/include/kinoplan/dynamics/model.hpp,
//   env
//   grid
//   planner  SPEC.md:333-457, PAPER.md:343-504 (Algorithms 1-4)
//
// Two arithmetic policies:
//   Faithful64 — Scalar = double exactly as types.hpp:11, plain a*b+c (the
//                reference builds with g++ -O2, no FMA contraction on x86-64),
//                std::sin/std::cos.  This is "the reference CPU planner" that
//                bench.py times as the CPU baseline.
//   Mirror32   — the same algorithm in fp32 with the pinned operation recipe the
//                device uses (explicit fma where the recipe says
//                MADD, IEEE div/sqrt, polynomial sincos).  Whole runs of the GPU
//                planner must be bit-identical to Mirror32 runs with workers = 1.
// Built with -ffp-contract=off so the compiler never fuses what the recipe
// keeps separate.
#pragma once

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace kpo {

// ---------------------------------------------------------------- errors ----
// errors.hpp:11-33 — the same five classes.
struct SchemaError : std::runtime_error { using std::runtime_error::runtime_error; };
struct InvalidProblemError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct GridTooFineError : std::runtime_error { using std::runtime_error::runtime_error; };
struct InvalidSegmentError : std::invalid_argument { using std::invalid_argument::invalid_argument; };

// ------------------------------------------------------------------ rng -----
// rng.hpp:12-31 SplitMix64.
struct SplitMix64 {
    uint64_t state;
    explicit SplitMix64(uint64_t seed) : state(seed) {}
    uint64_t operator()() {
        state += 0x9E3779B97F4A7C15ULL;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
};

// rng.hpp:34-39 mix64.
inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// rng.hpp:44-52 derive_stream.
inline uint64_t derive_stream(uint64_t seed, uint64_t iteration, uint64_t node_id, uint64_t branch) {
    uint64_t s = mix64(seed);
    s = mix64(s ^ iteration);
    s = mix64(s ^ node_id);
    s = mix64(s ^ branch);
    return s;
}

// rng.hpp:55-57 uniform_unit: 53-bit [0, 1).
inline double uniform_unit(SplitMix64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

// Philox4x32-10 (Salmon et al., SC'11; Random123 constants).  Counter
// (iteration, node id, branch, call), key (seed lo, seed hi).  DECISION
// (SURVEY.md §7 "RNG"): the north-star device RNG; SplitMix64 stays available.
inline void philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
        const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
        const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
        const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// ------------------------------------------------------------ policies ------
// Pinned fp32 sincos recipe: Cody-Waite reduction by pi/2 with
// a two-part constant, Taylor polynomials on |r| <= pi/4 evaluated by Horner
// with fma, quadrant select.  The device implements the same recipe.
inline void sincos_recipe_f32(float x, float* s_out, float* c_out) {
    const float j = std::rint(x * 0x1.45f306p-1f);          // 2/pi
    const int q = static_cast<int>(j);
    float r = std::fma(-j, 0x1.921fb4p+0f, x);               // pi/2 hi
    r = std::fma(-j, 0x1.4442d2p-24f, r);                    // pi/2 lo
    const float r2 = r * r;
    float ps = std::fma(r2, 0x1.71de3ap-19f, -0x1.a01a02p-13f);  // 1/9!, -1/7!
    ps = std::fma(r2, ps, 0x1.111112p-7f);                   // 1/5!
    ps = std::fma(r2, ps, -0x1.555556p-3f);                  // -1/3!
    const float s = std::fma(r * r2, ps, r);
    float pc = std::fma(r2, -0x1.27e4fcp-22f, 0x1.a01a02p-16f);  // -1/10!, 1/8!
    pc = std::fma(r2, pc, -0x1.6c16c2p-10f);                 // -1/6!
    pc = std::fma(r2, pc, 0x1.555556p-5f);                   // 1/4!
    pc = std::fma(r2, pc, -0.5f);
    const float c = std::fma(r2, pc, 1.0f);
    switch (q & 3) {
        case 0: *s_out = s; *c_out = c; break;
        case 1: *s_out = c; *c_out = -s; break;
        case 2: *s_out = -s; *c_out = -c; break;
        default: *s_out = -c; *c_out = s; break;
    }
}

struct Faithful64 {
    using R = double;
    using Enc = uint64_t;
    static R madd(R a, R b, R c) { return a * b + c; }  // two roundings (-ffp-contract=off)
    static constexpr bool kClosedFormDI = false;         // the reference's RK4 for every model
    static constexpr bool kRotatedDubins = false;
    static void sincos(R x, R* s, R* c) { *s = std::sin(x); *c = std::cos(x); }
    static Enc encode(R v) { Enc e; std::memcpy(&e, &v, sizeof e); return e; }
    static R decode(Enc e) { R v; std::memcpy(&v, &e, sizeof v); return v; }
    static constexpr R kPi = 3.14159265358979323846;
};

struct Mirror32 {
    using R = float;
    using Enc = uint32_t;
    static R madd(R a, R b, R c) { return std::fma(a, b, c); }
    static constexpr bool kClosedFormDI = true;  // device recipe: double integrator in closed form
    static constexpr bool kRotatedDubins = true;  // device recipe: Dubins stage trigonometry by rotation
    static void sincos(R x, R* s, R* c) { sincos_recipe_f32(x, s, c); }
    static Enc encode(R v) { Enc e; std::memcpy(&e, &v, sizeof e); return e; }
    static R decode(Enc e) { R v; std::memcpy(&v, &e, sizeof v); return v; }
    static constexpr R kPi = 3.14159265358979323846f;
};

// --------------------------------------------------------------- types -----
constexpr int kMaxStateDim = 12;  // types.hpp:15

template <class R>
struct Vec {  // fixed-max stack vector, as types.hpp:17 (Eigen Matrix<..., 12, 1>)
    R d[kMaxStateDim];
    int n = 0;
    R& operator[](int i) { return d[i]; }
    const R& operator[](int i) const { return d[i]; }
};

struct Interval {  // types.hpp:22-28 closed interval
    double lo = 0, hi = 0;
};

// types.hpp:49-58 wrap_angle to (-pi, pi].
template <class P>
typename P::R wrap_angle(typename P::R a) {
    using R = typename P::R;
    const R pi = P::kPi;
    a = std::fmod(a, 2 * pi);
    if (a <= -pi) a += 2 * pi;
    else if (a > pi) a -= 2 * pi;
    return a;
}

enum class ModelId { DI4 = 0, DI6 = 1, Dubins6 = 2, Quad12 = 3 };
enum class CostKind { PathLength = 0, ControlDuration = 1 };
enum Status : uint8_t { kActive = 0, kInactive = 1, kTerminal = 2 };

struct Obstacle {
    int type = 0;  // 0 box, 1 sphere
    double a[3] = {0, 0, 0};
    double b[3] = {0, 0, 0};
};

// Everything the planner reads, in double (problem values are immutable,
// SPEC.md:104,241).  Policies convert to R at the point of use.
struct ProblemDef {
    ModelId model = ModelId::DI6;
    int n = 6, m = 3;  // state / control dims
    std::vector<int> position_dims;  // model.hpp:33
    std::vector<int> angle_dims;     // model.hpp:36
    // model params (model.hpp:15-22; defaults)
    double mass = 1.0, gravity = 9.81, arm = 1.0, Ixx = 1.0, Iyy = 1.0, Izz = 2.0;
    std::vector<double> x_init;
    std::vector<Interval> state_bounds, control_bounds;
    int ws_dim = 3;
    std::vector<Interval> workspace;
    std::vector<Obstacle> obstacles;
    std::vector<int> goal_dims;
    std::vector<double> goal_center;
    double goal_radius = 0;
    CostKind cost = CostKind::PathLength;
    int cost_position_dims = 3;
    std::vector<int> grid_dims;
    std::vector<int64_t> grid_cells;  // resolved by build_grid
};

struct ConfigDef {
    int lambda = 32, i_max = 5;
    double t_max_s = 0;  // <= 0: unlimited
    double t_prop = 0.5, ode_step = 0.02, collision_step = 0.05;
    uint64_t capacity = 1 << 20, seed = 0, max_iterations = 0;
    int workers = 1;
    bool deactivate_after_expansion = false;
    int rng_kind = 0;  // 0 Philox, 1 SplitMix
    bool stop_at_first_solution = false;
};

// Model table (model.hpp:64-68).  Dubins6 and Quad12
// equations are PROPOSED pins (SPEC.md:170, :184 — the supplement is absent).
inline void model_shape(ModelId id, int* n, int* m, std::vector<int>* pos, std::vector<int>* ang) {
    switch (id) {
        case ModelId::DI4: *n = 4; *m = 2; *pos = {0, 1}; *ang = {}; break;
        case ModelId::DI6: *n = 6; *m = 3; *pos = {0, 1, 2}; *ang = {}; break;
        case ModelId::Dubins6: *n = 6; *m = 3; *pos = {0, 1, 2}; *ang = {3}; break;
        case ModelId::Quad12: *n = 12; *m = 4; *pos = {0, 1, 2}; *ang = {6, 7, 8}; break;
        default: throw SchemaError("unknown model id");
    }
}

// Per-policy constants of a problem, pre-rounded to R once (the device gets the
// same fp32 constants from the host).
template <class P>
struct Consts {
    using R = typename P::R;
    R slo[kMaxStateDim], shi[kMaxStateDim];
    R clo[4], chi[4], cw[4];
    R wlo[3], whi[3];
    std::vector<std::array<R, 6>> boxes;   // lo xyz, hi xyz
    std::vector<std::array<R, 4>> spheres; // c xyz, r^2
    R goal_c[kMaxStateDim];
    R goal_r2;
    R g_lo[8], g_side[8];
    int64_t g_cells[8], g_stride[8];
    R t_prop, h, coll, zero_rate;
    // quad
    R inv_m, grav, cx, cy, cz, inv_ix, inv_iy, inv_iz;
};

template <class P>
Consts<P> make_consts(const ProblemDef& pd, const ConfigDef& cf) {
    using R = typename P::R;
    Consts<P> k{};
    for (int i = 0; i < pd.n; ++i) { k.slo[i] = R(pd.state_bounds[i].lo); k.shi[i] = R(pd.state_bounds[i].hi); }
    for (int i = 0; i < pd.m; ++i) {
        k.clo[i] = R(pd.control_bounds[i].lo);
        k.chi[i] = R(pd.control_bounds[i].hi);
        k.cw[i] = k.chi[i] - k.clo[i];
    }
    for (int i = 0; i < pd.ws_dim; ++i) { k.wlo[i] = R(pd.workspace[i].lo); k.whi[i] = R(pd.workspace[i].hi); }
    for (const auto& o : pd.obstacles) {
        if (o.type == 0) {
            k.boxes.push_back({R(o.a[0]), R(o.a[1]), R(o.a[2]), R(o.b[0]), R(o.b[1]), R(o.b[2])});
        } else {
            const R r = R(o.b[0]);
            k.spheres.push_back({R(o.a[0]), R(o.a[1]), R(o.a[2]), r * r});
        }
    }
    for (size_t i = 0; i < pd.goal_dims.size(); ++i) k.goal_c[i] = R(pd.goal_center[i]);
    { const R r = R(pd.goal_radius); k.goal_r2 = r * r; }
    int64_t stride = 1;
    for (size_t j = 0; j < pd.grid_dims.size(); ++j) {
        const int d = pd.grid_dims[j];
        k.g_lo[j] = R(pd.state_bounds[d].lo);
        k.g_cells[j] = pd.grid_cells[j];
        k.g_side[j] = (R(pd.state_bounds[d].hi) - R(pd.state_bounds[d].lo)) / R(pd.grid_cells[j]);
        k.g_stride[j] = stride;
        stride *= pd.grid_cells[j];
    }
    k.t_prop = R(cf.t_prop);
    k.h = R(cf.ode_step);
    k.coll = R(cf.collision_step);
    k.zero_rate = R(1e-6);  // cost.hpp:30 kZeroDisplacementCostRate
    k.inv_m = R(1) / R(pd.mass);
    k.grav = R(pd.gravity);
    const R ix = R(pd.Ixx), iy = R(pd.Iyy), iz = R(pd.Izz);
    k.cx = (iy - iz) / ix; k.cy = (iz - ix) / iy; k.cz = (ix - iy) / iz;
    k.inv_ix = R(1) / ix; k.inv_iy = R(1) / iy; k.inv_iz = R(1) / iz;
    return k;
}

// ------------------------------------------------------------ dynamics -----
// DynamicsModel::derivative (model.hpp:42).
template <class P>
void derivative(const ProblemDef& pd, const Consts<P>& k, const Vec<typename P::R>& x,
                const Vec<typename P::R>& u, Vec<typename P::R>& out) {
    using R = typename P::R;
    out.n = pd.n;
    switch (pd.model) {
        case ModelId::DI4:  // (x, y, vx, vy), u = (ax, ay)
            out[0] = x[2]; out[1] = x[3]; out[2] = u[0]; out[3] = u[1];
            break;
        case ModelId::DI6:  // SPEC.md:126 (x,y,z,vx,vy,vz), u = accelerations
            out[0] = x[3]; out[1] = x[4]; out[2] = x[5];
            out[3] = u[0]; out[4] = u[1]; out[5] = u[2];
            break;
        case ModelId::Dubins6: {  // SPEC.md:127 (x,y,z,psi,gamma,v); u = (turn, pitch rate, accel)
            R sp, cp, sg, cg;
            P::sincos(x[3], &sp, &cp);
            P::sincos(x[4], &sg, &cg);
            const R vc = x[5] * cg;
            out[0] = vc * cp; out[1] = vc * sp; out[2] = x[5] * sg;
            out[3] = u[0]; out[4] = u[1]; out[5] = u[2];
            break;
        }
        case ModelId::Quad12: {  // SPEC.md:128; (p, v_world, phi theta psi, p q r); u = (T, tx, ty, tz)
            R sph, cph, sth, cth, sps, cps;
            P::sincos(x[6], &sph, &cph);
            P::sincos(x[7], &sth, &cth);
            P::sincos(x[8], &sps, &cps);
            const R a = u[0] * k.inv_m;
            const R t1 = cph * sth;
            out[0] = x[3]; out[1] = x[4]; out[2] = x[5];
            out[3] = a * P::madd(t1, cps, sph * sps);
            out[4] = a * P::madd(t1, sps, -(sph * cps));
            out[5] = P::madd(a, cph * cth, -k.grav);
            const R w = P::madd(x[10], sph, x[11] * cph);  // q sin(phi) + r cos(phi)
            const R ic = R(1) / cth;                          // sec(theta)
            out[6] = P::madd(w, sth * ic, x[9]);
            out[7] = P::madd(x[10], cph, -(x[11] * sph));
            out[8] = w * ic;
            out[9] = P::madd(k.cx, x[10] * x[11], u[1] * k.inv_ix);
            out[10] = P::madd(k.cy, x[9] * x[11], u[2] * k.inv_iy);
            out[11] = P::madd(k.cz, x[9] * x[10], u[3] * k.inv_iz);
            break;
        }
    }
}

// ----------------------------------------------------------- sampling ------
// sample_control + sample_duration for one
// work item.  DECISION: controls in axis order, then dt = t_prop * (1 - U)
// so dt in (0, t_prop].
template <class P>
void sample_item(const ProblemDef& pd, const ConfigDef& cf, const Consts<P>& k, uint64_t iteration,
                 uint64_t node_id, uint64_t branch, Vec<typename P::R>& u, typename P::R& dt) {
    using R = typename P::R;
    u.n = pd.m;
    if (cf.rng_kind == 1) {
        SplitMix64 rng(derive_stream(cf.seed, iteration, node_id, branch));
        for (int i = 0; i < pd.m; ++i) {
            const double U = uniform_unit(rng);
            const double lo = pd.control_bounds[i].lo, hi = pd.control_bounds[i].hi;
            u[i] = R(lo + (hi - lo) * U);
        }
        const double U = uniform_unit(rng);
        dt = R(cf.t_prop * (1.0 - U));
    } else {
        uint32_t r[8];
        const uint32_t key[2] = {static_cast<uint32_t>(cf.seed), static_cast<uint32_t>(cf.seed >> 32)};
        uint32_t ctr[4] = {static_cast<uint32_t>(iteration), static_cast<uint32_t>(node_id),
                           static_cast<uint32_t>(branch), 0u};
        philox4x32_10(ctr, key, r);
        if (pd.m + 1 > 4) { ctr[3] = 1u; philox4x32_10(ctr, key, r + 4); }
        for (int i = 0; i < pd.m; ++i) {
            const R U = R(r[i] >> 8) * R(0x1.0p-24);
            u[i] = P::madd(k.cw[i], U, k.clo[i]);
        }
        const R U = R(r[pd.m] >> 8) * R(0x1.0p-24);
        dt = k.t_prop * (R(1) - U);
    }
}

// ---------------------------------------------------------- integrator -----
// propagate_ode: classical RK4, ZOH control, samples at
// 0, h, 2h, ..., dt (last step shortened), angles wrapped after every step,
// non-finite -> diverged.  Returns false on divergence.
template <class P>
bool propagate_ode(const ProblemDef& pd, const Consts<P>& k, const Vec<typename P::R>& x0,
                   const Vec<typename P::R>& u, typename P::R dt, typename P::R h,
                   std::vector<Vec<typename P::R>>& samples) {
    using R = typename P::R;
    samples.clear();
    samples.push_back(x0);  // samples[0] = x, bit-exact
    const int n = pd.n;
    const R q = dt / h;
    int S = static_cast<int>(std::ceil(q));
    if (S < 1) S = 1;
    if constexpr (P::kClosedFormDI) {
        if (pd.model == ModelId::DI4 || pd.model == ModelId::DI6) {
            // RK4 with constant control is exact on the double integrator
            // (SPEC.md:138-139): the device evaluates every sample in closed
            // form from x0, p = MADD(u/2, t*t, MADD(v0, t, p0)), v = MADD(u, t, v0),
            // t = (s+1) h, the last sample at dt (skipped when dt - (S-1) h <= 0)
            const int D = n / 2;
            Vec<R> x;
            x.n = n;
            for (int s = 0; s < S; ++s) {
                R t = R(s + 1) * h;
                if (s + 1 == S) {
                    if (!(dt - R(S - 1) * h > R(0))) break;
                    t = dt;
                }
                const R tt = t * t;
                for (int i = 0; i < D; ++i) {
                    x[i] = P::madd(R(0.5) * u[i], tt, P::madd(x0[D + i], t, x0[i]));
                    x[D + i] = P::madd(u[i], t, x0[D + i]);
                }
                for (int i = 0; i < n; ++i)
                    if (!std::isfinite(x[i])) return false;
                samples.push_back(x);
            }
            return true;
        }
    }
    Vec<R> x = x0, k1, k2, k3, k4, t;
    t.n = n;
    for (int s = 0; s < S; ++s) {
        const R hk = (s + 1 < S) ? h : dt - R(S - 1) * h;
        if (!(hk > R(0))) break;
        const R half = R(0.5) * hk;
        if constexpr (P::kRotatedDubins) {
            if (pd.model == ModelId::Dubins6) {
                // the device recipe (kp_math.cuh rk4_step<2>): heading and
                // flight-path rates are the constant controls, so the stage angles'
                // sines / cosines are those of the step's start rotated by
                // {sin, cos}(hk/2 u) and {sin, cos}(hk u); stage 3 equals stage 2
                R rot[8];
                P::sincos(half * u[0], &rot[0], &rot[1]);
                P::sincos(hk * u[0], &rot[2], &rot[3]);
                P::sincos(half * u[1], &rot[4], &rot[5]);
                P::sincos(hk * u[1], &rot[6], &rot[7]);
                auto rot2 = [](R s, R c, R rs, R rc, R* so, R* co) {
                    *so = P::madd(s, rc, c * rs);
                    *co = P::madd(c, rc, -(s * rs));
                };
                auto slope = [&](R sp, R cp, R sg, R cg, R v, Vec<R>& f) {
                    f.n = n;
                    const R vc = v * cg;
                    f[0] = vc * cp; f[1] = vc * sp; f[2] = v * sg;
                    f[3] = u[0]; f[4] = u[1]; f[5] = u[2];
                };
                R sp, cp, sg, cg;
                P::sincos(x[3], &sp, &cp);
                P::sincos(x[4], &sg, &cg);
                slope(sp, cp, sg, cg, x[5], k1);
                R sp1, cp1, sg1, cg1;
                rot2(sp, cp, rot[0], rot[1], &sp1, &cp1);
                rot2(sg, cg, rot[4], rot[5], &sg1, &cg1);
                slope(sp1, cp1, sg1, cg1, P::madd(half, u[2], x[5]), k2);
                for (int i = 0; i < n; ++i) k1[i] = P::madd(R(2), k2[i], P::madd(R(2), k2[i], k1[i]));
                R sp2, cp2, sg2, cg2;
                rot2(sp, cp, rot[2], rot[3], &sp2, &cp2);
                rot2(sg, cg, rot[6], rot[7], &sg2, &cg2);
                slope(sp2, cp2, sg2, cg2, P::madd(hk, u[2], x[5]), k4);
                const R sixth = hk / R(6);
                for (int i = 0; i < n; ++i) x[i] = P::madd(sixth, k1[i] + k4[i], x[i]);
                for (int ad : pd.angle_dims) x[ad] = wrap_angle<P>(x[ad]);
                for (int i = 0; i < n; ++i)
                    if (!std::isfinite(x[i])) return false;
                samples.push_back(x);
                continue;
            }
        }
        // slopes accumulated in production order: acc = ((k1 + 2 k2) + 2 k3) + k4
        // (the device keeps only acc and the current stage live)
        Vec<R>& acc = k1;
        derivative<P>(pd, k, x, u, acc);
        for (int i = 0; i < n; ++i) t[i] = P::madd(half, acc[i], x[i]);
        derivative<P>(pd, k, t, u, k2);
        for (int i = 0; i < n; ++i) {
            t[i] = P::madd(half, k2[i], x[i]);
            acc[i] = P::madd(R(2), k2[i], acc[i]);
        }
        derivative<P>(pd, k, t, u, k3);
        for (int i = 0; i < n; ++i) {
            t[i] = P::madd(hk, k3[i], x[i]);
            acc[i] = P::madd(R(2), k3[i], acc[i]);
        }
        derivative<P>(pd, k, t, u, k4);
        const R sixth = hk / R(6);
        for (int i = 0; i < n; ++i) x[i] = P::madd(sixth, acc[i] + k4[i], x[i]);
        for (int ad : pd.angle_dims) x[ad] = wrap_angle<P>(x[ad]);
        for (int i = 0; i < n; ++i)
            if (!std::isfinite(x[i])) return false;
        samples.push_back(x);
    }
    return true;
}

// --------------------------------------------------------- environment -----
template <class P>
bool point_in_obstacle(const ProblemDef& pd, const Consts<P>& k, const typename P::R* p) {
    using R = typename P::R;
    const int w = pd.ws_dim;
    for (const auto& b : k.boxes) {  // closed box
        bool in = true;
        for (int i = 0; i < w; ++i) in = in && (p[i] >= b[i] && p[i] <= b[3 + i]);
        if (in) return true;
    }
    for (const auto& s : k.spheres) {
        R d2 = (p[0] - s[0]) * (p[0] - s[0]);
        for (int i = 1; i < w; ++i) { const R d = p[i] - s[i]; d2 = P::madd(d, d, d2); }
        if (d2 <= s[3]) return true;
    }
    return false;
}

// is_state_valid.
template <class P>
bool is_state_valid(const ProblemDef& pd, const Consts<P>& k, const Vec<typename P::R>& x) {
    using R = typename P::R;
    for (int i = 0; i < pd.n; ++i)
        if (!(x[i] >= k.slo[i] && x[i] <= k.shi[i])) return false;
    R p[3] = {0, 0, 0};
    for (int i = 0; i < pd.ws_dim; ++i) {
        p[i] = x[pd.position_dims[i]];
        if (!(p[i] >= k.wlo[i] && p[i] <= k.whi[i])) return false;
    }
    return !point_in_obstacle<P>(pd, k, p);
}

// Euclidean norm of the position difference, recipe: d2 = a0*a0, then
// d2 = MADD(ai, ai, d2), sqrt (cost.hpp:60 `.norm()`).
template <class P>
typename P::R pos_delta_norm(int m, const typename P::R* dlt) {
    using R = typename P::R;
    R d2 = dlt[0] * dlt[0];
    for (int i = 1; i < m; ++i) d2 = P::madd(dlt[i], dlt[i], d2);
    return std::sqrt(d2);
}

// is_segment_valid.  DECISION: between
// consecutive samples a, b with d = ||b - a|| > c, k is the smallest power of
// two with d / k <= c (dyadic, capped at 2^24) and the points
// p_j = MADD(j/k, b - a, a), j = 1..k-1, are obstacle-checked.  Dyadic points
// nest, so a finer collision_step re-checks every coarser point: the SPEC.md:231
// monotone-refinement property holds exactly (ceil(d/c) points would not nest).
template <class P>
bool is_segment_valid(const ProblemDef& pd, const Consts<P>& k,
                      const std::vector<Vec<typename P::R>>& samples) {
    using R = typename P::R;
    const int w = pd.ws_dim;
    for (size_t i = 0; i < samples.size(); ++i) {
        if (!is_state_valid<P>(pd, k, samples[i])) return false;
        if (i == 0) continue;
        R a[3], dl[3];
        for (int j = 0; j < w; ++j) {
            a[j] = samples[i - 1][pd.position_dims[j]];
            dl[j] = samples[i][pd.position_dims[j]] - a[j];
        }
        const R d = pos_delta_norm<P>(w, dl);
        if (d > k.coll) {
            int kk = 2;
            while (d / R(kk) > k.coll && kk < (1 << 24)) kk <<= 1;
            for (int jj = 1; jj < kk; ++jj) {
                const R t = R(jj) / R(kk);
                R p[3] = {0, 0, 0};
                for (int j = 0; j < w; ++j) p[j] = P::madd(t, dl[j], a[j]);
                if (point_in_obstacle<P>(pd, k, p)) return false;
            }
        }
    }
    return true;
}

// ---------------------------------------------------------------- cost -----
// segment_cost (cost.hpp:44-67).
template <class P>
typename P::R segment_cost(const ProblemDef& pd, const Consts<P>& k,
                           const std::vector<Vec<typename P::R>>& samples, typename P::R duration) {
    using R = typename P::R;
    if (samples.size() < 2) throw InvalidSegmentError("segment_cost: segment needs at least 2 samples");
    if (!(duration > 0)) throw InvalidSegmentError("segment_cost: segment duration must be positive");
    if (pd.cost == CostKind::ControlDuration) return duration;
    const int d = pd.cost_position_dims;
    if constexpr (P::kClosedFormDI) {
        if (pd.model == ModelId::DI4 || pd.model == ModelId::DI6) {
            // device recipe: segment lengths rounded to multiples
            // of 2^-40, summed exactly as a 64-bit integer, one rounding to R
            long long fx = 0;
            for (size_t i = 1; i < samples.size(); ++i) {
                R dl[kMaxStateDim];
                for (int j = 0; j < d; ++j) dl[j] = samples[i][j] - samples[i - 1][j];
                fx += std::llrint(static_cast<double>(pos_delta_norm<P>(d, dl)) * 0x1p40);
            }
            if (fx == 0) return k.zero_rate * duration;
            return static_cast<R>(fx) * R(0x1p-40);
        }
    }
    R total = 0;
    for (size_t i = 1; i < samples.size(); ++i) {
        R dl[kMaxStateDim];
        for (int j = 0; j < d; ++j) dl[j] = samples[i][j] - samples[i - 1][j];
        total += pos_delta_norm<P>(d, dl);
    }
    if (total == 0) return k.zero_rate * duration;
    return total;
}

// in_goal (cost.hpp:77-84), boundary inclusive.
template <class P>
bool in_goal(const ProblemDef& pd, const Consts<P>& k, const Vec<typename P::R>& x) {
    using R = typename P::R;
    const int g = static_cast<int>(pd.goal_dims.size());
    R dx = x[pd.goal_dims[0]] - k.goal_c[0];
    R d2 = dx * dx;
    for (int i = 1; i < g; ++i) { dx = x[pd.goal_dims[i]] - k.goal_c[i]; d2 = P::madd(dx, dx, d2); }
    return d2 <= k.goal_r2;
}

// ---------------------------------------------------------------- grid -----
// build_grid: cells_i = max(1, ceil((hi-lo)_i sqrt(n)/delta)).
inline void build_grid(ProblemDef& pd, const std::vector<int64_t>& cells, double delta,
                       uint64_t max_cells) {
    const int nd = static_cast<int>(pd.grid_dims.size());
    pd.grid_cells.assign(nd, 1);
    long double total = 1;
    for (int j = 0; j < nd; ++j) {
        const Interval& b = pd.state_bounds[pd.grid_dims[j]];
        int64_t c;
        if (!cells.empty()) c = cells[j];
        else c = std::max<int64_t>(1, static_cast<int64_t>(std::ceil((b.hi - b.lo) * std::sqrt(double(nd)) / delta)));
        if (c < 1) throw ConfigError("cells_per_dim must be >= 1");
        pd.grid_cells[j] = c;
        total *= c;
    }
    if (total > static_cast<long double>(max_cells))
        throw GridTooFineError("region grid would have " + std::to_string(static_cast<double>(total)) +
                               " cells, above the ceiling " + std::to_string(max_cells));
}

// region_index: clamp(floor((x - lo)/side), 0, cells-1),
// row-major, dim 0 fastest.
template <class P>
uint32_t region_index(const ProblemDef& pd, const Consts<P>& k, const Vec<typename P::R>& x) {
    using R = typename P::R;
    int64_t r = 0;
    for (size_t j = 0; j < pd.grid_dims.size(); ++j) {
        const R v = (x[pd.grid_dims[j]] - k.g_lo[j]) / k.g_side[j];
        const R fv = std::floor(v);
        int64_t i;
        if (fv < R(0)) i = 0;
        else if (fv > R(k.g_cells[j] - 1)) i = k.g_cells[j] - 1;
        else i = static_cast<int64_t>(fv);
        r += i * k.g_stride[j];
    }
    return static_cast<uint32_t>(r);
}

enum class Outcome { Improved = 0, Equal = 1, Worse = 2 };

// try_update_region_cost: CAS loop on the order-preserving
// encoding (nonnegative IEEE bit patterns are monotone as unsigned).
template <class P>
Outcome try_update(std::atomic<typename P::Enc>& cell, typename P::R c) {
    using Enc = typename P::Enc;
    const Enc e = P::encode(c);
    Enc old = cell.load(std::memory_order_relaxed);
    while (true) {
        if (e > old) return Outcome::Worse;
        if (e == old) return Outcome::Equal;
        if (cell.compare_exchange_weak(old, e, std::memory_order_acq_rel, std::memory_order_relaxed))
            return Outcome::Improved;
    }
}

// --------------------------------------------------------- worker pool -----
// worker_pool.cpp (absent): parallel-for with a barrier at the
// end of every pass; workers = 1 runs the same code path serially in order.
class WorkerPool {
public:
    explicit WorkerPool(int workers) : n_(std::max(1, workers)) {
        for (int t = 1; t < n_; ++t) threads_.emplace_back([this, t] { loop(t); });
    }
    ~WorkerPool() {
        { std::lock_guard<std::mutex> g(m_); stop_ = true; ++gen_; }
        cv_.notify_all();
        for (auto& th : threads_) th.join();
    }
    int size() const { return n_; }
    // fn(worker, begin, end) over [0, count) in n_ contiguous chunks; barrier on return.
    void parallel_for(size_t count, const std::function<void(int, size_t, size_t)>& fn) {
        if (n_ == 1 || count < 2) { fn(0, 0, count); return; }
        {
            std::lock_guard<std::mutex> g(m_);
            fn_ = &fn; count_ = count; pending_ = n_ - 1; ++gen_;
        }
        cv_.notify_all();
        run_chunk(0);
        std::unique_lock<std::mutex> lk(m_);
        done_cv_.wait(lk, [this] { return pending_ == 0; });
        fn_ = nullptr;
    }

private:
    void run_chunk(int t) {
        const size_t b = count_ * t / n_, e = count_ * (t + 1) / n_;
        if (b < e) (*fn_)(t, b, e);
    }
    void loop(int t) {
        uint64_t seen = 0;
        while (true) {
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
            }
            run_chunk(t);
            {
                std::lock_guard<std::mutex> g(m_);
                if (--pending_ == 0) done_cv_.notify_one();
            }
        }
    }
    int n_;
    std::vector<std::thread> threads_;
    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int, size_t, size_t)>* fn_ = nullptr;
    size_t count_ = 0;
    int pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// -------------------------------------------------------------- planner ----
struct Stats {  // PlannerStats
    uint64_t iterations = 0, attempted = 0, valid = 0, admitted = 0, committed = 0;
    uint64_t pruned_terminal = 0, deactivated = 0, reactivated = 0, dropped_capacity = 0;
    bool capacity_exhausted = false;
};

struct TimelineEntry {
    uint64_t iteration;
    double elapsed_s;
    double cost;
    int64_t leaf;
};

template <class P>
class Planner {
public:
    using R = typename P::R;
    using Enc = typename P::Enc;

    struct Node {
        Vec<R> state, u;
        R dt = 0, acc = 0;
        int64_t parent = -1;
        uint32_t region = 0;
        uint8_t status = kActive;
        uint32_t icnt = 0;
    };
    struct Candidate {  // V_U entry
        Vec<R> state, u;
        R dt, acc;
        int64_t parent;
        uint32_t region;
        uint64_t slot;
        bool goal;
    };

    Planner(const ProblemDef& pd, const ConfigDef& cf)
        : pd_(pd), cf_(cf), k_(make_consts<P>(pd, cf)), pool_(cf.workers) {
        int64_t total = 1;
        for (auto c : pd.grid_cells) total *= c;
        n_regions_ = static_cast<size_t>(total);
        table_ = std::vector<std::atomic<Enc>>(n_regions_);
        reset();
    }

    // Alg. 1 lines 1-5: root Active, grid +inf, best +inf.
    // DECISION: the root's region is seeded with cost 0 so the region-dominance
    // invariant holds for the root too.
    void reset() {
        const Enc inf = P::encode(std::numeric_limits<R>::infinity());
        for (auto& c : table_) c.store(inf, std::memory_order_relaxed);
        nodes_.clear();
        nodes_.reserve(std::min<uint64_t>(cf_.capacity, 1u << 22));
        Node root;
        root.state.n = pd_.n;
        for (int i = 0; i < pd_.n; ++i) root.state[i] = R(pd_.x_init[i]);
        root.u.n = pd_.m;
        for (int i = 0; i < pd_.m; ++i) root.u[i] = 0;
        root.region = region_index<P>(pd_, k_, root.state);
        nodes_.push_back(root);
        try_update<P>(table_[root.region], R(0));
        va_ = {0};
        best_cost_ = std::numeric_limits<R>::infinity();
        best_leaf_ = -1;
        best_iter_ = 0;
        best_t_ = 0;
        first_t_ = -1;
        first_iter_ = 0;
        first_cost_ = std::numeric_limits<R>::infinity();
        stats_ = Stats{};
        timeline_.clear();
        iteration_ = 0;
        elapsed_ = 0;
    }

    // One work item of Alg. 2; returns 0 valid, 1 invalid, 2 diverged.
    int propagate_item(const Vec<R>& parent_state, R parent_acc, uint64_t node_id, uint64_t branch,
                       uint64_t iteration, Candidate& c, std::vector<Vec<R>>& samples) const {
        sample_item<P>(pd_, cf_, k_, iteration, node_id, branch, c.u, c.dt);
        if (!propagate_ode<P>(pd_, k_, parent_state, c.u, c.dt, k_.h, samples)) return 2;
        if (!is_segment_valid<P>(pd_, k_, samples)) return 1;
        c.state = samples.back();
        c.acc = parent_acc + segment_cost<P>(pd_, k_, samples, c.dt);
        c.region = region_index<P>(pd_, k_, c.state);
        c.goal = in_goal<P>(pd_, k_, c.state);
        return 0;
    }

    // propagate_pass.
    void propagate_pass() {
        const size_t lam = static_cast<size_t>(cf_.lambda);
        const size_t items = va_.size() * lam;
        const int W = pool_.size();
        std::vector<std::vector<Candidate>> local(W);
        std::vector<uint64_t> valid(W, 0), admitted(W, 0);
        pool_.parallel_for(items, [&](int w, size_t b, size_t e) {
            std::vector<Vec<R>> samples;
            samples.reserve(64);
            for (size_t i = b; i < e; ++i) {
                const size_t f = i / lam;
                const uint64_t br = i % lam;
                const Node& x = nodes_[va_[f]];
                Candidate c;
                if (propagate_item(x.state, x.acc, va_[f], br, iteration_, c, samples) != 0) continue;
                ++valid[w];
                if (try_update<P>(table_[c.region], c.acc) != Outcome::Worse) {
                    c.parent = static_cast<int64_t>(va_[f]);
                    c.slot = i;
                    local[w].push_back(c);
                    ++admitted[w];
                }
            }
        });
        vu_.clear();
        for (int w = 0; w < W; ++w) {
            stats_.valid += valid[w];
            stats_.admitted += admitted[w];
            vu_.insert(vu_.end(), local[w].begin(), local[w].end());
        }
        // chunks are contiguous and in worker order, so vu_ is in slot order
        stats_.attempted += items;
    }

    R region_cost(uint32_t r) const { return P::decode(table_[r].load(std::memory_order_relaxed)); }

    // prune_pass with the SPEC.md:434-437 priority rules.
    void prune_pass() {
        const int W = pool_.size();
        std::vector<uint64_t> term(W, 0), deact(W, 0), react(W, 0);
        pool_.parallel_for(nodes_.size(), [&](int w, size_t b, size_t e) {
            for (size_t i = b; i < e; ++i) {
                Node& x = nodes_[i];
                if (x.status == kTerminal) continue;  // absorbing
                if (x.acc > region_cost(x.region)) {  // (1)
                    x.status = kTerminal;
                    ++term[w];
                } else if (x.status == kInactive) {  // (2)
                    x.icnt += 1;
                    if (x.icnt > static_cast<uint32_t>(cf_.i_max)) {
                        x.status = kActive;
                        x.icnt = 0;
                        ++react[w];
                    }
                } else if (x.status == kActive) {  // (3)
                    bool dominated = cf_.deactivate_after_expansion;
                    for (int64_t p = x.parent; p >= 0 && !dominated; p = nodes_[p].parent) {
                        const Node& a = nodes_[p];
                        if (a.acc > region_cost(a.region)) dominated = true;
                    }
                    if (dominated) {
                        x.status = kInactive;
                        x.icnt = 0;
                        ++deact[w];
                    }
                }
            }
        });
        for (int w = 0; w < W; ++w) {
            stats_.pruned_terminal += term[w];
            stats_.deactivated += deact[w];
            stats_.reactivated += react[w];
        }
    }

    // update_tree_pass; serial in slot order.
    void update_tree_pass() {
        for (const Candidate& c : vu_) {
            if (P::encode(c.acc) != table_[c.region].load(std::memory_order_relaxed)) continue;
            if (nodes_.size() >= cf_.capacity) {  // store full -> dropped
                stats_.capacity_exhausted = true;
                ++stats_.dropped_capacity;
                continue;
            }
            Node nd;
            nd.state = c.state; nd.u = c.u; nd.dt = c.dt; nd.acc = c.acc;
            nd.parent = c.parent; nd.region = c.region; nd.status = kActive; nd.icnt = 0;
            const int64_t id = static_cast<int64_t>(nodes_.size());
            nodes_.push_back(nd);
            ++stats_.committed;
            if (c.goal && c.acc < best_cost_) {  // Alg. 4 lines 5-7
                best_cost_ = c.acc;
                best_leaf_ = id;
            }
        }
        vu_.clear();
        // V_A for the next iteration: Active nodes in id order.
        va_.clear();
        for (size_t i = 0; i < nodes_.size(); ++i)
            if (nodes_[i].status == kActive) va_.push_back(i);
    }

    bool live() const {
        for (const auto& n : nodes_)
            if (n.status != kTerminal) return true;
        return false;
    }

    // plan: iterate until t_max / max_iterations.
    void run(double budget_s, uint64_t max_iters, bool stop_first) {
        const auto t0 = std::chrono::steady_clock::now();
        auto now_s = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
        const uint64_t start_iter = iteration_;
        while (true) {
            if (max_iters && iteration_ - start_iter >= max_iters) break;
            if (budget_s > 0 && now_s() >= budget_s) break;
            if (stop_first && best_leaf_ >= 0) break;
            if (va_.empty() && !live()) break;
            const R before = best_cost_;
            propagate_pass();
            prune_pass();
            update_tree_pass();
            ++iteration_;
            ++stats_.iterations;
            elapsed_ = now_s();
            if (best_cost_ < before) {
                best_t_ = elapsed_;
                best_iter_ = iteration_;
                timeline_.push_back({iteration_, elapsed_, double(best_cost_), best_leaf_});
                if (first_t_ < 0) { first_t_ = elapsed_; first_iter_ = iteration_; first_cost_ = best_cost_; }
            }
        }
    }

    const ProblemDef& problem() const { return pd_; }
    const Consts<P>& consts() const { return k_; }
    const std::vector<Node>& nodes() const { return nodes_; }
    const std::vector<std::atomic<Enc>>& table() const { return table_; }
    const Stats& stats() const { return stats_; }
    const std::vector<TimelineEntry>& timeline() const { return timeline_; }
    R best_cost() const { return best_cost_; }
    int64_t best_leaf() const { return best_leaf_; }
    double best_t() const { return best_t_; }
    uint64_t best_iter() const { return best_iter_; }
    double first_t() const { return first_t_; }
    uint64_t first_iter() const { return first_iter_; }
    R first_cost() const { return first_cost_; }
    double elapsed() const { return elapsed_; }
    uint64_t iteration() const { return iteration_; }
    size_t n_regions() const { return n_regions_; }

private:
    ProblemDef pd_;
    ConfigDef cf_;
    Consts<P> k_;
    WorkerPool pool_;
    size_t n_regions_ = 0;
    std::vector<std::atomic<Enc>> table_;
    std::vector<Node> nodes_;
    std::vector<uint64_t> va_;
    std::vector<Candidate> vu_;
    R best_cost_;
    int64_t best_leaf_ = -1;
    uint64_t best_iter_ = 0, first_iter_ = 0;
    double best_t_ = 0, first_t_ = -1;
    R first_cost_;
    Stats stats_;
    std::vector<TimelineEntry> timeline_;
    uint64_t iteration_ = 0;
    double elapsed_ = 0;
};

}  // namespace kpo
