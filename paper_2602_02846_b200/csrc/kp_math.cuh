// kp_math.cuh — per-work-item device arithmetic of the Kino-PAX+ iteration.
//
// This is the pinned fp32 operation recipe of DESIGN.md §4.  The whole
// library is compiled with --fmad=false, so `a * b + c` is two roundings and
// only the explicit fmaf() calls below fuse; division and sqrt are IEEE
// (-prec-div/-prec-sqrt defaults, no fast-math, no FTZ).  Under that recipe a
// work item's verdict, region, cost bits and final state are bit-identical to
// the reference restatement run in fp32 (oracle Mirror32 policy).
//
// Reference behaviour followed (file:line):
//   sampling      rng.hpp:12-57
//   dynamics      model.hpp:42 (derivative)
//   integrator    SPEC.md:132-140, :163-171; wrap_angle types.hpp:49-58
//   validity      SPEC.md:200-218, :236-237; contains types.hpp:22-39
//   cost          cost.hpp:44-67 (segment_cost), :77-84 (in_goal)
//   region
#pragma once
#include <stdint.h>

#include "kp_types.h"

#define KP_DEV __device__ __forceinline__

namespace kp {

#ifdef KP_CHECKS
__device__ unsigned int kp_check_code;
__device__ __noinline__ void check_fail(unsigned int code) { atomicCAS(&kp_check_code, 0u, code); }
#endif

// ------------------------------------------------------------------- RNG ---
KP_DEV uint64_t mix64(uint64_t z) {  // rng.hpp:34-39
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

KP_DEV uint64_t derive_stream(uint64_t seed, uint64_t it, uint64_t node, uint64_t br) {  // rng.hpp:44-52
    uint64_t s = mix64(seed);
    s = mix64(s ^ it);
    s = mix64(s ^ node);
    s = mix64(s ^ br);
    return s;
}

struct SplitMix64 {  // rng.hpp:12-31
    uint64_t state;
    KP_DEV uint64_t next() {
        state += 0x9E3779B97F4A7C15ULL;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    KP_DEV double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }  // rng.hpp:55-57
};

// Philox4x32-10, counter (c0..c3), key (k0, k1).
KP_DEV uint4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    return make_uint4(c0, c1, c2, c3);
}

// sample_control + sample_duration for one work item (controls in axis
// order, then dt = t_prop * (1 - U) in (0, t_prop]).
template <int M>
KP_DEV void sample_item(const KpProblem& P, uint64_t seed, uint32_t it, uint32_t node, uint32_t br, float* u,
                        float& dt) {
    if (P.rng_kind == 1) {
        SplitMix64 r{derive_stream(seed, it, node, br)};
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const double U = r.unit();
            u[i] = static_cast<float>(P.clo_d[i] + (P.chi_d[i] - P.clo_d[i]) * U);
        }
        const double U = r.unit();
        dt = static_cast<float>(P.t_prop_d * (1.0 - U));
    } else {
        const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
        const uint4 a = philox(it, node, br, 0u, k0, k1);
        uint32_t r[8] = {a.x, a.y, a.z, a.w, 0u, 0u, 0u, 0u};
        if (M + 1 > 4) {
            const uint4 b = philox(it, node, br, 1u, k0, k1);
            r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
        }
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const float U = static_cast<float>(r[i] >> 8) * 0x1.0p-24f;
            u[i] = fmaf(P.cw[i], U, P.clo[i]);
        }
        const float U = static_cast<float>(r[M] >> 8) * 0x1.0p-24f;
        dt = P.t_prop * (1.0f - U);
    }
}

// ----------------------------------------------------------------- math ---
// Pinned sincos recipe, identical to the oracle's.
KP_DEV void sincos_poly(float r, float& s, float& c) {  // |r| <= pi/4
    const float r2 = r * r;
    float ps = fmaf(r2, 0x1.71de3ap-19f, -0x1.a01a02p-13f);
    ps = fmaf(r2, ps, 0x1.111112p-7f);
    ps = fmaf(r2, ps, -0x1.555556p-3f);
    s = fmaf(r * r2, ps, r);
    float pc = fmaf(r2, -0x1.27e4fcp-22f, 0x1.a01a02p-16f);
    pc = fmaf(r2, pc, -0x1.6c16c2p-10f);
    pc = fmaf(r2, pc, 0x1.555556p-5f);
    pc = fmaf(r2, pc, -0.5f);
    c = fmaf(r2, pc, 1.0f);
}

// SMALL: an angle whose state bounds keep it inside (-pi/4, pi/4) (the
// quadcopter's roll and pitch, |phi|, |theta| <= 0.6; the airplane's flight
// path angle, |gamma| <= 0.5, and the per-segment Dubins shifts).  When
// |x * 2/pi| < 1/2, j = 0, r == x exactly (fma(-0, c, x) == x) and there is no
// quadrant fix-up: the same bits as the general path without its reduction and
// select instructions.  A plain per-lane test: for these angles it is
// warp-uniform in practice (a warp vote made it slower); headings (psi) always
// take the general path, where a divergent branch would run both.
template <bool SMALL = false>
KP_DEV void sincos_recipe(float x, float& s_out, float& c_out) {
    if constexpr (SMALL) {
        if (fabsf(x * 0x1.45f306p-1f) < 0.5f) {
            sincos_poly(x, s_out, c_out);
            return;
        }
    }
    // j = rint(x * 2/pi) with round-half-even via the 1.5 * 2^23 magic add (bit-identical
    // to rintf for |x * 2/pi| < 2^22) and the quadrant from the sum's integer bits: no
    // XU-pipe conversion instructions
    const float t = x * 0x1.45f306p-1f + 12582912.0f;
    const float j = t - 12582912.0f;
    const int q = __float_as_int(t) - 0x4B400000;
    float r = fmaf(-j, 0x1.921fb4p+0f, x);
    r = fmaf(-j, 0x1.4442d2p-24f, r);
    float s, c;
    sincos_poly(r, s, c);
    // quadrant select without branches: q&1 swaps (s, c) -> (c, -s); q&2 negates both
    float so = (q & 1) ? c : s;
    float co = (q & 1) ? -s : c;
    if (q & 2) { so = -so; co = -co; }
    s_out = so;
    c_out = co;
}

// wrap_angle (types.hpp:49-58) in fp32; only called outside (-pi, pi], where
// fmodf is exact, so the result equals calling it unconditionally.
KP_DEV float wrap_angle(float a) {
    const float pi = 3.14159265358979323846f;
    if (a > pi || a <= -pi) {
        a = fmodf(a, 2.0f * pi);
        if (a <= -pi) a += 2.0f * pi;
        else if (a > pi) a -= 2.0f * pi;
    }
    return a;
}

// Two small-range angles at once (the quadcopter's roll and pitch): one branch
// for both — the fast path when both have j = 0, else the general path for
// both (same bits either way).
KP_DEV void sincos2_small(float a, float b, float& sa, float& ca, float& sb, float& cb) {
    if (fmaxf(fabsf(a * 0x1.45f306p-1f), fabsf(b * 0x1.45f306p-1f)) < 0.5f) {
        sincos_poly(a, sa, ca);
        sincos_poly(b, sb, cb);
        return;
    }
    sincos_recipe(a, sa, ca);
    sincos_recipe(b, sb, cb);
}

// ------------------------------------------------------------ dynamics ----
template <int MODEL> struct Model;
template <> struct Model<0> { static constexpr int N = 4, M = 2, NA = 0, A0 = 0; };   // double_integrator_4d
template <> struct Model<1> { static constexpr int N = 6, M = 3, NA = 0, A0 = 0; };   // double_integrator_6d
template <> struct Model<2> { static constexpr int N = 6, M = 3, NA = 1, A0 = 3; };   // dubins_airplane_6d (psi)
template <> struct Model<3> { static constexpr int N = 12, M = 4, NA = 3, A0 = 6; };  // quadcopter_12d (phi,theta,psi)

// DynamicsModel::derivative (model.hpp:42).
template <int MODEL>
KP_DEV void derivative(const KpProblem& P, const float* x, const float* u, float* f) {
    if constexpr (MODEL == 0) {
        f[0] = x[2]; f[1] = x[3]; f[2] = u[0]; f[3] = u[1];
    } else if constexpr (MODEL == 1) {
        f[0] = x[3]; f[1] = x[4]; f[2] = x[5]; f[3] = u[0]; f[4] = u[1]; f[5] = u[2];
    } else if constexpr (MODEL == 2) {
        // (rk4_step evaluates this slope through dubins_slope, with the stage
        // trigonometry rotated from the step's start: DESIGN.md §4)
        float sp, cp, sg, cg;
        sincos_recipe(x[3], sp, cp);
        sincos_recipe<true>(x[4], sg, cg);
        const float vc = x[5] * cg;
        f[0] = vc * cp; f[1] = vc * sp; f[2] = x[5] * sg;
        f[3] = u[0]; f[4] = u[1]; f[5] = u[2];
    } else {
        float sph, cph, sth, cth, sps, cps;
        sincos2_small(x[6], x[7], sph, cph, sth, cth);
        sincos_recipe(x[8], sps, cps);
        const float a = u[0] * P.inv_m;
        const float t1 = cph * sth;
        f[0] = x[3]; f[1] = x[4]; f[2] = x[5];
        f[3] = a * fmaf(t1, cps, sph * sps);
        f[4] = a * fmaf(t1, sps, -(sph * cps));
        f[5] = fmaf(a, cph * cth, -P.grav);
        const float w = fmaf(x[10], sph, x[11] * cph);
        const float ic = 1.0f / cth;  // one IEEE division per evaluation (recipe)
        f[6] = fmaf(w, sth * ic, x[9]);
        f[7] = fmaf(x[10], cph, -(x[11] * sph));
        f[8] = w * ic;
        f[9] = fmaf(P.cx, x[10] * x[11], u[1] * P.inv_ix);
        f[10] = fmaf(P.cy, x[9] * x[11], u[2] * P.inv_iy);
        f[11] = fmaf(P.cz, x[9] * x[10], u[3] * P.inv_iz);
    }
}

// Per-segment factors of an RK4 step of length hk.  Dubins
// airplane: the heading and flight-path rates are the controls u0, u1,
// constant over a segment, so a step's stage angles are a, a + hk/2 u, a +
// hk/2 u (stages 2 and 3 alike) and a + hk u; their sines and cosines are
// those of a rotated by {sin, cos}(hk/2 u) and {sin, cos}(hk u), computed
// once per segment: ctx = {s, c of hk/2 u0, s, c of hk u0, the same for u1}.
template <int MODEL>
KP_DEV void step_ctx(const float* u, float hk, float* ctx) {
    if constexpr (MODEL == 2) {
        const float half = 0.5f * hk;
        sincos_recipe<true>(half * u[0], ctx[0], ctx[1]);
        sincos_recipe<true>(hk * u[0], ctx[2], ctx[3]);
        sincos_recipe<true>(half * u[1], ctx[4], ctx[5]);
        sincos_recipe<true>(hk * u[1], ctx[6], ctx[7]);
    } else {
        (void)u; (void)hk; (void)ctx;
    }
}

// (s, c) rotated by the angle whose sine / cosine are (rs, rc).
KP_DEV void rotate_sc(float s, float c, float rs, float rc, float& so, float& co) {
    so = fmaf(s, rc, c * rs);
    co = fmaf(c, rc, -(s * rs));
}

// Dubins airplane slope from its stage trigonometry (derivative<2> layout).
KP_DEV void dubins_slope(float sp, float cp, float sg, float cg, float v, const float* u, float* f) {
    const float vc = v * cg;
    f[0] = vc * cp; f[1] = vc * sp; f[2] = v * sg;
    f[3] = u[0]; f[4] = u[1]; f[5] = u[2];
}

// One classical RK4 step with constant control, then angle wrap.
// `sixth` must equal hk / 6.0f (IEEE division; hoisted by the caller for the
// full-length steps), ctx = step_ctx(u, hk).  Returns false when a coordinate
// is non-finite (propagation diverged).
template <int MODEL>
KP_DEV bool rk4_step(const KpProblem& P, float* x, const float* u, float hk, float sixth, const float* ctx) {
    constexpr int N = Model<MODEL>::N;
    // the stage slopes are accumulated as they are produced, acc = k1 + 2 k2 +
    // 2 k3 + k4 in that order: only acc and the current stage stay live (the
    // quadcopter's 12-dim step otherwise holds k1 and k2 across later stages)
    float k[N], acc[N], t[N];
    const float half = 0.5f * hk;
    if constexpr (MODEL == 2) {
        // stage trigonometry by rotation (step_ctx); the stage speeds are
        // x5 + hk/2 u2 (stages 2, 3) and x5 + hk u2, and positions do not enter
        // the slope, so stage 3 equals stage 2
        (void)t;
        float sp, cp, sg, cg;
        sincos_recipe(x[3], sp, cp);
        sincos_recipe<true>(x[4], sg, cg);
        dubins_slope(sp, cp, sg, cg, x[5], u, acc);
        float sp1, cp1, sg1, cg1;
        rotate_sc(sp, cp, ctx[0], ctx[1], sp1, cp1);
        rotate_sc(sg, cg, ctx[4], ctx[5], sg1, cg1);
        dubins_slope(sp1, cp1, sg1, cg1, fmaf(half, u[2], x[5]), u, k);
#pragma unroll
        for (int i = 0; i < N; ++i) acc[i] = fmaf(2.0f, k[i], fmaf(2.0f, k[i], acc[i]));  // + 2 k2 + 2 k3
        float sp2, cp2, sg2, cg2;
        rotate_sc(sp, cp, ctx[2], ctx[3], sp2, cp2);
        rotate_sc(sg, cg, ctx[6], ctx[7], sg2, cg2);
        dubins_slope(sp2, cp2, sg2, cg2, fmaf(hk, u[2], x[5]), u, k);
    } else {
    (void)ctx;
    derivative<MODEL>(P, x, u, acc);
#pragma unroll
    for (int i = 0; i < N; ++i) t[i] = fmaf(half, acc[i], x[i]);
    derivative<MODEL>(P, t, u, k);
#pragma unroll
    for (int i = 0; i < N; ++i) {
        t[i] = fmaf(half, k[i], x[i]);
        acc[i] = fmaf(2.0f, k[i], acc[i]);
    }
    derivative<MODEL>(P, t, u, k);
#pragma unroll
    for (int i = 0; i < N; ++i) {
        t[i] = fmaf(hk, k[i], x[i]);
        acc[i] = fmaf(2.0f, k[i], acc[i]);
    }
    derivative<MODEL>(P, t, u, k);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = fmaf(sixth, acc[i] + k[i], x[i]);
    if constexpr (Model<MODEL>::NA > 0) {
        // one test for every angle: wrap_angle only changes |a| >= pi (and
        // leaves pi itself and NaN unchanged), so wrapping all of them when
        // any is out of range gives the same bits as testing each
        float m = fabsf(x[Model<MODEL>::A0]);
#pragma unroll
        for (int i = 1; i < Model<MODEL>::NA; ++i) m = fmaxf(m, fabsf(x[Model<MODEL>::A0 + i]));
        if (m >= 3.14159265358979323846f) {
#pragma unroll
            for (int i = 0; i < Model<MODEL>::NA; ++i) x[Model<MODEL>::A0 + i] = wrap_angle(x[Model<MODEL>::A0 + i]);
        }
    }
    if (!P.check_finite) return true;  // finite bounds reject inf / NaN in within_bounds anyway
    bool ok = true;
#pragma unroll
    for (int i = 0; i < N; ++i) ok = ok && isfinite(x[i]);
    return ok;
}

template <int MODEL>
KP_DEV bool rk4_step(const KpProblem& P, float* x, const float* u, float hk) {
    float ctx[8];
    step_ctx<MODEL>(u, hk, ctx);
    return rk4_step<MODEL>(P, x, u, hk, hk / 6.0f, ctx);
}

// Double integrator in closed form: RK4 with constant control is exact on it
// (SPEC.md:138-139), so the sample at time t is evaluated directly,
// p(t) = p0 + v0 t + (u/2) t^2, v(t) = v0 + u t, with the fused recipe below
// (DESIGN.md §4).  Every sample depends only on the parent state, not on the
// previous sample: no rounding accumulates along the segment and the samples of
// one rollout can be evaluated in any order or in parallel.
template <int MODEL>
KP_DEV void di_sample(const float* x0, const float* u, float t, float* x) {
    constexpr int D = Model<MODEL>::N / 2;  // position dims, then the matching velocities
    const float tt = t * t;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        x[i] = fmaf(0.5f * u[i], tt, fmaf(x0[D + i], t, x0[i]));
        x[D + i] = fmaf(u[i], t, x0[D + i]);
    }
}

template <int MODEL>
__host__ __device__ constexpr bool closed_form() { return MODEL == 0 || MODEL == 1; }

// Path length of a closed-form rollout (DECISION): every segment
// length is rounded to a multiple of 2^-40 and the multiples are summed as a
// 64-bit integer, so the sum is exact and independent of the order in which
// segments are added (the sample-parallel path adds them from several threads);
// one rounding back to fp32 at the end.  d * 2^40 is exact in fp32.
KP_DEV long long len_fixed(float d) { return __float2ll_rn(d * 0x1p40f); }
KP_DEV float fixed_len(long long s) { return __ll2float_rn(s) * 0x1p-40f; }

// Frontier position of V_U slot i (slot = position * lambda + branch): a
// shift when lambda is a power of two (every bundled scene), else a division.
KP_DEV uint32_t frontier_pos(const KpProblem& P, uint32_t i) {
    return P.lam_shift >= 0 ? (i >> P.lam_shift) : i / static_cast<uint32_t>(P.lambda);
}

// Number of RK4 steps of a segment: samples at 0, h, ..., dt.
KP_DEV int step_count(const KpProblem& P, float dt) {
    const int S = static_cast<int>(ceilf(dt / P.h));
    return S < 1 ? 1 : S;
}

// --------------------------------------------------------- environment ----
// The environment blob (kp_types.h) lives in dynamic shared memory.  It is
// addressed through this extern __shared__ array (never through generic
// pointers), so every access compiles to a plain LDS with no per-access
// shared-window conversion.
extern __shared__ float4 kp_env_smem[];

struct Env {  // 32-bit shared-window base of kp_env_smem + byte offsets inside it
    uint32_t base, off_bhi, off_sph, off_cells, off_cids;
};

KP_DEV uint32_t env_saddr();

KP_DEV Env env_view(const KpProblem& P) {
    Env e;
    // once per kernel: the shared-window address of the blob involves a special
    // register read (S2R SR_CgaCtaId); the volatile copy keeps the compiler
    // from rematerialising that sequence at every use inside the step loop
    const uint32_t a = env_saddr();
    asm volatile("mov.b32 %0, %1;" : "=r"(e.base) : "r"(a));
    e.off_bhi = 16u * static_cast<uint32_t>(P.n_box);
    e.off_sph = 32u * static_cast<uint32_t>(P.n_box);
    e.off_cells = P.off_cells;
    e.off_cids = P.off_cids;
    return e;
}

// 32-bit shared-window address of the blob and typed ld.shared helpers
// (non-volatile: the compiler may still schedule / batch them).
KP_DEV uint32_t env_saddr() { return static_cast<uint32_t>(__cvta_generic_to_shared(kp_env_smem)); }
KP_DEV uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
KP_DEV uint32_t lds_u16(uint32_t a) {
    unsigned short v;
    asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
KP_DEV float4 lds_f4(uint32_t a) {
    float4 v;
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}

// Broad-phase cell of v along d: floor(v * inv + off) clamped to [0, n-1].
// Branch-free: an undivided dim has inv = off = 0 (cell 0; NaN converts to 0).
// The binning need not be exact: the host lists every obstacle in all cells
// its AABB touches with a margin of 1e-3 cell, far above this rounding.
KP_DEV int bg_cell(const KpProblem& P, float v, int d) {
    const int c = __float2int_rd(fmaf(v, P.bg_inv[d], P.bg_off[d]));
    return min(max(c, 0), P.bg_max[d]);
}

// Position inside some closed obstacle?  Broad phase: the
// point's cell list; narrow phase: the exact closed box / sphere test, boxes
// read as two float4 (no short-circuit chains of dependent loads).  nbox /
// nsph accumulate the narrow-phase tests executed (roofline accounting).
KP_DEV bool in_obstacle(const KpProblem& P, const Env& E, float px, float py, float pz, uint32_t& nbox,
                        uint32_t& nsph) {
    const int c = bg_cell(P, px, 0) + P.bg_n[0] * (bg_cell(P, py, 1) + P.bg_n[1] * bg_cell(P, pz, 2));
    const uint32_t base = E.base;
    KP_ASSERT(c >= 0 && c < P.n_cells, 1);
    const uint32_t range = lds_u32(base + E.off_cells + 4u * static_cast<uint32_t>(c));
    const int b = static_cast<int>(range & 0xFFFFu), e = static_cast<int>(range >> 16);
    KP_ASSERT(b <= e && e <= P.n_entries, 2);
    for (int k = b; k < e; ++k) {
        const int id = static_cast<int>(lds_u16(base + E.off_cids + 2u * static_cast<uint32_t>(k)));
        KP_ASSERT(id < P.n_box + P.n_sph, 3);
        if (id < P.n_box) {
            const float4 lo = lds_f4(base + 16u * static_cast<uint32_t>(id));
            const float4 hi = lds_f4(base + E.off_bhi + 16u * static_cast<uint32_t>(id));
            ++nbox;
            const bool in = (px >= lo.x) & (px <= hi.x) & (py >= lo.y) & (py <= hi.y) & (pz >= lo.z) & (pz <= hi.z);
            if (in) return true;
        } else {
            const float4 o = lds_f4(base + E.off_sph + 16u * static_cast<uint32_t>(id - P.n_box));
            ++nsph;
            const float dx = px - o.x, dy = py - o.y, dz = pz - o.z;
            float d2 = dx * dx;
            d2 = fmaf(dy, dy, d2);
            d2 = fmaf(dz, dz, d2);
            if (d2 <= o.w) return true;
        }
    }
    return false;
}

// is_state_valid minus the obstacle part, which the caller
// does on the (px, py, pz) projection.  vel = false skips the velocity dims of
// a closed-form model (checked once per item instead, vel_ok_at_end).
template <int MODEL>
KP_DEV bool within_bounds(const KpProblem& P, const float* x, bool vel = true) {
    constexpr int N = Model<MODEL>::N;
    constexpr int D = closed_form<MODEL>() ? N / 2 : N;  // dims checked at every sample when !vel
    // state bounds with the workspace bounds folded into the
    // position dims on the host: x >= max(lo_s, lo_w) <=> x >= lo_s && x >= lo_w.
    // Three independent compare chains (the predicate-accumulating FSETP form
    // is serial) combined at the end: shorter dependent path per RK4 step.
    bool ok0 = true, ok1 = true, ok2 = true;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        if (i >= D && !vel) break;
        const bool in = (x[i] >= P.blo[i]) & (x[i] <= P.bhi[i]);
        if (i % 3 == 0) ok0 = ok0 & in;
        else if (i % 3 == 1) ok1 = ok1 & in;
        else ok2 = ok2 & in;
    }
    return ok0 & ok1 & ok2;
}

// x[d] for a runtime d without spilling x to local memory (fully unrolled select).
template <int N>
KP_DEV float pick(const float* x, int d) {
    float v = x[0];
#pragma unroll
    for (int k = 1; k < N; ++k) v = (d == k) ? x[k] : v;
    return v;
}

// region_index.  IDENT: the decomposed dims are 0, 1, ...
// (every bundled scene): the coordinates are read directly instead of through
// the runtime-dimension select chain.
template <int N, bool IDENT>
KP_DEV uint32_t region_index_dims(const KpProblem& P, const float* x) {
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < KP_MAX_GRID; ++j) {
        if (j >= P.grid_n || (IDENT && j >= N)) break;
        const float xv = IDENT ? x[j < N ? j : 0] : pick<N>(x, P.grid_dims[j]);
        const float v = (xv - P.g_lo[j]) / P.g_side[j];
        const float fv = floorf(v);
        uint32_t i;
        if (fv < 0.0f) i = 0;
        else if (fv > static_cast<float>(P.g_cells[j] - 1)) i = static_cast<uint32_t>(P.g_cells[j] - 1);
        else i = static_cast<uint32_t>(fv);
        r += i * P.g_stride[j];
    }
    return r;
}

template <int N>
KP_DEV uint32_t region_index(const KpProblem& P, const float* x) {
    return P.grid_ident ? region_index_dims<N, true>(P, x) : region_index_dims<N, false>(P, x);
}

// in_goal (cost.hpp:77-84), boundary inclusive.  IDENT as region_index.
template <int N, bool IDENT>
KP_DEV bool in_goal_dims(const KpProblem& P, const float* x) {
    float d = (IDENT ? x[0] : pick<N>(x, P.goal_dims[0])) - P.goal_c[0];
    float d2 = d * d;
#pragma unroll
    for (int i = 1; i < N; ++i) {
        if (i >= P.goal_n) break;
        d = (IDENT ? x[i] : pick<N>(x, P.goal_dims[i])) - P.goal_c[i];
        d2 = fmaf(d, d, d2);
    }
    return d2 <= P.goal_r2;
}

template <int N>
KP_DEV bool in_goal(const KpProblem& P, const float* x) {
    return P.goal_ident ? in_goal_dims<N, true>(P, x) : in_goal_dims<N, false>(P, x);
}

// --------------------------------------------------------- work item ------
struct ItemOut {
    float acc;
    uint32_t region;
    uint32_t steps;    // RK4 steps executed
    uint32_t interp;   // interpolated points checked
    uint32_t nbox, nsph;  // primitive tests executed
    bool goal;
};

// Rollout + validity + cost of one work item whose (u, dt) are drawn (Alg. 2
// lines 4-7): RK4 rollout streamed in registers, every
// sample validated and every interpolated point (spacing <= collision_step)
// obstacle-checked, path length accumulated.  integrate_steps runs steps
// [s0, s1) of an item with S steps: x holds the state after step s0 on entry
// (the parent state for s0 = 0) and after the last step run on return, total
// the path length so far.  Returns 0 (no violation up to s1), 1 invalid,
// 2 diverged.  The parent (samples[0]) is not re-checked: it is a stored valid
// node.  Splitting [0, S) at any step is bit-identical to one call.
// Interpolated points between consecutive samples p and p + (dx, dy, dz),
// d = ||(dx, dy, dz)|| > collision_step: dyadic subdivision,
// k = the smallest power of two with d / k <= collision_step (nested points,
// SPEC.md:231).  d / k and j / k are exact, so multiplying by the exact
// power-of-two reciprocal equals the division bit-for-bit.  True when a point
// is inside an obstacle.
template <bool TWO_D>
KP_DEV bool segment_hit(const KpProblem& P, const Env& E, float px, float py, float pz, float dx, float dy, float dz,
                        float d, uint32_t& interp, uint32_t& nbox, uint32_t& nsph) {
    int k = 2;
    float rk = 0.5f;
    while (d * rk > P.coll && k < (1 << 24)) {
        k <<= 1;
        rk *= 0.5f;
    }
    for (int j = 1; j < k; ++j) {
        const float t = static_cast<float>(j) * rk;
        interp += 1;
        if (in_obstacle(P, E, fmaf(t, dx, px), fmaf(t, dy, py), TWO_D ? 0.0f : fmaf(t, dz, pz), nbox, nsph))
            return true;
    }
    return false;
}

// Sample s + 1 of a rollout with S steps: the closed form
// from the parent state x0 for the double integrator, otherwise one RK4 step
// of x (h6 = h / 6).  Returns 0, 1 when the shortened last step is empty
// (dt - (S-1) h <= 0: the rollout ends at sample S - 1), 2 when diverged.
template <int MODEL>
KP_DEV int advance(const KpProblem& P, const float* x0, float* x, const float* u, float dt, int S, int s, float h6,
                   const float* ctx) {
    if constexpr (closed_form<MODEL>()) {
        float t = static_cast<float>(s + 1) * P.h;
        if (s + 1 == S) {
            const float hk = dt - static_cast<float>(S - 1) * P.h;
            if (!(hk > 0.0f)) return 1;
            t = dt;
        }
        di_sample<MODEL>(x0, u, t, x);
        if (P.check_finite) {
            bool ok = true;
#pragma unroll
            for (int i = 0; i < Model<MODEL>::N; ++i) ok = ok && isfinite(x[i]);
            if (!ok) return 2;
        }
        return 0;
    } else {
        float hk = P.h, sixth = h6;
        if (s + 1 == S) {  // the shortened last step: only here the IEEE division
            hk = dt - static_cast<float>(S - 1) * P.h;
            if (!(hk > 0.0f)) return 1;
            // IEEE div.rn (== hk / 6.0f); volatile so it is not if-converted into every step
            asm volatile("div.rn.f32 %0, %1, %2;" : "=f"(sixth) : "f"(hk), "f"(6.0f));
        }
        if constexpr (MODEL == 2) {
            // the step factors of the shortened last step are its own; a separate
            // inlined step for it measured faster here (7.8 vs 7.2 G items/s)
            if (s + 1 == S) {
                float ctx_last[8];
                step_ctx<MODEL>(u, hk, ctx_last);
                return rk4_step<MODEL>(P, x, u, hk, sixth, ctx_last) ? 0 : 2;
            }
        }
        // one call site otherwise (two inlined RK4 steps: Quad12 -8 %)
        return rk4_step<MODEL>(P, x, u, hk, sixth, ctx) ? 0 : 2;
    }
}

// Closed-form models, velocity bounds once per item: v(t) = fma(u, t, v0) is
// monotone in t (fma is correctly rounded, hence monotone) and the sample
// times 0 < h < 2h < ... < t_last increase (t_last = dt when the last step is
// non-empty, dt > fl((S-1) h)), so with a valid parent (samples[0] is a stored
// node) every sample's velocity lies inside its interval bounds iff the last
// sample's does.  The per-sample checks then cover the position dims only;
// the verdict is the same as checking every sample.  Only
// for finite bounds (P.check_finite == 0), where no sample can diverge.
template <int MODEL>
KP_DEV bool vel_ok_at_end(const KpProblem& P, const float* x0, const float* u, float dt, int S, int seff) {
    constexpr int D = Model<MODEL>::N / 2;
    const float t = (seff == S) ? dt : static_cast<float>(seff) * P.h;
    bool ok = true;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        const float v = fmaf(u[i], t, x0[D + i]);
        ok = ok & (v >= P.blo[D + i]) & (v <= P.bhi[D + i]);
    }
    return ok;
}

// Samples of a rollout with S steps: S, or S - 1 when the shortened last step
// is empty (dt - (S-1) h <= 0).
KP_DEV int effective_samples(const KpProblem& P, float dt, int S) {
    return (S > 1 && !(dt - static_cast<float>(S - 1) * P.h > 0.0f)) ? S - 1 : S;
}

template <int MODEL>
KP_DEV int integrate_steps(const KpProblem& P, const Env& E, float* x, const float* u, float dt, int S, int s0, int s1,
                           float& total, ItemOut& o) {
    constexpr bool TWO_D = (MODEL == 0);
    constexpr int N = Model<MODEL>::N;
    float px = x[0], py = x[1], pz = TWO_D ? 0.0f : x[2];
    const float h6 = P.h / 6.0f;
    float x0[N];  // the parent state (closed form: every sample from it; s0 must be 0)
#pragma unroll
    for (int i = 0; i < N; ++i) x0[i] = x[i];
    long long fx = 0;  // closed form: fixed-point path length
    float ctx[8];      // per-segment step factors (step_ctx)
    step_ctx<MODEL>(u, P.h, ctx);
    bool vel = true;   // check the velocity dims at every sample
    if constexpr (closed_form<MODEL>()) {
        if (!P.check_finite) {
            if (!vel_ok_at_end<MODEL>(P, x0, u, dt, S, effective_samples(P, dt, S))) return 1;
            vel = false;
        }
    }
    for (int s = s0; s < s1; ++s) {
        const int st = advance<MODEL>(P, x0, x, u, dt, S, s, h6, ctx);
        if (st == 1) break;
        if (st == 2) return 2;
        o.steps += 1;
        const float nx = x[0], ny = x[1], nz = TWO_D ? 0.0f : x[2];
        // bounds and obstacle test without a branch in between (one exit per step;
        // the broad-phase cell index is clamped, so out-of-bounds states are safe)
        const bool inb = within_bounds<MODEL>(P, x, vel);
        const bool hit = in_obstacle(P, E, nx, ny, nz, o.nbox, o.nsph);
        if (!inb || hit) return 1;
        const float dx = nx - px, dy = ny - py, dz = nz - pz;
        float d2 = dx * dx;
        d2 = fmaf(dy, dy, d2);
        if (!TWO_D) d2 = fmaf(dz, dz, d2);
        const float d = sqrtf(d2);
        if (d2 > P.coll_d2 && segment_hit<TWO_D>(P, E, px, py, pz, dx, dy, dz, d, o.interp, o.nbox, o.nsph))
            return 1;
        // cost.hpp:59-61 (position head == workspace dims for every built-in model)
        if constexpr (closed_form<MODEL>()) fx += len_fixed(d);
        else total += d;
        px = nx; py = ny; pz = nz;
    }
    if constexpr (closed_form<MODEL>()) total = fixed_len(fx);
    return 0;
}

// Cost, region and goal flag of a valid end state x (Alg. 2 line 7).
template <int MODEL>
KP_DEV void finish_item(const KpProblem& P, const float* x, float dt, float total, float acc_parent, ItemOut& o) {
    float seg;
    if (P.cost_kind == 1) seg = dt;                        // control_duration
    else seg = (total == 0.0f) ? P.zero_rate * dt : total;  // cost.hpp:62
    o.acc = acc_parent + seg;
    o.region = region_index<Model<MODEL>::N>(P, x);
    o.goal = in_goal<Model<MODEL>::N>(P, x);
}

// A whole rollout: 0 valid (o.acc / o.region / o.goal set), 1 invalid, 2 diverged.
template <int MODEL>
KP_DEV int integrate_item(const KpProblem& P, const Env& E, float* x, const float* u, float dt, int S, float acc_parent,
                          ItemOut& o) {
    o.steps = 0;
    o.interp = 0;
    o.nbox = 0;
    o.nsph = 0;
    float total = 0.0f;
    const int rc = integrate_steps<MODEL>(P, E, x, u, dt, S, 0, S, total, o);
    if (rc == 0) finish_item<MODEL>(P, x, dt, total, acc_parent, o);
    return rc;
}

// One whole work item of Alg. 2 lines 3-7: sample (u, dt), then integrate.
template <int MODEL>
KP_DEV int propagate_item(const KpProblem& P, const Env& E, float* x, float acc_parent, uint64_t seed, uint32_t it,
                          uint32_t node, uint32_t br, float* u, float& dt, ItemOut& o) {
    sample_item<Model<MODEL>::M>(P, seed, it, node, br, u, dt);
    return integrate_item<MODEL>(P, E, x, u, dt, step_count(P, dt), acc_parent, o);
}

}  // namespace kp
