// kinoplan_host.cpp — host (fp64) building blocks of the reference API:
// propagate_ode / sample_control / sample_duration,
// is_state_valid / is_segment_valid, build_grid /
// region_index / try_update_region_cost / region_cost.
// They follow the SPEC in double precision for callers that set up, check or
// replay pieces of a plan on the CPU; the planner itself runs on the GPU.
#include <algorithm>
#include <bit>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>

#include "kinoplan_b200/kinoplan.hpp"

namespace kinoplan {

void invariant_failure(const char* expr, const char* file, int line, const std::string& msg) {
    std::fprintf(stderr, "kinoplan invariant violated: %s\n  at %s:%d\n  %s\n", expr, file, line, msg.c_str());
    std::abort();
}

// ---------------------------------------------------------------- dynamics
std::vector<State> propagate_ode(const State& x, const Control& u, Scalar dt, Scalar h, const DynamicsModel& model) {
    const int n = model.state_dim();
    if (static_cast<int>(x.size()) != n || static_cast<int>(u.size()) != model.control_dim())
        throw InvalidSegmentError("propagate_ode: state / control size does not match the model");
    if (!(dt > 0) || !(h > 0)) throw InvalidSegmentError("propagate_ode: dt and h must be positive");
    const int S = std::max(1, static_cast<int>(std::ceil(dt / h)));
    std::vector<State> out;
    out.reserve(static_cast<size_t>(S) + 1);
    out.push_back(x);  // samples[0] == x, bit-exact
    State cur = x, k1, k2, k3, k4, t(n);
    for (int s = 0; s < S; ++s) {
        const Scalar hk = (s + 1 == S) ? dt - static_cast<Scalar>(S - 1) * h : h;  // last step lands on dt
        if (!(hk > 0)) break;
        model.derivative(cur, u, k1);
        for (int i = 0; i < n; ++i) t[i] = cur[i] + 0.5 * hk * k1[i];
        model.derivative(t, u, k2);
        for (int i = 0; i < n; ++i) t[i] = cur[i] + 0.5 * hk * k2[i];
        model.derivative(t, u, k3);
        for (int i = 0; i < n; ++i) t[i] = cur[i] + hk * k3[i];
        model.derivative(t, u, k4);
        for (int i = 0; i < n; ++i) cur[i] += hk / 6.0 * (k1[i] + 2.0 * (k2[i] + k3[i]) + k4[i]);
        for (int a : model.angle_dims()) cur[a] = wrap_angle(cur[a]);  // types.hpp:49-58
        for (int i = 0; i < n; ++i)
            if (!std::isfinite(cur[i])) throw InvalidSegmentError("propagate_ode: propagation diverged (non-finite state)");
        out.push_back(cur);
    }
    return out;
}

Control sample_control(SplitMix64& rng, const Bounds& bounds) {
    Control u(bounds.size());
    for (size_t i = 0; i < bounds.size(); ++i) u[i] = bounds[i].lo + (bounds[i].hi - bounds[i].lo) * uniform_unit(rng);
    return u;
}

Scalar sample_duration(SplitMix64& rng, Scalar t_prop) {
    return t_prop * (1.0 - uniform_unit(rng));  // (0, t_prop]
}

// ------------------------------------------------------------- environment
namespace {

bool point_in_obstacle(const Environment& env, const Scalar* p, int wd) {
    for (const Obstacle& o : env.obstacles) {
        if (o.type == Obstacle::Type::Box) {
            bool in = true;
            for (int d = 0; d < wd; ++d) in = in && p[d] >= o.a[d] && p[d] <= o.b[d];  // closed
            if (in) return true;
        } else {
            Scalar d2 = 0;
            for (int d = 0; d < wd; ++d) d2 += (p[d] - o.a[d]) * (p[d] - o.a[d]);
            if (d2 <= o.b[0] * o.b[0]) return true;
        }
    }
    return false;
}

}  // namespace

bool is_state_valid(const State& x, const Environment& env, const DynamicsModel& model) {
    const int n = model.state_dim();
    for (int i = 0; i < n && i < static_cast<int>(env.state_bounds.size()); ++i)
        if (!env.state_bounds[i].contains(x[i])) return false;
    const int wd = static_cast<int>(env.workspace_bounds.size());
    for (int d = 0; d < wd; ++d)
        if (!env.workspace_bounds[d].contains(x[d])) return false;
    return !point_in_obstacle(env, x.data(), wd);
}

bool is_segment_valid(std::span<const State> samples, const Environment& env, const DynamicsModel& model,
                      Scalar collision_step) {
    const int wd = static_cast<int>(env.workspace_bounds.size());
    for (size_t s = 0; s < samples.size(); ++s) {
        if (!is_state_valid(samples[s], env, model)) return false;
        if (s == 0) continue;
        const State& a = samples[s - 1];
        const State& b = samples[s];
        Scalar d2 = 0;
        for (int d = 0; d < wd; ++d) d2 += (b[d] - a[d]) * (b[d] - a[d]);
        const Scalar dist = std::sqrt(d2);
        if (!(dist > collision_step)) continue;
        // dyadic interior points: k = smallest power of two with
        // dist / k <= collision_step; nested, so finer steps never un-detect
        uint64_t k = 2;
        while (dist / static_cast<Scalar>(k) > collision_step && k < (1ull << 40)) k <<= 1;
        Scalar p[3] = {0, 0, 0};
        for (uint64_t j = 1; j < k; ++j) {
            const Scalar t = static_cast<Scalar>(j) / static_cast<Scalar>(k);
            for (int d = 0; d < wd; ++d) p[d] = std::fma(t, b[d] - a[d], a[d]);
            if (point_in_obstacle(env, p, wd)) return false;
        }
    }
    return true;
}

// ----------------------------------------------------------- decomposition
namespace {

constexpr uint64_t kInfBits = 0x7FF0000000000000ull;  // encoding of +inf: above every finite cost

uint64_t encode(Scalar c) { return std::bit_cast<uint64_t>(c); }  // nonnegative doubles: order-isomorphic
Scalar decode(uint64_t b) { return std::bit_cast<Scalar>(b); }

}  // namespace

RegionGrid build_grid(const std::vector<int>& dims, const Bounds& bounds, std::optional<Scalar> delta,
                      const std::vector<int>& cells, uint64_t max_cells) {
    if (dims.empty() || dims.size() != bounds.size()) throw ConfigError("build_grid: dims / bounds size mismatch");
    for (const Interval& b : bounds)
        if (!(b.lo < b.hi)) throw ConfigError("build_grid: every bound needs lo < hi");
    RegionGrid g;
    g.dims = dims;
    g.bounds = bounds;
    const size_t nd = dims.size();
    if (delta) {
        if (!(*delta > 0)) throw ConfigError("build_grid: delta must be positive");
        const Scalar rn = std::sqrt(static_cast<Scalar>(nd));
        for (const Interval& b : bounds)
            g.cells.push_back(std::max(1, static_cast<int>(std::ceil(b.width() * rn / *delta))));  // as the planner's grid
    } else {
        if (cells.size() != nd) throw ConfigError("build_grid: cells / dims size mismatch");
        for (int c : cells)
            if (c < 1) throw ConfigError("build_grid: cells per dim must be >= 1");
        g.cells = cells;
    }
    const uint64_t ceiling = max_cells ? max_cells : (1ull << 28);
    long double total = 1;
    for (int c : g.cells) total *= c;
    if (total > static_cast<long double>(ceiling))
        throw GridTooFineError("build_grid: " + std::to_string(static_cast<unsigned long long>(total)) +
                               " regions exceed the ceiling of " + std::to_string(ceiling));
    g.n_regions = static_cast<uint64_t>(total);
    Scalar diag2 = 0;
    for (size_t d = 0; d < nd; ++d) {
        g.side.push_back(bounds[d].width() / g.cells[d]);
        diag2 += g.side[d] * g.side[d];
    }
    g.delta = std::sqrt(diag2);
    g.table = std::make_unique<std::atomic<uint64_t>[]>(g.n_regions);
    for (uint64_t i = 0; i < g.n_regions; ++i) g.table[i].store(kInfBits, std::memory_order_relaxed);
    return g;
}

uint64_t region_index(const State& x, const RegionGrid& g) {
    uint64_t idx = 0, stride = 1;
    for (size_t d = 0; d < g.dims.size(); ++d) {
        long long c = static_cast<long long>(std::floor((x[g.dims[d]] - g.bounds[d].lo) / g.side[d]));
        c = std::clamp<long long>(c, 0, g.cells[d] - 1);  // upper boundary -> last cell
        idx += static_cast<uint64_t>(c) * stride;
        stride *= static_cast<uint64_t>(g.cells[d]);
    }
    return idx;
}

UpdateOutcome try_update_region_cost(RegionGrid& g, uint64_t i, Scalar c) {
    KINO_CHECK(i < g.n_regions && std::isfinite(c) && c >= 0, "try_update_region_cost: index in range, finite cost >= 0");
    const uint64_t nb = encode(c == 0 ? 0.0 : c);  // -0 -> +0: one encoding per value
    uint64_t old = g.table[i].load(std::memory_order_relaxed);
    while (nb < old) {
        if (g.table[i].compare_exchange_weak(old, nb, std::memory_order_acq_rel, std::memory_order_relaxed))
            return UpdateOutcome::Improved;
    }
    return nb == old ? UpdateOutcome::Equal : UpdateOutcome::Worse;
}

Scalar region_cost(const RegionGrid& g, uint64_t i) {
    KINO_CHECK(i < g.n_regions, "region_cost: index in range");
    return decode(g.table[i].load(std::memory_order_acquire));
}

}  // namespace kinoplan
