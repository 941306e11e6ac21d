// Host (fp64) building blocks of the C++ drop-in API against the SPEC examples
// (SPEC.md:132-160, :200-228, :267-305).  No GPU: these run on the CPU.
// Prints "ok <n checks>" and exits 0, or reports the first failure and exits 1.
#include <kinoplan_b200/kinoplan.hpp>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

using namespace kinoplan;

static int checks = 0;
#define CHECK(c)                                                             \
    do {                                                                     \
        ++checks;                                                            \
        if (!(c)) {                                                          \
            std::fprintf(stderr, "FAILED %s at line %d\n", #c, __LINE__); \
            std::exit(1);                                                    \
        }                                                                    \
    } while (0)

template <class F>
static bool throws_schema(F f, const char* needle) {
    try {
        f();
    } catch (const SchemaError& e) {
        return std::string(e.what()).find(needle) != std::string::npos;
    }
    return false;
}

int main() {
    // ---- propagate_ode ----
    auto di = make_model("double_integrator_6d");
    {
        const State x{0, 0, 0, 1, 0, 0};
        auto s = propagate_ode(x, {0, 0, 0}, 1.0, 0.1, *di);
        CHECK(s.size() == 11 && s[0] == x);  // samples[0] bit-exact
        CHECK(std::fabs(s.back()[0] - 1.0) < 1e-12 && s.back()[3] == 1.0);
    }
    {
        auto s = propagate_ode(State(6, 0.0), {1, 0, 0}, 1.0, 0.1, *di);
        CHECK(std::fabs(s.back()[0] - 0.5) < 1e-12 && std::fabs(s.back()[3] - 1.0) < 1e-12);
    }
    {  // shortened last step lands exactly on dt
        auto s = propagate_ode(State(6, 0.0), {0, 0, 1}, 0.25, 0.1, *di);
        CHECK(s.size() == 4 && std::fabs(s.back()[5] - 0.25) < 1e-12 && std::fabs(s.back()[2] - 0.03125) < 1e-12);
    }
    {  // quadcopter from hover vs a fine explicit Euler oracle
        ModelParams mp;
        auto q = make_model("quadcopter_12d", mp);
        State x(12, 0.0);
        x[2] = 1.0;
        x[6] = 0.05;
        x[10] = 0.1;
        const Control u{9.81, 0.01, -0.02, 0.005};
        auto s = propagate_ode(x, u, 0.5, 0.01, *q);
        State e = x, f;
        const double h = 1e-5;
        for (int k = 0; k < 50000; ++k) {
            q->derivative(e, u, f);
            for (int i = 0; i < 12; ++i) e[i] += h * f[i];
        }
        for (int i = 0; i < 12; ++i) CHECK(std::fabs(s.back()[i] - e[i]) < 1e-4);
    }
    {  // Dubins RK4 order: halving h shrinks the error >= 12x
        auto d = make_model("dubins_airplane_6d");
        const State x{0, 0, 1, 0.3, 0.1, 1.5};
        const Control u{0.8, -0.2, 0.1};
        const auto ref = propagate_ode(x, u, 1.0, 1e-4, *d).back();
        auto err = [&](double h) {
            const auto r = propagate_ode(x, u, 1.0, h, *d).back();
            double m = 0;
            for (int i = 0; i < 6; ++i) m = std::max(m, std::fabs(r[i] - ref[i]));
            return m;
        };
        CHECK(err(0.1) / err(0.05) >= 12.0);
    }
    {  // divergence is an error
        bool thrown = false;
        try {
            (void)propagate_ode(State{0, 0, 0, 1e308, 0, 0}, {1e308, 0, 0}, 1.0, 0.1, *di);
        } catch (const InvalidSegmentError&) {
            thrown = true;
        }
        CHECK(thrown);
    }

    // ---- sampling ----
    {
        SplitMix64 r(derive_stream(7, 1, 2, 3));
        const Control c = sample_control(r, {{2.5, 2.5}, {-1, -1}});
        CHECK(c[0] == 2.5 && c[1] == -1.0);
        SplitMix64 a(11), b(11);
        CHECK(sample_control(a, {{-1, 1}, {-1, 1}, {-1, 1}}) == sample_control(b, {{-1, 1}, {-1, 1}, {-1, 1}}));
        SplitMix64 m(3);
        double su = 0, sd = 0, dmin = 1e9, dmax = 0;
        const int n = 100000;
        for (int i = 0; i < n; ++i) {
            su += sample_control(m, {{0, 1}})[0];
            const double d = sample_duration(m, 2.0);
            sd += d;
            dmin = std::min(dmin, d);
            dmax = std::max(dmax, d);
        }
        CHECK(std::fabs(su / n - 0.5) < 3 * std::sqrt(1.0 / 12 / n) && std::fabs(sd / n - 1.0) < 3 * 2 * std::sqrt(1.0 / 12 / n));
        CHECK(dmin > 0 && dmax <= 2.0);
    }

    // ---- environment ----
    {
        Environment env = load_environment(
            R"({"workspace_bounds": [[-2, 2], [-2, 2], [-2, 2]],
                "state_bounds": [[-2, 2], [-2, 2], [-2, 2], [-1, 1], [-1, 1], [-1, 1]],
                "obstacles": [{"type": "box", "min": [-0.5, -0.5, -0.5], "max": [0.5, 0.5, 0.5]},
                              {"type": "sphere", "center": [1.5, 1.5, 1.5], "radius": 0.25}]})");
        CHECK(env.obstacles.size() == 2 && env.state_bounds.size() == 6);
        CHECK(!is_state_valid({0, 0, 0, 0, 0, 0}, env, *di));           // inside the box
        CHECK(!is_state_valid({0.5, 0.1, 0.1, 0, 0, 0}, env, *di));     // boundary contact
        CHECK(is_state_valid({1, -1, 1, 0, 0, 0}, env, *di));
        CHECK(!is_state_valid({1, -1, 1, 1.0 + 1e-9, 0, 0}, env, *di));  // velocity bound
        CHECK(!is_state_valid({1.5, 1.5, 1.6, 0, 0, 0}, env, *di));      // sphere
        CHECK(!is_state_valid({2.1, 0, 0, 0, 0, 0}, env, *di));          // workspace
        // two samples straddling a thin box: only interpolation catches it
        Environment thin = load_environment(
            R"({"workspace_bounds": [[0, 10], [0, 10], [0, 10]],
                "obstacles": [{"type": "box", "min": [4.98, 0, 0], "max": [5.02, 10, 10]}]})");
        const std::vector<State> seg{{4.9, 5, 5, 0, 0, 0}, {5.1, 5, 5, 0, 0, 0}};
        CHECK(is_state_valid(seg[0], thin, *di) && is_state_valid(seg[1], thin, *di));
        CHECK(!is_segment_valid(seg, thin, *di, 0.03));
        for (double c : {0.02, 0.01, 0.005}) CHECK(!is_segment_valid(seg, thin, *di, c));  // monotone refinement
        CHECK(is_segment_valid(seg, thin, *di, 0.5));  // coarse checking misses it
        Environment none = load_environment(R"({"workspace_bounds": [[0, 1], [0, 1]]})");
        CHECK(none.obstacles.empty());
        CHECK(throws_schema([] { (void)load_environment(R"({"workspace_bounds": [[0, 1], [0, 1]], "obstacles": [{"type": "box", "min": [1, 0], "max": [0, 1]}]})"); },
                            "environment.obstacles[0]"));
        CHECK(throws_schema([] { (void)load_environment(R"({"workspace_bounds": [[0, 1], [0, 1]], "obstacles": [{"type": "sphere", "center": [0, 0], "radius": 0}]})"); },
                            "environment.obstacles[0].radius"));
        CHECK(throws_schema([] { (void)load_environment(R"({"obstacles": []})"); }, "environment.workspace_bounds"));
    }

    // ---- decomposition ----
    {
        RegionGrid g = build_grid({0, 1}, {{0, 1}, {0, 1}}, std::nullopt, {2, 2});
        CHECK(g.n_regions == 4 && g.side[0] == 0.5 && std::fabs(g.delta - 0.5 * std::sqrt(2.0)) < 1e-12);
        CHECK(region_index({0.25, 0.25}, g) == 0 && region_index({0.75, 0.25}, g) == 1 && region_index({1.0, 1.0}, g) == 3);
        RegionGrid g1 = build_grid({0}, {{0, 10}}, 1.0, {});
        CHECK(g1.n_regions == 10 && std::fabs(g1.delta - 1.0) < 1e-12);
        CHECK(std::isinf(region_cost(g, 2)));
        CHECK(try_update_region_cost(g, 2, 5.0) == UpdateOutcome::Improved && region_cost(g, 2) == 5.0);
        CHECK(try_update_region_cost(g, 2, 7.0) == UpdateOutcome::Worse && region_cost(g, 2) == 5.0);
        CHECK(try_update_region_cost(g, 2, 5.0) == UpdateOutcome::Equal);
        CHECK(try_update_region_cost(g, 2, 3.0) == UpdateOutcome::Improved && try_update_region_cost(g, 2, 2.0) == UpdateOutcome::Improved);
        CHECK(region_cost(g, 2) == 2.0);
        bool too_fine = false;
        try {
            (void)build_grid({0, 1, 2}, {{0, 1}, {0, 1}, {0, 1}}, 1e-4, {}, 1000000);
        } catch (const GridTooFineError&) {
            too_fine = true;
        }
        CHECK(too_fine);
        // concurrent updates: the final value is the minimum of all submissions
        RegionGrid s = build_grid({0}, {{0, 1}}, std::nullopt, {1000});
        std::vector<std::thread> th;
        for (int w = 0; w < 8; ++w)
            th.emplace_back([&, w] {
                for (int k = 0; k < 125000; ++k) {
                    const uint64_t r = (static_cast<uint64_t>(k) * 2654435761u + w) % 1000;
                    (void)try_update_region_cost(s, r, 1.0 + static_cast<double>((k * 7919 + w * 104729) % 1000003));
                }
            });
        for (auto& t : th) t.join();
        std::vector<double> mins(1000, INFINITY);
        for (int w = 0; w < 8; ++w)
            for (int k = 0; k < 125000; ++k) {
                const uint64_t r = (static_cast<uint64_t>(k) * 2654435761u + w) % 1000;
                mins[r] = std::min(mins[r], 1.0 + static_cast<double>((k * 7919 + w * 104729) % 1000003));
            }
        bool same = true;
        for (int r = 0; r < 1000; ++r) same = same && region_cost(s, r) == mins[r];
        CHECK(same);
    }
    std::printf("ok %d\n", checks);
    return 0;
}
