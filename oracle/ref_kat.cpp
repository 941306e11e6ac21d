// oracle/ref_kat.cpp — runs the REFERENCE's own shipped headers
// (/root/reference/proj/include/kinoplan/core/{rng,cost,types}.hpp, compiled
// in place against oracle/ref_shim/Eigen/Core) and prints known-answer vectors
// as JSON.  Built by oracle/Makefile into oracle/_ref/ref_kat (git-ignored).
// tests/golden/make_golden.py turns its output into tests/golden/reference_kat.json.
// TEST INFRASTRUCTURE ONLY.
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <numbers>
#include <vector>

#include "kinoplan/core/cost.hpp"
#include "kinoplan/core/rng.hpp"
#include "kinoplan/core/types.hpp"

using namespace kinoplan;

static State vec(std::initializer_list<double> v) {
    State s(static_cast<int>(v.size()));
    int i = 0;
    for (double x : v) s[i++] = x;
    return s;
}

int main() {
    std::printf("{\n");
    // SplitMix64 raw outputs and uniform_unit draws for a few seeds.
    std::printf("\"splitmix\": [");
    const uint64_t seeds[] = {0ull, 1ull, 7ull, 2602ull, 0xDEADBEEFCAFEBABEull};
    for (size_t s = 0; s < 5; ++s) {
        SplitMix64 a(seeds[s]), b(seeds[s]);
        std::printf("%s{\"seed\": \"%" PRIu64 "\", \"raw\": [", s ? ", " : "", seeds[s]);
        for (int i = 0; i < 8; ++i) std::printf("%s\"%" PRIu64 "\"", i ? ", " : "", a());
        std::printf("], \"unit\": [");
        for (int i = 0; i < 8; ++i) std::printf("%s%.17g", i ? ", " : "", uniform_unit(b));
        std::printf("]}");
    }
    std::printf("],\n");
    std::printf("\"mix64\": [");
    const uint64_t zs[] = {0ull, 1ull, 42ull, 0xFFFFFFFFFFFFFFFFull, 0x9E3779B97F4A7C15ull};
    for (size_t i = 0; i < 5; ++i) std::printf("%s[\"%" PRIu64 "\", \"%" PRIu64 "\"]", i ? ", " : "", zs[i], mix64(zs[i]));
    std::printf("],\n");
    // derive_stream over a grid of (seed, iteration, node, branch).
    std::printf("\"derive_stream\": [");
    bool first = true;
    for (uint64_t seed : {0ull, 7ull, 123456789ull})
        for (uint64_t it : {0ull, 1ull, 3ull, 1000ull})
            for (uint64_t node : {0ull, 42ull, 1048575ull})
                for (uint64_t br : {0ull, 5ull, 31ull}) {
                    const uint64_t s = derive_stream(seed, it, node, br);
                    SplitMix64 r(s);
                    const double u0 = uniform_unit(r), u1 = uniform_unit(r);
                    std::printf("%s[\"%" PRIu64 "\", \"%" PRIu64 "\", \"%" PRIu64 "\", \"%" PRIu64 "\", \"%" PRIu64 "\", %.17g, %.17g]",
                                first ? "" : ", ", seed, it, node, br, s, u0, u1);
                    first = false;
                }
    std::printf("],\n");
    // wrap_angle
    std::printf("\"wrap_angle\": [");
    const double pi = std::numbers::pi;
    const double as[] = {pi, -pi, 3 * pi, 7.0, -7.0, 0.0, 1e-300, 100.0, -100.5, 2 * pi, -2 * pi, pi + 1e-12, -pi - 1e-12};
    for (size_t i = 0; i < sizeof as / sizeof as[0]; ++i) std::printf("%s[%.17g, %.17g]", i ? ", " : "", as[i], wrap_angle(as[i]));
    std::printf("],\n");
    // segment_cost
    std::printf("\"segment_cost\": [");
    {
        CostMetric pl{CostKind::PathLength, 3, {}};
        CostMetric cd{CostKind::ControlDuration, 3, {}};
        std::vector<State> s1 = {vec({0, 0, 0}), vec({3, 4, 0})};
        std::printf("{\"name\": \"pythagorean\", \"value\": %.17g}", segment_cost(s1, State(), 1.0, pl));
        std::vector<State> s2 = {vec({1, 2, 3, 4}), vec({1, 2, 3, 9})};
        std::printf(", {\"name\": \"zero_displacement_dt0.5\", \"value\": %.17g}", segment_cost(s2, State(), 0.5, pl));
        std::printf(", {\"name\": \"control_duration_0.25\", \"value\": %.17g}", segment_cost(s1, State(), 0.25, cd));
        std::vector<State> q;
        for (int i = 0; i < 64; ++i) {
            const double t = (pi / 2) * i / 63.0;
            q.push_back(vec({std::cos(t), std::sin(t), 0}));
        }
        std::printf(", {\"name\": \"quarter_circle_64\", \"value\": %.17g}", segment_cost(q, State(), 1.0, pl));
        // deterministic pseudo-random polylines (SplitMix64 stream) for the oracle
        SplitMix64 r(2602);
        for (int k = 0; k < 20; ++k) {
            const int dim = 3 + (k % 4);
            const int pdim = 2 + (k % 2);
            const int ns = 2 + (k % 7);
            std::vector<State> s;
            std::printf(", {\"name\": \"poly%d\", \"dim\": %d, \"position_dims\": %d, \"samples\": [", k, dim, pdim);
            for (int i = 0; i < ns; ++i) {
                State x(dim);
                for (int j = 0; j < dim; ++j) x[j] = uniform_unit(r) * 10.0 - 5.0;
                s.push_back(x);
                std::printf("%s[", i ? ", " : "");
                for (int j = 0; j < dim; ++j) std::printf("%s%.17g", j ? ", " : "", x[j]);
                std::printf("]");
            }
            CostMetric m{CostKind::PathLength, pdim, {}};
            std::printf("], \"duration\": 0.3, \"value\": %.17g}", segment_cost(s, State(), 0.3, m));
        }
    }
    std::printf("],\n");
    // in_goal
    std::printf("\"in_goal\": [");
    {
        GoalRegion g{{0, 1, 2}, vec({9.5, 9.5, 5.0}), 0.5};
        const State c = vec({9.5, 9.5, 5.0, 0, 0, 0});
        const State on = vec({10.0, 9.5, 5.0, 0, 0, 0});
        const State out = vec({10.0 + 1e-12, 9.5, 5.0, 0, 0, 0});
        const State diag = vec({9.5 + 0.3, 9.5 + 0.4, 5.0, 1, 1, 1});
        std::printf("{\"name\": \"center\", \"value\": %d}", in_goal(c, g));
        std::printf(", {\"name\": \"at_radius\", \"value\": %d}", in_goal(on, g));
        std::printf(", {\"name\": \"radius_plus_eps\", \"value\": %d}", in_goal(out, g));
        std::printf(", {\"name\": \"diag_3_4_5\", \"value\": %d}", in_goal(diag, g));
    }
    std::printf("],\n");
    std::printf("\"cost_kind\": [\"%s\", \"%s\"],\n", std::string(to_string(CostKind::PathLength)).c_str(),
                std::string(to_string(CostKind::ControlDuration)).c_str());
    int threw = 0;
    try { (void)cost_kind_from_string("manhattan"); } catch (const SchemaError&) { threw = 1; }
    std::printf("\"unknown_cost_kind_throws_schema_error\": %d,\n", threw);
    int seg_threw = 0;
    try {
        std::vector<State> one = {vec({0, 0, 0})};
        (void)segment_cost(one, State(), 1.0, CostMetric{});
    } catch (const InvalidSegmentError&) { seg_threw = 1; }
    std::printf("\"one_sample_throws_invalid_segment\": %d\n", seg_threw);
    std::printf("}\n");
    return 0;
}
