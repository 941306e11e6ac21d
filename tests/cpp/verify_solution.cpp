// Plans each bundled scene on the GPU through the C++ drop-in API, then checks
// the returned trajectory with the host fp64 building blocks: every segment
// re-propagated in double precision (propagate_ode) lands on the stored fp32
// child state, the fp64 samples pass is_segment_valid, and the fp64 path
// length matches the planner's cost.  Prints one line per scene:
//   name segments max_state_err cost_rel_err valid
#include <kinoplan_b200/bench.hpp>

#include <algorithm>
#include <cmath>
#include <cstdio>

using namespace kinoplan;

int main(int argc, char** argv) {
    int bad = 0;
    for (int a = 1; a < argc; ++a) {
        Scenario s = load_scenario(argv[a]);
        s.config.t_max = 0.05;
        s.config.stop_at_first_solution = false;
        const PlanResult r = plan(s.problem, s.config);
        if (!r.trajectory) {
            std::printf("%s no-solution\n", s.name.c_str());
            ++bad;
            continue;
        }
        const Trajectory& t = *r.trajectory;
        const DynamicsModel& m = *s.problem.model;
        Environment env = s.problem.environment;
        env.state_bounds = s.problem.state_bounds;
        const double h = s.config.ode_step.value_or(std::min(s.config.t_prop / 10.0, 0.02));
        double max_err = 0, cost = 0;
        bool valid = true;
        for (size_t k = 1; k < t.states.size(); ++k) {
            const auto samples = propagate_ode(t.states[k - 1], t.controls[k], t.durations[k], h, m);
            for (int i = 0; i < m.state_dim(); ++i)
                max_err = std::max(max_err, std::fabs(samples.back()[i] - t.states[k][i]) /
                                                std::max(1.0, std::fabs(t.states[k][i])));
            valid = valid && is_segment_valid(samples, env, m, s.config.collision_step);
            cost += segment_cost(samples, t.controls[k], t.durations[k], s.problem.cost);
        }
        const double rel = std::fabs(cost - r.best.cost) / r.best.cost;
        std::printf("%s %zu %.3g %.3g %d\n", s.name.c_str(), t.states.size() - 1, max_err, rel, valid ? 1 : 0);
        if (!(max_err < 1e-4) || !(rel < 1e-4) || !valid) ++bad;
    }
    return bad ? 1 : 0;
}
