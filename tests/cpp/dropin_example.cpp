// The INTEGRATION.md example: the reference-shaped C++ API (namespace kinoplan)
// linked against libkinoplan_b200.so.  Prints "found cost iterations".
#include <cstdio>

#include <kinoplan_b200/kinoplan.hpp>

int main() {
    kinoplan::PlanningProblem pr;
    pr.model = kinoplan::make_model("double_integrator_6d");
    pr.environment.workspace_bounds = {{0, 10}, {0, 10}, {0, 10}};
    pr.environment.obstacles.push_back(kinoplan::Obstacle::box({4, 4, 0}, {5, 5, 10}));
    pr.x_init = {0.5, 0.5, 5, 0, 0, 0};
    pr.goal = {{0, 1, 2}, {9.5, 9.5, 5}, 0.5};
    pr.state_bounds = {{0, 10}, {0, 10}, {0, 10}, {-2, 2}, {-2, 2}, {-2, 2}};
    pr.control_bounds = {{-2, 2}, {-2, 2}, {-2, 2}};
    kinoplan::PlannerConfig cf;
    cf.decomposition.dims = {0, 1, 2};
    cf.decomposition.cells = {30, 30, 30};
    cf.t_max = 0.05;
    try {
        kinoplan::PlanningProblem bad = pr;
        bad.x_init = {4.5, 4.5, 5, 0, 0, 0};  // inside the box
        (void)kinoplan::plan(bad, cf);
        std::printf("expected InvalidProblemError\n");
        return 2;
    } catch (const kinoplan::InvalidProblemError&) {
    }
    const kinoplan::PlanResult r = kinoplan::plan(pr, cf);
    if (!r.best.leaf || !r.trajectory) return 3;
    const auto& t = *r.trajectory;
    // the re-integrated segment costs sum (fp32) to the leaf's accumulated cost
    std::printf("%d %.9g %llu %.9g %zu\n", 1, r.best.cost, static_cast<unsigned long long>(r.stats.iterations), t.cost,
                t.samples.size());
    return t.cost == r.best.cost ? 0 : 4;
}
