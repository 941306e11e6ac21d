// kinoplan.cpp — C++ drop-in API (include/kinoplan_b200/kinoplan.hpp) over the
// C-ABI (include/kinoplan_b200.h).  Host-side only: descriptor marshalling,
// status -> exception mapping (errors.hpp:11-33), result conversion.
#include "kinoplan_b200/kinoplan.hpp"

#include <limits>

#include "kinoplan_b200.h"

namespace kinoplan {

namespace {

[[noreturn]] void raise(int code, const std::string& msg) {
    switch (code) {
        case KP_ERR_SCHEMA: throw SchemaError(msg);
        case KP_ERR_INVALID_PROBLEM: throw InvalidProblemError(msg);
        case KP_ERR_CONFIG: throw ConfigError(msg);
        case KP_ERR_GRID_TOO_FINE: throw GridTooFineError(msg);
        case KP_ERR_INVALID_SEGMENT: throw InvalidSegmentError(msg);
        default: throw DeviceError(msg);
    }
}

void check(int rc, const kp_planner* h) {
    if (rc != KP_OK) raise(rc, kp_last_error(h));
}

}  // namespace

Scalar segment_cost(std::span<const State> samples, const Control&, Scalar duration, const CostMetric& metric) {
    if (samples.size() < 2) throw InvalidSegmentError("segment_cost: segment needs at least 2 samples");
    if (!(duration > 0)) throw InvalidSegmentError("segment_cost: segment duration must be positive");
    if (metric.kind == CostKind::ControlDuration) return duration;
    Scalar total = 0;
    for (size_t i = 1; i < samples.size(); ++i) {
        Scalar s = 0;
        for (int j = 0; j < metric.position_dims; ++j) {
            const Scalar d = samples[i][j] - samples[i - 1][j];
            s += d * d;
        }
        total += std::sqrt(s);
    }
    return total == 0 ? kZeroDisplacementCostRate * duration : total;
}

bool in_goal(const State& x, const GoalRegion& goal) noexcept {
    Scalar d2 = 0;
    for (size_t i = 0; i < goal.dims.size(); ++i) {
        const Scalar dx = x[goal.dims[i]] - goal.center[i];
        d2 += dx * dx;
    }
    return d2 <= goal.radius * goal.radius;
}

void DynamicsModel::derivative(const Vec& x, const Vec& u, Vec& f) const {
    f.assign(state_dim_, 0.0);
    switch (code_) {
        case KP_MODEL_DOUBLE_INTEGRATOR_4D:
            f[0] = x[2]; f[1] = x[3]; f[2] = u[0]; f[3] = u[1];
            break;
        case KP_MODEL_DOUBLE_INTEGRATOR_6D:
            f[0] = x[3]; f[1] = x[4]; f[2] = x[5]; f[3] = u[0]; f[4] = u[1]; f[5] = u[2];
            break;
        case KP_MODEL_DUBINS_AIRPLANE_6D: {
            const Scalar vc = x[5] * std::cos(x[4]);
            f[0] = vc * std::cos(x[3]); f[1] = vc * std::sin(x[3]); f[2] = x[5] * std::sin(x[4]);
            f[3] = u[0]; f[4] = u[1]; f[5] = u[2];
            break;
        }
        default: {
            const Scalar m = params_.get("mass", 1.0), g = params_.get("gravity", 9.81);
            const Scalar ix = params_.get("Ixx", 1.0), iy = params_.get("Iyy", 1.0), iz = params_.get("Izz", 2.0);
            const Scalar sph = std::sin(x[6]), cph = std::cos(x[6]), sth = std::sin(x[7]), cth = std::cos(x[7]);
            const Scalar sps = std::sin(x[8]), cps = std::cos(x[8]);
            const Scalar a = u[0] / m;
            f[0] = x[3]; f[1] = x[4]; f[2] = x[5];
            f[3] = a * (cph * sth * cps + sph * sps);
            f[4] = a * (cph * sth * sps - sph * cps);
            f[5] = a * cph * cth - g;
            const Scalar w = x[10] * sph + x[11] * cph;
            f[6] = x[9] + w * sth / cth;
            f[7] = x[10] * cph - x[11] * sph;
            f[8] = w / cth;
            f[9] = ((iy - iz) * x[10] * x[11] + u[1]) / ix;
            f[10] = ((iz - ix) * x[9] * x[11] + u[2]) / iy;
            f[11] = ((ix - iy) * x[9] * x[10] + u[3]) / iz;
        }
    }
}

std::shared_ptr<const DynamicsModel> make_model(const std::string& id, const ModelParams& params) {
    if (id == "double_integrator_4d")
        return std::make_shared<DynamicsModel>(id, KP_MODEL_DOUBLE_INTEGRATOR_4D, 4, 2, std::vector<int>{0, 1},
                                               std::vector<int>{}, params);
    if (id == "double_integrator_6d")
        return std::make_shared<DynamicsModel>(id, KP_MODEL_DOUBLE_INTEGRATOR_6D, 6, 3, std::vector<int>{0, 1, 2},
                                               std::vector<int>{}, params);
    if (id == "dubins_airplane_6d")
        return std::make_shared<DynamicsModel>(id, KP_MODEL_DUBINS_AIRPLANE_6D, 6, 3, std::vector<int>{0, 1, 2},
                                               std::vector<int>{3}, params);
    if (id == "quadcopter_12d")
        return std::make_shared<DynamicsModel>(id, KP_MODEL_QUADCOPTER_12D, 12, 4, std::vector<int>{0, 1, 2},
                                               std::vector<int>{6, 7, 8}, params);
    throw SchemaError("unknown dynamics model id: \"" + id + "\"");
}

Obstacle Obstacle::box(std::initializer_list<double> lo, std::initializer_list<double> hi) {
    Obstacle o;
    o.type = Type::Box;
    int i = 0;
    for (double v : lo) o.a[i++] = v;
    i = 0;
    for (double v : hi) o.b[i++] = v;
    return o;
}

Obstacle Obstacle::sphere(std::initializer_list<double> c, double r) {
    Obstacle o;
    o.type = Type::Sphere;
    int i = 0;
    for (double v : c) o.a[i++] = v;
    o.b[0] = r;
    return o;
}

Planner::Planner(const PlanningProblem& pr, const PlannerConfig& cf) {
    if (!pr.model) throw SchemaError("problem has no dynamics model");
    const DynamicsModel& md = *pr.model;
    n_ = md.state_dim();
    m_ = md.control_dim();
    if (static_cast<int>(pr.x_init.size()) != n_ || static_cast<int>(pr.state_bounds.size()) != n_ ||
        static_cast<int>(pr.control_bounds.size()) != m_)
        throw SchemaError("x_init / state_bounds / control_bounds size does not match the model");
    std::vector<std::string> pnames;
    std::vector<const char*> pptr;
    std::vector<double> pvals;
    for (const auto& [k, v] : md.params().values) {
        pnames.push_back(k);
        pvals.push_back(v);
    }
    for (const auto& s : pnames) pptr.push_back(s.c_str());
    std::vector<double> slo, shi, clo, chi, wlo, whi;
    for (const auto& b : pr.state_bounds) { slo.push_back(b.lo); shi.push_back(b.hi); }
    for (const auto& b : pr.control_bounds) { clo.push_back(b.lo); chi.push_back(b.hi); }
    for (const auto& b : pr.environment.workspace_bounds) { wlo.push_back(b.lo); whi.push_back(b.hi); }
    std::vector<kp_obstacle> obs;
    for (const auto& o : pr.environment.obstacles) {
        kp_obstacle k{};
        k.type = o.type == Obstacle::Type::Box ? KP_OBSTACLE_BOX : KP_OBSTACLE_SPHERE;
        for (int j = 0; j < 3; ++j) { k.a[j] = o.a[j]; k.b[j] = o.b[j]; }
        obs.push_back(k);
    }
    std::vector<int32_t> gdims(pr.goal.dims.begin(), pr.goal.dims.end());
    const Decomposition& dc = cf.decomposition;
    std::vector<int32_t> ddims(dc.dims.begin(), dc.dims.end()), dcells(dc.cells.begin(), dc.cells.end());
    kp_problem_desc d{};
    d.model = md.model_code();
    d.n_params = static_cast<int32_t>(pptr.size());
    d.param_names = pptr.data();
    d.param_values = pvals.data();
    d.state_dim = n_;
    d.control_dim = m_;
    d.x_init = pr.x_init.data();
    d.state_lo = slo.data();
    d.state_hi = shi.data();
    d.control_lo = clo.data();
    d.control_hi = chi.data();
    d.workspace_dim = static_cast<int32_t>(wlo.size());
    d.n_obstacles = static_cast<int32_t>(obs.size());
    d.workspace_lo = wlo.data();
    d.workspace_hi = whi.data();
    d.obstacles = obs.data();
    d.goal_n_dims = static_cast<int32_t>(gdims.size());
    d.goal_dims = gdims.data();
    d.goal_center = pr.goal.center.data();
    d.goal_radius = pr.goal.radius;
    d.cost_kind = pr.cost.kind == CostKind::PathLength ? KP_COST_PATH_LENGTH : KP_COST_CONTROL_DURATION;
    d.cost_position_dims = pr.cost.position_dims;
    d.grid_n_dims = static_cast<int32_t>(ddims.size());
    d.grid_dims = ddims.data();
    d.grid_cells = dcells.empty() ? nullptr : dcells.data();
    d.grid_delta = dc.delta.value_or(0.0);
    d.grid_max_cells = dc.max_cells;
    kp_config_desc c{};
    c.lambda = cf.lambda;
    c.i_max = cf.i_max;
    c.t_max_s = cf.t_max;
    c.t_prop = cf.t_prop;
    c.ode_step = cf.ode_step.value_or(0.0);
    c.collision_step = cf.collision_step;
    c.capacity = cf.capacity;
    c.seed = cf.seed;
    c.max_iterations = cf.max_iterations;
    c.workers = cf.workers;
    c.deactivate_after_expansion = cf.deactivate_after_expansion;
    c.rng_kind = static_cast<int32_t>(cf.rng);
    c.stop_at_first_solution = cf.stop_at_first_solution;
    c.max_slots = cf.max_slots;
    check(kp_create(&d, &c, cf.device, &h_), nullptr);
}

Planner::~Planner() { kp_destroy(h_); }

void Planner::reset(uint64_t seed) { check(kp_reset(h_, seed), h_); }

Trajectory Planner::extract_trajectory(int64_t leaf) {
    Trajectory t;
    size_t len = 0;
    check(kp_get_path(h_, leaf, nullptr, nullptr, nullptr, nullptr, 0, &len), h_);
    std::vector<double> st(len * n_), ct(len * m_), du(len), ac(len);
    check(kp_get_path(h_, leaf, st.data(), ct.data(), du.data(), ac.data(), len, &len), h_);
    for (size_t i = 0; i < len; ++i) {
        t.states.emplace_back(st.begin() + i * n_, st.begin() + (i + 1) * n_);
        t.controls.emplace_back(ct.begin() + i * m_, ct.begin() + (i + 1) * m_);
        t.durations.push_back(du[i]);
    }
    size_t ns = 0, nseg = 0;
    check(kp_get_trajectory(h_, leaf, nullptr, 0, &ns, nullptr, 0, &nseg), h_);
    std::vector<double> sm(ns * n_), sc(nseg);
    check(kp_get_trajectory(h_, leaf, sm.data(), ns, &ns, sc.data(), nseg, &nseg), h_);
    for (size_t i = 0; i < ns; ++i) t.samples.emplace_back(sm.begin() + i * n_, sm.begin() + (i + 1) * n_);
    t.segment_costs = sc;
    float run = 0.0f;  // fp32 running sum, the planner's own accumulation
    for (double s : sc) run = run + static_cast<float>(s);
    t.cost = run;
    return t;
}

PlanResult Planner::solve(double budget_s, uint64_t max_iterations, bool extract) {
    kp_result r{};
    check(kp_solve(h_, budget_s, max_iterations, &r), h_);
    PlanResult out;
    out.best.cost = r.best_cost;
    if (r.found) out.best.leaf = r.best_leaf;
    out.best.found_at = r.best_found_at_s;
    PlannerStats& s = out.stats;
    s.iterations = r.iterations;
    s.propagations_attempted = r.propagations_attempted;
    s.propagations_valid = r.propagations_valid;
    s.propagations_admitted = r.propagations_admitted;
    s.nodes_pruned_terminal = r.nodes_pruned_terminal;
    s.nodes_deactivated = r.nodes_deactivated;
    s.nodes_reactivated = r.nodes_reactivated;
    s.nodes_committed = r.nodes_committed;
    s.capacity_exhausted = r.capacity_exhausted;
    s.elapsed = r.elapsed_s;
    s.first_solution_iteration = r.first_solution_iteration;
    s.best_found_iteration = r.best_found_iteration;
    s.node_count = r.node_count;
    std::vector<kp_timeline_entry> tl(r.timeline_len);
    size_t len = 0;
    check(kp_get_timeline(h_, tl.data(), tl.size(), &len), h_);
    for (size_t i = 0; i < std::min(len, tl.size()); ++i) s.cost_timeline.emplace_back(tl[i].elapsed_s, tl[i].cost);
    if (r.found) s.first_solution = std::make_pair(r.first_solution_s, r.first_solution_cost);
    if (extract && r.found) out.trajectory = extract_trajectory(r.best_leaf);
    return out;
}

PlanResult plan(const PlanningProblem& problem, const PlannerConfig& config) {
    Planner p(problem, config);
    return p.solve(config.t_max > 0 ? config.t_max : -1, config.max_iterations, true);
}

}  // namespace kinoplan
