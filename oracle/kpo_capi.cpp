// oracle/kpo_capi.cpp — C entry points of the CPU oracle for the Python test
// harness (ctypes) and bench.py's CPU baseline.  TEST INFRASTRUCTURE ONLY: the
// product never links this library.
//
// The descriptors are the public POD structs of include/kinoplan_b200.h (the
// boundary definition), so the oracle and the device planner are driven from
// byte-identical problem/config values.
#include <cstdio>
#include <memory>
#include <string>

#include "../include/kinoplan_b200.h"
#include "kpo.hpp"

using namespace kpo;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return KP_OK;
    } catch (const SchemaError& e) {
        return fail(KP_ERR_SCHEMA, e.what());
    } catch (const InvalidProblemError& e) {
        return fail(KP_ERR_INVALID_PROBLEM, e.what());
    } catch (const ConfigError& e) {
        return fail(KP_ERR_CONFIG, e.what());
    } catch (const GridTooFineError& e) {
        return fail(KP_ERR_GRID_TOO_FINE, e.what());
    } catch (const InvalidSegmentError& e) {
        return fail(KP_ERR_INVALID_SEGMENT, e.what());
    } catch (const std::exception& e) {
        return fail(KP_ERR_ARGUMENT, e.what());
    }
}

// Descriptor -> ProblemDef/ConfigDef with the SPEC.md invariants
// (model.hpp:64-68).
void convert(const kp_problem_desc* p, const kp_config_desc* c, ProblemDef& pd, ConfigDef& cf) {
    if (!p || !c) throw std::invalid_argument("null descriptor");
    if (p->model < 0 || p->model > 3) throw SchemaError("unknown model id " + std::to_string(p->model));
    pd.model = static_cast<ModelId>(p->model);
    model_shape(pd.model, &pd.n, &pd.m, &pd.position_dims, &pd.angle_dims);
    if (p->state_dim != pd.n || p->control_dim != pd.m)
        throw SchemaError("state/control dimension does not match the model");
    for (int i = 0; i < p->n_params; ++i) {
        const std::string k = p->param_names[i];
        const double v = p->param_values[i];
        if (k == "mass") pd.mass = v;
        else if (k == "gravity") pd.gravity = v;
        else if (k == "arm_length") pd.arm = v;
        else if (k == "Ixx") pd.Ixx = v;
        else if (k == "Iyy") pd.Iyy = v;
        else if (k == "Izz") pd.Izz = v;
        else throw SchemaError("unknown model parameter \"" + k + "\"");
    }
    pd.x_init.assign(p->x_init, p->x_init + pd.n);
    pd.state_bounds.resize(pd.n);
    for (int i = 0; i < pd.n; ++i) {
        pd.state_bounds[i] = {p->state_lo[i], p->state_hi[i]};
        if (!(p->state_lo[i] <= p->state_hi[i])) throw SchemaError("state bound lo > hi");
    }
    pd.control_bounds.resize(pd.m);
    for (int i = 0; i < pd.m; ++i) {
        pd.control_bounds[i] = {p->control_lo[i], p->control_hi[i]};
        if (!(p->control_lo[i] <= p->control_hi[i])) throw SchemaError("control bound lo > hi");
    }
    pd.ws_dim = p->workspace_dim;
    if (pd.ws_dim != static_cast<int>(pd.position_dims.size()))
        throw SchemaError("workspace dimension does not match the model's position dims");
    pd.workspace.resize(pd.ws_dim);
    for (int i = 0; i < pd.ws_dim; ++i) {
        pd.workspace[i] = {p->workspace_lo[i], p->workspace_hi[i]};
        const Interval& sb = pd.state_bounds[pd.position_dims[i]];
        if (!(p->workspace_lo[i] <= p->workspace_hi[i])) throw SchemaError("workspace lo > hi");
        if (p->workspace_lo[i] < sb.lo || p->workspace_hi[i] > sb.hi)
            throw SchemaError("workspace_bounds not contained in state_bounds (SPEC.md:196)");
    }
    for (int i = 0; i < p->n_obstacles; ++i) {
        const kp_obstacle& o = p->obstacles[i];
        Obstacle ob;
        ob.type = o.type;
        for (int j = 0; j < 3; ++j) { ob.a[j] = o.a[j]; ob.b[j] = o.b[j]; }
        if (o.type == KP_OBSTACLE_BOX) {
            for (int j = 0; j < pd.ws_dim; ++j)
                if (!(o.a[j] <= o.b[j])) throw SchemaError("obstacle " + std::to_string(i) + ": box min > max");
        } else if (o.type == KP_OBSTACLE_SPHERE) {
            if (!(o.b[0] > 0)) throw SchemaError("obstacle " + std::to_string(i) + ": sphere radius <= 0");
        } else {
            throw SchemaError("obstacle " + std::to_string(i) + ": unknown type");
        }
        pd.obstacles.push_back(ob);
    }
    if (p->goal_n_dims < 1) throw SchemaError("goal needs at least one dimension");
    pd.goal_dims.assign(p->goal_dims, p->goal_dims + p->goal_n_dims);
    pd.goal_center.assign(p->goal_center, p->goal_center + p->goal_n_dims);
    pd.goal_radius = p->goal_radius;
    if (!(pd.goal_radius > 0)) throw SchemaError("goal radius must be > 0");
    for (int i = 0; i < p->goal_n_dims; ++i) {
        const int d = pd.goal_dims[i];
        if (d < 0 || d >= pd.n) throw SchemaError("goal dimension out of range");
        const Interval& sb = pd.state_bounds[d];
        if (!(pd.goal_center[i] >= sb.lo && pd.goal_center[i] <= sb.hi))
            throw InvalidProblemError("goal center outside state bounds (SPEC.md:62)");
    }
    pd.cost = static_cast<CostKind>(p->cost_kind);
    pd.cost_position_dims = p->cost_position_dims;
    if (p->cost_kind != 0 && p->cost_kind != 1) throw SchemaError("unknown cost metric kind");
    if (pd.cost_position_dims < 1 || pd.cost_position_dims > pd.n) throw SchemaError("bad cost position dims");
    if (p->grid_n_dims < 1 || p->grid_n_dims > KP_MAX_GRID_DIMS) throw SchemaError("bad decomposition dims");
    pd.grid_dims.assign(p->grid_dims, p->grid_dims + p->grid_n_dims);
    for (int d : pd.grid_dims)
        if (d < 0 || d >= pd.n) throw SchemaError("decomposition dimension out of range");
    std::vector<int64_t> cells;
    if (p->grid_cells) cells.assign(p->grid_cells, p->grid_cells + p->grid_n_dims);
    else if (!(p->grid_delta > 0)) throw ConfigError("decomposition needs delta > 0 or cells");
    for (int d : pd.grid_dims)
        if (!(pd.state_bounds[d].lo < pd.state_bounds[d].hi)) throw SchemaError("decomposed dim needs lo < hi");
    build_grid(pd, cells, p->grid_delta, p->grid_max_cells ? p->grid_max_cells : (1ull << 28));

    cf.lambda = c->lambda;
    cf.i_max = c->i_max;
    cf.t_max_s = c->t_max_s;
    cf.t_prop = c->t_prop;
    cf.ode_step = c->ode_step > 0 ? c->ode_step : std::min(c->t_prop / 10.0, 0.02);
    cf.collision_step = c->collision_step;
    cf.capacity = c->capacity;
    cf.seed = c->seed;
    cf.max_iterations = c->max_iterations;
    cf.workers = c->workers < 1 ? 1 : c->workers;
    cf.deactivate_after_expansion = c->deactivate_after_expansion != 0;
    cf.rng_kind = c->rng_kind;
    cf.stop_at_first_solution = c->stop_at_first_solution != 0;
    // SPEC.md:68
    if (cf.lambda < 1) throw ConfigError("lambda must be >= 1");
    if (cf.i_max < 1) throw ConfigError("i_max must be >= 1");
    if (cf.capacity < 1) throw ConfigError("capacity must be >= 1");
    if (!(cf.t_prop > 0)) throw ConfigError("t_prop must be > 0");
    if (!(cf.ode_step > 0) || cf.ode_step > cf.t_prop) throw ConfigError("need 0 < ode_step <= t_prop");
    if (!(cf.collision_step > 0)) throw ConfigError("collision_step must be > 0");
    if (cf.rng_kind != 0 && cf.rng_kind != 1) throw ConfigError("unknown rng kind");
}

struct Handle {
    ProblemDef pd;
    ConfigDef cf;
    int policy = 0;  // 0 Mirror32, 1 Faithful64
    std::unique_ptr<Planner<Mirror32>> m32;
    std::unique_ptr<Planner<Faithful64>> f64;
};

template <class P>
void validate_root(const Planner<P>& pl) {
    const auto& n0 = pl.nodes()[0];
    if (!is_state_valid<P>(pl.problem(), pl.consts(), n0.state))
        throw InvalidProblemError("x_init is not a valid state (SPEC.md:61, :374)");
}

template <class P>
void fill_result(const Planner<P>& pl, kp_result* r) {
    std::memset(r, 0, sizeof *r);
    const auto& s = pl.stats();
    r->found = pl.best_leaf() >= 0;
    r->capacity_exhausted = s.capacity_exhausted;
    r->best_cost = static_cast<double>(pl.best_cost());
    r->best_leaf = pl.best_leaf();
    r->best_found_at_s = pl.best_t();
    r->best_found_iteration = pl.best_iter();
    r->first_solution_s = pl.first_t();
    r->first_solution_cost = static_cast<double>(pl.first_cost());
    r->first_solution_iteration = pl.first_iter();
    r->elapsed_s = pl.elapsed();
    r->iterations = s.iterations;
    r->propagations_attempted = s.attempted;
    r->propagations_valid = s.valid;
    r->propagations_admitted = s.admitted;
    r->nodes_committed = s.committed;
    r->nodes_pruned_terminal = s.pruned_terminal;
    r->nodes_deactivated = s.deactivated;
    r->nodes_reactivated = s.reactivated;
    r->candidates_dropped_capacity = s.dropped_capacity;
    r->node_count = pl.nodes().size();
    r->timeline_len = pl.timeline().size();
}

template <class P>
void get_nodes(const Planner<P>& pl, double* states, double* controls, double* dts, double* acc,
               int64_t* parent, uint32_t* region, uint8_t* status, uint32_t* icnt, size_t cap, size_t* len) {
    const auto& nodes = pl.nodes();
    const int n = pl.problem().n, m = pl.problem().m;
    *len = nodes.size();
    const size_t k = std::min(cap, nodes.size());
    for (size_t i = 0; i < k; ++i) {
        const auto& x = nodes[i];
        if (states) for (int j = 0; j < n; ++j) states[i * n + j] = x.state[j];
        if (controls) for (int j = 0; j < m; ++j) controls[i * m + j] = x.u[j];
        if (dts) dts[i] = x.dt;
        if (acc) acc[i] = x.acc;
        if (parent) parent[i] = x.parent;
        if (region) region[i] = x.region;
        if (status) status[i] = x.status;
        if (icnt) icnt[i] = x.icnt;
    }
}

template <class P>
void get_table(const Planner<P>& pl, double* out, size_t cap, size_t* len) {
    const auto& t = pl.table();
    *len = t.size();
    for (size_t i = 0; i < std::min(cap, t.size()); ++i) out[i] = P::decode(t[i].load());
}

}  // namespace

extern "C" {

const char* kpo_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- planner ---
int kpo_create(const kp_problem_desc* p, const kp_config_desc* c, int policy, void** out) {
    *out = nullptr;
    return guard([&] {
        auto h = std::make_unique<Handle>();
        convert(p, c, h->pd, h->cf);
        h->policy = policy;
        if (policy == 0) {
            h->m32 = std::make_unique<Planner<Mirror32>>(h->pd, h->cf);
            validate_root(*h->m32);
        } else {
            h->f64 = std::make_unique<Planner<Faithful64>>(h->pd, h->cf);
            validate_root(*h->f64);
        }
        *out = h.release();
    });
}

void kpo_destroy(void* h) { delete static_cast<Handle*>(h); }

int kpo_reset(void* hv, uint64_t seed) {
    auto* h = static_cast<Handle*>(hv);
    return guard([&] {
        h->cf.seed = seed;
        if (h->m32) h->m32 = std::make_unique<Planner<Mirror32>>(h->pd, h->cf);
        if (h->f64) h->f64 = std::make_unique<Planner<Faithful64>>(h->pd, h->cf);
    });
}

int kpo_run(void* hv, double budget_s, uint64_t max_iters, int stop_first, kp_result* out) {
    auto* h = static_cast<Handle*>(hv);
    return guard([&] {
        const double b = budget_s >= 0 ? budget_s : h->cf.t_max_s;
        const uint64_t mi = max_iters ? max_iters : h->cf.max_iterations;
        const bool sf = stop_first >= 0 ? stop_first != 0 : h->cf.stop_at_first_solution;
        if (h->m32) { h->m32->run(b, mi, sf); fill_result(*h->m32, out); }
        else { h->f64->run(b, mi, sf); fill_result(*h->f64, out); }
    });
}

int kpo_get_nodes(void* hv, double* states, double* controls, double* dts, double* acc, int64_t* parent,
                  uint32_t* region, uint8_t* status, uint32_t* icnt, size_t cap, size_t* len) {
    auto* h = static_cast<Handle*>(hv);
    return guard([&] {
        if (h->m32) get_nodes(*h->m32, states, controls, dts, acc, parent, region, status, icnt, cap, len);
        else get_nodes(*h->f64, states, controls, dts, acc, parent, region, status, icnt, cap, len);
    });
}

int kpo_get_table(void* hv, double* out, size_t cap, size_t* len) {
    auto* h = static_cast<Handle*>(hv);
    return guard([&] {
        if (h->m32) get_table(*h->m32, out, cap, len);
        else get_table(*h->f64, out, cap, len);
    });
}

int kpo_get_timeline(void* hv, kp_timeline_entry* buf, size_t cap, size_t* len) {
    auto* h = static_cast<Handle*>(hv);
    return guard([&] {
        const std::vector<TimelineEntry>& t = h->m32 ? h->m32->timeline() : h->f64->timeline();
        *len = t.size();
        for (size_t i = 0; i < std::min(cap, t.size()); ++i)
            buf[i] = {t[i].iteration, t[i].elapsed_s, t[i].cost, t[i].leaf};
    });
}

int kpo_get_grid(void* hv, int64_t* cells, double* side, uint64_t* n_regions) {
    auto* h = static_cast<Handle*>(hv);
    return guard([&] {
        for (size_t j = 0; j < h->pd.grid_cells.size(); ++j) {
            cells[j] = h->pd.grid_cells[j];
            side[j] = h->m32 ? double(h->m32->consts().g_side[j]) : h->f64->consts().g_side[j];
        }
        *n_regions = h->m32 ? h->m32->n_regions() : h->f64->n_regions();
    });
}

// Per-work-item propagate (mirror of kp_debug_propagate).  valid: 1 valid,
// 0 invalid, 2 diverged.  States are double arrays (exact for fp32 values).
int kpo_propagate_items(void* hv, size_t count, const double* parent_states, const double* parent_acc,
                        const uint32_t* node_ids, const uint32_t* branches, uint32_t iteration,
                        uint8_t* valid, double* final_states, double* controls, double* durations,
                        double* acc, uint32_t* region, uint32_t* steps, uint8_t* goal) {
    auto* h = static_cast<Handle*>(hv);
    return guard([&] {
        auto run = [&](auto& pl) {
            using P = std::remove_reference_t<decltype(pl)>;
            using R = typename std::remove_reference_t<decltype(*pl)>::R;
            (void)sizeof(P);
            const int n = h->pd.n, m = h->pd.m;
            std::vector<Vec<R>> samples;
            for (size_t i = 0; i < count; ++i) {
                Vec<R> x;
                x.n = n;
                for (int j = 0; j < n; ++j) x[j] = R(parent_states[i * n + j]);
                typename std::remove_reference_t<decltype(*pl)>::Candidate c{};
                const int rc = pl->propagate_item(x, R(parent_acc[i]), node_ids[i], branches[i], iteration, c, samples);
                valid[i] = rc == 0 ? 1 : (rc == 1 ? 0 : 2);
                if (steps) steps[i] = static_cast<uint32_t>(samples.size() - 1);
                if (controls) for (int j = 0; j < m; ++j) controls[i * m + j] = c.u[j];
                if (durations) durations[i] = c.dt;
                if (rc == 0) {
                    if (final_states) for (int j = 0; j < n; ++j) final_states[i * n + j] = c.state[j];
                    if (acc) acc[i] = c.acc;
                    if (region) region[i] = c.region;
                    if (goal) goal[i] = c.goal;
                } else {
                    if (final_states) for (int j = 0; j < n; ++j) final_states[i * n + j] = 0;
                    if (acc) acc[i] = 0;
                    if (region) region[i] = 0;
                    if (goal) goal[i] = 0;
                }
            }
        };
        if (h->m32) run(h->m32);
        else run(h->f64);
    });
}

// ------------------------------------------------------------- single ops ---
uint64_t kpo_mix64(uint64_t z) { return mix64(z); }
uint64_t kpo_derive_stream(uint64_t s, uint64_t it, uint64_t node, uint64_t br) {
    return derive_stream(s, it, node, br);
}
// Draw `count` raw outputs / uniform_unit values from SplitMix64(seed).
void kpo_splitmix(uint64_t seed, size_t count, uint64_t* raw, double* unit) {
    SplitMix64 a(seed), b(seed);
    for (size_t i = 0; i < count; ++i) {
        if (raw) raw[i] = a();
        if (unit) unit[i] = uniform_unit(b);
    }
}
void kpo_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) { philox4x32_10(ctr, key, out); }
double kpo_wrap_angle(double a) { return wrap_angle<Faithful64>(a); }
float kpo_wrap_angle_f32(float a) { return wrap_angle<Mirror32>(a); }
void kpo_sincos_f32(float x, float* s, float* c) { sincos_recipe_f32(x, s, c); }

// segment_cost over explicit samples (cost.hpp:44-67), fp64 policy.
int kpo_segment_cost(const double* samples, size_t n_samples, int dim, int position_dims, int kind,
                     double duration, double* out) {
    return guard([&] {
        ProblemDef pd;
        pd.n = dim;
        pd.cost = static_cast<CostKind>(kind);
        pd.cost_position_dims = position_dims;
        Consts<Faithful64> k{};
        k.zero_rate = 1e-6;
        std::vector<Vec<double>> s(n_samples);
        for (size_t i = 0; i < n_samples; ++i) {
            s[i].n = dim;
            for (int j = 0; j < dim; ++j) s[i][j] = samples[i * dim + j];
        }
        *out = segment_cost<Faithful64>(pd, k, s, duration);
    });
}

// in_goal (cost.hpp:77-84), fp64.
int kpo_in_goal(const double* x, int dim, const int32_t* goal_dims, const double* center, int g, double radius) {
    ProblemDef pd;
    pd.n = dim;
    pd.goal_dims.assign(goal_dims, goal_dims + g);
    Consts<Faithful64> k{};
    for (int i = 0; i < g; ++i) k.goal_c[i] = center[i];
    k.goal_r2 = radius * radius;
    Vec<double> v;
    v.n = dim;
    for (int i = 0; i < dim; ++i) v[i] = x[i];
    return in_goal<Faithful64>(pd, k, v) ? 1 : 0;
}

// propagate_ode from an explicit (x, u, dt, h) with the handle's model.
int kpo_propagate_ode(void* hv, const double* x, const double* u, double dt, double h_step, double* samples,
                      size_t cap, size_t* n_samples) {
    auto* h = static_cast<Handle*>(hv);
    return guard([&] {
        auto run = [&](auto& pl) {
            using R = typename std::remove_reference_t<decltype(*pl)>::R;
            using PP = std::conditional_t<std::is_same_v<R, float>, Mirror32, Faithful64>;
            const int n = h->pd.n, m = h->pd.m;
            Vec<R> xv, uv;
            xv.n = n; uv.n = m;
            for (int j = 0; j < n; ++j) xv[j] = R(x[j]);
            for (int j = 0; j < m; ++j) uv[j] = R(u[j]);
            std::vector<Vec<R>> s;
            const bool ok = propagate_ode<PP>(h->pd, pl->consts(), xv, uv, R(dt), R(h_step), s);
            *n_samples = s.size();
            for (size_t i = 0; i < std::min(cap, s.size()); ++i)
                for (int j = 0; j < n; ++j) samples[i * n + j] = s[i][j];
            if (!ok) throw std::runtime_error("propagation diverged");
        };
        if (h->m32) run(h->m32);
        else run(h->f64);
    });
}

int kpo_derivative(void* hv, const double* x, const double* u, double* out) {
    auto* h = static_cast<Handle*>(hv);
    return guard([&] {
        auto run = [&](auto& pl) {
            using R = typename std::remove_reference_t<decltype(*pl)>::R;
            using PP = std::conditional_t<std::is_same_v<R, float>, Mirror32, Faithful64>;
            Vec<R> xv, uv, o;
            xv.n = h->pd.n; uv.n = h->pd.m;
            for (int j = 0; j < h->pd.n; ++j) xv[j] = R(x[j]);
            for (int j = 0; j < h->pd.m; ++j) uv[j] = R(u[j]);
            derivative<PP>(h->pd, pl->consts(), xv, uv, o);
            for (int j = 0; j < h->pd.n; ++j) out[j] = o[j];
        };
        if (h->m32) run(h->m32);
        else run(h->f64);
    });
}

int kpo_is_state_valid(void* hv, const double* x) {
    auto* h = static_cast<Handle*>(hv);
    int res = 0;
    auto run = [&](auto& pl) {
        using R = typename std::remove_reference_t<decltype(*pl)>::R;
        using PP = std::conditional_t<std::is_same_v<R, float>, Mirror32, Faithful64>;
        Vec<R> v;
        v.n = h->pd.n;
        for (int j = 0; j < h->pd.n; ++j) v[j] = R(x[j]);
        res = is_state_valid<PP>(h->pd, pl->consts(), v);
    };
    if (h->m32) run(h->m32);
    else run(h->f64);
    return res;
}

int kpo_is_segment_valid(void* hv, const double* samples, size_t n_samples) {
    auto* h = static_cast<Handle*>(hv);
    int res = 0;
    auto run = [&](auto& pl) {
        using R = typename std::remove_reference_t<decltype(*pl)>::R;
        using PP = std::conditional_t<std::is_same_v<R, float>, Mirror32, Faithful64>;
        std::vector<Vec<R>> s(n_samples);
        for (size_t i = 0; i < n_samples; ++i) {
            s[i].n = h->pd.n;
            for (int j = 0; j < h->pd.n; ++j) s[i][j] = R(samples[i * h->pd.n + j]);
        }
        res = is_segment_valid<PP>(h->pd, pl->consts(), s);
    };
    if (h->m32) run(h->m32);
    else run(h->f64);
    return res;
}

uint32_t kpo_region_index(void* hv, const double* x) {
    auto* h = static_cast<Handle*>(hv);
    uint32_t res = 0;
    auto run = [&](auto& pl) {
        using R = typename std::remove_reference_t<decltype(*pl)>::R;
        using PP = std::conditional_t<std::is_same_v<R, float>, Mirror32, Faithful64>;
        Vec<R> v;
        v.n = h->pd.n;
        for (int j = 0; j < h->pd.n; ++j) v[j] = R(x[j]);
        res = region_index<PP>(h->pd, pl->consts(), v);
    };
    if (h->m32) run(h->m32);
    else run(h->f64);
    return res;
}

// try_update_region_cost on a standalone fp64 table:
// applies `count` (region, cost) updates with `workers` threads in
// interleaved chunks; writes outcomes and the final table.
int kpo_atomic_min_stress(size_t n_regions, size_t count, const uint32_t* regions, const double* costs,
                          int workers, double* final_table, uint8_t* outcomes) {
    return guard([&] {
        std::vector<std::atomic<uint64_t>> t(n_regions);
        for (auto& c : t) c.store(Faithful64::encode(std::numeric_limits<double>::infinity()));
        std::vector<std::thread> th;
        const int W = std::max(1, workers);
        for (int w = 0; w < W; ++w) {
            th.emplace_back([&, w] {
                for (size_t i = w; i < count; i += W) {
                    const Outcome o = try_update<Faithful64>(t[regions[i]], costs[i]);
                    if (outcomes) outcomes[i] = static_cast<uint8_t>(o);
                }
            });
        }
        for (auto& x : th) x.join();
        for (size_t i = 0; i < n_regions; ++i) final_table[i] = Faithful64::decode(t[i].load());
    });
}

}  // extern "C"
