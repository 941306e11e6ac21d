// kinoplan_b200/kinoplan.hpp — C++ drop-in API of the B200 planner.
//
// Mirrors the reference library `kinoplan` (namespace kinoplan, C++20):
//   errors        proj/include/kinoplan/core/errors.hpp:11-33 (same class names)
//   types         proj/include/kinoplan/core/types.hpp:11-58 (Scalar, Interval, Bounds, wrap_angle)
//   cost          proj/include/kinoplan/core/cost.hpp:13-92 (CostKind, CostMetric, GoalRegion, segment_cost, in_goal)
//   dynamics      proj/include/kinoplan/dynamics/model.hpp:15-68 (ModelParams, DynamicsModel, make_model)
//   problem/plan  SPEC.md:58-69 (PlanningProblem, PlannerConfig), SPEC.md:355-378 (BestSolution,
//                 PlannerStats, plan), SPEC.md:414-422 (extract_trajectory)
// Vectors are std::vector<double> instead of Eigen fixed-max vectors (Eigen is
// not a dependency of the GPU build).  Every call goes through the C-ABI in
// include/kinoplan_b200.h; planning runs on the GPU only.
#pragma once

#include <atomic>
#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <numbers>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

struct kp_planner;

namespace kinoplan {

// ---- errors.hpp:11-33 ----
struct SchemaError : std::runtime_error { using std::runtime_error::runtime_error; };
struct InvalidProblemError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct GridTooFineError : std::runtime_error { using std::runtime_error::runtime_error; };
struct InvalidSegmentError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };  // no reference counterpart

[[noreturn]] void invariant_failure(const char* expr, const char* file, int line, const std::string& msg);
}  // namespace kinoplan

// Internal invariants abort: a bug, not a recoverable condition (errors.hpp:35-48).
#define KINO_CHECK(cond, msg)                                                         \
    do {                                                                              \
        if (!(cond)) ::kinoplan::invariant_failure(#cond, __FILE__, __LINE__, (msg)); \
    } while (0)

namespace kinoplan {

// ---- types.hpp ----
using Scalar = double;
inline constexpr int kMaxStateDim = 12;
using Vec = std::vector<Scalar>;
using State = Vec;
using Control = Vec;

struct Interval {
    Scalar lo = 0;
    Scalar hi = 0;
    [[nodiscard]] bool contains(Scalar v) const noexcept { return v >= lo && v <= hi; }
    [[nodiscard]] Scalar width() const noexcept { return hi - lo; }
};
using Bounds = std::vector<Interval>;

[[nodiscard]] inline Scalar wrap_angle(Scalar a) noexcept {  // types.hpp:49-58
    constexpr Scalar pi = std::numbers::pi_v<Scalar>;
    a = std::fmod(a, 2 * pi);
    if (a <= -pi) a += 2 * pi;
    else if (a > pi) a -= 2 * pi;
    return a;
}

// ---- cost.hpp ----
enum class CostKind { PathLength, ControlDuration };
inline constexpr Scalar kZeroDisplacementCostRate = 1e-6;

struct CostMetric {
    CostKind kind = CostKind::PathLength;
    int position_dims = 3;
    std::optional<Scalar> lipschitz_hint;
};

struct GoalRegion {
    std::vector<int> dims;
    Vec center;
    Scalar radius = 0;
};

[[nodiscard]] Scalar segment_cost(std::span<const State> samples, const Control& control, Scalar duration,
                                  const CostMetric& metric);
[[nodiscard]] bool in_goal(const State& x, const GoalRegion& goal) noexcept;

// ---- model.hpp ----
struct ModelParams {
    std::map<std::string, Scalar> values;
    [[nodiscard]] Scalar get(const std::string& key, Scalar fallback) const {
        const auto it = values.find(key);
        return it == values.end() ? fallback : it->second;
    }
};

class DynamicsModel {
public:
    DynamicsModel(std::string id, int model_code, int state_dim, int control_dim, std::vector<int> position_dims,
                  std::vector<int> angle_dims, ModelParams params)
        : id_(std::move(id)), code_(model_code), state_dim_(state_dim), control_dim_(control_dim),
          position_dims_(std::move(position_dims)), angle_dims_(std::move(angle_dims)), params_(std::move(params)) {}
    [[nodiscard]] const std::string& id() const noexcept { return id_; }
    [[nodiscard]] int model_code() const noexcept { return code_; }
    [[nodiscard]] int state_dim() const noexcept { return state_dim_; }
    [[nodiscard]] int control_dim() const noexcept { return control_dim_; }
    [[nodiscard]] std::span<const int> position_dims() const noexcept { return position_dims_; }
    [[nodiscard]] std::span<const int> angle_dims() const noexcept { return angle_dims_; }
    [[nodiscard]] const ModelParams& params() const noexcept { return params_; }
    /// Host fp64 evaluation of dx/dt = f(x, u) (model.hpp:42).  The planner's
    /// device code evaluates the same equations in fp32.
    void derivative(const Vec& x, const Vec& u, Vec& out) const;

private:
    std::string id_;
    int code_;
    int state_dim_, control_dim_;
    std::vector<int> position_dims_, angle_dims_;
    ModelParams params_;
};

/// make_model (model.hpp:64-68): double_integrator_4d, double_integrator_6d,
/// dubins_airplane_6d, quadcopter_12d.  Throws SchemaError for unknown ids.
[[nodiscard]] std::shared_ptr<const DynamicsModel> make_model(const std::string& id, const ModelParams& params = {});

// ---- environment ----
struct Obstacle {
    enum class Type { Box, Sphere } type = Type::Box;
    double a[3] = {0, 0, 0};  // box min / sphere center
    double b[3] = {0, 0, 0};  // box max / sphere radius in b[0]
    static Obstacle box(std::initializer_list<double> lo, std::initializer_list<double> hi);
    static Obstacle sphere(std::initializer_list<double> c, double r);
};

struct Environment {
    Bounds workspace_bounds;
    std::vector<Obstacle> obstacles;
    Bounds state_bounds;  // SPEC.md:192 full-state limits (is_state_valid); the planner takes PlanningProblem::state_bounds
};

// ---- problem / config ----
struct PlanningProblem {
    std::shared_ptr<const DynamicsModel> model;
    Environment environment;
    State x_init;
    GoalRegion goal;
    CostMetric cost;
    Bounds state_bounds;
    Bounds control_bounds;
};

struct Decomposition {
    std::vector<int> dims;          // decomposed state dims
    std::optional<double> delta;    // region diagonal, or
    std::vector<int> cells;         // cells per dim
    uint64_t max_cells = 0;         // GridTooFineError ceiling (0 = 2^28)
};

enum class RngKind { Philox = 0, SplitMix = 1 };

struct PlannerConfig {
    Decomposition decomposition;
    int lambda = 32;
    int i_max = 5;
    double t_max = 0.1;             // seconds
    double t_prop = 0.5;
    uint64_t capacity = 1u << 20;
    uint64_t seed = 0;
    int workers = 1;                // accepted, ignored on the GPU (deterministic)
    std::optional<double> ode_step; // default min(t_prop/10, 0.02)
    double collision_step = 0.05;
    uint64_t max_iterations = 0;
    bool deactivate_after_expansion = false;
    RngKind rng = RngKind::Philox;
    bool stop_at_first_solution = false;
    uint64_t max_slots = 0;         // per-iteration V_U slot buffer (0 = min(lambda*capacity, 2^25))
    int device = 0;
};

// ---- results ----
struct BestSolution {
    Scalar cost = std::numeric_limits<Scalar>::infinity();
    std::optional<int64_t> leaf;
    Scalar found_at = 0;  // seconds
};

struct PlannerStats {
    uint64_t iterations = 0, propagations_attempted = 0, propagations_valid = 0, propagations_admitted = 0;
    uint64_t nodes_pruned_terminal = 0, nodes_deactivated = 0, nodes_reactivated = 0, nodes_committed = 0;
    std::vector<std::pair<Scalar, Scalar>> cost_timeline;  // (elapsed s, best cost)
    std::optional<std::pair<Scalar, Scalar>> first_solution;
    bool capacity_exhausted = false;
    Scalar elapsed = 0;
    uint64_t first_solution_iteration = 0;  // iteration boundary that first set best < inf
    uint64_t best_found_iteration = 0;
    uint64_t node_count = 0;
};

struct Trajectory {
    std::vector<State> states;         // root .. leaf node states
    std::vector<Control> controls;     // incoming control per node (root: zeros)
    std::vector<Scalar> durations;     // incoming duration per node (root: 0)
    std::vector<State> samples;        // re-integrated dense samples root -> leaf
    std::vector<Scalar> segment_costs; // per segment; running sum == leaf acc (fp32, bit-exact)
    Scalar cost = 0;
};

struct PlanResult {
    BestSolution best;
    std::optional<Trajectory> trajectory;
    PlannerStats stats;
};

/// A reusable GPU planner instance (single owner).
class Planner {
public:
    Planner(const PlanningProblem& problem, const PlannerConfig& config);
    ~Planner();
    Planner(const Planner&) = delete;
    Planner& operator=(const Planner&) = delete;
    void reset(uint64_t seed);
    /// Runs until budget_s (< 0: config.t_max) / max_iterations (0: config value).
    PlanResult solve(double budget_s = -1, uint64_t max_iterations = 0, bool extract = true);
    [[nodiscard]] Trajectory extract_trajectory(int64_t leaf);

private:
    kp_planner* h_ = nullptr;
    int n_ = 0, m_ = 0;
};

/// plan(problem, config): one fresh run with config.seed.
PlanResult plan(const PlanningProblem& problem, const PlannerConfig& config);

// ---------------------------------------------------------------------------
// Host (fp64) building blocks of the reference API, for callers that set up,
// check or replay pieces of a plan on the CPU.  The planner itself runs on the
// GPU (fp32 recipe); these follow the SPEC in double precision.
// ---------------------------------------------------------------------------

// ---- rng.hpp:12-57 ----
class SplitMix64 {
public:
    using result_type = uint64_t;
    explicit constexpr SplitMix64(uint64_t seed) noexcept : state_(seed) {}
    static constexpr result_type min() noexcept { return 0; }
    static constexpr result_type max() noexcept { return ~result_type{0}; }
    constexpr result_type operator()() noexcept {
        state_ += 0x9E3779B97F4A7C15ULL;
        uint64_t z = state_;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }

private:
    uint64_t state_;
};

[[nodiscard]] constexpr uint64_t mix64(uint64_t z) noexcept {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

[[nodiscard]] constexpr uint64_t derive_stream(uint64_t seed, uint64_t iteration, uint64_t node_id,
                                               uint64_t branch) noexcept {
    uint64_t s = mix64(seed);
    s = mix64(s ^ iteration);
    s = mix64(s ^ node_id);
    s = mix64(s ^ branch);
    return s;
}

[[nodiscard]] inline Scalar uniform_unit(SplitMix64& rng) noexcept {
    return static_cast<Scalar>(rng() >> 11) * 0x1.0p-53;
}

// ---- dynamics ----
/// Samples at 0, h, ..., dt (last step shortened), classical RK4 under constant
/// u, angles wrapped after every step; samples[0] == x bit-exact.  A
/// non-finite state throws InvalidSegmentError ("propagation diverged").
[[nodiscard]] std::vector<State> propagate_ode(const State& x, const Control& u, Scalar dt, Scalar h,
                                               const DynamicsModel& model);
/// Each axis uniform on [lo, hi] (controls in axis order).
[[nodiscard]] Control sample_control(SplitMix64& rng, const Bounds& bounds);
/// Uniform on (0, t_prop].
[[nodiscard]] Scalar sample_duration(SplitMix64& rng, Scalar t_prop);

// ---- environment ----
/// Within env.state_bounds (every coordinate, when given) and the workspace
/// (position dims), outside every closed obstacle.
[[nodiscard]] bool is_state_valid(const State& x, const Environment& env, const DynamicsModel& model);
/// Every sample valid, plus the dyadic interior points (spacing <= collision_step)
/// of consecutive samples farther apart than collision_step obstacle-free.
[[nodiscard]] bool is_segment_valid(std::span<const State> samples, const Environment& env,
                                    const DynamicsModel& model, Scalar collision_step);
/// Environment fragment of a scenario file (keys workspace_bounds,
/// state_bounds, obstacles); SchemaError names the offending primitive.
[[nodiscard]] Environment load_environment(const std::string& json_fragment);

// ---- decomposition ----
enum class UpdateOutcome { Improved, Equal, Worse };

/// Region grid over the decomposed state dims with an atomically updatable
/// cost table (order-preserving u64 encoding of the fp64 cost, +inf initial).
class RegionGrid {
public:
    std::vector<int> dims;        // decomposed state dims
    Bounds bounds;                // per decomposed dim
    std::vector<int> cells;       // cells per dim
    std::vector<Scalar> side;     // cell widths
    Scalar delta = 0;             // cell diagonal
    uint64_t n_regions = 0;
    RegionGrid() = default;
    RegionGrid(RegionGrid&&) noexcept = default;
    RegionGrid& operator=(RegionGrid&&) noexcept = default;
    std::unique_ptr<std::atomic<uint64_t>[]> table;
};

/// cells_i = max(1, ceil((hi-lo)_i sqrt(n) / delta)) when delta is given, else
/// `cells`; GridTooFineError above max_cells (0 = 2^28).
[[nodiscard]] RegionGrid build_grid(const std::vector<int>& dims, const Bounds& bounds,
                                    std::optional<Scalar> delta, const std::vector<int>& cells,
                                    uint64_t max_cells = 0);
/// clamp(floor((x_d - lo) / side), 0, cells - 1), row-major with dim 0 fastest.
[[nodiscard]] uint64_t region_index(const State& x, const RegionGrid& grid);
/// Atomic min via CAS on the encoding; Improved / Equal / Worse vs the old value.
UpdateOutcome try_update_region_cost(RegionGrid& grid, uint64_t i, Scalar c);
[[nodiscard]] Scalar region_cost(const RegionGrid& grid, uint64_t i);

}  // namespace kinoplan
