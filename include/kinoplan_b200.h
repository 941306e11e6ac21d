/*
 * kinoplan_b200.h — C-ABI drop-in boundary of the B200-native Kino-PAX+ planner.
 *
 * The reference (/root/reference) is a C++20 library `kinoplan` whose planner
 * sources are absent; its interface is fixed by the shipped headers and SPEC.md.
 * Every entry point below cites the reference interface it replaces.  No C++
 * types, exceptions or torch types cross this boundary: plain pointers, sizes
 * and POD structs only.  Errors map 1:1 onto the reference exception classes
 * (proj/include/kinoplan/core/errors.hpp:11-33) via kp_status, with the message
 * available from kp_last_error().
 *
 * Threading ("plan is single-owner"): one host thread per handle
 * at a time; handles on different devices are independent.
 */
#ifndef KINOPLAN_B200_H
#define KINOPLAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KP_ABI_VERSION 1
#define KP_MAX_STATE_DIM 12   /* types.hpp:15 kMaxStateDim */
#define KP_MAX_CONTROL_DIM 4  /* quadcopter_12d has the widest control */
#define KP_MAX_GRID_DIMS 6
#define KP_MAX_OBSTACLES 4096

/* Status codes.  Nonzero values map onto errors.hpp exception classes. */
typedef enum kp_status {
    KP_OK = 0,
    KP_ERR_SCHEMA = 1,            /* errors.hpp:11  SchemaError (unknown model id, bad geometry) */
    KP_ERR_INVALID_PROBLEM = 2,   /* errors.hpp:16  InvalidProblemError (x_init invalid, goal outside) */
    KP_ERR_CONFIG = 3,            /* errors.hpp:21  ConfigError (SPEC.md:68 invariants) */
    KP_ERR_GRID_TOO_FINE = 4,     /* errors.hpp:26  GridTooFineError */
    KP_ERR_INVALID_SEGMENT = 5,   /* errors.hpp:31  InvalidSegmentError (cost.hpp:47-52) */
    KP_ERR_CUDA = 6,              /* device / runtime failure (no reference counterpart) */
    KP_ERR_ARGUMENT = 7,          /* null pointer / short buffer at the ABI */
    KP_ERR_SLOT_OVERFLOW = 8      /* lambda*|V_A| exceeded the per-iteration slot buffer */
} kp_status;

/* model.hpp:64-68 make_model ids. */
typedef enum kp_model_id {
    KP_MODEL_DOUBLE_INTEGRATOR_4D = 0,
    KP_MODEL_DOUBLE_INTEGRATOR_6D = 1,
    KP_MODEL_DUBINS_AIRPLANE_6D = 2,
    KP_MODEL_QUADCOPTER_12D = 3
} kp_model_id;

/* cost.hpp:13-16 CostKind. */
typedef enum kp_cost_kind { KP_COST_PATH_LENGTH = 0, KP_COST_CONTROL_DURATION = 1 } kp_cost_kind;

typedef enum kp_obstacle_type { KP_OBSTACLE_BOX = 0, KP_OBSTACLE_SPHERE = 1 } kp_obstacle_type;

/* Per-work-item random stream.  SPLITMIX is rng.hpp:44-57 derive_stream +
 * uniform_unit verbatim; PHILOX is Philox4x32-10 keyed by the seed with counter
 * (iteration, node id, branch, call) — the north-star device RNG. */
typedef enum kp_rng_kind { KP_RNG_PHILOX = 0, KP_RNG_SPLITMIX = 1 } kp_rng_kind;

/* Environment primitive: box {a = min corner, b = max corner} or
 * sphere {a = center, b[0] = radius}.  Unused coordinates of 2-D scenes are 0. */
typedef struct kp_obstacle {
    int32_t type;
    int32_t reserved;
    double a[3];
    double b[3];
} kp_obstacle;

/* PlanningProblem + Environment + RegionGrid
 * spec + ModelParams (model.hpp:15-22).  Copied at kp_create. */
typedef struct kp_problem_desc {
    int32_t model;              /* kp_model_id */
    int32_t n_params;           /* ModelParams overrides (model.hpp:15) */
    const char* const* param_names;
    const double* param_values;
    int32_t state_dim;          /* must equal the model's state_dim */
    int32_t control_dim;        /* must equal the model's control_dim */
    const double* x_init;       /* [state_dim] */
    const double* state_lo;     /* [state_dim] state_bounds */
    const double* state_hi;
    const double* control_lo;   /* [control_dim] control_bounds */
    const double* control_hi;
    int32_t workspace_dim;      /* 2 or 3 */
    int32_t n_obstacles;
    const double* workspace_lo; /* [workspace_dim] */
    const double* workspace_hi;
    const kp_obstacle* obstacles;
    int32_t goal_n_dims;        /* GoalRegion (cost.hpp:70-74) */
    int32_t reserved0;
    const int32_t* goal_dims;
    const double* goal_center;
    double goal_radius;
    int32_t cost_kind;          /* kp_cost_kind (cost.hpp:32-39) */
    int32_t cost_position_dims; /* CostMetric::position_dims (cost.hpp:36) */
    int32_t grid_n_dims;        /* decomposition dims */
    int32_t reserved1;
    const int32_t* grid_dims;   /* [grid_n_dims] state indices */
    const int32_t* grid_cells;  /* [grid_n_dims] cells_per_dim, or NULL to use grid_delta */
    double grid_delta;          /* region diagonal when grid_cells == NULL */
    uint64_t grid_max_cells;    /* GridTooFineError ceiling; 0 = default 2^28 */
} kp_problem_desc;

/* PlannerConfig (keys SPEC.md:518). */
typedef struct kp_config_desc {
    int32_t lambda;             /* branching factor >= 1 */
    int32_t i_max;              /* inactivity threshold >= 1 */
    double t_max_s;             /* wall budget; <= 0 means unlimited (use max_iterations) */
    double t_prop;              /* max propagation duration > 0 */
    double ode_step;            /* RK4 step h; <= 0 selects min(t_prop/10, 0.02) */
    double collision_step;      /* max spacing of validity samples */
    uint64_t capacity;          /* node store capacity t_e >= 1 */
    uint64_t seed;
    uint64_t max_iterations;    /* 0 = unlimited */
    int32_t workers;            /* accepted and ignored on the GPU (deterministic by construction) */
    int32_t deactivate_after_expansion; /* SPEC.md:436 ablation flag */
    int32_t rng_kind;           /* kp_rng_kind */
    int32_t stop_at_first_solution; /* stop at the first iteration boundary with best < inf */
    uint64_t max_slots;         /* per-iteration V_U slot buffer; 0 = min(lambda*capacity, 2^25) */
} kp_config_desc;

/* BestSolution + PlannerStats. */
typedef struct kp_result {
    int32_t found;                  /* success: best cost < inf */
    int32_t capacity_exhausted;
    double best_cost;               /* +inf when none */
    int64_t best_leaf;              /* -1 when none */
    double best_found_at_s;         /* elapsed s at the iteration boundary that set it */
    uint64_t best_found_iteration;
    double first_solution_s;        /* TTFS: device time, solve start -> first boundary with best < inf */
    double first_solution_cost;
    uint64_t first_solution_iteration;
    double elapsed_s;               /* device time, solve start -> last iteration boundary */
    uint64_t iterations;
    uint64_t propagations_attempted;
    uint64_t propagations_valid;
    uint64_t propagations_admitted; /* V_U admissions (order-dependent under races) */
    uint64_t nodes_committed;
    uint64_t nodes_pruned_terminal;
    uint64_t nodes_deactivated;
    uint64_t nodes_reactivated;
    uint64_t candidates_dropped_capacity;
    uint64_t node_count;
    uint64_t timeline_len;
} kp_result;

/* cost_timeline entry, one per iteration boundary that improved best. */
typedef struct kp_timeline_entry {
    uint64_t iteration;
    double elapsed_s;
    double cost;
    int64_t leaf;
} kp_timeline_entry;

typedef struct kp_planner kp_planner;

/* ---- lifecycle ---------------------------------------------------------- */

/* Replaces make_model (model.hpp:67) + PlanningProblem validation
 * + build_grid.  Copies the descriptors, allocates every device
 * buffer on `device` and validates.  On error *out is NULL and the message is
 * available from kp_last_error(NULL). */
int kp_create(const kp_problem_desc* problem, const kp_config_desc* config, int device,
              kp_planner** out);

void kp_destroy(kp_planner* planner);

/* Message of the last failing call on this handle (or of the last failing
 * kp_create when planner == NULL).  Never NULL. */
const char* kp_last_error(const kp_planner* planner);

/* Re-seed and clear the tree/grid/best so the next kp_solve starts a fresh run
 * ("trial k uses seed = base_seed + k"). */
int kp_reset(kp_planner* planner, uint64_t seed);

/* One query = (seed, start state).  Like kp_reset, but also replaces x_init
 * with the host array x_init[state_dim] (copied host->device; NULL keeps the
 * current start).  The new start is validated (InvalidProblemError,
 * SPEC.md:61, :374). */
int kp_reset_query(kp_planner* planner, uint64_t seed, const double* x_init);

/* Toggle PlannerConfig.stop_at_first_solution for later kp_solve calls. */
int kp_set_stop_at_first_solution(kp_planner* planner, int enabled);

/* ---- solve -------------------------------------------------------------- */

/* Replaces plan(problem, config).  Runs Alg. 1 iterations
 * (propagate -> prune -> update) on the device from the current (reset) state
 * until budget_s elapses (checked at iteration boundaries), or
 * max_iterations, or the first solution when stop_at_first_solution.  A
 * negative budget / zero max_iterations means "use the config value".  Blocks.
 * "No solution" is not an error: found = 0, best_cost = +inf. */
int kp_solve(kp_planner* planner, double budget_s, uint64_t max_iterations, kp_result* out);

/* PlannerStats::cost_timeline.  Copies up to cap entries. */
int kp_get_timeline(kp_planner* planner, kp_timeline_entry* buf, size_t cap, size_t* len);

/* extract_trajectory: root->leaf chain.  Writes up to cap
 * nodes: states [cap][state_dim], the incoming controls [cap][control_dim] and
 * durations [cap] (root: zeros), and accumulated costs [cap].  leaf < 0 selects
 * the best leaf.  *len receives the chain length (even if > cap). */
int kp_get_path(kp_planner* planner, int64_t leaf, double* states, double* controls,
                double* durations, double* acc_costs, size_t cap, size_t* len);

/* Re-integrated trajectory: every RK4 sample of every segment of
 * the root->leaf chain, concatenated (segment k contributes its samples 1..S_k),
 * recomputed on the device with the same fp32 arithmetic as propagation, plus
 * the per-segment costs whose running sum equals the leaf's acc_cost bit-exactly. */
int kp_get_trajectory(kp_planner* planner, int64_t leaf, double* samples, size_t cap_samples,
                      size_t* n_samples, double* segment_costs, size_t cap_segments,
                      size_t* n_segments);

/* ---- introspection (tests / parity) -------------------------------------- */

/* Node store snapshot.  Any pointer may be NULL.  Writes
 * min(cap, node_count) nodes; *len receives node_count.
 * states [n][state_dim] fp32, controls [n][control_dim] fp32, durations [n],
 * acc [n] fp32, parent [n] (-1 root), region [n], status [n]
 * (0 Active, 1 Inactive, 2 Terminal), icount [n]. */
int kp_get_nodes(kp_planner* planner, float* states, float* controls, float* durations,
                 float* acc, int32_t* parent, uint32_t* region, uint8_t* status,
                 uint8_t* icount, size_t cap, size_t* len);

/* Region cost table as encoded u32 (fp32 bits; +inf = 0x7F800000). */
int kp_get_region_table(kp_planner* planner, uint32_t* out, size_t cap, size_t* len);

/* Grid facts derived by build_grid: cells per dim, side (fp32) and
 * total region count. */
int kp_get_grid(kp_planner* planner, int32_t* cells, float* side, uint64_t* n_regions);

/* One propagate work item per entry, on the device, with explicit inputs —
 * exactly the arithmetic of the propagate kernel (Alg. 2 lines 3-7).  Used to
 * check per-work-item parity.  Inputs: parent states [n][state_dim]
 * fp32, parent acc [n], node ids [n], branches [n], one iteration number.
 * Outputs (any may be NULL): valid [n] (1 valid, 0 invalid, 2 diverged), final
 * states [n][state_dim], controls [n][control_dim], durations [n],
 * acc [n], region [n], steps [n], in_goal [n].  The region table is NOT touched. */
int kp_debug_propagate(kp_planner* planner, size_t n, const float* parent_states,
                       const float* parent_acc, const uint32_t* node_ids,
                       const uint32_t* branches, uint32_t iteration, uint8_t* valid,
                       float* final_states, float* controls, float* durations, float* acc,
                       uint32_t* region, uint32_t* steps, uint8_t* in_goal);

/* Work and timing counters for roofline accounting (bench.py).  Device
 * counters are cumulative since the last kp_reset; kernel_launches /
 * graph_launches since kp_create; the per-class CUDA-event times are only
 * collected while profiling is on (kp_set_profiling), one launch at a time. */
typedef struct kp_profile {
    uint64_t kernel_launches;   /* kernels enqueued by the library (graph nodes counted individually) */
    uint64_t graph_launches;
    double t_propagate_s, t_select_s, t_scatter_s;
    uint64_t n_propagate, n_select, n_scatter;
    uint64_t items;             /* propagate work items (== propagations_attempted) */
    uint64_t rk4_steps;         /* RK4 steps executed (valid + invalid items) */
    uint64_t samples_checked;   /* integration samples validity-checked */
    uint64_t interp_points;     /* interpolated points obstacle-checked */
    uint64_t box_tests;         /* point-vs-box tests executed */
    uint64_t sphere_tests;      /* point-vs-sphere tests executed */
    uint64_t live_scanned;      /* live nodes visited by the prune pass */
    uint64_t ancestor_hops;     /* parent hops of the ancestor-domination walks */
    uint64_t slots_scanned;     /* V_U slots visited by select */
    uint64_t admitted_checked;  /* admitted slots commit-tested */
} kp_profile;

int kp_set_profiling(kp_planner* planner, int enabled);
int kp_get_profile(kp_planner* planner, kp_profile* out);

/* Per-iteration trace (tracing aux subsystem): one record per iteration
 * boundary since the last reset, newest KP_TRACE_CAP kept.  t_ns is device
 * time since solve start (%globaltimer); items = lambda*|V_A| propagated in
 * that iteration; live / frontier / nodes are the counts after it. */
#define KP_TRACE_CAP 8192
typedef struct kp_trace_entry {
    uint64_t t_ns;
    uint32_t iteration, items, live, frontier, nodes, committed;
    /* in-graph kernel stamps, ns since solve start: block-0 entry of
     * propagate / select_reduce, entry of the select_scatter block that
     * closes the iteration (t_sel_end == t_scat; t_ns = the boundary) */
    uint32_t t_prop, t_sel, t_sel_end, t_scat;
} kp_trace_entry;

int kp_get_trace(kp_planner* planner, kp_trace_entry* buf, size_t cap, size_t* len);

/* The CUDA stream (cudaStream_t) every kernel of this handle is launched on,
 * so a caller can bracket work with its own CUDA events. */
int kp_get_stream(kp_planner* planner, void** stream);

/* Diagnostics of a library built with -DKP_STAMPS (scripts/stamps.py): the
 * %globaltimer phase stamps of the last 64 iterations, 64 x 32 uint64 (row =
 * iteration mod 64; columns in kp_kernels.cu).  KP_ERR_CONFIG otherwise. */
int kp_debug_stamps(kp_planner* planner, uint64_t* out_64x32);

/* ---- propagation sweep (BASELINE config 5) -------------------------------- */

/* Replace the tree by a synthetic frontier of n_nodes valid states: positions
 * uniform in the workspace (seeded, rejection-sampled against the obstacles),
 * every other coordinate as x_init ("hover-ish"), all Active, so that one propagate launch processes
 * n_nodes * lambda work items.  Needs capacity >= n_nodes and max_slots >=
 * n_nodes * lambda.  The planner must be kp_reset before a normal solve. */
int kp_sweep_setup(kp_planner* planner, uint64_t n_nodes, uint64_t seed);

/* Launch the propagate kernel alone `launches` times on the synthetic frontier
 * (region table reset to +inf before each launch, so every launch does the
 * same work) and return the mean device time per launch (CUDA events) and
 * the work counters of one launch. */
int kp_sweep_run(kp_planner* planner, uint32_t launches, double* ms_per_launch, kp_profile* one_launch);

/* ---- batched independent queries (BASELINE config 4) -------- */

/* Solve K independent seeded queries of the same problem on one device, one
 * query after another on the handle's stream.  results[K]. */
int kp_solve_batch(kp_planner* planner, const uint64_t* seeds, size_t k, double budget_s,
                   uint64_t max_iterations, kp_result* results);

/* Concurrent batch engine: `lanes` independent planner instances (own device
 * buffers, stream and CUDA graph each) on one device, fed by one asynchronous
 * host scheduler, so the kernels of different queries overlap on the GPU.
 * Queries share nothing (replicas-only semantics). */
typedef struct kp_batch kp_batch;
int kp_batch_create(const kp_problem_desc* problem, const kp_config_desc* config, int device, int lanes,
                    kp_batch** out);
void kp_batch_destroy(kp_batch* batch);
const char* kp_batch_last_error(const kp_batch* batch);
/* Solve queries seeds[0..k) (each with budget_s / max_iterations as
 * kp_solve); results[k] in seed order; *wall_s = host wall time of the batch. */
int kp_batch_solve(kp_batch* batch, const uint64_t* seeds, size_t k, double budget_s, uint64_t max_iterations,
                   kp_result* results, double* wall_s);

int kp_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* KINOPLAN_B200_H */
