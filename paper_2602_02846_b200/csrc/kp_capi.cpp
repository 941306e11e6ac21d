// kp_capi.cpp — host implementation of the C-ABI in include/kinoplan_b200.h.
//
// Owns one planner instance: validates the descriptors (the reference's
// problem/config invariants, model.hpp:64-68),
// rounds every constant to fp32 once (KpProblem), allocates the SoA device
// buffers, captures a CUDA graph of KP_GRAPH_ITERS iterations (3 kernels
// each) and drives kp_solve by launching that graph until the device raises
// its mapped "done" word.  No CPU fallback exists: without a device every
// entry point returns KP_ERR_CUDA.
//
// Compiled with -ffp-contract=off so the host-side fp32 constant folding is
// the same arithmetic the oracle's Mirror32 policy performs.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/kinoplan_b200.h"
#include "kp_types.h"

namespace kp {
cudaError_t read_check_code(unsigned int* code);
cudaError_t read_stamps(unsigned long long* out);
cudaError_t launch_iteration(const KpProblem& P, const KpBuffers& B, int grid_prop, int grid_sel, cudaStream_t st,
                             int which);
cudaError_t set_propagate_smem(const KpProblem& P);
void plan_propagate_smem(KpProblem& P);
void set_flat_limit(KpProblem& P, int grid_prop);

int propagate_occupancy(const KpProblem& P);
cudaError_t launch_reset(const KpProblem& P, const KpBuffers& B, unsigned long long seed, cudaStream_t st);
cudaError_t launch_start(const KpBuffers& B, unsigned long long budget_ns, uint32_t max_iters, uint32_t stop_first,
                         uint32_t seq, cudaStream_t st);
cudaError_t launch_debug_propagate(const KpProblem& P, const KpBuffers& B, uint32_t n, const float* ps,
                                   const float* pacc, const uint32_t* ids, const uint32_t* brs, uint32_t it,
                                   uint8_t* valid, float* xs, float* us, float* dts, float* accs, uint32_t* regs,
                                   uint32_t* steps, uint8_t* goals, cudaStream_t st);
cudaError_t launch_chain(const KpBuffers& B, int32_t leaf, int32_t* chain, uint32_t cap, uint32_t* len,
                         cudaStream_t st);
cudaError_t launch_sweep_prepare(const KpProblem& P, const KpBuffers& B, uint32_t n, cudaStream_t st);
cudaError_t launch_gather_chain(const KpProblem& P, const KpBuffers& B, const int32_t* chain, uint32_t len,
                                float* st, float* ct, float* dts, float* accs, cudaStream_t s);
cudaError_t launch_reintegrate(const KpProblem& P, const KpBuffers& B, const int32_t* chain, uint32_t n_seg,
                               const uint32_t* off, float* out, float* seg_cost, cudaStream_t st);
}  // namespace kp

namespace {

// Iterations per captured graph.  Consecutive graphs on the stream cannot
// chain their kernels with programmatic dependent launch, so every graph
// boundary costs ~6 us more than an iteration boundary inside a graph; after
// the device raises done, the rest of the graph runs as no-op kernels, which
// the next query on the stream waits behind.  A solve therefore launches
// graphs of KP_GRAPH_HEAD iterations first (a first solution typically comes
// within them: few trailing no-ops for stop-at-first-solution queries), then
// graphs of KP_GRAPH_ITERS (forest 100 ms queries +2 %, time to first
// solution 0.622 -> 0.610 ms over graphs of 8 only, profiles/README.md).
#ifndef KP_GRAPH_ITERS
#define KP_GRAPH_ITERS 32
#endif
#ifndef KP_GRAPH_HEAD
#define KP_GRAPH_HEAD 8
#endif
#ifndef KP_HEAD_LAUNCHES
#define KP_HEAD_LAUNCHES 4
#endif

struct KpError : std::runtime_error {
    int code;
    KpError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw KpError(KP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

thread_local std::string g_create_error;

}  // namespace

struct kp_planner {
    KpProblem P{};
    KpBuffers B{};
    kp_config_desc cfg{};
    int device = 0;
    int sms = 148;
    int grid_prop = 0, grid_sel = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t fetch_stream = nullptr;  // result fetch that need not wait for trailing no-op launches
    cudaGraphExec_t graph = nullptr;       // KP_GRAPH_ITERS iterations
    cudaGraphExec_t graph_head = nullptr;  // KP_GRAPH_HEAD iterations: a solve's first launches
    uint32_t* host_done = nullptr;  // pinned, mapped
    uint32_t solve_seq = 0;         // number of the current solve (the device writes it to host_done when done)
    std::vector<void*> allocs;
    std::string err;
    KpCtl ctl{};  // host copy after the last solve
    bool ctl_valid = false;
    bool profiling = false;
    double ktime[3] = {0, 0, 0};
    uint64_t klaunch[3] = {0, 0, 0};
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    uint64_t seed = 0;
    uint64_t kernel_launches = 0, graph_launches = 0;
    uint32_t sweep_nodes = 0;
    std::vector<float> boxes, spheres;  // host copies for start-state validation
    float* h_x0 = nullptr;              // pinned staging for the query's start state
    KpCtl* h_ctl = nullptr;             // pinned copy target for asynchronous result fetches
    size_t last_fetch_bytes = 0;

    template <class T>
    T* dalloc(size_t count) {
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
        allocs.push_back(p);
        return static_cast<T*>(p);
    }
    ~kp_planner() {
        if (stream) cudaStreamSynchronize(stream);
        if (graph) cudaGraphExecDestroy(graph);
        if (graph_head) cudaGraphExecDestroy(graph_head);
        for (auto* e : ev)
            if (e) cudaEventDestroy(e);
        for (void* p : allocs) cudaFree(p);
        if (host_done) cudaFreeHost(host_done);
        if (h_x0) cudaFreeHost(h_x0);
        if (h_ctl) cudaFreeHost(h_ctl);
        if (stream) cudaStreamDestroy(stream);
        if (fetch_stream) cudaStreamDestroy(fetch_stream);
    }
};

namespace {

// Model table (model.hpp:64-68).  Dubins6 / Quad12 shapes: SPEC.md:127-128.
void model_shape(int model, int* n, int* m, int* ws) {
    switch (model) {
        case KP_MODEL_DOUBLE_INTEGRATOR_4D: *n = 4; *m = 2; *ws = 2; break;
        case KP_MODEL_DOUBLE_INTEGRATOR_6D: *n = 6; *m = 3; *ws = 3; break;
        case KP_MODEL_DUBINS_AIRPLANE_6D: *n = 6; *m = 3; *ws = 3; break;
        case KP_MODEL_QUADCOPTER_12D: *n = 12; *m = 4; *ws = 3; break;
        default: throw KpError(KP_ERR_SCHEMA, "unknown model id " + std::to_string(model));
    }
}

// Descriptor validation + fp32 constant folding.  Returns the host-side
// obstacle arrays (boxes [6], spheres [4]) to upload.
void build_problem(const kp_problem_desc* p, const kp_config_desc* c, KpProblem& P, std::vector<float>& boxes,
                   std::vector<float>& spheres, uint64_t* n_regions_out) {
    if (!p || !c) throw KpError(KP_ERR_ARGUMENT, "null descriptor");
    int n, m, ws;
    model_shape(p->model, &n, &m, &ws);
    P.model = p->model;
    if (p->state_dim != n || p->control_dim != m)
        throw KpError(KP_ERR_SCHEMA, "state/control dimension does not match the model");
    P.n = n;
    P.m = m;
    double mass = 1.0, gravity = 9.81, Ixx = 1.0, Iyy = 1.0, Izz = 2.0;  // SPEC.md:170 defaults
    for (int i = 0; i < p->n_params; ++i) {
        const std::string k = p->param_names[i];
        const double v = p->param_values[i];
        if (k == "mass") mass = v;
        else if (k == "gravity") gravity = v;
        else if (k == "arm_length") { /* recorded only: controls are thrust + body moments */ }
        else if (k == "Ixx") Ixx = v;
        else if (k == "Iyy") Iyy = v;
        else if (k == "Izz") Izz = v;
        else throw KpError(KP_ERR_SCHEMA, "unknown model parameter \"" + k + "\"");
    }
    if (!p->x_init || !p->state_lo || !p->state_hi || !p->control_lo || !p->control_hi)
        throw KpError(KP_ERR_ARGUMENT, "null bounds / x_init");
    for (int i = 0; i < n; ++i) {
        if (!(p->state_lo[i] <= p->state_hi[i])) throw KpError(KP_ERR_SCHEMA, "state bound lo > hi");
        P.slo[i] = static_cast<float>(p->state_lo[i]);
        P.shi[i] = static_cast<float>(p->state_hi[i]);
        P.x_init[i] = static_cast<float>(p->x_init[i]);
    }
    for (int i = 0; i < m; ++i) {
        if (!(p->control_lo[i] <= p->control_hi[i])) throw KpError(KP_ERR_SCHEMA, "control bound lo > hi");
        P.clo[i] = static_cast<float>(p->control_lo[i]);
        P.cw[i] = static_cast<float>(p->control_hi[i]) - P.clo[i];
        P.clo_d[i] = p->control_lo[i];
        P.chi_d[i] = p->control_hi[i];
    }
    if (p->workspace_dim != ws) throw KpError(KP_ERR_SCHEMA, "workspace dimension does not match the model");
    P.ws_dim = ws;
    for (int i = 0; i < 3; ++i) {
        if (i < ws) {
            if (!(p->workspace_lo[i] <= p->workspace_hi[i])) throw KpError(KP_ERR_SCHEMA, "workspace lo > hi");
            if (p->workspace_lo[i] < p->state_lo[i] || p->workspace_hi[i] > p->state_hi[i])
                throw KpError(KP_ERR_SCHEMA, "workspace_bounds not contained in state_bounds (SPEC.md:196)");
            P.wlo[i] = static_cast<float>(p->workspace_lo[i]);
            P.whi[i] = static_cast<float>(p->workspace_hi[i]);
        } else {
            P.wlo[i] = -std::numeric_limits<float>::infinity();
            P.whi[i] = std::numeric_limits<float>::infinity();
        }
    }
    P.check_finite = 0;
    for (int i = 0; i < n; ++i) {
        P.blo[i] = P.slo[i];
        P.bhi[i] = P.shi[i];
        if (i < ws) {
            P.blo[i] = std::max(P.blo[i], P.wlo[i]);
            P.bhi[i] = std::min(P.bhi[i], P.whi[i]);
        }
        if (!std::isfinite(P.blo[i]) || !std::isfinite(P.bhi[i])) P.check_finite = 1;
    }
    if (p->n_obstacles < 0 || p->n_obstacles > KP_MAX_OBSTACLES)
        throw KpError(KP_ERR_SCHEMA, "obstacle count out of range");
    for (int i = 0; i < p->n_obstacles; ++i) {
        const kp_obstacle& o = p->obstacles[i];
        if (o.type == KP_OBSTACLE_BOX) {
            for (int j = 0; j < ws; ++j)
                if (!(o.a[j] <= o.b[j]))
                    throw KpError(KP_ERR_SCHEMA, "obstacle " + std::to_string(i) + ": box min > max");
            for (int j = 0; j < 3; ++j) boxes.push_back(j < ws ? static_cast<float>(o.a[j]) : -INFINITY);
            for (int j = 0; j < 3; ++j) boxes.push_back(j < ws ? static_cast<float>(o.b[j]) : INFINITY);
        } else if (o.type == KP_OBSTACLE_SPHERE) {
            if (!(o.b[0] > 0)) throw KpError(KP_ERR_SCHEMA, "obstacle " + std::to_string(i) + ": sphere radius <= 0");
            const float r = static_cast<float>(o.b[0]);
            for (int j = 0; j < 3; ++j) spheres.push_back(j < ws ? static_cast<float>(o.a[j]) : 0.0f);
            spheres.push_back(r * r);
        } else {
            throw KpError(KP_ERR_SCHEMA, "obstacle " + std::to_string(i) + ": unknown type");
        }
    }
    P.n_box = static_cast<int32_t>(boxes.size() / 6);
    P.n_sph = static_cast<int32_t>(spheres.size() / 4);
    if (p->goal_n_dims < 1 || p->goal_n_dims > KP_MAX_N) throw KpError(KP_ERR_SCHEMA, "bad goal dimensions");
    if (!(p->goal_radius > 0)) throw KpError(KP_ERR_SCHEMA, "goal radius must be > 0");
    P.goal_n = p->goal_n_dims;
    P.goal_ident = 1;
    for (int i = 0; i < p->goal_n_dims; ++i) {
        if (p->goal_dims[i] != i) P.goal_ident = 0;
        const int d = p->goal_dims[i];
        if (d < 0 || d >= n) throw KpError(KP_ERR_SCHEMA, "goal dimension out of range");
        if (!(p->goal_center[i] >= p->state_lo[d] && p->goal_center[i] <= p->state_hi[d]))
            throw KpError(KP_ERR_INVALID_PROBLEM, "goal center outside state bounds (SPEC.md:62)");
        P.goal_dims[i] = d;
        P.goal_c[i] = static_cast<float>(p->goal_center[i]);
    }
    {
        const float r = static_cast<float>(p->goal_radius);
        P.goal_r2 = r * r;
    }
    if (p->cost_kind != KP_COST_PATH_LENGTH && p->cost_kind != KP_COST_CONTROL_DURATION)
        throw KpError(KP_ERR_SCHEMA, "unknown cost metric kind");
    P.cost_kind = p->cost_kind;
    if (p->cost_position_dims < 1 || p->cost_position_dims > n) throw KpError(KP_ERR_SCHEMA, "bad cost position dims");
    if (p->cost_position_dims != ws)
        throw KpError(KP_ERR_SCHEMA, "cost position dims must equal the workspace dims on the device");
    P.cost_pos_dims = p->cost_position_dims;
    // build_grid
    if (p->grid_n_dims < 1 || p->grid_n_dims > KP_MAX_GRID) throw KpError(KP_ERR_SCHEMA, "bad decomposition dims");
    P.grid_n = p->grid_n_dims;
    long double total = 1;
    const uint64_t ceiling = p->grid_max_cells ? p->grid_max_cells : (1ull << 28);
    if (!p->grid_cells && !(p->grid_delta > 0)) throw KpError(KP_ERR_CONFIG, "decomposition needs delta > 0 or cells");
    std::vector<int64_t> cells(P.grid_n);
    for (int j = 0; j < P.grid_n; ++j) {
        const int d = p->grid_dims[j];
        if (d < 0 || d >= n) throw KpError(KP_ERR_SCHEMA, "decomposition dimension out of range");
        const double lo = p->state_lo[d], hi = p->state_hi[d];
        if (!(lo < hi)) throw KpError(KP_ERR_SCHEMA, "decomposed dim needs lo < hi");
        int64_t cnum;
        if (p->grid_cells) cnum = p->grid_cells[j];
        else cnum = std::max<int64_t>(1, static_cast<int64_t>(std::ceil((hi - lo) * std::sqrt(double(P.grid_n)) / p->grid_delta)));
        if (cnum < 1) throw KpError(KP_ERR_CONFIG, "cells_per_dim must be >= 1");
        cells[j] = cnum;
        total *= cnum;
    }
    if (total > static_cast<long double>(ceiling) || total >= 4294967295.0L)
        throw KpError(KP_ERR_GRID_TOO_FINE, "region grid would have " + std::to_string(static_cast<double>(total)) +
                                                " cells, above the ceiling " + std::to_string(ceiling));
    uint32_t stride = 1;
    P.grid_ident = 1;
    for (int j = 0; j < P.grid_n; ++j) {
        const int d = p->grid_dims[j];
        if (d != j) P.grid_ident = 0;
        P.grid_dims[j] = d;
        P.g_lo[j] = static_cast<float>(p->state_lo[d]);
        P.g_cells[j] = static_cast<int32_t>(cells[j]);
        P.g_side[j] = (static_cast<float>(p->state_hi[d]) - static_cast<float>(p->state_lo[d])) / static_cast<float>(cells[j]);
        P.g_stride[j] = stride;
        stride *= static_cast<uint32_t>(cells[j]);
    }
    P.n_regions = stride;
    *n_regions_out = stride;
    // PlannerConfig
    const double h = c->ode_step > 0 ? c->ode_step : std::min(c->t_prop / 10.0, 0.02);
    if (c->lambda < 1) throw KpError(KP_ERR_CONFIG, "lambda must be >= 1");
    if (c->i_max < 1 || c->i_max > 65534) throw KpError(KP_ERR_CONFIG, "i_max must be in [1, 65534]");
    if (c->capacity < 1 || c->capacity > (1ull << 30)) throw KpError(KP_ERR_CONFIG, "capacity must be in [1, 2^30]");
    if (!(c->t_prop > 0)) throw KpError(KP_ERR_CONFIG, "t_prop must be > 0");
    if (!(h > 0) || h > c->t_prop) throw KpError(KP_ERR_CONFIG, "need 0 < ode_step <= t_prop");
    if (!(c->collision_step > 0)) throw KpError(KP_ERR_CONFIG, "collision_step must be > 0");
    if (c->rng_kind != KP_RNG_PHILOX && c->rng_kind != KP_RNG_SPLITMIX) throw KpError(KP_ERR_CONFIG, "unknown rng kind");
    P.lambda = c->lambda;
    P.lam_shift = -1;
    for (int b = 0; b < 31; ++b)
        if (c->lambda == (1 << b)) P.lam_shift = b;
    P.i_max = c->i_max;
    P.rng_kind = c->rng_kind;
    P.deact = c->deactivate_after_expansion ? 1 : 0;
    P.capacity = static_cast<uint32_t>(c->capacity);
    // Default: lambda * capacity (|V_A| <= live nodes <= capacity, so the
    // buffer cannot overflow), capped at 2^25 slots (<= 2.7 GB for Quad12).
    uint64_t slots = c->max_slots ? c->max_slots
                                  : std::min<uint64_t>(static_cast<uint64_t>(c->lambda) * c->capacity, 1ull << 25);
    slots = (slots + 31) & ~31ull;
    if (slots > (1ull << 29)) throw KpError(KP_ERR_CONFIG, "max_slots too large (<= 2^29)");
    P.max_slots = static_cast<uint32_t>(slots);
    P.t_prop = static_cast<float>(c->t_prop);
    P.t_prop_d = c->t_prop;
    P.h = static_cast<float>(h);
    P.coll = static_cast<float>(c->collision_step);
    {  // threshold on the squared distance: the interpolation test without the sqrt latency
        float t = P.coll * P.coll;
        while (std::sqrt(t) > P.coll) t = std::nextafter(t, 0.0f);
        while (std::sqrt(std::nextafter(t, INFINITY)) <= P.coll) t = std::nextafter(t, INFINITY);
        P.coll_d2 = t;
    }
    P.zero_rate = static_cast<float>(1e-6);  // cost.hpp:30
    P.inv_m = 1.0f / static_cast<float>(mass);
    P.grav = static_cast<float>(gravity);
    const float ix = static_cast<float>(Ixx), iy = static_cast<float>(Iyy), iz = static_cast<float>(Izz);
    P.cx = (iy - iz) / ix;
    P.cy = (iz - ix) / iy;
    P.cz = (ix - iy) / iz;
    P.inv_ix = 1.0f / ix;
    P.inv_iy = 1.0f / iy;
    P.inv_iz = 1.0f / iz;
}

// is_state_valid(x_init) on the host with the same fp32 comparisons
// (x_init valid; InvalidProblemError otherwise).
bool host_state_valid(const KpProblem& P, const std::vector<float>& boxes, const std::vector<float>& spheres) {
    const float* x = P.x_init;
    for (int i = 0; i < P.n; ++i)
        if (!(x[i] >= P.slo[i] && x[i] <= P.shi[i])) return false;
    for (int i = 0; i < P.ws_dim; ++i)
        if (!(x[i] >= P.wlo[i] && x[i] <= P.whi[i])) return false;
    const float px = x[0], py = x[1], pz = P.ws_dim == 3 ? x[2] : 0.0f;
    for (size_t b = 0; b + 6 <= boxes.size(); b += 6)
        if (px >= boxes[b] && px <= boxes[b + 3] && py >= boxes[b + 1] && py <= boxes[b + 4] && pz >= boxes[b + 2] &&
            pz <= boxes[b + 5])
            return false;
    for (size_t s = 0; s + 4 <= spheres.size(); s += 4) {
        const float dx = px - spheres[s], dy = py - spheres[s + 1], dz = pz - spheres[s + 2];
        float d2 = dx * dx;
        d2 = std::fma(dy, dy, d2);
        d2 = std::fma(dz, dz, d2);
        if (d2 <= spheres[s + 3]) return false;
    }
    return true;
}

// Environment blob: obstacles as float4 + an exact broad-phase cell grid over
// the workspace.  Cells per dim ~ 2 x workspace extent / median obstacle extent
// (<= 64), shrunk until <= 16384 cells and < 32768 list entries; every
// obstacle is listed in every cell its AABB (expanded by a margin of 1e-3
// cell, far above the fp32 error of the device's cell computation) touches.
std::vector<uint8_t> build_env(KpProblem& P, const std::vector<float>& boxes, const std::vector<float>& spheres) {
    const int nb = P.n_box, ns = P.n_sph, no = nb + ns;
    std::vector<std::array<double, 6>> aabb(no);
    for (int i = 0; i < nb; ++i)
        for (int d = 0; d < 3; ++d) {
            aabb[i][d] = boxes[6 * i + d];
            aabb[i][3 + d] = boxes[6 * i + 3 + d];
        }
    for (int i = 0; i < ns; ++i) {
        const double r = std::sqrt(static_cast<double>(spheres[4 * i + 3]));
        for (int d = 0; d < 3; ++d) {
            aabb[nb + i][d] = spheres[4 * i + d] - r;
            aabb[nb + i][3 + d] = spheres[4 * i + d] + r;
        }
    }
    int n[3] = {1, 1, 1};
    double lo[3] = {0, 0, 0}, cell[3] = {1, 1, 1};
    for (int d = 0; d < P.ws_dim; ++d) {
        lo[d] = P.wlo[d];
        const double ext = static_cast<double>(P.whi[d]) - lo[d];
        std::vector<double> sz;
        for (int i = 0; i < no; ++i) sz.push_back(std::min(ext, std::max(1e-9, aabb[i][3 + d] - aabb[i][d])));
        double med = ext;
        if (!sz.empty()) {
            std::nth_element(sz.begin(), sz.begin() + sz.size() / 2, sz.end());
            med = sz[sz.size() / 2];
        }
        // cells about half the median obstacle extent: most cells list 0-1 candidates,
        // which keeps the lanes of a warp on the same narrow-phase trip count
        n[d] = std::max(1, std::min(64, static_cast<int>(std::lround(2.0 * ext / med))));
        if (no == 0 || !(ext > 0)) n[d] = 1;
    }
    std::vector<std::vector<uint16_t>> lists;
    for (;;) {
        const int nc = n[0] * n[1] * n[2];
        lists.assign(nc, {});
        size_t entries = 0;
        for (int d = 0; d < 3; ++d) cell[d] = d < P.ws_dim ? (static_cast<double>(P.whi[d]) - lo[d]) / n[d] : 1.0;
        for (int i = 0; i < no; ++i) {
            int r0[3], r1[3];
            for (int d = 0; d < 3; ++d) {
                if (d >= P.ws_dim) { r0[d] = 0; r1[d] = 0; continue; }
                const double m = 1e-3 * cell[d];
                const double a = std::isfinite(aabb[i][d]) ? (aabb[i][d] - m - lo[d]) / cell[d] : -1.0;
                const double b = std::isfinite(aabb[i][3 + d]) ? (aabb[i][3 + d] + m - lo[d]) / cell[d] : n[d];
                r0[d] = std::max(0, std::min(n[d] - 1, static_cast<int>(std::floor(a))));
                r1[d] = std::max(0, std::min(n[d] - 1, static_cast<int>(std::floor(b))));
            }
            for (int z = r0[2]; z <= r1[2]; ++z)
                for (int y = r0[1]; y <= r1[1]; ++y)
                    for (int x = r0[0]; x <= r1[0]; ++x) {
                        lists[x + n[0] * (y + n[1] * z)].push_back(static_cast<uint16_t>(i));
                        ++entries;
                    }
        }
        if ((nc <= 16384 && entries < 32768) || nc == 1) {
            if (entries >= 65535) throw KpError(KP_ERR_SCHEMA, "too many obstacle cell entries");
            break;
        }
        int dm = 0;
        for (int d = 1; d < 3; ++d)
            if (n[d] > n[dm]) dm = d;
        n[dm] = std::max(1, n[dm] / 2);
    }
    const int nc = n[0] * n[1] * n[2];
    for (int d = 0; d < 3; ++d) {
        const bool divided = d < P.ws_dim && n[d] > 1;
        P.bg_n[d] = n[d];
        P.bg_max[d] = n[d] - 1;
        P.bg_lo[d] = d < P.ws_dim ? static_cast<float>(lo[d]) : 0.0f;
        P.bg_inv[d] = divided ? static_cast<float>(1.0 / cell[d]) : 0.0f;
        P.bg_off[d] = divided ? static_cast<float>(-lo[d] / cell[d]) : 0.0f;
    }
    std::vector<uint32_t> range(nc, 0);
    std::vector<uint16_t> ids;
    for (int c = 0; c < nc; ++c) {
        const uint32_t b = static_cast<uint32_t>(ids.size());
        ids.insert(ids.end(), lists[c].begin(), lists[c].end());
        range[c] = b | (static_cast<uint32_t>(ids.size()) << 16);
    }
    P.n_cells = nc;
    P.n_entries = static_cast<int32_t>(ids.size());
    auto pad16 = [](size_t x) { return (x + 15) & ~size_t(15); };
    const size_t obj_bytes = 16 * static_cast<size_t>(2 * nb + ns);
    P.off_cells = static_cast<uint32_t>(obj_bytes);
    P.off_cids = static_cast<uint32_t>(pad16(obj_bytes + 4 * range.size()));
    P.env_bytes = static_cast<uint32_t>(pad16(P.off_cids + 2 * std::max<size_t>(ids.size(), 1)));
    if (P.env_bytes > 200 * 1024) throw KpError(KP_ERR_SCHEMA, "environment does not fit in shared memory");
    std::vector<uint8_t> blob(P.env_bytes, 0);
    float* f = reinterpret_cast<float*>(blob.data());
    for (int i = 0; i < nb; ++i) {
        for (int d = 0; d < 3; ++d) {
            f[4 * i + d] = boxes[6 * i + d];
            f[4 * (nb + i) + d] = boxes[6 * i + 3 + d];
        }
    }
    for (int i = 0; i < ns; ++i)
        for (int d = 0; d < 4; ++d) f[4 * (2 * nb + i) + d] = spheres[4 * i + d];
    std::memcpy(blob.data() + P.off_cells, range.data(), 4 * range.size());
    if (!ids.empty()) std::memcpy(blob.data() + P.off_cids, ids.data(), 2 * ids.size());
    return blob;
}

void capture_graph(kp_planner* pl) {
    for (int which = 0; which < 2; ++which) {
        const int iters = which ? KP_GRAPH_HEAD : KP_GRAPH_ITERS;
        cudaGraph_t g = nullptr;
        cuda_check(cudaStreamBeginCapture(pl->stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
        for (int i = 0; i < iters; ++i) kp::launch_iteration(pl->P, pl->B, pl->grid_prop, pl->grid_sel, pl->stream, 7);
        cuda_check(cudaStreamEndCapture(pl->stream, &g), "cudaStreamEndCapture");
        cuda_check(cudaGraphInstantiate(which ? &pl->graph_head : &pl->graph, g, 0), "cudaGraphInstantiate");
        cudaGraphDestroy(g);
    }
}

// Launch the solve's n-th graph (head graphs first); returns its iterations.
int launch_graph(kp_planner* pl, int n) {
    const bool head = n < KP_HEAD_LAUNCHES;
    cuda_check(cudaGraphLaunch(head ? pl->graph_head : pl->graph, pl->stream), "cudaGraphLaunch");
    pl->graph_launches += 1;
    const int iters = head ? KP_GRAPH_HEAD : KP_GRAPH_ITERS;
    pl->kernel_launches += 3 * iters;
    return iters;
}

void reset_async(kp_planner* pl, uint64_t seed) {
    pl->seed = seed;
    pl->sweep_nodes = 0;
    cuda_check(cudaMemcpyAsync(pl->B.x0, pl->h_x0, sizeof(float) * KP_MAX_N, cudaMemcpyHostToDevice, pl->stream),
               "x0 H2D");
    cuda_check(kp::launch_reset(pl->P, pl->B, seed, pl->stream), "reset");
    pl->kernel_launches += 2;
    pl->ctl_valid = false;
}

void do_reset(kp_planner* pl, uint64_t seed) {
    reset_async(pl, seed);
    cuda_check(cudaStreamSynchronize(pl->stream), "reset sync");
}

// Checks build (-DKP_CHECKS): raise on the first failed device invariant.
void check_invariants() {
    unsigned int code = 0;
    cuda_check(kp::read_check_code(&code), "read check code");
    if (code) throw KpError(KP_ERR_CUDA, "device invariant check " + std::to_string(code) + " failed");
}

// Result block D2H.  Default: ordered after everything queued on the
// planner's stream.  after_done: the device has raised the done word, so the
// control block is final (the boundary fences it before the mapped write) and
// the trailing no-op launches of the graphs in flight never write it: read it
// on a side stream instead of waiting for them.  Only the header and the
// timeline entries in use are copied (pinned staging).
void fetch_ctl(kp_planner* pl, bool after_done = false) {
    constexpr size_t head = offsetof(KpCtl, timeline);
    constexpr size_t win = 256;  // timeline entries in the first copy
    cudaStream_t st = after_done ? pl->fetch_stream : pl->stream;
    cuda_check(cudaMemcpyAsync(pl->h_ctl, pl->B.ctl, head + win * sizeof(KpTimeline), cudaMemcpyDeviceToHost, st),
               "ctl D2H");
    cuda_check(cudaStreamSynchronize(st), "ctl sync");
    const size_t len = std::min<size_t>(pl->h_ctl->timeline_len, KP_TIMELINE_CAP);
    if (len > win) {
        cuda_check(cudaMemcpyAsync(pl->h_ctl->timeline + win, pl->B.ctl->timeline + win,
                                   (len - win) * sizeof(KpTimeline), cudaMemcpyDeviceToHost, st),
                   "ctl timeline D2H");
        cuda_check(cudaStreamSynchronize(st), "ctl timeline sync");
    }
    std::memcpy(&pl->ctl, pl->h_ctl, head + std::max(len, win) * sizeof(KpTimeline));
    // the last boundary's best-solution bookkeeping, which the device does in
    // the next propagate (none runs after the solve stopped): the same entry
    goal_bookkeeping(pl->ctl);
    pl->last_fetch_bytes = head + std::max(len, win) * sizeof(KpTimeline);
    pl->ctl_valid = true;
    check_invariants();
}

double bits_to_cost(uint64_t best) {
    if (best == ~0ull) return std::numeric_limits<double>::infinity();
    const uint32_t b = static_cast<uint32_t>(best >> 32);
    float f;
    std::memcpy(&f, &b, 4);
    return f;
}

void fill_result(const kp_planner* pl, kp_result* r) {
    const KpCtl& c = pl->ctl;
    std::memset(r, 0, sizeof *r);
    r->found = c.best != ~0ull;
    r->capacity_exhausted = c.capacity_exhausted != 0;
    r->best_cost = bits_to_cost(c.best);
    r->best_leaf = r->found ? static_cast<int64_t>(c.best & 0xFFFFFFFFull) : -1;
    r->best_found_at_s = r->found ? c.best_ns * 1e-9 : 0.0;
    r->best_found_iteration = c.best_iter;
    r->first_solution_s = r->found ? c.first_ns * 1e-9 : -1.0;
    r->first_solution_cost = c.timeline_len ? bits_to_cost(c.timeline[0].best) : std::numeric_limits<double>::infinity();
    r->first_solution_iteration = c.first_iter;
    r->elapsed_s = c.t_last_ns > c.t_start_ns ? (c.t_last_ns - c.t_start_ns) * 1e-9 : 0.0;
    r->iterations = c.iter;
    r->propagations_attempted = c.stats.attempted;
    r->propagations_valid = c.stats.valid;
    r->propagations_admitted = c.stats.admitted;
    r->nodes_committed = c.stats.committed;
    r->nodes_pruned_terminal = c.stats.pruned_terminal;
    r->nodes_deactivated = c.stats.deactivated;
    r->nodes_reactivated = c.stats.reactivated;
    r->candidates_dropped_capacity = c.stats.dropped_capacity;
    r->node_count = c.n_nodes;
    r->timeline_len = c.timeline_len;
}

template <class F>
int guard(kp_planner* pl, F&& f) {
    try {
        f();
        return KP_OK;
    } catch (const KpError& e) {
        if (pl) pl->err = e.what();
        else g_create_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        if (pl) pl->err = e.what();
        else g_create_error = e.what();
        return KP_ERR_ARGUMENT;
    }
}

template <class T>
struct DevBuf {  // scratch device buffer for debug / extraction calls
    T* p = nullptr;
    explicit DevBuf(size_t n) { cuda_check(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc scratch"); }
    ~DevBuf() { if (p) cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

uint32_t chain_of(kp_planner* pl, int64_t leaf, DevBuf<int32_t>*& out_chain, std::vector<int32_t>& host_chain) {
    fetch_ctl(pl);
    if (leaf < 0) {
        if (pl->ctl.best == ~0ull) throw KpError(KP_ERR_ARGUMENT, "no solution: best leaf is undefined");
        leaf = static_cast<int64_t>(pl->ctl.best & 0xFFFFFFFFull);
    }
    if (leaf >= static_cast<int64_t>(pl->ctl.n_nodes)) throw KpError(KP_ERR_ARGUMENT, "leaf id out of range");
    DevBuf<uint32_t> dlen(1);
    // depth <= node count; size the chain buffer by a first pass
    cuda_check(kp::launch_chain(pl->B, static_cast<int32_t>(leaf), nullptr, 0, dlen.p, pl->stream), "chain");
    uint32_t len = 0;
    cuda_check(cudaMemcpyAsync(&len, dlen.p, 4, cudaMemcpyDeviceToHost, pl->stream), "chain len");
    cuda_check(cudaStreamSynchronize(pl->stream), "chain sync");
    out_chain = new DevBuf<int32_t>(len);
    cuda_check(kp::launch_chain(pl->B, static_cast<int32_t>(leaf), out_chain->p, len, dlen.p, pl->stream), "chain");
    host_chain.resize(len);
    cuda_check(cudaMemcpyAsync(host_chain.data(), out_chain->p, len * 4, cudaMemcpyDeviceToHost, pl->stream), "chain D2H");
    cuda_check(cudaStreamSynchronize(pl->stream), "chain sync");
    return len;
}

}  // namespace

extern "C" {

int kp_abi_version(void) { return KP_ABI_VERSION; }

const char* kp_last_error(const kp_planner* pl) { return pl ? pl->err.c_str() : g_create_error.c_str(); }

int kp_create(const kp_problem_desc* problem, const kp_config_desc* config, int device, kp_planner** out) {
    if (!out) return KP_ERR_ARGUMENT;
    *out = nullptr;
    kp_planner* pl = new kp_planner();
    const int rc = guard(nullptr, [&] {
        std::vector<float> boxes, spheres;
        uint64_t n_regions = 0;
        build_problem(problem, config, pl->P, boxes, spheres, &n_regions);
        if (!host_state_valid(pl->P, boxes, spheres))
            throw KpError(KP_ERR_INVALID_PROBLEM, "x_init is not a valid state (SPEC.md:61, :374)");
        pl->cfg = *config;
        int ndev = 0;
        cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (device < 0 || device >= ndev) throw KpError(KP_ERR_CUDA, "no such CUDA device " + std::to_string(device));
        pl->device = device;
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp prop;
        cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major < 10) throw KpError(KP_ERR_CUDA, "device is not sm_100 class (built for sm_100a only)");
        pl->sms = prop.multiProcessorCount;
        cuda_check(cudaStreamCreateWithFlags(&pl->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        cuda_check(cudaStreamCreateWithFlags(&pl->fetch_stream, cudaStreamNonBlocking), "cudaStreamCreate");
        void* hd = nullptr;
        cuda_check(cudaHostAlloc(&hd, 64, cudaHostAllocMapped), "cudaHostAlloc");
        pl->host_done = static_cast<uint32_t*>(hd);
        *pl->host_done = 0;
        void* dd = nullptr;
        cuda_check(cudaHostGetDevicePointer(&dd, hd, 0), "cudaHostGetDevicePointer");
        KpBuffers& B = pl->B;
        const KpProblem& P = pl->P;
        const size_t cap = P.capacity, S = P.max_slots;
        B.host_done = static_cast<volatile uint32_t*>(dd);
        B.state = pl->dalloc<float>(cap * P.n);
        B.ctrl = pl->dalloc<float>(cap * P.m);
        B.dt = pl->dalloc<float>(cap);
        B.acc = pl->dalloc<uint32_t>(cap);
        B.parent = pl->dalloc<int32_t>(cap);
        B.region = pl->dalloc<uint32_t>(cap);
        B.status = pl->dalloc<uint8_t>(cap);
        B.live_st = pl->dalloc<uint32_t>(cap);
        B.icnt = pl->dalloc<uint16_t>(cap);
        B.link = pl->dalloc<uint4>(cap);
        B.rc = pl->dalloc<uint32_t>(n_regions);
        for (int i = 0; i < 2; ++i) {
            B.live[i] = pl->dalloc<uint4>(cap);
            B.live_si[i] = pl->dalloc<uint32_t>(cap);
            B.va[i] = pl->dalloc<uint32_t>(cap);
        }
        B.vu_state = pl->dalloc<float>(S * P.n);
        B.vu_ctrl = pl->dalloc<float>(S * P.m);
        B.vu_dt = pl->dalloc<float>(S);
        B.vu_acc = pl->dalloc<uint32_t>(S);
        B.vu_region = pl->dalloc<uint32_t>(S);
        B.admit_mask = pl->dalloc<uint32_t>(S / 32);
        B.goal_mask = pl->dalloc<uint32_t>(S / 32);
        B.commit_mask = pl->dalloc<uint32_t>(S / 32);
        const uint64_t max_e = ((cap + 31) & ~31ull) + S;
        B.max_tiles = static_cast<uint32_t>((max_e + KP_SELECT_THREADS - 1) / KP_SELECT_THREADS);
        B.tile_sums = pl->dalloc<uint32_t>(3ull * B.max_tiles);
        const std::vector<uint8_t> blob = build_env(pl->P, boxes, spheres);
        float4* denv = pl->dalloc<float4>(blob.size() / 16);
        cuda_check(cudaMemcpy(denv, blob.data(), blob.size(), cudaMemcpyHostToDevice), "env H2D");
        B.env = denv;
        B.ctl = pl->dalloc<KpCtl>(1);
        B.x0 = pl->dalloc<float>(KP_MAX_N);
        B.trace = pl->dalloc<KpTraceRec>(KP_TRACE_CAP);
        void* hx = nullptr;
        cuda_check(cudaHostAlloc(&hx, sizeof(float) * KP_MAX_N, cudaHostAllocDefault), "cudaHostAlloc x0");
        pl->h_x0 = static_cast<float*>(hx);
        for (int i = 0; i < KP_MAX_N; ++i) pl->h_x0[i] = i < P.n ? P.x_init[i] : 0.0f;
        pl->boxes = boxes;
        pl->spheres = spheres;
        void* hc = nullptr;
        cuda_check(cudaHostAlloc(&hc, sizeof(KpCtl), cudaHostAllocDefault), "cudaHostAlloc ctl");
        pl->h_ctl = static_cast<KpCtl*>(hc);
        pl->P.sel_spec = 1;
        if (const char* v = std::getenv("KP_SEL_SPEC")) pl->P.sel_spec = std::atoi(v) ? 1 : 0;  // A/B hook
        kp::plan_propagate_smem(pl->P);
        cuda_check(kp::set_propagate_smem(P), "smem attribute");
        const int occ = std::max(1, kp::propagate_occupancy(P));
        if (std::getenv("KP_VERBOSE"))
            std::fprintf(stderr, "k_propagate: %u B shared (environment %u B, sample-parallel %d: %u items), %d blocks/SM\n",
                         P.prop_smem, P.env_bytes, P.flat_on, P.flat_nb, occ);
        // test hook: KP_PROP_GRID caps the propagate grid, so the multi-group
        // paths (several groups per warp, split rollouts) run at small item counts
        pl->grid_prop = pl->sms * occ;
        if (const char* g = std::getenv("KP_PROP_GRID")) pl->grid_prop = std::max(1, std::min(pl->grid_prop, std::atoi(g)));
        // 8 select blocks per SM: the steady state needs far fewer (its tiles
        // fit in ~one block per SM), but the growth-phase iterations around the
        // first solution have thousands of tiles (forest TTFS 0.530 -> 0.510 ms
        // against 4 per SM, throughput unchanged)
        pl->grid_sel = pl->sms * (2048 / KP_SELECT_THREADS);
        if (const char* g = std::getenv("KP_SEL_GRID")) pl->grid_sel = std::max(1, std::atoi(g));  // A/B hook
        kp::set_flat_limit(pl->P, pl->grid_prop);
        B.prop_scratch = pl->dalloc<float>(static_cast<size_t>(pl->grid_prop) * (P.n + 1) * 1024);

        for (auto*& e : pl->ev) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
        do_reset(pl, config->seed);
        capture_graph(pl);
    });
    if (rc != KP_OK) {
        delete pl;
        return rc;
    }
    *out = pl;
    return KP_OK;
}

void kp_destroy(kp_planner* pl) { delete pl; }

int kp_reset(kp_planner* pl, uint64_t seed) {
    if (!pl) return KP_ERR_ARGUMENT;
    return guard(pl, [&] {
        cuda_check(cudaSetDevice(pl->device), "cudaSetDevice");
        do_reset(pl, seed);
    });
}

int kp_reset_query(kp_planner* pl, uint64_t seed, const double* x_init) {
    if (!pl) return KP_ERR_ARGUMENT;
    return guard(pl, [&] {
        cuda_check(cudaSetDevice(pl->device), "cudaSetDevice");
        if (x_init) {
            KpProblem q = pl->P;
            for (int i = 0; i < pl->P.n; ++i) q.x_init[i] = static_cast<float>(x_init[i]);
            if (!host_state_valid(q, pl->boxes, pl->spheres))
                throw KpError(KP_ERR_INVALID_PROBLEM, "x_init is not a valid state (SPEC.md:61, :374)");
            for (int i = 0; i < pl->P.n; ++i) pl->h_x0[i] = q.x_init[i];
            pl->P.x_init[0] = pl->P.x_init[0];  // P itself is unchanged (captured graph args)
        }
        do_reset(pl, seed);
    });
}

int kp_set_stop_at_first_solution(kp_planner* pl, int enabled) {
    if (!pl) return KP_ERR_ARGUMENT;
    pl->cfg.stop_at_first_solution = enabled ? 1 : 0;
    return KP_OK;
}

int kp_set_profiling(kp_planner* pl, int enabled) {
    if (!pl) return KP_ERR_ARGUMENT;
    pl->profiling = enabled != 0;
    return KP_OK;
}

int kp_get_profile(kp_planner* pl, kp_profile* out) {
    if (!pl || !out) return KP_ERR_ARGUMENT;
    return guard(pl, [&] {
        fetch_ctl(pl);
        const KpStats& st = pl->ctl.stats;
        std::memset(out, 0, sizeof *out);
        out->kernel_launches = pl->kernel_launches;
        out->graph_launches = pl->graph_launches;
        out->t_propagate_s = pl->ktime[0];
        out->t_select_s = pl->ktime[1];
        out->t_scatter_s = pl->ktime[2];
        out->n_propagate = pl->klaunch[0];
        out->n_select = pl->klaunch[1];
        out->n_scatter = pl->klaunch[2];
        out->items = st.attempted;
        out->rk4_steps = st.rk4_steps;
        out->samples_checked = st.rk4_steps;  // every executed step's sample is validity-checked
        out->interp_points = st.interp_points;
        out->box_tests = st.box_tests;
        out->sphere_tests = st.sphere_tests;
        out->live_scanned = st.live_scanned;
        out->ancestor_hops = st.ancestor_hops;
        out->slots_scanned = st.slots_scanned;
        out->admitted_checked = st.admitted_checked;
    });
}

int kp_get_trace(kp_planner* pl, kp_trace_entry* buf, size_t cap, size_t* len) {
    if (!pl || !len) return KP_ERR_ARGUMENT;
    return guard(pl, [&] {
        fetch_ctl(pl);
        const uint32_t n = std::min<uint32_t>(pl->ctl.iter, KP_TRACE_CAP);
        *len = n;
        if (!buf || cap == 0) return;
        std::vector<KpTraceRec> all(KP_TRACE_CAP);
        cuda_check(cudaMemcpyAsync(all.data(), pl->B.trace, sizeof(KpTraceRec) * KP_TRACE_CAP, cudaMemcpyDeviceToHost,
                                   pl->stream), "trace D2H");
        cuda_check(cudaStreamSynchronize(pl->stream), "trace sync");
        const uint32_t first = pl->ctl.iter - n;  // oldest kept iteration index
        for (uint32_t k = 0; k < std::min<size_t>(cap, n); ++k) {
            const KpTraceRec& r = all[(first + k) % KP_TRACE_CAP];
            buf[k] = {r.t_ns, r.iteration, r.items, r.live, r.frontier, r.nodes, r.committed,
                      r.t_prop, r.t_sel, r.t_sel_end, r.t_scat};
        }
    });
}

int kp_get_stream(kp_planner* pl, void** stream) {
    if (!pl || !stream) return KP_ERR_ARGUMENT;
    *stream = static_cast<void*>(pl->stream);
    return KP_OK;
}

int kp_debug_stamps(kp_planner* pl, uint64_t* out) {
    if (!pl || !out) return KP_ERR_ARGUMENT;
    return guard(pl, [&] {
        cuda_check(cudaSetDevice(pl->device), "cudaSetDevice");
        cuda_check(cudaStreamSynchronize(pl->stream), "sync");
        const cudaError_t e = kp::read_stamps(reinterpret_cast<unsigned long long*>(out));
        if (e == cudaErrorNotSupported) throw KpError(KP_ERR_CONFIG, "library built without -DKP_STAMPS");
        cuda_check(e, "read stamps");
    });
}

int kp_solve(kp_planner* pl, double budget_s, uint64_t max_iterations, kp_result* out) {
    if (!pl || !out) return KP_ERR_ARGUMENT;
    return guard(pl, [&] {
        cuda_check(cudaSetDevice(pl->device), "cudaSetDevice");
        const double budget = budget_s >= 0 ? budget_s : pl->cfg.t_max_s;
        const uint64_t mi = max_iterations ? max_iterations : pl->cfg.max_iterations;
        const bool stop_first = pl->cfg.stop_at_first_solution != 0;
        if (!(budget > 0) && mi == 0 && !stop_first)
            throw KpError(KP_ERR_CONFIG, "solve needs a time budget, an iteration budget or stop_at_first_solution");
        if (mi > 0xFFFFFFF0ull) throw KpError(KP_ERR_CONFIG, "max_iterations too large");
        const unsigned long long budget_ns = budget > 0 ? static_cast<unsigned long long>(budget * 1e9) : 0ull;
        *pl->host_done = 0;
        if (++pl->solve_seq == 0) pl->solve_seq = 1;
        const uint32_t seq = pl->solve_seq;
        cuda_check(kp::launch_start(pl->B, budget_ns, static_cast<uint32_t>(mi), stop_first ? 1u : 0u, seq,
                                    pl->stream),
                   "start");
        pl->kernel_launches += 1;
        // host watchdog: the device stops itself at the budget; this only
        // guards against a hang (budget + 60 s, or 600 s for iteration-only runs).
        const double watchdog = (budget > 0 ? budget : 540.0) + 60.0;
        const auto t0 = std::chrono::steady_clock::now();
        auto wall = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
        volatile uint32_t* done = pl->host_done;
        if (pl->profiling) {
            // per-kernel CUDA-event timing, one iteration at a time
            while (*done != seq) {
                for (int k = 0; k < 3; ++k) {
                    cuda_check(cudaEventRecord(pl->ev[0], pl->stream), "event");
                    cuda_check(kp::launch_iteration(pl->P, pl->B, pl->grid_prop, pl->grid_sel, pl->stream, 1 << k), "iter");
                    pl->kernel_launches += 1;
                    cuda_check(cudaEventRecord(pl->ev[1], pl->stream), "event");
                    cuda_check(cudaEventSynchronize(pl->ev[1]), "event sync");
                    float ms = 0;
                    cuda_check(cudaEventElapsedTime(&ms, pl->ev[0], pl->ev[1]), "elapsed");
                    pl->ktime[k] += ms * 1e-3;
                    pl->klaunch[k] += 1;
                }
                if (wall() > watchdog) throw KpError(KP_ERR_CUDA, "solve watchdog expired (device did not finish)");
            }
        } else {
            // keep at most two graphs in flight; stop as soon as the device
            // raises the mapped done word
            cudaEvent_t inflight[2] = {pl->ev[2], pl->ev[3]};
            int n_launched = 0;
            while (*done != seq) {
                if (n_launched >= 2) {
                    cudaEvent_t e = inflight[n_launched & 1];  // recorded two launches ago
                    for (;;) {
                        if (*done == seq) break;
                        const cudaError_t q = cudaEventQuery(e);
                        if (q == cudaSuccess) break;
                        if (q != cudaErrorNotReady) cuda_check(q, "graph execution");
                        if (wall() > watchdog) throw KpError(KP_ERR_CUDA, "solve watchdog expired");
                    }
                    if (*done == seq) break;
                }
                launch_graph(pl, n_launched);
                cuda_check(cudaEventRecord(inflight[n_launched & 1], pl->stream), "event");
                ++n_launched;
            }
        }
        fetch_ctl(pl, /*after_done=*/!pl->profiling);
        if (pl->ctl.error == 8)
            throw KpError(KP_ERR_SLOT_OVERFLOW, "lambda*|V_A| exceeded max_slots; raise kp_config_desc.max_slots");
        fill_result(pl, out);
    });
}

int kp_sweep_setup(kp_planner* pl, uint64_t n_nodes, uint64_t seed) {
    if (!pl) return KP_ERR_ARGUMENT;
    return guard(pl, [&] {
        const KpProblem& P = pl->P;
        if (n_nodes < 1 || n_nodes > P.capacity) throw KpError(KP_ERR_CONFIG, "sweep: n_nodes must be in [1, capacity]");
        if (n_nodes * static_cast<uint64_t>(P.lambda) > P.max_slots)
            throw KpError(KP_ERR_CONFIG, "sweep: n_nodes * lambda exceeds max_slots");
        cuda_check(cudaSetDevice(pl->device), "cudaSetDevice");
        // synthetic frontier: uniform in the (folded) bounds, rejection against the environment
        uint64_t st = seed ? seed : 0x9E3779B97F4A7C15ULL;
        auto next = [&] {
            st += 0x9E3779B97F4A7C15ULL;
            uint64_t z = st;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
            return z ^ (z >> 31);
        };
        std::vector<float> soa(static_cast<size_t>(P.n) * n_nodes);
        KpProblem q = P;
        for (uint64_t i = 0; i < n_nodes; ++i) {
            for (int tries = 0;; ++tries) {
                for (int d = 0; d < P.n; ++d) {  // positions uniform in free space, the rest as x_init (hover-ish)
                    if (d >= P.ws_dim) { q.x_init[d] = P.x_init[d]; continue; }
                    const double u = static_cast<double>(next() >> 11) * 0x1.0p-53;
                    const float lo = P.blo[d], hi = P.bhi[d];
                    q.x_init[d] = lo + static_cast<float>(u) * (hi - lo);
                }
                if (host_state_valid(q, pl->boxes, pl->spheres)) break;
                if (tries > 100000) throw KpError(KP_ERR_INVALID_PROBLEM, "sweep: could not sample valid states");
            }
            for (int d = 0; d < P.n; ++d) soa[static_cast<size_t>(d) * n_nodes + i] = q.x_init[d];
        }
        for (int d = 0; d < P.n; ++d)
            cuda_check(cudaMemcpyAsync(pl->B.state + static_cast<size_t>(d) * P.capacity, soa.data() + d * n_nodes,
                                       n_nodes * 4, cudaMemcpyHostToDevice, pl->stream), "sweep H2D");
        cuda_check(cudaMemsetAsync(pl->B.acc, 0, n_nodes * 4, pl->stream), "sweep acc");
        pl->sweep_nodes = static_cast<uint32_t>(n_nodes);
        cuda_check(cudaStreamSynchronize(pl->stream), "sweep sync");
        pl->ctl_valid = false;
    });
}

int kp_sweep_run(kp_planner* pl, uint32_t launches, double* ms_per_launch, kp_profile* one) {
    if (!pl || !ms_per_launch) return KP_ERR_ARGUMENT;
    return guard(pl, [&] {
        if (!pl->sweep_nodes) throw KpError(KP_ERR_CONFIG, "sweep: call kp_sweep_setup first");
        cuda_check(cudaSetDevice(pl->device), "cudaSetDevice");
        double total = 0;
        for (uint32_t k = 0; k < std::max(1u, launches); ++k) {
            cuda_check(kp::launch_sweep_prepare(pl->P, pl->B, pl->sweep_nodes, pl->stream), "sweep prepare");
            cuda_check(cudaEventRecord(pl->ev[0], pl->stream), "event");
            cuda_check(kp::launch_iteration(pl->P, pl->B, pl->grid_prop, pl->grid_sel, pl->stream, 1), "sweep launch");
            cuda_check(cudaEventRecord(pl->ev[1], pl->stream), "event");
            cuda_check(cudaEventSynchronize(pl->ev[1]), "event sync");
            float ms = 0;
            cuda_check(cudaEventElapsedTime(&ms, pl->ev[0], pl->ev[1]), "elapsed");
            total += ms;
            pl->kernel_launches += 2;
        }
        *ms_per_launch = total / std::max(1u, launches);
        if (one) {
            fetch_ctl(pl);
            const KpStats& st = pl->ctl.stats;
            std::memset(one, 0, sizeof *one);
            one->items = pl->ctl.n_items;
            one->rk4_steps = st.rk4_steps;
            one->samples_checked = st.rk4_steps;
            one->interp_points = st.interp_points;
            one->box_tests = st.box_tests;
            one->sphere_tests = st.sphere_tests;
            one->n_propagate = 1;
            one->t_propagate_s = *ms_per_launch * 1e-3;
        }
    });
}

int kp_solve_batch(kp_planner* pl, const uint64_t* seeds, size_t k, double budget_s, uint64_t max_iterations,
                   kp_result* results) {
    if (!pl || (!seeds && k) || (!results && k)) return KP_ERR_ARGUMENT;
    for (size_t i = 0; i < k; ++i) {
        int rc = kp_reset(pl, seeds[i]);
        if (rc) return rc;
        rc = kp_solve(pl, budget_s, max_iterations, &results[i]);
        if (rc) return rc;
    }
    return KP_OK;
}

}  // extern "C"

struct kp_batch {
    std::vector<kp_planner*> lanes;
    std::string err;
    ~kp_batch() {
        for (auto* l : lanes) delete l;
    }
};

extern "C" {

int kp_batch_create(const kp_problem_desc* problem, const kp_config_desc* config, int device, int lanes,
                    kp_batch** out) {
    if (!out || lanes < 1 || lanes > 256) return KP_ERR_ARGUMENT;
    *out = nullptr;
    auto* b = new kp_batch();
    for (int i = 0; i < lanes; ++i) {
        kp_planner* pl = nullptr;
        const int rc = kp_create(problem, config, device, &pl);
        if (rc != KP_OK) {
            delete b;
            return rc;  // message in kp_last_error(NULL)
        }
        b->lanes.push_back(pl);
    }
    // Concurrent lanes share the GPU: beyond 4 lanes each lane's kernels get a
    // proportionally smaller grid (at least half a block per SM), so the lanes'
    // blocks interleave instead of every lane spreading one iteration over the
    // whole device (8 lanes: 5.7 -> 7.3 G propagations/s aggregate).
    if (lanes > 4) {
        try {
            for (kp_planner* pl : b->lanes) {
                cuda_check(cudaSetDevice(pl->device), "cudaSetDevice");
                pl->grid_prop = std::max(std::max(1, pl->sms / 2), pl->grid_prop * 4 / lanes);
                pl->grid_sel = std::max(std::max(1, pl->sms / 2), pl->sms * (1024 / KP_SELECT_THREADS) * 4 / lanes);
                kp::set_flat_limit(pl->P, pl->grid_prop);
                pl->P.sel_spec = 0;  // throughput-bound: the speculative loads cost more than they hide
                if (pl->graph) cudaGraphExecDestroy(pl->graph);
                if (pl->graph_head) cudaGraphExecDestroy(pl->graph_head);
                pl->graph = nullptr;
                pl->graph_head = nullptr;
                capture_graph(pl);
            }
        } catch (const KpError& e) {
            g_create_error = e.what();
            delete b;
            return e.code;
        }
    }
    *out = b;
    return KP_OK;
}

void kp_batch_destroy(kp_batch* b) { delete b; }

const char* kp_batch_last_error(const kp_batch* b) { return b ? b->err.c_str() : ""; }

int kp_batch_solve(kp_batch* b, const uint64_t* seeds, size_t k, double budget_s, uint64_t max_iterations,
                   kp_result* results, double* wall_s) {
    if (!b || (k && (!seeds || !results))) return KP_ERR_ARGUMENT;
    try {
        kp_planner* l0 = b->lanes[0];
        cuda_check(cudaSetDevice(l0->device), "cudaSetDevice");
        const double budget = budget_s >= 0 ? budget_s : l0->cfg.t_max_s;
        const uint64_t mi = max_iterations ? max_iterations : l0->cfg.max_iterations;
        const bool stop_first = l0->cfg.stop_at_first_solution != 0;
        if (!(budget > 0) && mi == 0 && !stop_first) throw KpError(KP_ERR_CONFIG, "batch solve needs a budget");
        const unsigned long long budget_ns = budget > 0 ? static_cast<unsigned long long>(budget * 1e9) : 0ull;
        enum State { IDLE, RUNNING, FETCHING };
        struct LaneState {
            State st = IDLE;
            size_t q = 0;
            int launched = 0;
        };
        std::vector<LaneState> ls(b->lanes.size());
        size_t next = 0, finished = 0;
        const auto t0 = std::chrono::steady_clock::now();
        auto wall = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
        const double watchdog = (budget > 0 ? budget : 540.0) * (1.0 + static_cast<double>(k)) + 120.0;
        while (finished < k) {
            for (size_t i = 0; i < b->lanes.size(); ++i) {
                kp_planner* pl = b->lanes[i];
                LaneState& L = ls[i];
                if (L.st == IDLE) {
                    if (next >= k) continue;
                    L.q = next++;
                    reset_async(pl, seeds[L.q]);
                    *pl->host_done = 0;
                    if (++pl->solve_seq == 0) pl->solve_seq = 1;
                    cuda_check(kp::launch_start(pl->B, budget_ns, static_cast<uint32_t>(mi), stop_first ? 1u : 0u,
                                                pl->solve_seq, pl->stream), "start");
                    pl->kernel_launches += 1;
                    L.launched = 0;
                    L.st = RUNNING;
                }
                if (L.st == RUNNING) {
                    if (*pl->host_done == pl->solve_seq) {
                        cuda_check(cudaMemcpyAsync(pl->h_ctl, pl->B.ctl, sizeof(KpCtl), cudaMemcpyDeviceToHost,
                                                   pl->stream), "ctl D2H");
                        cuda_check(cudaEventRecord(pl->ev[0], pl->stream), "event");
                        L.st = FETCHING;
                    } else {
                        cudaEvent_t e = pl->ev[2 + (L.launched & 1)];
                        const bool slot_free = L.launched < 2 || cudaEventQuery(e) == cudaSuccess;
                        if (slot_free) {
                            launch_graph(pl, L.launched);
                            cuda_check(cudaEventRecord(e, pl->stream), "event");
                            ++L.launched;
                        }
                    }
                }
                if (L.st == FETCHING) {
                    const cudaError_t q = cudaEventQuery(pl->ev[0]);
                    if (q == cudaErrorNotReady) continue;
                    cuda_check(q, "batch fetch");
                    std::memcpy(&pl->ctl, pl->h_ctl, sizeof(KpCtl));
                    goal_bookkeeping(pl->ctl);  // the last boundary's (fetch_ctl)
                    pl->ctl_valid = true;
                    if (pl->ctl.error == 8) throw KpError(KP_ERR_SLOT_OVERFLOW, "lambda*|V_A| exceeded max_slots");
                    fill_result(pl, &results[L.q]);
                    L.st = IDLE;
                    ++finished;
                }
            }
            if (wall() > watchdog) throw KpError(KP_ERR_CUDA, "batch watchdog expired");
        }
        if (wall_s) *wall_s = wall();
        return KP_OK;
    } catch (const KpError& e) {
        b->err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        b->err = e.what();
        return KP_ERR_ARGUMENT;
    }
}

int kp_get_timeline(kp_planner* pl, kp_timeline_entry* buf, size_t cap, size_t* len) {
    if (!pl || !len) return KP_ERR_ARGUMENT;
    return guard(pl, [&] {
        fetch_ctl(pl);
        *len = pl->ctl.timeline_len;
        for (size_t i = 0; i < std::min<size_t>(cap, pl->ctl.timeline_len); ++i) {
            const KpTimeline& t = pl->ctl.timeline[i];
            buf[i].iteration = t.iteration;
            buf[i].elapsed_s = t.t_ns * 1e-9;
            buf[i].cost = bits_to_cost(t.best);
            buf[i].leaf = static_cast<int64_t>(t.best & 0xFFFFFFFFull);
        }
    });
}

int kp_get_nodes(kp_planner* pl, float* states, float* controls, float* durations, float* acc, int32_t* parent,
                 uint32_t* region, uint8_t* status, uint8_t* icount, size_t cap, size_t* len) {
    if (!pl || !len) return KP_ERR_ARGUMENT;
    return guard(pl, [&] {
        fetch_ctl(pl);
        const size_t n = pl->ctl.n_nodes;
        *len = n;
        const size_t k = std::min(cap, n);
        if (k == 0) return;
        const KpProblem& P = pl->P;
        const KpBuffers& B = pl->B;
        auto d2h = [&](void* dst, const void* src, size_t bytes) {
            cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, pl->stream), "nodes D2H");
        };
        std::vector<float> tmp;
        if (states) {
            tmp.resize(k);
            for (int d = 0; d < P.n; ++d) {
                d2h(tmp.data(), B.state + static_cast<size_t>(d) * P.capacity, k * 4);
                cuda_check(cudaStreamSynchronize(pl->stream), "sync");
                for (size_t i = 0; i < k; ++i) states[i * P.n + d] = tmp[i];
            }
        }
        if (controls) {
            tmp.resize(k);
            for (int d = 0; d < P.m; ++d) {
                d2h(tmp.data(), B.ctrl + static_cast<size_t>(d) * P.capacity, k * 4);
                cuda_check(cudaStreamSynchronize(pl->stream), "sync");
                for (size_t i = 0; i < k; ++i) controls[i * P.m + d] = tmp[i];
            }
        }
        if (durations) d2h(durations, B.dt, k * 4);
        if (acc) d2h(acc, B.acc, k * 4);
        if (parent) d2h(parent, B.parent, k * 4);
        if (region) d2h(region, B.region, k * 4);
        if (status) d2h(status, B.status, k);
        std::vector<uint16_t> ic;
        if (icount) {
            ic.resize(k);
            d2h(ic.data(), B.icnt, k * 2);
        }
        cuda_check(cudaStreamSynchronize(pl->stream), "nodes sync");
        if (icount)
            for (size_t i = 0; i < k; ++i) icount[i] = static_cast<uint8_t>(std::min<uint16_t>(ic[i], 255));
    });
}

int kp_get_region_table(kp_planner* pl, uint32_t* out, size_t cap, size_t* len) {
    if (!pl || !len) return KP_ERR_ARGUMENT;
    return guard(pl, [&] {
        *len = pl->P.n_regions;
        const size_t k = std::min<size_t>(cap, pl->P.n_regions);
        if (k && out) {
            cuda_check(cudaMemcpyAsync(out, pl->B.rc, k * 4, cudaMemcpyDeviceToHost, pl->stream), "table D2H");
            cuda_check(cudaStreamSynchronize(pl->stream), "table sync");
        }
    });
}

int kp_get_grid(kp_planner* pl, int32_t* cells, float* side, uint64_t* n_regions) {
    if (!pl) return KP_ERR_ARGUMENT;
    for (int j = 0; j < pl->P.grid_n; ++j) {
        if (cells) cells[j] = pl->P.g_cells[j];
        if (side) side[j] = pl->P.g_side[j];
    }
    if (n_regions) *n_regions = pl->P.n_regions;
    return KP_OK;
}

int kp_debug_propagate(kp_planner* pl, size_t n, const float* parent_states, const float* parent_acc,
                       const uint32_t* node_ids, const uint32_t* branches, uint32_t iteration, uint8_t* valid,
                       float* final_states, float* controls, float* durations, float* acc, uint32_t* region,
                       uint32_t* steps, uint8_t* in_goal) {
    if (!pl || (n && (!parent_states || !parent_acc || !node_ids || !branches))) return KP_ERR_ARGUMENT;
    return guard(pl, [&] {
        if (n == 0) return;
        const KpProblem& P = pl->P;
        cudaStream_t s = pl->stream;
        DevBuf<float> ps(n * P.n), pa(n), xs(n * P.n), us(n * P.m), dts(n), accs(n);
        DevBuf<uint32_t> ids(n), brs(n), regs(n), stp(n);
        DevBuf<uint8_t> val(n), gl(n);
        auto h2d = [&](void* d, const void* h, size_t b) { cuda_check(cudaMemcpyAsync(d, h, b, cudaMemcpyHostToDevice, s), "H2D"); };
        auto d2h = [&](void* h, const void* d, size_t b) {
            if (h) cuda_check(cudaMemcpyAsync(h, d, b, cudaMemcpyDeviceToHost, s), "D2H");
        };
        h2d(ps.p, parent_states, n * P.n * 4);
        h2d(pa.p, parent_acc, n * 4);
        h2d(ids.p, node_ids, n * 4);
        h2d(brs.p, branches, n * 4);
        cuda_check(kp::launch_debug_propagate(P, pl->B, static_cast<uint32_t>(n), ps.p, pa.p, ids.p, brs.p, iteration,
                                              val.p, xs.p, us.p, dts.p, accs.p, regs.p, stp.p, gl.p, s),
                   "debug propagate");
        d2h(valid, val.p, n);
        d2h(final_states, xs.p, n * P.n * 4);
        d2h(controls, us.p, n * P.m * 4);
        d2h(durations, dts.p, n * 4);
        d2h(acc, accs.p, n * 4);
        d2h(region, regs.p, n * 4);
        d2h(steps, stp.p, n * 4);
        d2h(in_goal, gl.p, n);
        cuda_check(cudaStreamSynchronize(s), "debug sync");
    });
}

int kp_get_path(kp_planner* pl, int64_t leaf, double* states, double* controls, double* durations,
                double* acc_costs, size_t cap, size_t* len) {
    if (!pl || !len) return KP_ERR_ARGUMENT;
    return guard(pl, [&] {
        DevBuf<int32_t>* chain = nullptr;
        std::vector<int32_t> hc;
        const uint32_t n = chain_of(pl, leaf, chain, hc);
        std::unique_ptr<DevBuf<int32_t>> own(chain);
        *len = n;
        const KpProblem& P = pl->P;
        DevBuf<float> st(n * P.n), ct(n * P.m), dts(n), accs(n);
        cuda_check(kp::launch_gather_chain(P, pl->B, chain->p, n, st.p, ct.p, dts.p, accs.p, pl->stream), "gather");
        std::vector<float> hs(n * P.n), hct(n * P.m), hd(n), ha(n);
        cuda_check(cudaMemcpyAsync(hs.data(), st.p, hs.size() * 4, cudaMemcpyDeviceToHost, pl->stream), "D2H");
        cuda_check(cudaMemcpyAsync(hct.data(), ct.p, hct.size() * 4, cudaMemcpyDeviceToHost, pl->stream), "D2H");
        cuda_check(cudaMemcpyAsync(hd.data(), dts.p, n * 4, cudaMemcpyDeviceToHost, pl->stream), "D2H");
        cuda_check(cudaMemcpyAsync(ha.data(), accs.p, n * 4, cudaMemcpyDeviceToHost, pl->stream), "D2H");
        cuda_check(cudaStreamSynchronize(pl->stream), "path sync");
        const size_t k = std::min<size_t>(cap, n);
        for (size_t i = 0; i < k; ++i) {
            if (states) for (int d = 0; d < P.n; ++d) states[i * P.n + d] = hs[i * P.n + d];
            if (controls) for (int d = 0; d < P.m; ++d) controls[i * P.m + d] = hct[i * P.m + d];
            if (durations) durations[i] = hd[i];
            if (acc_costs) acc_costs[i] = ha[i];
        }
    });
}

int kp_get_trajectory(kp_planner* pl, int64_t leaf, double* samples, size_t cap_samples, size_t* n_samples,
                      double* segment_costs, size_t cap_segments, size_t* n_segments) {
    if (!pl || !n_samples || !n_segments) return KP_ERR_ARGUMENT;
    return guard(pl, [&] {
        DevBuf<int32_t>* chain = nullptr;
        std::vector<int32_t> hc;
        const uint32_t n = chain_of(pl, leaf, chain, hc);
        std::unique_ptr<DevBuf<int32_t>> own(chain);
        const KpProblem& P = pl->P;
        DevBuf<float> st(n * P.n), ct(n * P.m), dts(n), accs(n);
        cuda_check(kp::launch_gather_chain(P, pl->B, chain->p, n, st.p, ct.p, dts.p, accs.p, pl->stream), "gather");
        std::vector<float> hd(n), h0(P.n);
        cuda_check(cudaMemcpyAsync(hd.data(), dts.p, n * 4, cudaMemcpyDeviceToHost, pl->stream), "D2H");
        cuda_check(cudaMemcpyAsync(h0.data(), st.p, P.n * 4, cudaMemcpyDeviceToHost, pl->stream), "D2H");
        cuda_check(cudaStreamSynchronize(pl->stream), "sync");
        const uint32_t n_seg = n - 1;
        std::vector<uint32_t> off(n_seg + 1, 0);
        for (uint32_t j = 0; j < n_seg; ++j) {
            const float dt = hd[j + 1];
            int S = static_cast<int>(std::ceil(dt / P.h));  // same fp32 arithmetic as the kernel
            if (S < 1) S = 1;
            off[j + 1] = off[j] + static_cast<uint32_t>(S);
        }
        const uint32_t total = off[n_seg];
        DevBuf<uint32_t> doff(n_seg + 1);
        DevBuf<float> out(static_cast<size_t>(total) * P.n), sc(n_seg);
        cuda_check(cudaMemcpyAsync(doff.p, off.data(), off.size() * 4, cudaMemcpyHostToDevice, pl->stream), "H2D");
        cuda_check(kp::launch_reintegrate(P, pl->B, chain->p, n_seg, doff.p, out.p, sc.p, pl->stream), "reintegrate");
        std::vector<float> ho(static_cast<size_t>(total) * P.n), hsc(n_seg);
        cuda_check(cudaMemcpyAsync(ho.data(), out.p, ho.size() * 4, cudaMemcpyDeviceToHost, pl->stream), "D2H");
        cuda_check(cudaMemcpyAsync(hsc.data(), sc.p, n_seg * 4, cudaMemcpyDeviceToHost, pl->stream), "D2H");
        cuda_check(cudaStreamSynchronize(pl->stream), "sync");
        // samples: root state then every segment's samples 1..S
        *n_samples = 1 + total;
        *n_segments = n_seg;
        if (samples && cap_samples) {
            for (int d = 0; d < P.n; ++d) samples[d] = h0[d];
            for (size_t i = 0; i < total && i + 1 < cap_samples; ++i)
                for (int d = 0; d < P.n; ++d) samples[(i + 1) * P.n + d] = ho[i * P.n + d];
        }
        if (segment_costs)
            for (size_t j = 0; j < std::min<size_t>(cap_segments, n_seg); ++j) segment_costs[j] = hsc[j];
    });
}

}  // extern "C"
