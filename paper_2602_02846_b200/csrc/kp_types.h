// kp_types.h — host/device layout of one B200 planner instance.
//
// Everything the kernels read lives in two places:
//   KpProblem  — immutable problem/config constants, pre-rounded to fp32 on the
//                host once (the same fp32 constants the Mirror32 recipe uses);
//                passed to every kernel by value (kernel parameter space).
//   KpCtl      — the mutable control block in device memory: list sizes,
//                iteration counter, best solution, stats, timeline, done flag.
// Node store, region table, V_U slots and the frontier/live lists are separate
// SoA buffers (KpBuffers) so every per-node field is a coalesced stream.
#pragma once
#include <stdint.h>

#define KP_MAX_N 12
#define KP_MAX_M 4
#define KP_MAX_GRID 6
#define KP_TIMELINE_CAP 4096
#ifndef KP_SELECT_THREADS
#define KP_SELECT_THREADS 256
#endif

// Device invariant checks (`make checks`: -DKP_CHECKS): index bounds of every
// indirect access on the iteration's path.  A failed check records its code in
// kp_check_code (first failure wins) and the host raises after the solve; the
// product build compiles them out.
#ifdef KP_CHECKS
#define KP_ASSERT(cond, code) \
    do {                      \
        if (!(cond)) kp::check_fail(code); \
    } while (0)
#else
#define KP_ASSERT(cond, code) \
    do {                      \
    } while (0)
#endif

enum KpStatus : uint8_t { KP_ST_ACTIVE = 0, KP_ST_INACTIVE = 1, KP_ST_TERMINAL = 2 };

struct KpProblem {
    int32_t model;           // kp_model_id
    int32_t n, m;            // state / control dims
    int32_t ws_dim;          // 2 or 3 (device always tests 3-D; 2-D scenes pad z)
    int32_t n_box, n_sph;
    int32_t n_angle;
    int32_t angle_dims[3];
    int32_t goal_n;
    int32_t goal_ident;      // goal_dims[i] == i for every i (read coordinates directly)
    int32_t goal_dims[KP_MAX_N];
    float goal_c[KP_MAX_N];
    float goal_r2;
    int32_t cost_kind;       // 0 path length, 1 control duration
    int32_t cost_pos_dims;
    float slo[KP_MAX_N], shi[KP_MAX_N];
    float blo[KP_MAX_N], bhi[KP_MAX_N];  // state bounds with the workspace folded into the position dims
    int32_t check_finite;                // some folded bound is infinite: keep the explicit finite test
    float clo[KP_MAX_M], cw[KP_MAX_M];
    double clo_d[KP_MAX_M], chi_d[KP_MAX_M];
    float wlo[3], whi[3];
    int32_t grid_n;
    int32_t grid_ident;      // grid_dims[j] == j for every j
    int32_t grid_dims[KP_MAX_GRID];
    float g_lo[KP_MAX_GRID], g_side[KP_MAX_GRID];
    int32_t g_cells[KP_MAX_GRID];
    uint32_t g_stride[KP_MAX_GRID];
    uint32_t n_regions;
    float t_prop, h, coll, zero_rate;
    float coll_d2;           // sqrtf(x) > coll  <=>  x > coll_d2 (largest x with sqrtf(x) <= coll)
    double t_prop_d;
    float inv_m, grav, cx, cy, cz, inv_ix, inv_iy, inv_iz;
    int32_t lambda, i_max, rng_kind, deact;
    int32_t lam_shift;       // log2(lambda) when lambda is a power of two, else -1
    uint32_t capacity;       // t_e
    uint32_t max_slots;      // V_U slot buffer (multiple of 32)
    float x_init[KP_MAX_N];
    // environment blob (staged into shared memory by k_propagate):
    //   float4 box_lo[n_box], float4 box_hi[n_box], float4 sph[n_sph] (c xyz, r^2),
    //   uint32 cell_range[n_cells] (start | end << 16), uint16 cell_ids[n_entries]
    // cell grid = exact broad phase: every obstacle whose (margin-expanded)
    // AABB overlaps a cell is listed in it, so the narrow-phase verdict equals
    // testing every obstacle ("outside every obstacle").
    float bg_lo[3], bg_inv[3], bg_off[3];  // cell = floor(v * bg_inv + bg_off), bg_off = -bg_lo * bg_inv
    int32_t bg_n[3], bg_max[3];
    int32_t n_cells, n_entries;
    uint32_t env_bytes;        // multiple of 16
    uint32_t off_cells, off_cids;  // byte offsets inside the blob
    // propagate's shared-memory arrays follow the blob (byte offsets from its start)
    uint32_t prop_smem;        // total dynamic shared memory of k_propagate
    uint32_t seq_base;         // step-sorted path: PropSmem<MODEL>
    // sample-parallel path (double integrator, kp_kernels.cu flat_phase): item
    // records, sample offsets, invalid flags, fixed-point path lengths
    int32_t sel_spec;          // select_reduce loads its first tile's live entries before the control block
                               // (latency win for a lone query; off for concurrent batch lanes)
    int32_t flat_on;
    uint32_t flat_max;         // launches of at most this many items take the sample-parallel path
    uint32_t flat_nb;          // items per batch
    uint32_t flat_rec, flat_offs, flat_bad, flat_len, flat_idx;
};

struct KpStats {
    unsigned long long attempted, valid, admitted, committed;
    unsigned long long pruned_terminal, deactivated, reactivated, dropped_capacity;
    // roofline accounting (valid + invalid items)
    unsigned long long rk4_steps, samples_checked, interp_points, box_tests, sphere_tests;
    unsigned long long live_scanned, ancestor_hops, slots_scanned, admitted_checked;
};

#ifdef __CUDACC__
#define KP_HD __host__ __device__
#else
#define KP_HD
#endif

struct KpCtl;
KP_HD inline void goal_bookkeeping(KpCtl& c);

struct KpTimeline {
    unsigned long long iteration;
    unsigned long long t_ns;
    unsigned long long best;  // (cost bits << 32) | leaf
};

#define KP_TRACE_CAP 8192
struct KpTraceRec {
    unsigned long long t_ns;
    uint32_t iteration, items, live, frontier, nodes, committed;
    // in-graph kernel timestamps (ns since solve start): block 0 entry of
    // propagate and select_reduce, entry of the select_scatter block that
    // closes the iteration (t_sel_end == t_scat); the boundary itself is t_ns
    uint32_t t_prop, t_sel, t_sel_end, t_scat;
};

struct KpCtl {
    // current iteration's lists (parity = iter & 1)
    uint32_t iter;            // iterations completed since reset
    uint32_t done;            // 1 = stop (budget / iterations / first solution / no live nodes)
    uint32_t error;           // nonzero = device error (slot overflow)
    uint32_t n_live, n_va, n_nodes, n_items;
    uint32_t capacity_exhausted;
    // produced by select_reduce for select_scatter
    uint32_t n_tiles;
    uint32_t tot_keep, tot_va, tot_commit, accepted;
    uint32_t ticket_b;        // (unused since the early boundary)
    uint32_t prop_cursor;     // dynamic chunk cursor of k_propagate (reset at every boundary)
    uint32_t n_adm_iter;      // slots admitted by this iteration's propagate (reset at every boundary);
                              // selects the select kernels' element layout (per slot / per mask word)
    uint32_t n_valid_iter;    // valid rollouts of this iteration's propagate (reset at every boundary)
    uint32_t split;           // 1: the next propagate splits its rollouts (>= 1/4 of the last iteration's were invalid)
    // The iteration boundary is written by select_scatter's block 0 as soon as
    // it has the totals, while the other blocks may still read the control
    // block: they read this iteration's view (parity = iteration & 1), which
    // the boundary writes for the next one, and the iteration number from
    // cur_iter (written by propagate).  done_iter: the iteration count at
    // which `done` was raised (a scatter skips only iterations after it).
    uint32_t cur_iter, done_iter;
    uint32_t solve_seq;       // kp_solve call number: the value the device writes to the host's done word
    uint32_t n_adm_p[2];      // slots admitted by propagate, per iteration parity (cleared by the previous boundary)
    uint32_t view_live[2], view_items[2], view_nodes[2];
    // run bookkeeping
    uint32_t max_iter_abs;    // stop when iter >= this (0 = unlimited)
    uint32_t stop_first;
    uint32_t timeline_len;
    uint32_t first_iter, best_iter;
    unsigned long long seed;  // run seed (kept here so captured graphs survive kp_reset)
    unsigned long long best;  // (cost bits << 32) | leaf ; init ~0
    unsigned long long tl_best;  // best of the last timeline entry (init ~0): no dependent load at the boundary
    unsigned long long t_start_ns, deadline_ns, t_last_ns;
    unsigned long long first_ns, best_ns;
    unsigned long long t_prop_ns, t_sel_ns, t_sel_end_ns, t_scat_ns;  // current iteration stamps
    KpStats stats;
    KpTimeline timeline[KP_TIMELINE_CAP];
};

// Best-solution bookkeeping of the last iteration boundary (SPEC.md:362-367,
// :440): a strict improvement of `best` over the last timeline entry appends
// an entry stamped with that boundary's time and iteration count, and sets
// the first / latest solution time.  Run by the next propagate (block 0,
// before anything else) and, for the last boundary of a solve, on the host
// copy of the control block (fetch_ctl): the same result either way.
KP_HD inline void goal_bookkeeping(KpCtl& c) {
    const unsigned long long best = c.best;
    if (!(best < c.tl_best)) return;
    const unsigned long long t = c.t_last_ns - c.t_start_ns;
    const uint32_t it = c.iter;
    if (c.timeline_len < KP_TIMELINE_CAP) {
        KpTimeline& e = c.timeline[c.timeline_len];
        e.iteration = it;
        e.t_ns = t;
        e.best = best;
        c.timeline_len += 1;
        c.tl_best = best;
    }
    if (c.first_ns == 0) {
        c.first_ns = t;
        c.first_iter = it;
    }
    c.best_ns = t;
    c.best_iter = it;
}


// Device buffer set of one planner.
struct KpBuffers {
    // node store, SoA [dim][capacity]
    float* state;
    float* ctrl;
    float* dt;
    uint32_t* acc;       // fp32 cost bits
    int32_t* parent;
    uint32_t* region;
    uint8_t* status;
    uint32_t* live_st;   // [capacity] status | i_count << 8 after this iteration's prune, by live-list position
    uint16_t* icnt;
    // region table [n_regions], encoded fp32 bits (+inf = 0x7F800000)
    uint32_t* rc;
    uint4* link;         // [capacity] {parent, region, acc bits, 0}: one 16-byte load per ancestor hop
    // lists, double-buffered [2][capacity]
    // live list entries carry what the prune pass needs (no gathers by id):
    // {id, region, acc bits, parent} and status | i_count << 8
    uint4* live[2];
    uint32_t* live_si[2];
    uint32_t* va[2];
    // V_U slots, SoA [dim][max_slots]
    float* vu_state;
    float* vu_ctrl;
    float* vu_dt;
    uint32_t* vu_acc;
    uint32_t* vu_region;
    uint32_t* admit_mask;   // [max_slots/32]
    uint32_t* goal_mask;    // [max_slots/32]
    uint32_t* commit_mask;  // [max_slots/32]
    // select scratch
    uint32_t* tile_sums;    // [3][max_tiles] per-tile counts (keep, active, commit)
    uint32_t max_tiles;
    float* prop_scratch;    // [propagate grid][n + 1][1024]: per-block parked rollouts (state, path length)
    const float4* env;      // environment blob (see KpProblem)
    KpTraceRec* trace;      // [KP_TRACE_CAP] ring, one record per iteration boundary
    float* x0;              // [KP_MAX_N] current query's start state (H2D per query)
    KpCtl* ctl;
    volatile uint32_t* host_done;  // mapped pinned word (device writes the solve's sequence number at termination)
};
