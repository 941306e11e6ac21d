// kp_kernels.cu — the three per-iteration kernels of the B200 Kino-PAX+ planner
// plus reset/start/debug/trajectory helpers.
//
// One iteration (Alg. 1 lines 6-9) = three launches on one
// stream, captured 8 / 32 iterations at a time into CUDA graphs with
// programmatic dependent launch between the kernels (kp_capi.cpp):
//
//   k_propagate<MODEL>   Alg. 2: per V_U slot (frontier
//                        position x branch) a Philox/SplitMix draw, the
//                        rollout (RK4 in registers; closed form for the double
//                        integrator), per-sample validity against the
//                        obstacles staged in shared memory, path length,
//                        region, atomicMin on the encoded region cost;
//                        admitted slots write their record and admit / goal
//                        bit.  Two paths: step-sorted (a block sorts its chunk
//                        by step count, a thread per slot; quadcopter rollouts
//                        split in two passes with compaction) and, for the
//                        double integrator's launches of up to two batches per
//                        block, sample-parallel (flat_phase: a batch of items
//                        flattened into 2-sample chunks).  The environment blob
//                        arrives by one bulk (TMA) copy on an mbarrier.
//   k_select_reduce      Alg. 3 + the commit test of Alg. 4.
//                        Element space = [live nodes] ++ [slots, or 32-slot
//                        mask words when few are admitted].  Live nodes: prune
//                        rules in SPEC.md:434-437 priority order; slots: commit
//                        iff admitted and acc bits == region minimum.
//                        Per-tile counts (keep, active, commit).
//   k_select_scatter     Re-derives each element's flags, block scan + tile
//                        prefix -> positions.  Survivors go to the next live /
//                        frontier lists in id order; committed slots get node
//                        ids count + rank in slot order (so ids equal the
//                        reference's workers=1 serial order), their records
//                        are written to the SoA node store, goal leaves do a
//                        64-bit atomicMin on (cost bits << 32 | id).  Block 0
//                        closes the iteration as soon as its tile prefix gives
//                        it the totals: counts, stats, termination (the other
//                        blocks read a per-parity view of the control block);
//                        the best / timeline / TTFS bookkeeping, which needs
//                        every goal commit, is the next propagate's first step.
//
// No kernel waits on another block: cross-block results flow through kernel
// boundaries (PDL), never a spin; the one in-block wait is the split
// rollouts' second pass behind a block barrier.
#include <cuda_runtime.h>
#include <stdint.h>
#include <cmath>
#include <cstdlib>

#include "kp_math.cuh"
#include "kp_types.h"

namespace kp {

KP_DEV unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Programmatic dependent launch (sm_90+): a kernel may start while its
// predecessor drains; griddepcontrol.wait blocks until the predecessor grid
// has completed and its memory is visible, so nothing before it may read data
// the predecessor writes.  launch_dependents lets the successor launch early.
KP_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
KP_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Diagnostic build only (-DKP_STAMPS, scripts/stamps.py): %globaltimer stamps
// of kernel phases per iteration (a ring of 64 iterations x 32 points) — block
// 0's entry / PDL release / control-block arrival and the latest block exit
// of each kernel, the scatter's iteration boundary.
#ifdef KP_STAMPS
__device__ unsigned long long kp_stamps[64][32];
#define KP_STAMP_B0(it, k, t)                                                        \
    do {                                                                            \
        if (blockIdx.x == 0 && threadIdx.x == 0) kp_stamps[(it) & 63][k] = (t);     \
    } while (0)
#define KP_STAMP_MAX(it, k)                                                          \
    do {                                                                            \
        if (threadIdx.x == 0) atomicMax(&kp_stamps[(it) & 63][k], globaltimer());   \
    } while (0)
#define KP_T0 const unsigned long long kp_t_entry = globaltimer()
#define KP_T1 const unsigned long long kp_t_pdl = globaltimer()
#else
#define KP_STAMP_B0(it, k, t) \
    do {                      \
    } while (0)
#define KP_STAMP_MAX(it, k) \
    do {                    \
    } while (0)
#define KP_T0 \
    do {      \
    } while (0)
#define KP_T1 \
    do {      \
    } while (0)
#endif

// Stage the environment blob into shared memory (16-byte vector copies).
KP_DEV Env stage_env(const KpProblem& P, const KpBuffers& B) {
    for (uint32_t i = threadIdx.x; i < P.env_bytes / 16; i += blockDim.x) kp_env_smem[i] = B.env[i];
    __syncthreads();
    return env_view(P);
}

// The propagate kernels stage the blob with the bulk-copy (TMA) engine
// instead: thread 0 arms an mbarrier with the blob's byte count and issues
// cp.async.bulk global -> shared; the block waits on the barrier (env_wait)
// only before its first obstacle test, so the copy overlaps the PDL wait,
// the control-block round trip and the sampling, and no thread spends issue
// slots on the copy.
__shared__ __align__(8) unsigned long long kp_env_bar;

KP_DEV uint32_t env_bar_addr() { return static_cast<uint32_t>(__cvta_generic_to_shared(&kp_env_bar)); }

KP_DEV Env stage_env_async(const KpProblem& P, const KpBuffers& B) {
    if (threadIdx.x == 0) {
        const uint32_t bar = env_bar_addr();
        const uint32_t dst = env_saddr();
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(P.env_bytes) : "memory");
        constexpr uint32_t CHUNK = 32768;  // bytes per bulk copy (multiples of 16)
        for (uint32_t off = 0; off < P.env_bytes; off += CHUNK) {
            const uint32_t n = min(CHUNK, P.env_bytes - off);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst + off),
                "l"(reinterpret_cast<const unsigned char*>(B.env) + off), "r"(n), "r"(bar)
                : "memory");
        }
    }
    __syncthreads();  // the barrier is initialised before any thread waits on it
    return env_view(P);
}

// Wait for the environment's bulk copy (phase 0 of the barrier: returns at
// once after the first completion, so repeated calls are free).
KP_DEV void env_wait() {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "ENV_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        "@!p bra ENV_WAIT_%=;\n"
        "}\n" ::"r"(env_bar_addr())
        : "memory");
}

// Propagate (Alg. 2).  Work is claimed by blocks in chunks of 256*G slots
// (dynamic cursor).  Per chunk: (1) every thread draws (u, dt) for G slots
// (convergent RNG) into shared memory; (2) block counting sort of the chunk
// by RK4 step count S, longest first; (3) each warp integrates groups of 32
// consecutive sorted slots, so lanes of a warp run nearly the same number of
// steps (SIMT efficiency) — the result of a slot does not depend on which
// lane runs it.  Admitted slots write their record and set their admit/goal
// bit with atomicOr (the consumers zero the words after use).
// Propagate block shape per model: 512 threads for the 4D/6D models (a larger
// step-count sort pool, so a 32-slot group spans fewer step counts), 256 for
// the register-heavy quadcopter (3 blocks/SM); chunks of at most 1024 slots.
template <int MODEL>
struct PropCfg {
#ifndef KP_QUAD_MINB
#define KP_QUAD_MINB 3
#endif
#ifndef KP_DUBINS_T
#define KP_DUBINS_T 512
#define KP_DUBINS_MINB 2
#endif
    static constexpr int T = MODEL == 3 ? 256 : (MODEL == 2 ? KP_DUBINS_T : 512);  // threads per block
    static constexpr int MAXG = 1024 / T;                                          // slot rounds per chunk
#ifndef KP_DI_MINB
#define KP_DI_MINB 2
#endif
    static constexpr int MIN_BLOCKS = MODEL == 3 ? KP_QUAD_MINB : (MODEL == 2 ? KP_DUBINS_MINB : KP_DI_MINB);
    // Steps of the first pass of a split rollout (0: never split).  Only the
    // quadcopter splits: ~55 % of its items stop early (invalid), and a first
    // pass of 8 steps cuts its warp-steps by ~22 % (scripts/split_sim.py); for
    // the 4D/6D models the split measured slower (profiles/README.md), and the
    // closed-form double integrator cannot resume from a parked state (its
    // samples derive from the parent state).  -DKP_SPLIT_Q/-DKP_SPLIT_D: A/B builds.
#ifdef KP_SPLIT_Q
    static constexpr int SPLIT = MODEL == 3 ? KP_SPLIT_Q : (closed_form<MODEL>() ? 0 : KP_SPLIT_D);
#else
    static constexpr int SPLIT = MODEL == 3 ? 8 : 0;
#endif
};

#define KP_SORT_BUCKETS 64

// the split rollouts' per-group masks (32 entries) and the per-block scratch
// (1024 slots) bound a chunk at 1024 slots in 32 groups
static_assert(PropCfg<0>::T * PropCfg<0>::MAXG <= 1024 && PropCfg<1>::T * PropCfg<1>::MAXG <= 1024 &&
                  PropCfg<2>::T * PropCfg<2>::MAXG <= 1024 && PropCfg<3>::T * PropCfg<3>::MAXG <= 1024,
              "propagate chunks hold at most 1024 slots");

template <int MODEL>
struct PropSmem {
    float u[Model<MODEL>::M][PropCfg<MODEL>::T * PropCfg<MODEL>::MAXG];
    float dt[PropCfg<MODEL>::T * PropCfg<MODEL>::MAXG];
    uint32_t node[PropCfg<MODEL>::T * PropCfg<MODEL>::MAXG];
    uint16_t steps[PropCfg<MODEL>::T * PropCfg<MODEL>::MAXG];
    uint16_t perm[PropCfg<MODEL>::T * PropCfg<MODEL>::MAXG];
    uint16_t slist[PropCfg<MODEL>::T * PropCfg<MODEL>::MAXG];  // survivors of the first pass (sorted positions)
    uint32_t hist[KP_SORT_BUCKETS];
    uint32_t gmask[32];  // per 32-slot group: lanes still running after the first pass
    uint32_t gbase[32];
    uint32_t n_surv, claim;
    uint32_t chunk;
    uint32_t cnt[6];
};

// The control-block fields every propagate block reads, in one round trip.
struct PropCtl {
    uint32_t done, n_items, it, split, stop_first, seq;
    unsigned long long seed, best, tl_best;
};

KP_DEV PropCtl load_prop_ctl(const KpCtl* ctl) {
    PropCtl c;
    c.done = ctl->done;
    c.n_items = ctl->n_items;
    c.it = ctl->iter;
    c.split = ctl->split;
    c.stop_first = ctl->stop_first;
    c.seq = ctl->solve_seq;
    c.seed = ctl->seed;
    c.best = ctl->best;
    c.tl_best = ctl->tl_best;
    return c;
}

// Work counters of a propagate launch: warp-aggregated (one REDUX per
// counter), then block-aggregated, then one atomic per counter and block.
KP_DEV void count_flush(KpCtl* ctl, uint32_t* c, uint32_t* cnt, int lane, uint32_t it) {
#pragma unroll
    for (int k = 0; k < 6; ++k) c[k] = __reduce_add_sync(0xFFFFFFFFu, c[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 6; ++k)
            if (c[k]) atomicAdd(&cnt[k], c[k]);  // 32-bit: a native shared atomic
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (cnt[0]) {
            atomicAdd(&ctl->stats.valid, static_cast<unsigned long long>(cnt[0]));
            atomicAdd(&ctl->n_valid_iter, cnt[0]);
        }
        if (cnt[1]) {
            atomicAdd(&ctl->stats.admitted, static_cast<unsigned long long>(cnt[1]));
            atomicAdd(&ctl->n_adm_p[it & 1], cnt[1]);
        }
        if (cnt[2]) atomicAdd(&ctl->stats.rk4_steps, static_cast<unsigned long long>(cnt[2]));
        if (cnt[3]) atomicAdd(&ctl->stats.interp_points, static_cast<unsigned long long>(cnt[3]));
        if (cnt[4]) atomicAdd(&ctl->stats.box_tests, static_cast<unsigned long long>(cnt[4]));
        if (cnt[5]) atomicAdd(&ctl->stats.sphere_tests, static_cast<unsigned long long>(cnt[5]));
    }
}

template <int MODEL>
KP_DEV void propagate_phase(const KpProblem& P, const KpBuffers& B, PropSmem<MODEL>& sh, const Env& E,
                            const PropCtl& pc) {
    constexpr int N = Model<MODEL>::N;
    constexpr int M = Model<MODEL>::M;
    constexpr uint32_t KP_PROP_THREADS = PropCfg<MODEL>::T;
    constexpr uint32_t KP_PROP_MAXG = PropCfg<MODEL>::MAXG;
    KpCtl* ctl = B.ctl;
    // the control block was read once by the kernel (PropCtl)
    const uint32_t n_items = pc.n_items, it = pc.it, split_on = pc.split;
    const unsigned long long seed = pc.seed;
    if (threadIdx.x < 6) sh.cnt[threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->t_prop_ns = globaltimer();
    // Chunk of slots per block: one block width while the launch fits in one
    // wave; beyond that, the items are spread evenly over every block (CH a
    // multiple of 32, so a few warps per block run a second, short group)
    // instead of doubling the chunk and leaving half the blocks idle.
    const uint32_t CH = min(KP_PROP_THREADS * KP_PROP_MAXG, ((n_items + gridDim.x - 1) / gridDim.x + 31u) & ~31u);
    const uint32_t G = (CH + KP_PROP_THREADS - 1) / KP_PROP_THREADS;  // sampling rounds / group rounds
    const uint32_t n_chunks = (n_items + CH - 1) / CH;
    if (blockIdx.x >= n_chunks) return;  // nothing for this block this iteration
    const uint32_t* va = B.va[it & 1];
    const uint32_t cap = P.capacity, S_cap = P.max_slots;
    const uint32_t lam = static_cast<uint32_t>(P.lambda);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t c[6] = {0, 0, 0, 0, 0, 0};  // valid, admitted, steps, interp, box tests, sphere tests
    if (threadIdx.x == 0) sh.chunk = blockIdx.x;  // first chunk is static, the rest dynamic
    __syncthreads();
    for (;;) {
        const uint32_t chunk = sh.chunk;
        if (chunk >= n_chunks) break;
        const uint32_t c0 = chunk * CH;
        if (threadIdx.x < KP_SORT_BUCKETS) sh.hist[threadIdx.x] = 0;
        __syncthreads();
        // (1) draw (u, dt) and the step count of every slot of the chunk
        for (uint32_t k = 0; k < G; ++k) {
            const uint32_t p = k * KP_PROP_THREADS + threadIdx.x;
            const uint32_t i = c0 + p;
            uint32_t key = 0;
            if (p < CH && i < n_items) {
                const uint32_t f = frontier_pos(P, i);
                const uint32_t br = i - f * lam;
                KP_ASSERT(f < ctl->n_va, 10);
                const uint32_t node = va[f];
                KP_ASSERT(node < ctl->n_nodes, 11);
                float u[M], dt;
                sample_item<M>(P, seed, it, node, br, u, dt);
                const int S = step_count(P, dt);
#pragma unroll
                for (int d = 0; d < M; ++d) sh.u[d][p] = u[d];
                sh.dt[p] = dt;
                sh.node[p] = node;
                sh.steps[p] = static_cast<uint16_t>(min(S, 65535));
                key = static_cast<uint32_t>(min(S, KP_SORT_BUCKETS - 1));
            }
            sh.perm[p] = static_cast<uint16_t>(key);  // temporarily the bucket key
            atomicAdd(&sh.hist[KP_SORT_BUCKETS - 1 - key], 1u);
        }
        __syncthreads();
        // (2) exclusive scan of the 64 buckets (descending S), then scatter
        if (warp == 0) {
            uint32_t a = sh.hist[2 * lane], b = sh.hist[2 * lane + 1];
            uint32_t x = a + b;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, off);
                if (lane >= off) x += y;
            }
            const uint32_t excl = x - a - b;
            sh.hist[2 * lane] = excl;
            sh.hist[2 * lane + 1] = excl + a;
        }
        __syncthreads();
        uint32_t keys[KP_PROP_MAXG];
        for (uint32_t k = 0; k < G; ++k) keys[k] = sh.perm[k * KP_PROP_THREADS + threadIdx.x];
        __syncthreads();
        for (uint32_t k = 0; k < G; ++k) {
            const uint32_t p = k * KP_PROP_THREADS + threadIdx.x;
            const uint32_t pos = atomicAdd(&sh.hist[KP_SORT_BUCKETS - 1 - keys[k]], 1u);
            sh.perm[pos] = static_cast<uint16_t>(p);
        }
        __syncthreads();
        env_wait();
        // (3) integrate groups of 32 consecutive sorted slots per warp.  When a
        // warp has several groups (the launch spans more than one wave) and at
        // least a quarter of the previous iteration's rollouts were invalid, the
        // rollout is split: every slot first runs at most SPLIT steps; the slots
        // still running (state + path length parked in this block's scratch) are
        // compacted in sorted order and finished in full groups claimed longest
        // first, so the lanes of items that stop early (invalid) do not idle
        // until the end of a group.  Bit-identical to one pass (integrate_steps).
        constexpr uint32_t NW = KP_PROP_THREADS / 32;
        constexpr uint32_t SCR = KP_PROP_THREADS * KP_PROP_MAXG;  // scratch stride (slots per chunk)
        constexpr int SPLIT = PropCfg<MODEL>::SPLIT;
        const bool split = SPLIT > 0 && G >= 2 && split_on;
        float* const scr = B.prop_scratch + static_cast<size_t>(blockIdx.x) * (N + 1) * SCR;
        uint32_t n_surv = 0;
        for (uint32_t job = 0;; ++job) {
            if (job == G) {
                if (!split) break;
                // compact the survivors of the first pass (sorted order kept)
                __syncthreads();
                if (warp == 0) {
                    const uint32_t v = lane < G * NW ? __popc(sh.gmask[lane]) : 0u;
                    uint32_t x = v;
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, off);
                        if (lane >= off) x += y;
                    }
                    sh.gbase[lane] = x - v;
                    if (lane == 31) {
                        sh.n_surv = x;
                        sh.claim = 0;
                    }
                }
                __syncthreads();
                for (uint32_t g = warp; g < G * NW; g += NW) {
                    const uint32_t m = sh.gmask[g];
                    if ((m >> lane) & 1u) sh.slist[sh.gbase[g] + __popc(m & ((1u << lane) - 1u))] = static_cast<uint16_t>(g * 32 + lane);
                }
                __syncthreads();
                n_surv = sh.n_surv;
            }
            const bool resume = job >= G;  // second pass: a compacted survivor
            uint32_t k = job, wk = 0, q;
            if (!resume) {
                // snake assignment of the step-sorted groups: round k even hands the
                // longest groups to the highest warp ids (the arbiter issues highest
                // warp id first), odd rounds reverse, so each warp's total step count
                // over its groups is about the same
                wk = (k & 1u) ? static_cast<uint32_t>(warp) : NW - 1 - static_cast<uint32_t>(warp);
                q = (k * NW + wk) * 32 + lane;
            } else {
                // second pass: warps claim the compacted groups longest first
                uint32_t g = 0;
                if (lane == 0) g = atomicAdd(&sh.claim, 1u);
                g = __shfl_sync(0xFFFFFFFFu, g, 0);
                if (g * 32 >= n_surv) break;
                q = g * 32 + lane;
            }
            uint32_t pos = q;
            bool have;
            if (resume) {
                have = q < n_surv;
                pos = have ? sh.slist[q] : 0u;
            }
            const uint32_t p = sh.perm[pos];
            const uint32_t i = c0 + p;
            if (!resume) have = p < CH && i < n_items;
            // loads guarded by `have`; the rollout below is warp-uniform control flow
            const uint32_t node = have ? sh.node[p] : 0u;
            const int S = have ? sh.steps[p] : 0;
            float x[N], u[M], total = 0.0f;
            if (have) {
                if (resume) {
#pragma unroll
                    for (int d = 0; d < N; ++d) x[d] = scr[d * SCR + pos];
                    total = scr[N * SCR + pos];
                } else {
#pragma unroll
                    for (int d = 0; d < N; ++d) x[d] = B.state[static_cast<size_t>(d) * cap + node];
                }
            }
#pragma unroll
            for (int d = 0; d < M; ++d) u[d] = sh.u[d][p];
            const float dt = sh.dt[p];
            ItemOut o;
            o.steps = o.interp = o.nbox = o.nsph = 0;
            const int s0 = resume ? SPLIT : 0;
            const int s1 = (split && !resume) ? min(S, SPLIT) : S;
            int rc = 1;
            if (have) rc = integrate_steps<MODEL>(P, E, x, u, dt, S, s0, s1, total, o);
            const bool running = rc == 0 && s1 < S;
            const bool ok = rc == 0 && s1 >= S;
            c[2] += o.steps;
            c[3] += o.interp;
            c[4] += o.nbox;
            c[5] += o.nsph;
            if (running) {  // park it for the second pass
#pragma unroll
                for (int d = 0; d < N; ++d) scr[d * SCR + pos] = x[d];
                scr[N * SCR + pos] = total;
            }
            if (split && !resume) {
                const uint32_t m = __ballot_sync(0xFFFFFFFFu, running);
                if (lane == 0) sh.gmask[k * NW + wk] = m;
            }
            if (ok) {
                finish_item<MODEL>(P, x, dt, total, __uint_as_float(B.acc[node]), o);
                ++c[0];
                const uint32_t bits = __float_as_uint(o.acc);
                KP_ASSERT(o.region < P.n_regions, 12);
                KP_ASSERT(i < S_cap, 13);
                const uint32_t old = atomicMin(B.rc + o.region, bits);
                if (bits <= old) {  // Improved / Equal admitted, Worse discarded
                    ++c[1];
#pragma unroll
                    for (int d = 0; d < N; ++d) B.vu_state[static_cast<size_t>(d) * S_cap + i] = x[d];
#pragma unroll
                    for (int d = 0; d < M; ++d) B.vu_ctrl[static_cast<size_t>(d) * S_cap + i] = u[d];
                    B.vu_dt[i] = dt;
                    B.vu_acc[i] = bits;
                    B.vu_region[i] = o.region;
                    atomicOr(B.admit_mask + (i >> 5), 1u << (i & 31));
                    if (o.goal) atomicOr(B.goal_mask + (i >> 5), 1u << (i & 31));
                }
            }
        }
        if (n_chunks <= gridDim.x) break;  // every chunk was assigned statically
        __syncthreads();
        if (threadIdx.x == 0) sh.chunk = gridDim.x + atomicAdd(&ctl->prop_cursor, 1u);
        __syncthreads();
    }
    count_flush(ctl, c, sh.cnt, lane, it);
}

// One sample of a closed-form rollout (the sequential loop's per-step checks,
// integrate_steps): finite state (when a bound is infinite), state bounds,
// obstacles, and the interpolated points of the segment from the previous
// sample position (px, py, pz); d = the segment length.  c: the work
// counters (samples, interpolated points, box / sphere tests at 2..5).
template <int MODEL>
KP_DEV bool check_sample(const KpProblem& P, const Env& E, const float* xs, float px, float py, float pz, float& d,
                         uint32_t* c) {
    constexpr int N = Model<MODEL>::N;
    constexpr bool TWO_D = (MODEL == 0);
    ++c[2];
    bool ok = true;
    if (P.check_finite) {
#pragma unroll
        for (int k = 0; k < N; ++k) ok = ok && isfinite(xs[k]);
    }
    const float nx = xs[0], ny = xs[1], nz = TWO_D ? 0.0f : xs[2];
    // closed form with finite bounds: velocities were checked once per item (vel_ok_at_end)
    const bool inb = within_bounds<MODEL>(P, xs, !(closed_form<MODEL>() && !P.check_finite));
    const bool hit = in_obstacle(P, E, nx, ny, nz, c[4], c[5]);
    ok = ok && inb && !hit;
    const float dx = nx - px, dy = ny - py, dz = nz - pz;
    float d2 = dx * dx;
    d2 = fmaf(dy, dy, d2);
    if (!TWO_D) d2 = fmaf(dz, dz, d2);
    d = sqrtf(d2);
    if (ok && d2 > P.coll_d2 && segment_hit<TWO_D>(P, E, px, py, pz, dx, dy, dz, d, c[3], c[4], c[5])) ok = false;
    return ok;
}

#ifndef KP_FLAT_ITEMS
#define KP_FLAT_ITEMS 512u  // items per sample-parallel batch (a multiple of the block size)
#endif
#ifndef KP_FLAT_K
#define KP_FLAT_K 2u        // samples per chunk of the sample-parallel path
#endif

// Sample-parallel propagate for the double integrator (closed form, §4 of
// DESIGN.md), used for one-wave launches (at most flat_nb items per block).
// Its samples do not depend on one another, so a batch of items is flattened
// into chunks of K consecutive samples and the whole block checks them: the
// batch takes about (sum of chunk counts) / threads rounds instead of the
// longest item's step count, which bounds a one-wave launch in the
// step-sorted path.  Per batch: (1) one item per thread draws (u, dt), stages
// the parent state, checks the velocity bounds once (vel_ok_at_end: an item
// failing them gets no chunks) and counts its chunks; (2) block scan of the
// counts; (3) chunks interleaved over the block: bounds, obstacles,
// interpolated points and segment lengths of each sample; an item with a
// failed sample is flagged and its remaining chunks skipped; each chunk adds
// its fixed-point length to its item once (order-independent, §4); (4) the
// owner thread converts the length, computes region and goal, and admits the
// candidate.  K = 2 measured fastest (K = 4 and 8, one sample per thread
// interleaved, and contiguous runs per thread were all slower: the shorter a
// chunk, the less the lanes of a warp wait on each other's chunk tails).
template <int MODEL>
KP_DEV void flat_phase(const KpProblem& P, const KpBuffers& B, const Env& E, unsigned char* dyn, const PropCtl& pc) {
    constexpr int N = Model<MODEL>::N;
    constexpr int M = Model<MODEL>::M;
    constexpr uint32_t T = PropCfg<MODEL>::T;
    constexpr uint32_t NWARP = T / 32;
    constexpr uint32_t IPT = (KP_FLAT_ITEMS + T - 1) / T;  // items per thread in a batch
    constexpr uint32_t FB = IPT * T;                        // items per batch (== P.flat_nb)
    constexpr int RW = (N + M + 3 + 3) / 4;  // float4 words per item record: x0, u, dt, S, seff
    constexpr bool TWO_D = (MODEL == 0);
    constexpr uint32_t K = KP_FLAT_K;
    __shared__ uint32_t fcnt[6];
    __shared__ uint32_t wsum[NWARP];
    __shared__ uint32_t fchunk;
    float4* const rec = reinterpret_cast<float4*>(dyn + P.flat_rec);
    uint32_t* const off = reinterpret_cast<uint32_t*>(dyn + P.flat_offs);           // [FB + 1]
    volatile uint32_t* const bad = reinterpret_cast<uint32_t*>(dyn + P.flat_bad);   // [FB]
    // fixed-point path lengths as two 32-bit limbs (native shared atomics):
    // len = hi << 24 + lo, every run adding its low 24 bits to lo and the rest to hi
    uint32_t* const len_lo = reinterpret_cast<uint32_t*>(dyn + P.flat_len);  // [FB]
    uint32_t* const len_hi = len_lo + FB;                                   // [FB]
    KpCtl* ctl = B.ctl;
    const uint32_t n_items = pc.n_items, it = pc.it;
    const unsigned long long seed = pc.seed;
    if (threadIdx.x < 6) fcnt[threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->t_prop_ns = globaltimer();
    const uint32_t CH = min(T * PropCfg<MODEL>::MAXG, ((n_items + gridDim.x - 1) / gridDim.x + 31u) & ~31u);
    const uint32_t n_chunks = (n_items + CH - 1) / CH;
    if (blockIdx.x >= n_chunks) return;
    const uint32_t* va = B.va[it & 1];
    const uint32_t cap = P.capacity, S_cap = P.max_slots;
    const uint32_t lam = static_cast<uint32_t>(P.lambda);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t c[6] = {0, 0, 0, 0, 0, 0};  // valid, admitted, samples, interp, box tests, sphere tests
    if (threadIdx.x == 0) fchunk = blockIdx.x;
    __syncthreads();
    for (;;) {
        const uint32_t chunk = fchunk;
        if (chunk >= n_chunks) break;
        const uint32_t cend = min(chunk * CH + CH, n_items);
        for (uint32_t b0 = chunk * CH; b0 < cend; b0 += FB) {
            // (1) IPT consecutive items per thread: draw (u, dt), stage the parent state
            uint32_t node[IPT], seffk[IPT];
            float acc_p[IPT];
            uint32_t seff = 0;  // this thread's samples
#pragma unroll
            for (uint32_t k = 0; k < IPT; ++k) {
                const uint32_t p = threadIdx.x * IPT + k;
                const uint32_t i = b0 + p;
                node[k] = 0;
                seffk[k] = 0;
                acc_p[k] = 0.0f;
                uint32_t vbad = 0u;
                if (i < cend) {
                    const uint32_t f = frontier_pos(P, i);
                    const uint32_t br = i - f * lam;
                    KP_ASSERT(f < ctl->n_va, 10);
                    node[k] = va[f];
                    KP_ASSERT(node[k] < ctl->n_nodes, 11);
                    float r[RW * 4];
#pragma unroll
                    for (int w = 0; w < RW * 4; ++w) r[w] = 0.0f;
#pragma unroll
                    for (int d = 0; d < N; ++d) r[d] = B.state[static_cast<size_t>(d) * cap + node[k]];
                    acc_p[k] = __uint_as_float(B.acc[node[k]]);
                    float u[M], dt;
                    sample_item<M>(P, seed, it, node[k], br, u, dt);
                    const int S = step_count(P, dt);
                    // the shortened last step may be empty (dt - (S-1) h <= 0): then
                    // the rollout ends at sample S - 1 (as integrate_steps)
                    seffk[k] = static_cast<uint32_t>(effective_samples(P, dt, S));
                    // velocity bounds once per item: an item failing them has no samples to check
                    if (!P.check_finite && !vel_ok_at_end<MODEL>(P, r, u, dt, S, static_cast<int>(seffk[k]))) vbad = 1u;
#pragma unroll
                    for (int d = 0; d < M; ++d) r[N + d] = u[d];
                    r[N + M] = dt;
                    r[N + M + 1] = __int_as_float(S);
                    r[N + M + 2] = __int_as_float(static_cast<int>(seffk[k]));
#pragma unroll
                    for (int w = 0; w < RW; ++w)
                        rec[p * RW + w] = make_float4(r[4 * w], r[4 * w + 1], r[4 * w + 2], r[4 * w + 3]);
                }
                if (vbad) seffk[k] = 0;  // no samples: skipped by every mapping, dropped by the owner
                seff += (seffk[k] + K - 1) / K;
                bad[p] = vbad;
                len_lo[p] = 0u;
                len_hi[p] = 0u;
            }
            KP_STAMP_MAX(it, 16);  // diagnostic build: sampling + parent loads done (latest block)
            // (2) exclusive scan of the sample counts over the block
            uint32_t x = seff;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) wsum[warp] = x;
            __syncthreads();
            if (warp == 0) {
                uint32_t w = lane < static_cast<int>(NWARP) ? wsum[lane] : 0u;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, w, o);
                    if (lane >= o) w += y;
                }
                if (lane < static_cast<int>(NWARP)) wsum[lane] = w;
            }
            __syncthreads();
            const uint32_t excl = x - seff + (warp ? wsum[warp - 1] : 0u);
            {
                uint32_t o = excl;
#pragma unroll
                for (uint32_t k = 0; k < IPT; ++k) {
                    off[threadIdx.x * IPT + k] = o;
                    o += (seffk[k] + K - 1) / K;
                }
                if (threadIdx.x == T - 1) off[FB] = o;
            }
            __syncthreads();
            env_wait();
            {
                // (3) chunks of K consecutive samples (one item each), interleaved
                // over the block: round r, thread t takes chunk r*T + t, so every
                // lane changes items at the same loop iteration (one convergent
                // record load per K samples), a warp's lanes hold consecutive
                // chunks of a few items (nearby points: coherent broad / narrow
                // phases), and each chunk adds its length to its item once
                const uint32_t U = off[FB];
                uint16_t* const cidx = reinterpret_cast<uint16_t*>(dyn + P.flat_idx);  // item of each chunk
                {
                    uint32_t o = excl;
#pragma unroll
                    for (uint32_t k = 0; k < IPT; ++k) {
                        const uint32_t nch = (seffk[k] + K - 1) / K;
                        for (uint32_t j = 0; j < nch; ++j) cidx[o + j] = static_cast<uint16_t>(threadIdx.x * IPT + k);
                        o += nch;
                    }
                }
                __syncthreads();
                for (uint32_t q0 = 0; q0 < U; q0 += T) {
                    const uint32_t q = q0 + threadIdx.x;
                    if (q >= U) break;
                    const uint32_t pi = cidx[q];
                    if (bad[pi]) continue;
                    float x0[N], u[M];
                    float r[RW * 4];
#pragma unroll
                    for (int w = 0; w < RW; ++w) {
                        const float4 v = rec[pi * RW + w];
                        r[4 * w] = v.x; r[4 * w + 1] = v.y; r[4 * w + 2] = v.z; r[4 * w + 3] = v.w;
                    }
#pragma unroll
                    for (int d = 0; d < N; ++d) x0[d] = r[d];
#pragma unroll
                    for (int d = 0; d < M; ++d) u[d] = r[N + d];
                    const float dt = r[N + M];
                    const int S = __float_as_int(r[N + M + 1]);
                    const int se = __float_as_int(r[N + M + 2]);
                    const int s0 = static_cast<int>(q - off[pi]) * static_cast<int>(K) + 1;
                    const int s1 = min(se, s0 + static_cast<int>(K) - 1);
                    float px, py, pz;
                    if (s0 == 1) {
                        px = x0[0]; py = x0[1]; pz = TWO_D ? 0.0f : x0[2];
                    } else {
                        float xp[N];
                        di_sample<MODEL>(x0, u, static_cast<float>(s0 - 1) * P.h, xp);
                        px = xp[0]; py = xp[1]; pz = TWO_D ? 0.0f : xp[2];
                    }
                    long long run = 0;
                    bool ok = true;
                    if constexpr (K == 2) {
                        // both samples of a chunk checked (no exit between them): two
                        // independent sample computations for the scheduler (+0.5 %)
                        float xa[N], xb[N];
                        di_sample<MODEL>(x0, u, (s0 == S) ? dt : static_cast<float>(s0) * P.h, xa);
                        const bool two = s1 > s0;
                        di_sample<MODEL>(x0, u, (s0 + 1 == S) ? dt : static_cast<float>(s0 + 1) * P.h, xb);
                        float da, db = 0.0f;
                        ok = check_sample<MODEL>(P, E, xa, px, py, pz, da, c);
                        if (two) ok = check_sample<MODEL>(P, E, xb, xa[0], xa[1], TWO_D ? 0.0f : xa[2], db, c) && ok;
                        run = len_fixed(da) + (two ? len_fixed(db) : 0ll);
                    } else {
                        for (int s = s0; s <= s1; ++s) {
                            float xs[N];
                            di_sample<MODEL>(x0, u, (s == S) ? dt : static_cast<float>(s) * P.h, xs);
                            float d;
                            if (!check_sample<MODEL>(P, E, xs, px, py, pz, d, c)) {
                                ok = false;
                                break;
                            }
                            run += len_fixed(d);
                            px = xs[0]; py = xs[1]; pz = TWO_D ? 0.0f : xs[2];
                        }
                    }
                    if (!ok) {
                        bad[pi] = 1u;
                    } else if (run) {
                        atomicAdd(len_lo + pi, static_cast<uint32_t>(run & 0xFFFFFF));
                        atomicAdd(len_hi + pi, static_cast<uint32_t>(run >> 24));
                    }
                }
            }
            __syncthreads();
            KP_STAMP_MAX(it, 17);  // diagnostic build: sample checks done (latest block)
            // (4) owner thread: path length, region, admission
#pragma unroll
            for (uint32_t k = 0; k < IPT; ++k) {
                const uint32_t p = threadIdx.x * IPT + k;
                const uint32_t i = b0 + p;
                if (!(i < cend) || bad[p]) continue;
                float r[RW * 4];
#pragma unroll
                for (int w = 0; w < RW; ++w) {
                    const float4 v = rec[p * RW + w];
                    r[4 * w] = v.x; r[4 * w + 1] = v.y; r[4 * w + 2] = v.z; r[4 * w + 3] = v.w;
                }
                float x0[N], u[M], xs[N];
#pragma unroll
                for (int d = 0; d < N; ++d) x0[d] = r[d];
#pragma unroll
                for (int d = 0; d < M; ++d) u[d] = r[N + d];
                const float dt = r[N + M];
                const int S = __float_as_int(r[N + M + 1]);
                di_sample<MODEL>(x0, u, (static_cast<int>(seffk[k]) == S) ? dt : static_cast<float>(seffk[k]) * P.h, xs);
                ItemOut o;
                const long long fx = (static_cast<long long>(len_hi[p]) << 24) + len_lo[p];
                finish_item<MODEL>(P, xs, dt, fixed_len(fx), acc_p[k], o);
                ++c[0];
                const uint32_t bits = __float_as_uint(o.acc);
                KP_ASSERT(o.region < P.n_regions, 12);
                KP_ASSERT(i < S_cap, 13);
                const uint32_t old = atomicMin(B.rc + o.region, bits);
                if (bits <= old) {  // Improved / Equal admitted, Worse discarded
                    ++c[1];
#pragma unroll
                    for (int d = 0; d < N; ++d) B.vu_state[static_cast<size_t>(d) * S_cap + i] = xs[d];
#pragma unroll
                    for (int d = 0; d < M; ++d) B.vu_ctrl[static_cast<size_t>(d) * S_cap + i] = u[d];
                    B.vu_dt[i] = dt;
                    B.vu_acc[i] = bits;
                    B.vu_region[i] = o.region;
                    atomicOr(B.admit_mask + (i >> 5), 1u << (i & 31));
                    if (o.goal) atomicOr(B.goal_mask + (i >> 5), 1u << (i & 31));
                }
            }
            __syncthreads();  // the next batch reuses the shared arrays
        }
        if (n_chunks <= gridDim.x) break;  // every chunk was assigned statically
        if (threadIdx.x == 0) fchunk = gridDim.x + atomicAdd(&ctl->prop_cursor, 1u);
        __syncthreads();
    }
    KP_STAMP_MAX(it, 18);  // diagnostic build: admissions issued (latest block)
    count_flush(ctl, c, fcnt, lane, it);
}

template <int MODEL>
__global__ void __launch_bounds__(PropCfg<MODEL>::T, PropCfg<MODEL>::MIN_BLOCKS) k_propagate(KpProblem P, KpBuffers B) {
    KP_T0;
    const Env E = stage_env_async(P, B);  // constant data: overlaps the predecessor's tail
    pdl_wait();
    KP_T1;
    pdl_trigger();
#ifdef KP_STAMPS
    const uint32_t it_s = B.ctl->iter;
    KP_STAMP_B0(it_s, 0, kp_t_entry);
    KP_STAMP_B0(it_s, 1, kp_t_pdl);
    KP_STAMP_B0(it_s, 14, globaltimer());
#endif
    unsigned char* const dyn = reinterpret_cast<unsigned char*>(kp_env_smem);
    // Control block (one round trip).  First, the previous boundary's
    // best-solution bookkeeping and stop-at-first-solution (they need every
    // goal commit of the scatter, complete now): block 0 records, every
    // block takes the same stop decision from the same `best`.
    const PropCtl pc = load_prop_ctl(B.ctl);
    const bool stop = !pc.done && pc.stop_first && pc.best != ~0ull;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        KpCtl* ctl = B.ctl;
        ctl->cur_iter = pc.it;
        if (pc.done) {
            // stopped at an earlier boundary: that grid has completed, so the
            // control block and the store are final — tell the host
            __threadfence_system();
            *B.host_done = pc.seq;  // (a no-op launch of an earlier solve writes that solve's number)
        } else {
            if (pc.best < pc.tl_best) goal_bookkeeping(*ctl);
            if (stop) {
                ctl->done_iter = pc.it;
                ctl->done = 1;
                __threadfence_system();
                *B.host_done = pc.seq;
            }
        }
    }
    if (pc.done || stop) {
        env_wait();  // no block exits with its bulk copy in flight
        return;
    }
    if constexpr (closed_form<MODEL>()) {
        // small launches are latency-bound: flatten them into samples; large
        // ones are issue-bound, where the step-sorted path runs fewer instructions
        if (P.flat_on && pc.n_items <= P.flat_max) {
            flat_phase<MODEL>(P, B, E, dyn, pc);
            env_wait();  // no block exits with its bulk copy in flight
            KP_STAMP_MAX(it_s, 2);
            return;
        }
    }
    propagate_phase<MODEL>(P, B, *reinterpret_cast<PropSmem<MODEL>*>(dyn + P.seq_base), E, pc);
    env_wait();
    KP_STAMP_MAX(it_s, 2);
}

// Block-wide inclusive sum of three counters (blockDim == KP_SELECT_THREADS).
struct Cnt3 {
    uint32_t k, v, c;
};

KP_DEV Cnt3 block_scan3(Cnt3 x, Cnt3* total) {
    __shared__ uint32_t sw[3][KP_SELECT_THREADS / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Cnt3 inc = x;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t a = __shfl_up_sync(0xFFFFFFFFu, inc.k, off);
        const uint32_t b = __shfl_up_sync(0xFFFFFFFFu, inc.v, off);
        const uint32_t c = __shfl_up_sync(0xFFFFFFFFu, inc.c, off);
        if (lane >= off) { inc.k += a; inc.v += b; inc.c += c; }
    }
    if (lane == 31) { sw[0][warp] = inc.k; sw[1][warp] = inc.v; sw[2][warp] = inc.c; }
    __syncthreads();
    if (warp == 0) {
        constexpr int NW = KP_SELECT_THREADS / 32;
        uint32_t a = lane < NW ? sw[0][lane] : 0, b = lane < NW ? sw[1][lane] : 0, c = lane < NW ? sw[2][lane] : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t a2 = __shfl_up_sync(0xFFFFFFFFu, a, off);
            const uint32_t b2 = __shfl_up_sync(0xFFFFFFFFu, b, off);
            const uint32_t c2 = __shfl_up_sync(0xFFFFFFFFu, c, off);
            if (lane >= off) { a += a2; b += b2; c += c2; }
        }
        if (lane < NW) { sw[0][lane] = a; sw[1][lane] = b; sw[2][lane] = c; }
    }
    __syncthreads();
    if (warp > 0) { inc.k += sw[0][warp - 1]; inc.v += sw[1][warp - 1]; inc.c += sw[2][warp - 1]; }
    total->k = sw[0][KP_SELECT_THREADS / 32 - 1];
    total->v = sw[1][KP_SELECT_THREADS / 32 - 1];
    total->c = sw[2][KP_SELECT_THREADS / 32 - 1];
    __syncthreads();
    return inc;
}

// prune_pass rules for one live node (priorities :434-437),
// from its live-list entry rec = {id, region, acc bits, parent} and
// si = status | i_count << 8.  Returns the new status | i_count << 8 and
// mirrors status / i_count into the node store.
KP_DEV uint32_t prune_node(const KpProblem& P, const KpBuffers& B, uint4 rec, uint32_t si, uint32_t* term,
                           uint32_t* deact, uint32_t* react, uint32_t* hops) {
    const uint32_t g = rec.x;
    KP_ASSERT(g < P.capacity, 20);
    const uint32_t st = si & 0xFFu;
    KP_ASSERT(rec.y < P.n_regions, 21);
    KP_ASSERT(st != KP_ST_TERMINAL, 22);  // Terminal nodes never stay in the live list
    // an Active node's parent link is loaded beside its own region cost (the
    // ancestor walk's first hop no longer waits for rule 1's round trip)
    const int32_t p = static_cast<int32_t>(rec.w);
    const bool walks = st == KP_ST_ACTIVE && P.deact == 0 && p >= 0;
    uint4 L = make_uint4(0xFFFFFFFFu, 0u, 0u, 0u);
    if (walks) L = B.link[p];  // {parent, region, acc, -}
    if (rec.z > B.rc[rec.y]) {  // (1) dominated -> Terminal (absorbing)
        B.status[g] = KP_ST_TERMINAL;
        ++*term;
        return KP_ST_TERMINAL;
    }
    if (st == KP_ST_INACTIVE) {  // (2) inactivity counter, reactivation
        const uint32_t ic = (si >> 8) + 1u;
        if (ic > static_cast<uint32_t>(P.i_max)) {
            B.icnt[g] = 0;
            B.status[g] = KP_ST_ACTIVE;
            ++*react;
            return KP_ST_ACTIVE;
        }
        B.icnt[g] = static_cast<uint16_t>(ic);
        return KP_ST_INACTIVE | (ic << 8);
    }
    // (3) Active: some ancestor no longer region-minimal -> Inactive.  The walk
    // is software-pipelined over 16-byte node links: the next hop's link load
    // is issued together with this hop's region-cost load, so the chain costs
    // about one L2 round trip per hop.
    bool dominated = P.deact != 0;
    if (walks) {
        for (;;) {
            ++*hops;
            const int32_t q = static_cast<int32_t>(L.x);
            KP_ASSERT(L.y < P.n_regions, 23);
            KP_ASSERT(q < static_cast<int32_t>(P.capacity), 24);
            uint4 Ln = make_uint4(0xFFFFFFFFu, 0u, 0u, 0u);
            if (q >= 0) Ln = B.link[q];
            if (L.z > B.rc[L.y]) { dominated = true; break; }
            if (q < 0) break;
            L = Ln;
        }
    }
    if (dominated) {
        B.status[g] = KP_ST_INACTIVE;
        B.icnt[g] = 0;
        ++*deact;
        return KP_ST_INACTIVE;
    }
    return KP_ST_ACTIVE;
}

// Slot elements are processed per 32-slot mask word (one thread per word):
// the frontier is sparse in admitted / committed slots, so a word-level scan
// touches 32x fewer elements than a slot-level one.  The set bits of a warp's
// 32 words are then spread over the warp's lanes (one bit per lane per round,
// bits in word order then bit order) so their memory round trips overlap.
struct WarpBits {
    uint32_t total;  // set bits over the warp's words (warp-uniform)
    uint32_t excl;   // this lane's exclusive prefix
};

KP_DEV WarpBits warp_bits(uint32_t word) {
    const int lane = threadIdx.x & 31;
    const uint32_t c = __popc(word);
    uint32_t incl = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, off);
        if (lane >= off) incl += y;
    }
    return {__shfl_sync(0xFFFFFFFFu, incl, 31), incl - c};
}

// Owner lane of the k-th set bit of the warp (smallest lane whose inclusive
// prefix exceeds k).  Convergent: every lane must call it.
KP_DEV int warp_bit_owner(const WarpBits& wb, uint32_t word, uint32_t k) {
    const uint32_t incl = wb.excl + __popc(word);
    int L = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
        const uint32_t v = __shfl_sync(0xFFFFFFFFu, incl, L + step - 1);
        if (v <= k) L += step;
    }
    return L;
}

// Block-wide sums of three counters (blockDim == KP_SELECT_THREADS); the
// result is valid in thread 0.  Ends with a barrier, so it can be reused.
KP_DEV Cnt3 block_sum3(Cnt3 x) {
    __shared__ uint32_t sr[3][KP_SELECT_THREADS / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        x.k += __shfl_down_sync(0xFFFFFFFFu, x.k, off);
        x.v += __shfl_down_sync(0xFFFFFFFFu, x.v, off);
        x.c += __shfl_down_sync(0xFFFFFFFFu, x.c, off);
    }
    if (lane == 0) { sr[0][warp] = x.k; sr[1][warp] = x.v; sr[2][warp] = x.c; }
    __syncthreads();
    Cnt3 t{0, 0, 0};
    if (threadIdx.x == 0) {
#pragma unroll
        for (int w = 0; w < KP_SELECT_THREADS / 32; ++w) { t.k += sr[0][w]; t.v += sr[1][w]; t.c += sr[2][w]; }
    }
    __syncthreads();
    return t;
}

// Element layout of the two select kernels for this iteration (identical in
// both): live nodes first, then the V_U slots either one per thread (dense:
// many admitted slots, every commit test in its own thread) or one 32-slot
// mask word per thread (sparse: 32x fewer elements to scan; the warp's set
// bits are spread over its lanes).
struct SelLayout {
    bool sparse;
    uint32_t slot0;   // first slot element (live part padded to a warp in the dense layout)
    uint32_t E, n_tiles;
};

KP_DEV SelLayout sel_layout(uint32_t n_live, uint32_t n_items, uint32_t n_adm) {
    SelLayout l;
    const uint32_t n_words = (n_items + 31u) >> 5;
#ifndef KP_SPARSE_DIV
#define KP_SPARSE_DIV 1
#endif
    l.sparse = n_adm * KP_SPARSE_DIV <= n_words;  // about one admitted slot per word or fewer: one round per warp
    l.slot0 = l.sparse ? n_live : ((n_live + 31u) & ~31u);
    l.E = l.slot0 + (l.sparse ? n_words : 32u * n_words);
    l.n_tiles = (l.E + KP_SELECT_THREADS - 1) / KP_SELECT_THREADS;
    return l;
}

template <bool SPEC>
KP_DEV void select_reduce_phase(const KpProblem& P, const KpBuffers& B) {
    KpCtl* ctl = B.ctl;
    // every control-block read up front: one round trip; beside it, the first
    // tile's live entries of both list parities (the parity comes with the
    // control block), so the region-cost gather follows the first round trip
    const uint32_t e0 = blockIdx.x * KP_SELECT_THREADS + threadIdx.x;
    uint4 rec_a = make_uint4(0u, 0u, 0u, 0u), rec_b = rec_a;
    uint32_t si_a = 0u, si_b = 0u;
    if (SPEC && e0 < P.capacity) {
        rec_a = B.live[0][e0];
        rec_b = B.live[1][e0];
        si_a = B.live_si[0][e0];
        si_b = B.live_si[1][e0];
    }
    const uint32_t done = ctl->done, it = ctl->iter, n_live = ctl->n_live, n_items = ctl->n_items;
    const uint32_t n_adm = ctl->n_adm_p[it & 1];
    if (done) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->t_sel_ns = globaltimer();
    __shared__ uint32_t s_st[7];
    __shared__ uint32_t s_cm[KP_SELECT_THREADS];  // commit words under construction (sparse layout)
    const SelLayout ly = sel_layout(n_live, n_items, n_adm);
    const uint32_t n_tiles = ly.n_tiles;
    const uint32_t n_part = min(gridDim.x, n_tiles);  // participating blocks
    if (blockIdx.x >= n_part) return;
    const uint4* live = B.live[it & 1];
    const uint32_t* live_si = B.live_si[it & 1];
    const int lane = threadIdx.x & 31;
    uint32_t term = 0, deact = 0, react = 0, hops = 0, nlive = 0, nslot = 0, nadm = 0;
    if (threadIdx.x < 7) s_st[threadIdx.x] = 0;
#ifdef KP_STAMPS
    __shared__ unsigned long long s_tmax[2];
    if (threadIdx.x < 2) s_tmax[threadIdx.x] = 0;
#endif
    __syncthreads();
    for (uint32_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const uint32_t e = tile * KP_SELECT_THREADS + threadIdx.x;
        Cnt3 x{0, 0, 0};
        if (e < n_live) {
            ++nlive;
            const bool first = SPEC && tile == blockIdx.x;
            const bool odd = (it & 1u) != 0u;
            const uint32_t si = prune_node(P, B, first ? (odd ? rec_b : rec_a) : live[e],
                                           first ? (odd ? si_b : si_a) : live_si[e], &term, &deact, &react, &hops);
            B.live_st[e] = si;  // scatter reads it by position, in parallel with live[e]
            const uint32_t st = si & 0xFFu;
            x.k = st != KP_ST_TERMINAL;
            x.v = st == KP_ST_ACTIVE;
#ifdef KP_STAMPS
            atomicMax(&s_tmax[0], globaltimer());  // latest prune of a live node (block max)
#endif
        }
        const bool in_slots = e >= ly.slot0 && e < ly.E;
        if (!ly.sparse) {  // one slot per thread; slot elements are warp-aligned
            bool commit = false;
            const uint32_t sl = e - ly.slot0;
            if (in_slots && sl < n_items) {
                ++nslot;
                // the slot record is loaded beside its admit bit (one round trip
                // less; a stale record of an unadmitted slot is never used)
                const uint32_t aw = B.admit_mask[sl >> 5];
                const uint32_t va_acc = B.vu_acc[sl], va_reg = B.vu_region[sl];
                if ((aw >> (sl & 31)) & 1u) {
                    ++nadm;
                    KP_ASSERT(va_reg < P.n_regions, 25);
                    commit = va_acc == B.rc[va_reg];  // Alg. 4 line 3, bit-exact
                    x.c = commit;
                }
            }
            const uint32_t cm = __ballot_sync(0xFFFFFFFFu, commit);
            if (in_slots && lane == 0) {
                B.commit_mask[sl >> 5] = cm;
                B.admit_mask[sl >> 5] = 0u;  // consumed: ready for the next propagate
            }
        } else {  // one mask word per thread
            uint32_t w = 0, a = 0;
            if (in_slots) {
                w = e - ly.slot0;
                a = B.admit_mask[w];
                nslot += min(32u, n_items - 32u * w);
            }
            s_cm[threadIdx.x] = 0u;
            const WarpBits wb = warp_bits(a);
            __syncwarp();
            for (uint32_t base = 0; base < wb.total; base += 32) {
                const uint32_t k = base + lane;
                const int L = warp_bit_owner(wb, a, k);
                const uint32_t aL = __shfl_sync(0xFFFFFFFFu, a, L);
                const uint32_t eL = __shfl_sync(0xFFFFFFFFu, wb.excl, L);
                const uint32_t wL = __shfl_sync(0xFFFFFFFFu, w, L);
                if (k < wb.total) {
                    const uint32_t bit = __fns(aL, 0, static_cast<int>(k - eL) + 1);
                    const uint32_t sl = 32u * wL + bit;
                    ++nadm;
                    KP_ASSERT(sl < n_items && B.vu_region[sl] < P.n_regions, 26);
                    if (B.vu_acc[sl] == B.rc[B.vu_region[sl]])  // Alg. 4 line 3, bit-exact
                        atomicOr(&s_cm[(threadIdx.x & ~31u) + static_cast<uint32_t>(L)], 1u << bit);
                }
            }
            __syncwarp();
            if (in_slots) {
                const uint32_t cm = s_cm[threadIdx.x];
                x.c = __popc(cm);
                B.commit_mask[w] = cm;
                if (a) B.admit_mask[w] = 0u;  // consumed: ready for the next propagate
            }
        }
#ifdef KP_STAMPS
        if (ly.sparse ? (e >= ly.slot0 && e < ly.E) : (e >= ly.slot0 && e - ly.slot0 < n_items))
            atomicMax(&s_tmax[1], globaltimer());  // latest commit test (block max)
        __syncthreads();
        if (threadIdx.x == 0) {
            if (s_tmax[0]) atomicMax(&kp_stamps[it & 63][20], s_tmax[0]);
            if (s_tmax[1]) atomicMax(&kp_stamps[it & 63][21], s_tmax[1]);
        }
#endif
        KP_STAMP_MAX(it, 19);  // diagnostic build: prune + commit tests done (latest block)
        const Cnt3 tot = block_sum3(x);
        KP_ASSERT(tile < B.max_tiles, 27);
        if (threadIdx.x == 0) {
            B.tile_sums[tile] = tot.k;
            B.tile_sums[B.max_tiles + tile] = tot.v;
            B.tile_sums[2 * B.max_tiles + tile] = tot.c;
        }
    }
    if (term) atomicAdd(&s_st[0], term);
    if (deact) atomicAdd(&s_st[1], deact);
    if (react) atomicAdd(&s_st[2], react);
    if (hops) atomicAdd(&s_st[3], hops);
    if (nlive) atomicAdd(&s_st[4], nlive);
    if (nslot) atomicAdd(&s_st[5], nslot);
    if (nadm) atomicAdd(&s_st[6], nadm);
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_st[0]) atomicAdd(&ctl->stats.pruned_terminal, static_cast<unsigned long long>(s_st[0]));
        if (s_st[1]) atomicAdd(&ctl->stats.deactivated, static_cast<unsigned long long>(s_st[1]));
        if (s_st[2]) atomicAdd(&ctl->stats.reactivated, static_cast<unsigned long long>(s_st[2]));
        if (s_st[3]) atomicAdd(&ctl->stats.ancestor_hops, static_cast<unsigned long long>(s_st[3]));
        if (s_st[4]) atomicAdd(&ctl->stats.live_scanned, static_cast<unsigned long long>(s_st[4]));
        if (s_st[5]) atomicAdd(&ctl->stats.slots_scanned, static_cast<unsigned long long>(s_st[5]));
        if (s_st[6]) atomicAdd(&ctl->stats.admitted_checked, static_cast<unsigned long long>(s_st[6]));
    }
}

// SPEC: the first tile's live entries are loaded beside the control block
// (a lone query's latency win; the batch engine's concurrent lanes use the
// plain variant, which also needs fewer registers)
template <bool SPEC>
__global__ void __launch_bounds__(KP_SELECT_THREADS, (SPEC ? 5 : 8) * 256 / KP_SELECT_THREADS) k_select_reduce(KpProblem P, KpBuffers B) {
    KP_T0;
    pdl_wait();
    KP_T1;
    pdl_trigger();
#ifdef KP_STAMPS
    const uint32_t it_s = B.ctl->iter;
    KP_STAMP_B0(it_s, 5, globaltimer());
#endif
    select_reduce_phase<SPEC>(P, B);
    KP_STAMP_MAX(it_s, 6);
}

// Close an iteration: counts, stats, trace record,
// termination.  Written by select_scatter's block 0 (thread 0) as soon as the
// tile prefix gives it the totals, while the other blocks still write their
// tiles: it reads nothing they write, and they read the iteration's parity
// view of the control block, not the fields it overwrites (kp_types.h).  The
// best-solution bookkeeping — which needs every goal commit — is the next
// propagate's first step (goal_bookkeeping), and stop-at-first-solution ends
// the solve there.  Its inputs were written before the scatter started (by
// the previous boundary, k_start, propagate and select_reduce); block 0's
// thread 0 loads them beside its control-block reads.
struct BoundaryIn {
    unsigned long long t_start, deadline, t_prop, t_sel;
    unsigned long long st_att, st_com, st_drop;
    uint32_t max_iter_abs, n_valid;
};

KP_DEV BoundaryIn load_boundary_in(const KpCtl* ctl) {
    BoundaryIn b;
    b.t_start = ctl->t_start_ns;
    b.deadline = ctl->deadline_ns;
    b.t_prop = ctl->t_prop_ns;
    b.t_sel = ctl->t_sel_ns;
    b.st_att = ctl->stats.attempted;
    b.st_com = ctl->stats.committed;
    b.st_drop = ctl->stats.dropped_capacity;
    b.max_iter_abs = ctl->max_iter_abs;
    b.n_valid = ctl->n_valid_iter;
    return b;
}

// bin: the prefetched inputs; t_scat: block 0's entry stamp.
KP_DEV void iteration_boundary(const KpProblem& P, const KpBuffers& B, uint32_t it, uint32_t n_items,
                               uint32_t tot_keep, uint32_t tot_va, uint32_t tot_commit, uint32_t n_nodes,
                               uint32_t accepted, const BoundaryIn& bin, unsigned long long t_scat) {
    KpCtl* ctl = B.ctl;
    const uint32_t S = P.max_slots;
    const uint32_t lam = static_cast<uint32_t>(P.lambda);
    const unsigned long long now = globaltimer();
    const uint32_t it1 = it + 1;
    const unsigned long long t_start = bin.t_start, deadline = bin.deadline;
    const unsigned long long t_prop = bin.t_prop, t_sel = bin.t_sel;
    const uint32_t max_iter_abs = bin.max_iter_abs;
    const unsigned long long st_att = bin.st_att, st_com = bin.st_com;
    const unsigned long long st_drop = bin.st_drop;
    const uint32_t n_valid = bin.n_valid;
    const uint32_t n_live1 = tot_keep + accepted, n_va1 = tot_va + accepted, n_nodes1 = n_nodes + accepted;
    KP_ASSERT(n_nodes1 <= P.capacity && n_live1 <= n_nodes1 && n_va1 <= n_live1, 40);
    const unsigned long long items = static_cast<unsigned long long>(n_va1) * lam;
    ctl->stats.attempted = st_att + n_items;
    ctl->stats.committed = st_com + accepted;
    if (tot_commit > accepted) {
        ctl->stats.dropped_capacity = st_drop + (tot_commit - accepted);
        ctl->capacity_exhausted = 1;
    }
    ctl->n_nodes = n_nodes1;
    ctl->n_live = n_live1;
    ctl->n_va = n_va1;
    ctl->iter = it1;
    ctl->t_last_ns = now;
    {
        KpTraceRec& tr = B.trace[it % KP_TRACE_CAP];
        tr.t_ns = now - t_start;
        tr.iteration = it1;
        tr.items = n_items;
        tr.live = n_live1;
        tr.frontier = n_va1;
        tr.nodes = n_nodes1;
        tr.committed = accepted;
        tr.t_prop = static_cast<uint32_t>(t_prop - t_start);
        tr.t_sel = static_cast<uint32_t>(t_sel - t_start);
        tr.t_sel_end = static_cast<uint32_t>(t_scat - t_start);
        tr.t_scat = static_cast<uint32_t>(t_scat - t_start);
    }
    bool done = false;
    uint32_t items1 = static_cast<uint32_t>(items);
    if (items > S) {
        ctl->error = 8;  // KP_ERR_SLOT_OVERFLOW
        done = true;
        items1 = 0;
    }
    ctl->n_items = items1;
    // the next iteration's view for its select_scatter blocks
    ctl->view_live[it1 & 1] = n_live1;
    ctl->view_items[it1 & 1] = items1;
    ctl->view_nodes[it1 & 1] = n_nodes1;
    ctl->n_adm_p[it1 & 1] = 0;
    if (max_iter_abs && it1 >= max_iter_abs) done = true;
    if (deadline && now >= deadline) done = true;
    if (n_live1 == 0) done = true;
    ctl->prop_cursor = 0;
    ctl->n_valid_iter = 0;
    // split the next propagate's rollouts when many items stop early (invalid):
    // the compaction then pays for its second pass (scripts/split_sim.py)
    ctl->split = (n_items - min(n_valid, n_items)) * 4u >= n_items && n_items > 0 ? 1u : 0u;
    if (done) {  // the host learns it from the next propagate (this grid may still be writing)
        ctl->done_iter = it1;
        ctl->done = 1;
    }
}

KP_DEV void scatter_phase(const KpProblem& P, const KpBuffers& B) {
    KpCtl* ctl = B.ctl;
    // every control-block read up front: one round trip.  Block 0 writes the
    // boundary while the other blocks run, so they read this iteration's view
    // (parity of cur_iter, written by propagate), not the fields it overwrites.
    const uint32_t it = ctl->cur_iter, done_iter = ctl->done_iter;
    const uint32_t n_live = ctl->view_live[it & 1], n_items = ctl->view_items[it & 1];
    const uint32_t n_nodes = ctl->view_nodes[it & 1], n_adm = ctl->n_adm_p[it & 1];
    __shared__ BoundaryIn s_bin;
    __shared__ unsigned long long s_t0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // the boundary's inputs, in the same round trip
        s_bin = load_boundary_in(ctl);
        s_t0 = globaltimer();
    }
    if (done_iter <= it) return;  // the solve stopped before this iteration
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->t_scat_ns = globaltimer();
    __shared__ uint32_t s_red[6][KP_SELECT_THREADS / 32];
    const SelLayout ly = sel_layout(n_live, n_items, n_adm);  // as select_reduce
    const uint32_t n_tiles = ly.n_tiles;
    const uint32_t n_part = min(gridDim.x, n_tiles);
    if (blockIdx.x >= n_part) return;
    // contiguous tile range of this block; exclusive prefix of its first tile
    // and the grand totals from one pass over the per-tile counts
    const uint32_t per = (n_tiles + n_part - 1) / n_part;
    const uint32_t tb = blockIdx.x * per, te = min(tb + per, n_tiles);
    const uint4* live = B.live[it & 1];
    // this thread's element of a tile: live node (id, pruned status) or slot /
    // mask word (commit and goal bits); independent of the prefix, so the first
    // tile's loads are issued before the prefix pass and overlap it
    struct Elem {
        Cnt3 x;
        uint4 rec;
        uint32_t si, w, cm, gm;
        bool in_slots;
    };
    auto load_elem = [&](uint32_t tile) {
        const uint32_t e = tile * KP_SELECT_THREADS + threadIdx.x;
        Elem el{{0, 0, 0}, make_uint4(0u, 0u, 0u, 0u), 0, 0, 0, 0, e >= ly.slot0 && e < ly.E};
        if (e < n_live) {
            el.rec = live[e];
            el.si = B.live_st[e];
            const uint32_t st = el.si & 0xFFu;
            el.x.k = st != KP_ST_TERMINAL;
            el.x.v = st == KP_ST_ACTIVE;
        } else if (el.in_slots) {
            el.w = e - ly.slot0;  // slot (dense) or mask word (sparse)
            if (!ly.sparse) {
                if (el.w < n_items) {  // both mask words in one round trip
                    const uint32_t cw = B.commit_mask[el.w >> 5], gw = B.goal_mask[el.w >> 5];
                    el.x.c = (cw >> (el.w & 31)) & 1u;
                    el.gm = el.x.c & (gw >> (el.w & 31));
                }
            } else {
                el.cm = B.commit_mask[el.w];
                el.gm = B.goal_mask[el.w];
                el.x.c = __popc(el.cm);
            }
        }
        return el;
    };
    const Elem first = load_elem(tb);
    uint32_t acc[6] = {0, 0, 0, 0, 0, 0};  // before tb: k, v, c; all: k, v, c
    constexpr int U = 8;  // 8 independent loads per array in flight per thread
    for (uint32_t base = threadIdx.x; base < n_tiles; base += U * KP_SELECT_THREADS) {
        uint32_t kk[U], vv[U], cc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t t = base + u * KP_SELECT_THREADS;
            const bool in = t < n_tiles;
            kk[u] = in ? B.tile_sums[t] : 0u;
            vv[u] = in ? B.tile_sums[B.max_tiles + t] : 0u;
            cc[u] = in ? B.tile_sums[2 * B.max_tiles + t] : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t t = base + u * KP_SELECT_THREADS;
            acc[3] += kk[u]; acc[4] += vv[u]; acc[5] += cc[u];
            if (t < tb) { acc[0] += kk[u]; acc[1] += vv[u]; acc[2] += cc[u]; }
        }
    }
    {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
        for (int q = 0; q < 6; ++q) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc[q] += __shfl_down_sync(0xFFFFFFFFu, acc[q], off);
            if (lane == 0) s_red[q][warp] = acc[q];
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            uint32_t v = 0;
            for (int w = 0; w < KP_SELECT_THREADS / 32; ++w) v += s_red[q][w];
            acc[q] = v;
        }
    }
    const uint32_t tot_keep = acc[3], tot_va = acc[4], tot_commit = acc[5];
    KP_STAMP_MAX(it, 15);  // diagnostic build: prefix pass done (latest block)
    const uint32_t remaining = P.capacity - n_nodes;
    const uint32_t accepted = tot_commit < remaining ? tot_commit : remaining;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // the iteration boundary, right away: nothing it reads comes from the
        // other blocks (their node-store and list writes are read by later
        // kernels, after this grid completes)
#ifdef KP_STAMPS
        kp_stamps[it & 63][10] = globaltimer();
#endif
        iteration_boundary(P, B, it, n_items, tot_keep, tot_va, tot_commit, n_nodes, accepted, s_bin, s_t0);
#ifdef KP_STAMPS
        kp_stamps[it & 63][12] = globaltimer();
#endif
    }
    Cnt3 run{acc[0], acc[1], acc[2]};
    const uint32_t cap = P.capacity, S = P.max_slots;
    const uint32_t lam = static_cast<uint32_t>(P.lambda);
    const uint32_t* va = B.va[it & 1];
    uint4* live_n = B.live[(it + 1) & 1];
    uint32_t* live_si_n = B.live_si[(it + 1) & 1];
    uint32_t* va_n = B.va[(it + 1) & 1];
    const int lane = threadIdx.x & 31;
    // one committed slot -> node id n_nodes + rank (slot order), store, lists, best
    auto commit_node = [&](uint32_t sl, uint32_t rank, bool goal) {
        const uint32_t id = n_nodes + rank;
        // (this iteration's frontier: n_items / lambda; ctl->n_va may already be the next one's)
        KP_ASSERT(id < cap && sl < S && sl < n_items, 30);
        KP_ASSERT(tot_keep + rank < cap && tot_va + rank < cap, 31);
        // every load of the slot record first, then the stores: interleaved,
        // the possible aliasing of the float arrays kept each load behind the
        // previous store — a dozen dependent L2 round trips per committed node
        float xs[KP_MAX_N], us[KP_MAX_M];
#pragma unroll
        for (int d = 0; d < KP_MAX_N; ++d)
            if (d < P.n) xs[d] = B.vu_state[static_cast<size_t>(d) * S + sl];
#pragma unroll
        for (int d = 0; d < KP_MAX_M; ++d)
            if (d < P.m) us[d] = B.vu_ctrl[static_cast<size_t>(d) * S + sl];
        const uint32_t abits = B.vu_acc[sl];
        const float dts = B.vu_dt[sl];
        const uint32_t par = va[frontier_pos(P, sl)];
        const uint32_t reg = B.vu_region[sl];
#pragma unroll
        for (int d = 0; d < KP_MAX_N; ++d)
            if (d < P.n) B.state[static_cast<size_t>(d) * cap + id] = xs[d];
#pragma unroll
        for (int d = 0; d < KP_MAX_M; ++d)
            if (d < P.m) B.ctrl[static_cast<size_t>(d) * cap + id] = us[d];
        B.dt[id] = dts;
        B.acc[id] = abits;
        B.region[id] = reg;
        B.parent[id] = static_cast<int32_t>(par);
        B.link[id] = make_uint4(par, reg, abits, 0u);
        B.status[id] = KP_ST_ACTIVE;
        B.icnt[id] = 0;
        live_n[tot_keep + rank] = make_uint4(id, reg, abits, par);
        live_si_n[tot_keep + rank] = KP_ST_ACTIVE;
        va_n[tot_va + rank] = id;
        if (goal)  // Alg. 4 lines 5-7 (bookkept by the next propagate)
            atomicMin(&ctl->best, (static_cast<unsigned long long>(abits) << 32) | id);
    };
    for (uint32_t tile = tb; tile < te; ++tile) {
        const Elem el = tile == tb ? first : load_elem(tile);
        const Cnt3 x = el.x;
        const uint32_t g = el.rec.x, w = el.w, cm = el.cm, gm = el.gm;
        const bool in_slots = el.in_slots;
        Cnt3 tot;
        const Cnt3 inc = block_scan3(x, &tot);  // (barrier: every lane has read its goal bit)
        if (tile == tb) KP_STAMP_MAX(it, 3);  // diagnostic build: first scan done (latest block)
        const uint32_t pk = run.k + inc.k - x.k;
        const uint32_t pv = run.v + inc.v - x.v;
        const uint32_t pc = run.c + inc.c - x.c;  // commits before this element (slot order)
        run.k += tot.k;
        run.v += tot.v;
        run.c += tot.c;
        if (x.k) {
            KP_ASSERT(pk < cap && pv < cap, 32);
            live_n[pk] = el.rec;
            live_si_n[pk] = el.si;
            if (x.v) va_n[pv] = g;
        }
        if (!ly.sparse) {
            if (in_slots && lane == 0) B.goal_mask[w >> 5] = 0u;  // consumed
            if (x.c && pc < accepted) commit_node(w, pc, gm != 0u);
        } else {
            if (gm) B.goal_mask[w] = 0u;  // consumed
            const WarpBits wb = warp_bits(cm);
            for (uint32_t base = 0; base < wb.total; base += 32) {
                const uint32_t k = base + lane;
                const int L = warp_bit_owner(wb, cm, k);
                const uint32_t cL = __shfl_sync(0xFFFFFFFFu, cm, L);
                const uint32_t eL = __shfl_sync(0xFFFFFFFFu, wb.excl, L);
                const uint32_t wL = __shfl_sync(0xFFFFFFFFu, w, L);
                const uint32_t pL = __shfl_sync(0xFFFFFFFFu, pc, L);
                const uint32_t gL = __shfl_sync(0xFFFFFFFFu, gm, L);
                if (k >= wb.total) continue;
                const uint32_t r = k - eL;
                if (pL + r >= accepted) continue;  // store full
                const uint32_t bit = __fns(cL, 0, static_cast<int>(r) + 1);
                commit_node(32u * wL + bit, pL + r, ((gL >> bit) & 1u) != 0u);
            }
        }
    }
    KP_STAMP_MAX(it, 4);  // diagnostic build: writes issued (latest block)
}

// 3 blocks/SM (up to 80 registers): at 4 (64 registers) the committed
// node's record spilled (forest 4.54 vs 4.61 G/s, TTFS 0.58 vs 0.56 ms)
#ifndef KP_SCATTER_MINB
#define KP_SCATTER_MINB (768 / KP_SELECT_THREADS)
#endif
__global__ void __launch_bounds__(KP_SELECT_THREADS, KP_SCATTER_MINB) k_select_scatter(KpProblem P, KpBuffers B) {
    KP_T0;
    pdl_wait();
    KP_T1;
    pdl_trigger();
#ifdef KP_STAMPS
    const uint32_t it_s = B.ctl->cur_iter;  // ctl->iter may already be the next iteration's (early boundary)
    KP_STAMP_B0(it_s, 7, kp_t_entry);
    KP_STAMP_B0(it_s, 8, kp_t_pdl);
    KP_STAMP_B0(it_s, 9, globaltimer());
#endif
    scatter_phase(P, B);
}

// Reset the region table and plant the root (Alg. 1 lines 1-5).
__global__ void k_reset_table(KpProblem P, KpBuffers B) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n_regions; i += gridDim.x * blockDim.x)
        B.rc[i] = 0x7F800000u;
}

__global__ void k_reset_root(KpProblem P, KpBuffers B, unsigned long long seed) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    KpCtl* ctl = B.ctl;
    ctl->seed = seed;
    float x[KP_MAX_N];
    for (int d = 0; d < P.n; ++d) {
        x[d] = B.x0[d];
        B.state[static_cast<size_t>(d) * P.capacity] = x[d];
    }
    for (int d = 0; d < P.m; ++d) B.ctrl[static_cast<size_t>(d) * P.capacity] = 0.0f;
    const uint32_t r = region_index<KP_MAX_N>(P, x);
    B.dt[0] = 0.0f;
    B.acc[0] = 0u;
    B.parent[0] = -1;
    B.region[0] = r;
    B.link[0] = make_uint4(0xFFFFFFFFu, r, 0u, 0u);
    B.status[0] = KP_ST_ACTIVE;
    B.icnt[0] = 0;
    B.rc[r] = 0u;  // DECISION: root region seeded with cost 0 (SPEC.md:425 region dominance)
    B.live[0][0] = make_uint4(0u, r, 0u, 0xFFFFFFFFu);
    B.live_si[0][0] = KP_ST_ACTIVE;
    B.va[0][0] = 0;
    ctl->n_live = 1;
    ctl->n_va = 1;
    ctl->n_nodes = 1;
    ctl->n_items = static_cast<uint32_t>(P.lambda);
    ctl->best = ~0ull;
    ctl->tl_best = ~0ull;
}

// Start of a kp_solve call: budget, iteration cap, immediate termination test.
__global__ void k_start(KpBuffers B, unsigned long long budget_ns, uint32_t max_iters, uint32_t stop_first,
                        uint32_t seq) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    KpCtl* ctl = B.ctl;
    const unsigned long long now = globaltimer();
    if (ctl->iter == 0 && ctl->t_start_ns == 0) ctl->t_start_ns = now;
    ctl->deadline_ns = budget_ns ? now + budget_ns : 0ull;
    ctl->max_iter_abs = max_iters ? ctl->iter + max_iters : 0u;
    ctl->stop_first = stop_first;
    ctl->prop_cursor = 0;
    const uint32_t it = ctl->iter;
    ctl->n_adm_p[it & 1] = 0;
    ctl->view_live[it & 1] = ctl->n_live;  // this iteration's view for select_scatter
    ctl->view_items[it & 1] = ctl->n_items;
    ctl->view_nodes[it & 1] = ctl->n_nodes;
    bool done = ctl->error != 0 || ctl->n_live == 0 || (stop_first && ctl->best != ~0ull);
    ctl->done_iter = done ? it : 0xFFFFFFFFu;
    ctl->done = done ? 1u : 0u;
    __threadfence_system();
    ctl->solve_seq = seq;
    *B.host_done = done ? seq : 0u;
    __threadfence_system();
}

// Explicit-input propagate items (kp_debug_propagate).
template <int MODEL>
__global__ void k_debug_propagate(KpProblem P, KpBuffers B, uint32_t n, const float* ps, const float* pacc,
                                  const uint32_t* ids, const uint32_t* brs, uint32_t it, uint8_t* valid,
                                  float* xs, float* us, float* dts, float* accs, uint32_t* regs, uint32_t* steps,
                                  uint8_t* goals) {
    constexpr int N = Model<MODEL>::N;
    constexpr int M = Model<MODEL>::M;
    const Env E = stage_env(P, B);
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float x[N], u[M], dt;
    for (int d = 0; d < N; ++d) x[d] = ps[static_cast<size_t>(i) * N + d];
    ItemOut o;
    const int rc = propagate_item<MODEL>(P, E, x, pacc[i], B.ctl->seed, it, ids[i], brs[i], u, dt, o);
    valid[i] = rc == 0 ? 1 : (rc == 1 ? 0 : 2);
    for (int d = 0; d < N; ++d) xs[static_cast<size_t>(i) * N + d] = rc == 0 ? x[d] : 0.0f;
    for (int d = 0; d < M; ++d) us[static_cast<size_t>(i) * M + d] = u[d];
    dts[i] = dt;
    accs[i] = rc == 0 ? o.acc : 0.0f;
    regs[i] = rc == 0 ? o.region : 0u;
    steps[i] = o.steps;
    goals[i] = rc == 0 ? o.goal : 0;
}

// extract_trajectory, step 1: root->leaf chain on the device.
__global__ void k_chain(KpBuffers B, int32_t leaf, int32_t* chain, uint32_t cap, uint32_t* len) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint32_t n = 0;
    for (int32_t p = leaf; p >= 0; p = B.parent[p]) ++n;
    *len = n;
    uint32_t k = n;
    for (int32_t p = leaf; p >= 0; p = B.parent[p]) {
        --k;
        if (k < cap) chain[k] = p;
    }
}

// Step 1b: gather the chain's node records into compact row-major buffers.
__global__ void k_gather_chain(KpProblem P, KpBuffers B, const int32_t* chain, uint32_t len, float* st, float* ct,
                               float* dts, float* accs) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= len) return;
    const uint32_t g = static_cast<uint32_t>(chain[j]);
    for (int d = 0; d < P.n; ++d) st[static_cast<size_t>(j) * P.n + d] = B.state[static_cast<size_t>(d) * P.capacity + g];
    for (int d = 0; d < P.m; ++d) ct[static_cast<size_t>(j) * P.m + d] = B.ctrl[static_cast<size_t>(d) * P.capacity + g];
    dts[j] = B.dt[g];
    accs[j] = __uint_as_float(B.acc[g]);
}

// Step 2: re-integrate segment j (chain[j] -> chain[j+1]) with the exact
// propagate arithmetic; samples 1..S of each segment at out[off[j] ..].
template <int MODEL>
__global__ void k_reintegrate(KpProblem P, KpBuffers B, const int32_t* chain, uint32_t n_seg, const uint32_t* off,
                              float* out, float* seg_cost) {
    constexpr int N = Model<MODEL>::N;
    constexpr int M = Model<MODEL>::M;
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_seg) return;
    const uint32_t a = static_cast<uint32_t>(chain[j]), b = static_cast<uint32_t>(chain[j + 1]);
    float x[N], u[M];
    for (int d = 0; d < N; ++d) x[d] = B.state[static_cast<size_t>(d) * P.capacity + a];
    for (int d = 0; d < M; ++d) u[d] = B.ctrl[static_cast<size_t>(d) * P.capacity + b];
    const float dt = B.dt[b];
    const float q = dt / P.h;
    int S = static_cast<int>(ceilf(q));
    if (S < 1) S = 1;
    float total = 0.0f;
    long long fx = 0;
    float px = x[0], py = x[1], pz = N >= 3 && MODEL != 0 ? x[2] : 0.0f;
    float x0[N];
    for (int d = 0; d < N; ++d) x0[d] = x[d];
    float ctx[8];
    step_ctx<MODEL>(u, P.h, ctx);
    uint32_t w = off[j];
    for (int s = 0; s < S; ++s) {
        if (advance<MODEL>(P, x0, x, u, dt, S, s, P.h / 6.0f, ctx) == 1) break;
        for (int d = 0; d < N; ++d) out[static_cast<size_t>(w) * N + d] = x[d];
        ++w;
        const float nx = x[0], ny = x[1], nz = MODEL != 0 ? x[2] : 0.0f;
        const float dx = nx - px, dy = ny - py, dz = nz - pz;
        float d2 = dx * dx;
        d2 = fmaf(dy, dy, d2);
        if (MODEL != 0) d2 = fmaf(dz, dz, d2);
        if constexpr (closed_form<MODEL>()) fx += len_fixed(sqrtf(d2));
        else total += sqrtf(d2);
        px = nx; py = ny; pz = nz;
    }
    if constexpr (closed_form<MODEL>()) total = fixed_len(fx);
    seg_cost[j] = P.cost_kind == 1 ? dt : (total == 0.0f ? P.zero_rate * dt : total);
}

}  // namespace kp

// ------------------------------------------------------------------------
// Launch wrappers (C++ linkage, used by kp_capi.cpp).
// ------------------------------------------------------------------------
namespace kp {

size_t propagate_smem(const KpProblem& P) { return P.prop_smem; }

// Shared-memory layout of k_propagate after the environment blob: the
// step-sorted path's PropSmem and (double integrator) the sample-parallel
// path's arrays share one area (a larger reservation than the step-sorted
// path's would keep the next kernel's blocks from becoming resident early
// under PDL).  A sample-parallel batch holds KP_FLAT_ITEMS item records,
// sample offsets, invalid flags and fixed-point path lengths.  KP_FLAT=0
// turns the sample-parallel path off.
#ifndef KP_FLAT_SMEM_KB
#define KP_FLAT_SMEM_KB 96  // propagate's shared memory with the sample-parallel arrays (2 blocks/SM)
#endif
#ifndef KP_FLAT_BATCHES
#define KP_FLAT_BATCHES 2u  // largest sample-parallel launch: batches per block of the grid
#endif
void plan_propagate_smem(KpProblem& P) {
    auto pad16 = [](size_t b) { return (b + 15) & ~static_cast<size_t>(15); };
    size_t seq = 0;
    uint32_t T = 0;
    switch (P.model) {
        case 0: seq = sizeof(PropSmem<0>); T = PropCfg<0>::T; break;
        case 1: seq = sizeof(PropSmem<1>); T = PropCfg<1>::T; break;
        case 2: seq = sizeof(PropSmem<2>); T = PropCfg<2>::T; break;
        default: seq = sizeof(PropSmem<3>); T = PropCfg<3>::T; break;
    }
    const size_t base = pad16(P.env_bytes);
    P.seq_base = static_cast<uint32_t>(base);
    size_t area = pad16(seq);
    P.flat_on = 0;
    P.flat_max = 0;
    const char* env = std::getenv("KP_FLAT");
    if ((P.model == 0 || P.model == 1) && !(env && env[0] == '0')) {
        const uint32_t nb = (KP_FLAT_ITEMS + T - 1) / T * T;
        const uint32_t rw = static_cast<uint32_t>((P.n + P.m + 3 + 3) / 4);
        const size_t rec = pad16(static_cast<size_t>(nb) * rw * 16);
        const size_t offs = pad16((nb + 1) * 4ull), badb = pad16(nb * 4ull), lenb = pad16(2 * nb * 4ull);
        const uint32_t smax = static_cast<uint32_t>(std::ceil(static_cast<double>(P.t_prop) / P.h)) + 1u;
        // chunk -> item index
        const size_t idxb = pad16(static_cast<size_t>(nb) * ((smax + KP_FLAT_K - 1) / KP_FLAT_K) * 2);
        const size_t flat = rec + offs + badb + lenb + idxb;
        if (base + flat <= KP_FLAT_SMEM_KB * 1024) {
            P.flat_on = 1;
            P.flat_nb = nb;
            P.flat_rec = static_cast<uint32_t>(base);
            P.flat_offs = static_cast<uint32_t>(base + rec);
            P.flat_bad = static_cast<uint32_t>(base + rec + offs);
            P.flat_len = static_cast<uint32_t>(base + rec + offs + badb);
            P.flat_idx = static_cast<uint32_t>(base + rec + offs + badb + lenb);
            area = std::max(area, flat);
        }
    }
    P.prop_smem = static_cast<uint32_t>(base + area);
}

// Largest launch on the sample-parallel path: two batches per block of the
// propagate grid (small launches are latency-bound; the sample-parallel path
// also won up to two batches per block — the DI growth phase around the first
// solution: forest time to first solution 0.64 -> 0.61 ms, building6d +10 %
// queries — while the step-sorted path runs fewer instructions per sample at
// saturation, and long rollouts, zigzag6d, lost beyond that).  KP_FLAT_MAX
// overrides.
void set_flat_limit(KpProblem& P, int grid_prop) {
    if (!P.flat_on) return;
    const char* fm = std::getenv("KP_FLAT_MAX");
    P.flat_max = fm ? static_cast<uint32_t>(std::strtoul(fm, nullptr, 10))
                    : KP_FLAT_BATCHES * P.flat_nb * static_cast<uint32_t>(grid_prop);
}

static bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("KP_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename Kern>
static cudaError_t launch_k(Kern kernel, int grid, int block, size_t smem, cudaStream_t st, const KpProblem& P,
                            const KpBuffers& B) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, P, B);
}

// The scatter grid never exceeds what is resident at once (3 blocks/SM at its
// 80 registers): blocks of a second wave would start only after the first
// wave's, and a growth-phase iteration with more tiles than blocks measured
// its tile prefix ~7 µs late; a resident block takes several tiles in turn.
static int scatter_grid(int grid_sel) {
    static const int resident = [] {
        int dev = 0, sms = 0, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_select_scatter, KP_SELECT_THREADS, 0);
        return std::max(1, sms * occ);
    }();
    return std::min(grid_sel, resident);
}

cudaError_t launch_iteration(const KpProblem& P, const KpBuffers& B, int grid_prop, int grid_sel, cudaStream_t st,
                             int which) {
    const size_t smem = propagate_smem(P);
    cudaError_t e = cudaSuccess;
    if (which & 1) {
        switch (P.model) {
            case 0: e = launch_k(k_propagate<0>, grid_prop, PropCfg<0>::T, smem, st, P, B); break;
            case 1: e = launch_k(k_propagate<1>, grid_prop, PropCfg<1>::T, smem, st, P, B); break;
            case 2: e = launch_k(k_propagate<2>, grid_prop, PropCfg<2>::T, smem, st, P, B); break;
            default: e = launch_k(k_propagate<3>, grid_prop, PropCfg<3>::T, smem, st, P, B); break;
        }
        if (e != cudaSuccess) return e;
    }
    if (which & 2) {
        e = P.sel_spec ? launch_k(k_select_reduce<true>, grid_sel, KP_SELECT_THREADS, 0, st, P, B)
                       : launch_k(k_select_reduce<false>, grid_sel, KP_SELECT_THREADS, 0, st, P, B);
        if (e != cudaSuccess) return e;
    }
    if (which & 4) e = launch_k(k_select_scatter, scatter_grid(grid_sel), KP_SELECT_THREADS, 0, st, P, B);
    return e;
}

cudaError_t set_propagate_smem(const KpProblem& P) {
    const int smem = static_cast<int>(propagate_smem(P));
    cudaError_t e = cudaSuccess;
    switch (P.model) {
        case 0: e = cudaFuncSetAttribute(k_propagate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); break;
        case 1: e = cudaFuncSetAttribute(k_propagate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); break;
        case 2: e = cudaFuncSetAttribute(k_propagate<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); break;
        default: e = cudaFuncSetAttribute(k_propagate<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); break;
    }

    return e;
}

int propagate_occupancy(const KpProblem& P) {
    int nb = 0;
    const size_t smem = propagate_smem(P);
    switch (P.model) {
        case 0: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_propagate<0>, PropCfg<0>::T, smem); break;
        case 1: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_propagate<1>, PropCfg<1>::T, smem); break;
        case 2: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_propagate<2>, PropCfg<2>::T, smem); break;
        default: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_propagate<3>, PropCfg<3>::T, smem); break;
    }
    return nb;
}

cudaError_t launch_reset(const KpProblem& P, const KpBuffers& B, unsigned long long seed, cudaStream_t st) {
    cudaMemsetAsync(B.ctl, 0, sizeof(KpCtl), st);
    cudaMemsetAsync(B.admit_mask, 0, sizeof(uint32_t) * (P.max_slots / 32), st);
    cudaMemsetAsync(B.goal_mask, 0, sizeof(uint32_t) * (P.max_slots / 32), st);
    k_reset_table<<<148 * 4, 256, 0, st>>>(P, B);
    k_reset_root<<<1, 32, 0, st>>>(P, B, seed);
    return cudaGetLastError();
}

cudaError_t launch_start(const KpBuffers& B, unsigned long long budget_ns, uint32_t max_iters, uint32_t stop_first,
                         uint32_t seq, cudaStream_t st) {
    k_start<<<1, 32, 0, st>>>(B, budget_ns, max_iters, stop_first, seq);
    return cudaGetLastError();
}

cudaError_t launch_debug_propagate(const KpProblem& P, const KpBuffers& B, uint32_t n, const float* ps,
                                   const float* pacc, const uint32_t* ids, const uint32_t* brs, uint32_t it,
                                   uint8_t* valid, float* xs, float* us, float* dts, float* accs, uint32_t* regs,
                                   uint32_t* steps, uint8_t* goals, cudaStream_t st) {
    const size_t smem = P.env_bytes;  // the environment only (sequential per-item path)
    const int grid = static_cast<int>((n + 127) / 128);
    if (n == 0) return cudaSuccess;
    switch (P.model) {
        case 0: k_debug_propagate<0><<<grid, 128, smem, st>>>(P, B, n, ps, pacc, ids, brs, it, valid, xs, us, dts, accs, regs, steps, goals); break;
        case 1: k_debug_propagate<1><<<grid, 128, smem, st>>>(P, B, n, ps, pacc, ids, brs, it, valid, xs, us, dts, accs, regs, steps, goals); break;
        case 2: k_debug_propagate<2><<<grid, 128, smem, st>>>(P, B, n, ps, pacc, ids, brs, it, valid, xs, us, dts, accs, regs, steps, goals); break;
        default: k_debug_propagate<3><<<grid, 128, smem, st>>>(P, B, n, ps, pacc, ids, brs, it, valid, xs, us, dts, accs, regs, steps, goals); break;
    }
    return cudaGetLastError();
}

// Sweep support: frontier = nodes 0..n-1 (the store's first n nodes, so
// kp_get_nodes returns the synthetic states), iteration counter fixed, region
// table +inf, counters cleared (one launch = n * lambda work items).
__global__ void k_sweep_prepare(KpProblem P, KpBuffers B, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t r = i; r < P.n_regions; r += gridDim.x * blockDim.x) B.rc[r] = 0x7F800000u;
    for (uint32_t k = i; k < n; k += gridDim.x * blockDim.x) B.va[0][k] = k;
    for (uint32_t w = i; w < P.max_slots / 32; w += gridDim.x * blockDim.x) {
        B.admit_mask[w] = 0u;
        B.goal_mask[w] = 0u;
    }
    if (i == 0) {
        KpCtl* c = B.ctl;
        c->done = 0;
        c->stop_first = 0;  // propagate's stop-at-first-solution test must not end a sweep launch
        c->iter = 0;
        c->n_va = n;
        c->n_nodes = n;
        c->n_items = n * static_cast<uint32_t>(P.lambda);
        c->prop_cursor = 0;
        c->n_adm_p[0] = 0;
        c->n_valid_iter = 0;
        c->split = 0;  // no previous iteration to measure the invalid share on
        c->stats = KpStats{};
    }
}

cudaError_t launch_sweep_prepare(const KpProblem& P, const KpBuffers& B, uint32_t n, cudaStream_t st) {
    k_sweep_prepare<<<148 * 4, 256, 0, st>>>(P, B, n);
    return cudaGetLastError();
}

cudaError_t launch_chain(const KpBuffers& B, int32_t leaf, int32_t* chain, uint32_t cap, uint32_t* len,
                         cudaStream_t st) {
    k_chain<<<1, 32, 0, st>>>(B, leaf, chain, cap, len);
    return cudaGetLastError();
}

cudaError_t launch_gather_chain(const KpProblem& P, const KpBuffers& B, const int32_t* chain, uint32_t len,
                                float* st, float* ct, float* dts, float* accs, cudaStream_t s) {
    if (len == 0) return cudaSuccess;
    k_gather_chain<<<(len + 127) / 128, 128, 0, s>>>(P, B, chain, len, st, ct, dts, accs);
    return cudaGetLastError();
}

cudaError_t launch_reintegrate(const KpProblem& P, const KpBuffers& B, const int32_t* chain, uint32_t n_seg,
                               const uint32_t* off, float* out, float* seg_cost, cudaStream_t st) {
    if (n_seg == 0) return cudaSuccess;
    const int grid = static_cast<int>((n_seg + 127) / 128);
    switch (P.model) {
        case 0: k_reintegrate<0><<<grid, 128, 0, st>>>(P, B, chain, n_seg, off, out, seg_cost); break;
        case 1: k_reintegrate<1><<<grid, 128, 0, st>>>(P, B, chain, n_seg, off, out, seg_cost); break;
        case 2: k_reintegrate<2><<<grid, 128, 0, st>>>(P, B, chain, n_seg, off, out, seg_cost); break;
        default: k_reintegrate<3><<<grid, 128, 0, st>>>(P, B, chain, n_seg, off, out, seg_cost); break;
    }
    return cudaGetLastError();
}

}  // namespace kp

namespace kp {
// Stamps build: copy the 64 x 32 phase stamps (KP_STAMPS), else an error.
cudaError_t read_stamps(unsigned long long* out) {
#ifdef KP_STAMPS
    return cudaMemcpyFromSymbol(out, kp_stamps, sizeof(kp_stamps));
#else
    (void)out;
    return cudaErrorNotSupported;
#endif
}

// Checks build: first failed device invariant (0 = none), cleared on read.
cudaError_t read_check_code(unsigned int* code) {
#ifdef KP_CHECKS
    cudaError_t e = cudaMemcpyFromSymbol(code, kp_check_code, sizeof(unsigned int));
    if (e != cudaSuccess) return e;
    const unsigned int z = 0;
    return cudaMemcpyToSymbol(kp_check_code, &z, sizeof z);
#else
    *code = 0;
    return cudaSuccess;
#endif
}
}  // namespace kp
