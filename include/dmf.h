/*
 * dmf.h -- C ABI of libdmf.so, a B200-native (sm_100a) dynamic max-flow engine
 * implementing the data-parallel hot path of arXiv 2511.05895, "Efficient Dynamic
 * MaxFlow Computation on GPUs" (citations "P:n" are lines of the paper's LaTeX
 * source, PAPER.md; "S:n" lines of SPEC.md; "§8(c) Rk" readings in DESIGN.md).
 *
 * Problem: directed graph G=(V,E), capacities c(u,v) >= 0, source s,
 * sink t; maximise |f| subject to 0 <= f <= c and conservation on V\{s,t}.
 * The engine keeps a residual graph (c_f(u,v) = c(u,v) - f(u,v) + f(v,u))
 * and a pseudoflow excess e(v) on the device, solves it from scratch with the
 * GPU-Static-Maxflow loop (Alg.1) and repairs it after a batch of
 * capacity changes with Dynamic Push-Relabel (Alg.4-5) or Dynamic
 * Push-Pull (Alg.6-8).
 *
 * Conventions for every entry point
 *  - Return value: DMF_OK (0) or a negative dmf_status; dmf_last_error() gives a
 *    thread-local one-line message for the most recent failure.
 *  - Vertex ids are int32 in [0, n).  Capacities are int32 in [0, DMF_CAP_MAX].
 *    Excess and flow values are int64 (grid configs exceed 2^31).
 *  - Pointers marked "host or device" may be plain host memory, pinned host memory
 *    or device memory of the handle's GPU (detected with cudaPointerGetAttributes).
 *    All caller buffers are caller-owned; the library copies what it needs.
 *  - All device work is ordered on the handle's stream (dmf_options.stream).  Every
 *    call returns only when its results are ready (it synchronises that stream).
 *  - A handle is not thread-safe; distinct handles are independent.
 */
#ifndef DMF_H
#define DMF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dmf_graph dmf_graph;   /* opaque: owns every device array of one instance */

typedef enum {
    DMF_OK = 0,
    DMF_EINVAL = -1,     /* bad argument: id out of range, self-loop, s == t, cap < 0 or > DMF_CAP_MAX */
    DMF_ENOSLOT = -2,    /* batch entry (u,v) names no slot (neither an input edge nor the reverse of one) */
    DMF_EDUP = -3,       /* batch names the same (u,v) twice */
    DMF_ESTATE = -4,     /* DMF_DYN_PP without a previous converged solve */
    DMF_ENOMEM = -5,     /* device allocation failed */
    DMF_ECUDA = -6,      /* CUDA runtime error (message in dmf_last_error) */
    DMF_EOVERFLOW = -7,  /* merged capacity of a pair exceeds DMF_CAP_MAX, or too many slots (>= 2^31) */
    DMF_ENOCONV = -8,    /* iteration cap reached (never expected; Thm P:318-330 bounds the work).
                            The handle then holds a valid but NOT converged pseudoflow: flow / cut
                            queries and DMF_DYN_PP return DMF_ESTATE until a dmf_static_solve or a
                            DMF_DYN_PR repair (which converges from any valid pseudoflow) succeeds. */
    DMF_ECHECK = -9      /* check_level > 0 and a device invariant check failed (a bug; the handle
                            is marked not converged as for DMF_ENOCONV) */
} dmf_status;

typedef enum {
    DMF_DYN_PR = 0,      /* Dynamic Push-Relabel, Alg.4 */
    DMF_DYN_PP = 1       /* Dynamic Push-Pull, Alg.8 */
} dmf_algo;

/* Upper bound of any capacity, so that c(u,v) + c(v,u) < 2^31 always holds and a
 * residual fits int32. */
#define DMF_CAP_MAX 1073741823

/* Discharge schedules (dmf_options.schedule).  Every schedule computes the same F,
 * S_min and S_max; they differ only in how active vertices are found and ordered. */
typedef enum {
    DMF_SCHED_AUTO = 0,      /* repairs: ASYNC; static solve: ROUNDS (topology auto-switch: topo_div) */
    DMF_SCHED_ASYNC = 1,     /* data-driven worklist seeding a device-wide ring queue: a vertex
                                made active by a push is processed at once (the property P:647 credits
                                to the topology-driven schedule) */
    DMF_SCHED_ROUNDS = 2,    /* data-driven worklist, barrier-separated rounds */
    DMF_SCHED_TOPOLOGY = 3   /* topology-driven rounds: every round sweeps all vertices of the
                                domain and discharges the active ones in place; no worklist */
} dmf_schedule;

typedef struct {
    int32_t kernel_cycles;  /* KERNELCYCLES of Alg.2/Alg.6; 0 => max(1, floor(m/n)) (R17) */
    int32_t algo;           /* default algorithm for dmf_apply_batch when its algo argument is < 0 */
    int32_t max_iters;      /* cap on outer loop iterations per call; 0 => 4*n + 64 */
    int32_t grid_blocks;    /* 0 => occupancy-derived cooperative grid (multiple of the SM count) */
    void *stream;           /* cudaStream_t for all work; NULL => a stream owned by the handle.
                               cudaStreamLegacy ((void*)1) selects the legacy default stream. */
    /* Optional device allocator (e.g. the torch caching allocator); NULL => cudaMalloc.
     * alloc returns a device pointer of >= bytes (256-byte aligned) or NULL. */
    void *(*alloc)(size_t bytes, void *ctx);
    void (*free)(void *ptr, size_t bytes, void *ctx);
    void *alloc_ctx;
    /* ---- engine knobs, per handle.  0 selects the default.  None of them changes a
     * result (F, S_min, S_max are unique); they change the work schedule only.  The
     * environment variable in brackets, when set, overrides the field (experiments). */
    int32_t schedule;       /* dmf_schedule [DMF_SCHED] */
    int32_t async_warps;    /* consumer warps per CTA in the ASYNC phase, 1..16; 0 => 8 [DMF_ASYNC_WARPS] */
    int32_t budget_mul;     /* discharge work allowed between two global relabels, in units of one
                               whole-graph BFS (S + 6n slot visits); 0 => 1; < 0 divides the unit
                               by -budget_mul (tests force budget stops with it) [DMF_BUDGET_MUL] */
    int32_t tail_items;     /* progress stop of an ASYNC phase: once at most 64 items are pending, this
                               many further item completions hand the rest to a global relabel;
                               0 => 2048, < 0 => never [DMF_TAIL_ITEMS] */
    int32_t local_gap;      /* R14 form 2, the local gap exit inside a discharge phase (per-level
                               counts): 0 => on, < 0 => off [DMF_LOCAL_GAP] */
    int32_t warm;           /* DYN_PP after DYN_PP starts from the previous call's labels: 0 => on,
                               < 0 => off (every repair starts with a fresh global relabel) [DMF_WARM] */
    int32_t topo_div;       /* auto-switch: a discharge phase runs topology-driven when more than
                               n / topo_div vertices are active; <= 0 => never (default: the worklist
                               won every A/B on B200) [DMF_TOPO_DIV] */
    int32_t check_level;    /* 0 => off; 1 => after every solve / repair the device checks the cheap
                               invariants (0 <= res <= cap + cap_rev, res[i] + res[rev[i]] = cap[i] +
                               cap[rev[i]], mirror consistency, sum of e = 0) and the call fails with
                               DMF_ECHECK if one is violated [DMF_CHECK_LEVEL] */
    int32_t certify;        /* DYN_PP after DYN_PP: after the warm discharge iteration, test convergence
                               with the universal certificate (reading R9: a fresh backward BFS from
                               {t} u {deficient vertices} reaches no excess vertex and s reaches none of
                               its labels); when it holds the call ends there (partition = that BFS's
                               reach, R15) and S_min is computed by dmf_min_cut_source_side on demand.
                               The certificate runs in k_reach; a failed one hands over to a second
                               k_solve launch (decided on the device, no host round trip).
                               0 => on, < 0 => off (always the full Alg.8 stage 1 / P / stage 2) [DMF_CERTIFY] */
    int32_t reserved[7];    /* must be zero */
} dmf_options;

typedef struct {
    int64_t n, m, S;           /* vertices; merged input edges; slots (m + materialised reverses) */
    int32_t kernel_cycles;     /* effective KERNELCYCLES */
    int32_t grid_blocks, block_threads;
    /* counters of the LAST solve / apply call */
    int64_t iterations;        /* outer loop iterations (each = BFS + discharge + RIE), all stages */
    int64_t bfs_levels;        /* BFS frontier levels over all global relabels */
    int64_t bfs_vertices;      /* frontier vertices expanded */
    int64_t bfs_slots;         /* slots scanned by BFS expansion */
    int64_t discharge_vertices;/* worklist entries discharged */
    int64_t discharge_slots;   /* slots scanned by discharge (argmin + push passes) */
    int64_t pushes;            /* push / pull operations (Alg.2 l.16-19, Alg.6 l.16-19) */
    int64_t relabels;          /* lift operations (Alg.2 l.21, Alg.6 l.21) */
    int64_t rie_slots;         /* slots scanned by RemoveInvalidEdges */
    int64_t rie_saturations;   /* edges saturated by RemoveInvalidEdges (Alg.3/Alg.7) */
    int64_t batch_entries;     /* k of the last batch */
    int64_t stage2_vertices;   /* |P| of the last push-pull stage 2 (Alg.8 l.29-34) */
    int64_t stage2_iterations;
    int64_t rounds;            /* discharge rounds (a round = discharge + RIE over the queued vertices) */
    int64_t activations;       /* vertices queued for the next round because a push made them active */
    int64_t reset_vertices;    /* vertices whose heights were reset for a global relabel */
    int64_t budget_stops;      /* discharge round sequences cut short by the work budget (-> global relabel) */
    int64_t bottom_up_levels;  /* BFS levels expanded bottom-up (direction-optimising BFS) */
    int64_t kernel_launches;   /* CUMULATIVE kernels launched by solve/apply/cut calls since dmf_create */
    float   device_ms;         /* device time of the last call's kernel(s), CUDA events */
    /* in-kernel phase clock (%globaltimer, block 0), microseconds, last call:
     * prologue = batch validate/apply/clamp + source / S->T saturation,
     * epilogue = P extraction, partitions, flow reduction, cut masks */
    float   t_prologue_us, t_reset_us, t_bfs_us, t_discharge_us, t_rie_us, t_epilogue_us;
    int64_t gap_levels;        /* R14 form 2: height levels found emptied by a lift (local gap) */
    int64_t gap_skips;         /* discharges stopped because the vertex sat above an emptied level */
    int64_t topology_rounds;   /* discharge rounds run topology-driven */
    int64_t tail_stops;        /* ASYNC phases ended by the progress stop (tail_items) */
    int64_t stage2_skipped;    /* DYN_PP: stage 2 / the P-reach skipped (P holds no deficit / no excess) */
    int64_t certified;         /* DYN_PP: 1 if the warm iteration was certified converged (options.certify) */
    float   query_ms;          /* device time of the last dmf_min_cut_source_side / dmf_max_cut_source_side
                                  launch (0 when S_min was already cached by the last DYN_PP call) */
    int64_t query_bfs_vertices;/* that query's BFS: vertices labelled and slots scanned */
    int64_t query_bfs_slots;
} dmf_stats;

/* Fill *opt with defaults (all zero / NULL; algo = DMF_DYN_PP). */
void dmf_default_options(dmf_options *opt);

/* Build the Bi-CSR residual graph ("Bi-Directional CSR ... zero-capacity
 * entries to address any missing reverse edges ... an additional array ... stores
 * the offset of the reverse edges").
 *  n        number of vertices (>= 2)
 *  row_ptr  int64[n+1], host or device: CSR offsets of the input edges
 *  col      int32[row_ptr[n]], host or device: heads
 *  cap      int32[row_ptr[n]], host or device: capacities in [0, DMF_CAP_MAX]
 *  s, t     source and sink, s != t
 * Duplicate (u,v) input entries are merged by summing; zero-capacity input
 * edges are kept (they are the insertion pool).  Self-loops, ids out of
 * range, s == t or a negative capacity -> DMF_EINVAL; a merged pair above
 * DMF_CAP_MAX or >= 2^31 slots -> DMF_EOVERFLOW.  The new state is the zero flow
 * (not yet solved).  On success *out owns all device memory (dmf_destroy frees it). */
int dmf_create(int32_t n, const int64_t *row_ptr, const int32_t *col, const int32_t *cap,
               int32_t s, int32_t t, const dmf_options *opt, dmf_graph **out);

/* GPU-Static-Maxflow (Alg.1) on the current capacities, from the zero
 * flow: c_f = c, e = 0, saturate s's out-edges, then loop {global relabel by
 * backward BFS from the sink set, PushRelabel x KERNELCYCLES on the active
 * worklist, RemoveInvalidEdges} until a fresh BFS reaches no active vertex
 * (readings R1, R2, R9 of DESIGN.md: the sink set is {t} u deficient vertices). */
int dmf_static_solve(dmf_graph *g);

/* Static push-pull variant: as dmf_static_solve, but the
 * initial preflow also saturates every in-edge (v,t) of the sink, so the tails start
 * deficient and act as secondary sinks (roots of every global relabel, reading R2)
 * while the excess from s is pushed into them.  Same F, S_min, S_max and converged
 * state semantics as dmf_static_solve (F by reading R8); a following DYN_PP batch
 * starts from its final partition. */
int dmf_static_solve_pp(dmf_graph *g);

/* Apply a batch of k capacity updates (SET semantics, all entries simultaneous,
 * P:342 "each batch is a set of edges whose new capacities may be either higher or
 * lower") and repair the state to convergence with `algo` (DMF_DYN_PR = Alg.4,
 * DMF_DYN_PP = Alg.8; < 0 => options.algo).
 *  u, v, new_cap  int32[k], host or device
 * The whole batch is validated on the device BEFORE any mutation: an entry whose
 * (u,v) is not a slot -> DMF_ENOSLOT, a repeated (u,v) -> DMF_EDUP, ids out of range
 * -> DMF_EINVAL, new_cap outside [0, DMF_CAP_MAX] -> DMF_EOVERFLOW; on any error the
 * residual/excess/capacity state is unchanged.  DMF_DYN_PP needs a previous
 * converged solve on this handle (else DMF_ESTATE).  k = 0 is allowed. */
int dmf_apply_batch(dmf_graph *g, int64_t k, const int32_t *u, const int32_t *v,
                    const int32_t *new_cap, int32_t algo);

/* Maximum-flow value of the converged state: F = e(t) + sum_{v not in {s,t}}
 * min(e(v), 0) (Alg.4 final loop P:381-386 / Alg.8; reading R8). */
int dmf_flow_value(const dmf_graph *g, int64_t *out);

/* Minimal min-cut source side S_min (unique): mask[v] = 1 iff v is reachable in the
 * residual graph from {s} u {v not in {s,t} : e(v) > 0} (reading R19; equals
 * the residual reach of s for any true maximum flow).  mask: uint8[n], host or device.
 * Cached when the last DYN_PP computed it (the full stage-1 path); otherwise one launch
 * of the dedicated BFS kernel k_reach (csrc/reach.cuh), which also refreshes h- with the
 * exact forward distances used by the next DYN_PP warm start. */
int dmf_min_cut_source_side(dmf_graph *g, uint8_t *mask);

/* Maximal min-cut source side S_max: mask[v] = 1 iff v cannot reach {t} u {deficient}
 * in the residual graph -- the paper's certificate S = {h = |V|} (Thm 3, P:245-248;
 * Note 1).  mask: uint8[n], host or device. */
int dmf_max_cut_source_side(dmf_graph *g, uint8_t *mask);

/* Counters of the last call (see dmf_stats). */
int dmf_get_stats(const dmf_graph *g, dmf_stats *out);

/* Phase tracing (aux/debug): capacity > 0 allocates a device ring of `capacity`
 * records; every later call records one record per grid phase of its kernel:
 * {phase, iteration, level-or-round, items, extra, duration_ns, slow_ns, slow_info}
 * (int32 x 8; slow_* = the slowest vertex discharge of the phase: ns and
 * (degree << 8 | cycles)) where
 * phase is 0 prologue, 1 reset, 2 bfs level expansion, 3 discharge round, 4 rie,
 * 5 epilogue, 6 bfs bottom-up pass B, 7 bfs compaction.  capacity = 0 disables tracing. */
int dmf_set_trace(dmf_graph *g, int32_t capacity);

/* Copy the trace of the LAST call: *count = records written; up to `capacity`
 * records are copied to `records` (host or device, int32[8 * capacity]). */
int dmf_get_trace(const dmf_graph *g, int32_t *records, int32_t capacity, int32_t *count);

/* Per-CTA view of the same trace (load-balance diagnostics): for record r and CTA b,
 * busy_ns[r * grid + b] = ns from CTA b's previous grid-barrier exit to its arrival
 * at the barrier that ends record r's phase.  *grid = CTAs of the persistent kernel;
 * up to `capacity` records are copied (busy_ns: host or device, uint32[capacity *
 * grid]; NULL only queries *grid). */
int dmf_get_trace_cta(const dmf_graph *g, uint32_t *busy_ns, int32_t capacity, int32_t *grid);

/* Sizes: *n vertices, *S slots, *m merged input edges (any may be NULL). */
int dmf_sizes(const dmf_graph *g, int32_t *n, int64_t *S, int64_t *m);

/* Copy the device state to caller buffers (host or device; any may be NULL):
 * row_ptr int64[n+1], dst/rev/cap/res int32[S] (slot form: rows sorted by head,
 * rev[i] = slot of the reverse pair), excess int64[n].  For checkers. */
int dmf_export_state(const dmf_graph *g, int64_t *row_ptr, int32_t *dst, int32_t *rev,
                     int32_t *cap, int32_t *res, int64_t *excess);

/* Checkpoint restore (SURVEY §5 "Checkpoint / resume": the converged residual graph IS
 * the state carried between batches).  cap, res: int32[S] and excess: int64[n]
 * (host or device) in the slot order of dmf_export_state of a handle built from the
 * SAME input graph (same n, row_ptr, col; capacities may differ).  The imported state
 * is validated on the device with the invariant check of check_level 1 plus
 * e(v) = sum over the slots j of v of (res[j] - cap[j]) (net inflow);
 * DMF_EINVAL if it fails, with the handle's previous state restored.  On success the
 * handle holds a valid pseudoflow that is NOT yet known to be converged: flow and cut
 * queries return DMF_ESTATE until dmf_static_solve or a DMF_DYN_PR batch (k = 0 is
 * allowed) has repaired it -- a Dynamic Push-Relabel repair converges from any valid
 * pseudoflow (the sink set {t} u deficient vertices, reading R2). */
int dmf_import_state(dmf_graph *g, const int32_t *cap, const int32_t *res, const int64_t *excess);

/* Run the device invariant check of check_level 1 on the current state now:
 * 0 <= res <= cap + cap_rev, res[i] + res[rev[i]] = cap[i] + cap[rev[i]], rres[i] =
 * res[rev[i]], e(v) = sum_{slots j of v} (res[j] - cap[j]), sum of e = 0.  DMF_OK or
 * DMF_ECHECK (message names the first violated invariant and a witness). */
int dmf_check_state(dmf_graph *g);

/* Stage (ii): turn the converged pseudoflow
 * into a true maximum flow in place.  Stuck excess is returned to s (every vertex with
 * excess reaches s in the residual graph, Lemma 4) and every deficit is
 * filled from t, with the same device engine (roots {s}, then {t}).  F,
 * S_min and S_max are unchanged; afterwards e(v) = 0 for every v not in {s,t} and
 * e(t) = -e(s) = F.  The next DYN_PP call starts with a full global relabel (the warm
 * labels are gone).  DMF_ESTATE before any solve; DMF_ENOCONV if a vertex keeps
 * excess or deficit (not expected: the lemmas guarantee the paths). */
int dmf_to_flow(dmf_graph *g);

/* Per-slot flow of the current state: flow[i] = max(0, cap[i] - res[i]) for slot i =
 * (u, dst[i]) (the net flow of the pair {u, dst[i]} in that direction; the reverse
 * slot holds the other direction, so at most one of the two is positive).  After
 * dmf_to_flow this is a feasible maximum flow.  flow: int32[S], host or device,
 * slot order of dmf_export_state. */
int dmf_edge_flow(dmf_graph *g, int32_t *flow);

/* Copy the engine's labels after the last call (host or device buffers; any may be
 * NULL): hp/hm int32[n] (h+ / h- heights, in [0, |V|+1]: |V| = unreached by the last
 * global relabel, |V|+1 = outside the track's region), part uint8[n] (1 = S, 2 = T,
 * 3 = P of Alg.8), rres int32[S] (the residual mirror rres[i] =
 * c_f(dst[i], u) of slot i = (u, dst[i]); equal to res[rev[i]] whenever no call is
 * running).  Inspection / invariant checks only: the labels are not part of the
 * result. */
int dmf_export_labels(const dmf_graph *g, int32_t *hp, int32_t *hm, uint8_t *part, int32_t *rres);

/* Free every device array of the handle (NULL is a no-op). */
void dmf_destroy(dmf_graph *g);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char *dmf_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* DMF_H */
