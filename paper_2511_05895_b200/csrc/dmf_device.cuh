// dmf_device.cuh -- device-side state layout and cooperative-group primitives of
// libdmf (B200 / sm_100a).  See DESIGN.md §3 for the HBM layout and §4 for the
// kernels.  Nothing here is shared with oracle/ (the CPU oracle).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

namespace dmf {

namespace cg = cooperative_groups;

// Persistent cooperative kernel geometry: 512 threads, >= 2 CTAs per SM
// (registers <= 64), grid = resident CTAs (a multiple of the 148 SMs).
constexpr int NT = 512;
constexpr int WPB = NT / 32;
constexpr int MIN_BLOCKS = 2;

// Worklist degree bins: thread / warp / CTA per vertex, and a
// "huge" bin whose rows are split over the whole grid where the phase allows it.
constexpr int NB = 4;
constexpr int32_t BIN0_MAX = 16;
constexpr int32_t BIN1_MAX = 512;
constexpr int32_t BIN2_MAX = 8192;

// Entries of queues / worklists carry the track in bit 31 (vertex ids < 2^31).
constexpr uint32_t TRACK_BIT = 0x80000000u;

// dmin sentinel (memset byte 0x7f): above every height (heights are <= |V|+1 < 2^31-1)
constexpr int32_t DMIN_NONE = 0x7f7f7f7f;
constexpr long long AQ_EMPTY = -1;

// Partition labels of Alg.8.  S'/T' are stored as S/T.
enum : uint8_t { PART_NONE = 0, PART_S = 1, PART_T = 2, PART_P = 3 };

enum Mode : int32_t {
  MODE_STATIC = 0,   // Alg.1 from the zero flow
  MODE_PR = 1,       // batch + Alg.4
  MODE_PP = 2,       // batch + Alg.8
  MODE_MINCUT = 3,   // forward reach of {s} u Exc  (S_min)
  MODE_MAXCUT = 4,   // complement of backward reach of {t} u Def (S_max)
  MODE_FLOW = 5,     // stage (ii): pseudoflow -> true maximum flow (excess back to s, deficits from t)
  MODE_PP_CONT = 6,  // DYN_PP after a failed k_reach certificate: full Alg.8 stage 1 from fresh
                     // labels, P, stage 2, S_min (exits at once when the certificate held)
};

enum Stat : int {
  ST_ITERS, ST_LEVELS, ST_BFS_V, ST_BFS_SLOTS, ST_DIS_V, ST_DIS_SLOTS, ST_PUSHES,
  ST_RELABELS, ST_RIE_SLOTS, ST_RIE_SAT, ST_S2_V, ST_S2_ITERS, ST_ROUNDS, ST_ACTIVATIONS, ST_RESET_V, ST_BUDGET_STOPS, ST_BU_LEVELS,
  ST_GAP_LEVELS, ST_GAP_SKIPS, ST_TOPO_ROUNDS, ST_TAIL_STOPS, ST_S2_SKIP,
  ST_T_PRO, ST_T_RESET, ST_T_BFS, ST_T_DIS, ST_T_RIE, ST_T_EPI, ST_T_BFS_BU, ST_T_BFS_CMP, ST_N
};

// Local gap (R14 form 2): per-track counts of the vertices at each height h < GAPW.
// Heights >= GAPW are not counted (no gap is ever reported there).
constexpr int32_t GAPW = 1024;

// Control block in device memory (zeroed by the host before every launch).
struct Ctl {
  int32_t qc[3 * NB];   // BFS frontier counts [level % 3][degree bin]
  int32_t wlc[3 * NB];  // active worklist counts [round % 3][degree bin]
  int32_t rlc[NB];      // relabelled-vertex list counts [degree bin] (one list per iteration)
  int32_t pcnt;         // |P| (push-pull stage 2 region)
  int32_t ntrace;       // trace records written
  int32_t status;       // dmf_status of the call (0 = OK)
  int32_t err_entry;    // first offending batch entry
  int32_t iters;
  int32_t pad;
  long long flow;       // F
  unsigned long long work[3];   // discharge work per round [round % 3]
  unsigned long long slow;      // trace mode: slowest discharge since the last trace record
  int32_t claim[9];             // dynamic work claims of a discharge round [round % 3][CTA/warp/tile]
  unsigned long long fs[6];     // frontier slot counts [level % 3][track] (direction-optimising BFS)
  int32_t bulc[4];              // bottom-up candidate queue counts [level & 1][warp/CTA bin]
  unsigned long long mu[2];     // slots of the still-unlabelled vertices per track (BFS direction choice)
  unsigned long long stat[ST_N];
  // asynchronous discharge phase: ring queue of activations
  unsigned long long aw;        // (ring tail << 32) | items pending (queued or in progress)
  int32_t ahead;                // next item index to claim (initial worklist first, then the ring)
  int32_t astop;                // work budget spent: stop claiming
  unsigned long long awork;     // discharge work of the phase
  int32_t atail;                // async: item completions while <= TAIL_PEND items were pending
  int32_t gtop[2];              // local gap per track: 0 = none, else GAPW - (lowest emptied level)
  int32_t tact[3];              // topology round r: some vertex became (or stayed) active [r % 3]
  int32_t tcq[3 * NB];          // topology round r: counts of the sweep's chunk list [r % 3][bin]
  int32_t check;                // invariant check: first violated check (0 = none) and a witness
  int32_t check_at;
  int32_t pdef, pexc;           // DYN_PP: deficit / excess vertices in P (stage 2 / P-reach skip)
  int32_t sreach;               // DYN_PP certificate: s reaches a vertex labelled by the backward BFS
  int32_t lazy_ok;              // DYN_PP: converged by the certificate (no S_min mask computed)
  // S_min query (k_reach, reach.cuh): per level % 3
  int32_t rcnt[3];              // frontier items of the level
  int32_t rnv[3];               // vertices labelled with the level
  int32_t rbq[3];               // bottom-up: rows queued for the warp pass
  unsigned long long rfs[3];    // slots of the level's vertices
  unsigned long long rmu;       // slots of the vertices not labelled at level 0
  int32_t rfail;                // k_reach certificate: an excess vertex is labelled / s reaches a label
  int32_t rfl[3];               // the same, per level % 3 (read at the top of the next level)
};

// Everything a kernel needs, passed by value.  Slot arrays are SoA int32[S]:
//   row[u]..row[u+1]  slots of u, sorted by dst (binary-searchable)
//   dst[i]            head of slot i
//   rev[i]            slot of the reverse pair (involution)
//   cap[i]            c(u,v)
//   res[i]            c_f(u,v)
//   rres[i]           mirror res[rev[i]] = c_f(v,u), kept in lock-step so that the
//                     backward BFS and the pull track read it coalesced
struct Dev {
  int32_t n, s, t, kc, max_iters;
  int32_t batch_id;
  int32_t warm;              // MODE_PP: hp/hm/part are the previous DYN_PP call's final labels (warm start)
  long long work_budget;     // discharge work (slots scanned) allowed between two global relabels
  int64_t S, k;
  const int32_t *__restrict__ row;
  const int32_t *__restrict__ dst;
  const int32_t *__restrict__ rev;
  int32_t *cap, *res, *rres;
  long long *e;              // excess e(v), int64
  int32_t *hp, *hm;          // h+ (push heights), h- (pull heights), in [0, n]
  uint8_t *part;             // PART_*
  int32_t *q0, *q1;          // BFS frontier ping-pong
  int32_t *wl;               // active worklists [2 rounds][NB bins][n]
  int32_t *rl;               // relabelled vertices [NB bins][n] (RemoveInvalidEdges scope, R13)
  int32_t *inq;              // per-vertex "queued for the next discharge round" flag
  uint8_t *rlf;              // per-vertex "already in the relabelled list" flag
  int32_t *bul;              // bottom-up candidate queue [2 bins][n]
  long long *cq0, *cq1, *cqr; // chunk queues of the frontier ping-pong and of the relabelled list
  long long *cw0, *cw1;      // chunk queues of the discharge worklist ping-pong (vertices of > BIN1_MAX slots)
  int32_t *dcnt;             // chunked discharge: chunks of u finished in the current round
  int32_t *dmin;             // chunked discharge: lowest height among u's slots left residual (DMIN_NONE if none)
  int32_t *arc;              // chunked discharge: current-arc chunk of u (the last chunk that pushed); NULL: no probes
  long long *aq;             // asynchronous discharge ring (AQ_EMPTY when free), aq_mask + 1 entries
  int32_t aq_mask;
  int32_t async;             // 1: asynchronous discharge phase, 0: barrier-separated rounds
  int32_t async_warps;       // consumer warps per CTA in the asynchronous phase
  int32_t static_pp;         // MODE_STATIC: static push-pull initialisation (also saturate t's in-edges)
  int32_t bu_alpha;          // BFS: bottom-up when frontier slots x bu_alpha > unvisited slots (BU_ALPHA)
  int32_t dense_div;         // BFS: top-down by stores + compaction when frontier slots x dense_div >= S (DENSE_DIV)
  int32_t async_sleep_ns;    // back-off of a warp waiting for a ring item
  int32_t *cnt;              // local gap: [2 tracks][GAPW] vertices per height (this call)
  int32_t *cnt_next;         // DYN_PP: the final labels' histogram for the next call's warm start
  int32_t local_gap;         // 1: local gap exit on (R14 form 2)
  int32_t topo_div;          // topology-driven phase when > n / topo_div vertices are active (0: never)
  int32_t tail_items;        // async progress stop (<= 0: off)
  int32_t check_level;
  int32_t imm_act;           // async discharge: activate a pushed head at the push (returning atomic) instead of after the item
  int32_t dmaxch;            // discharge: at most this many chunk items per big-vertex activation (0: CH-slot chunks)
  int32_t scan2;             // chunked discharge: two-pass scan (list admissible slots, one claim, push)
  int32_t split;             // DYN_PP warm start: the certificate runs in k_reach (the PP launch stops
                             // after the warm iteration; MODE_PP_CONT continues if it fails)
  int32_t lazy;              // DYN_PP warm start: certify with the universal backward BFS (no pull BFS / stage 2)
  int32_t *plist;            // region P of push-pull stage 2
  int32_t *stamp;            // per-slot batch stamp (duplicate detection)
  const int32_t *bu, *bv, *bc;  // batch entries
  int32_t *bslot;            // slot of each batch entry
  int32_t *brec;             // per batch entry: residual delta, clamp, S->T saturation (undo of an invalid batch)
  const int4 *htab;          // (u,v) -> slot table {u, v, slot, rev[slot]}, x = -1 empty
  int32_t hmask;
  uint8_t *mask;             // cut output
  Ctl *ctl;
  volatile int32_t *dbg;     // mapped pinned host words: progress beacon for the host watchdog
  int32_t *trace;            // per-phase trace records (8 ints each), NULL unless tracing
  uint32_t *trace_cta;       // per-phase, per-CTA busy time (ns from the CTA's previous barrier exit to its arrival)
  int32_t trace_cap;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// progress beacon: block 0 / thread 0 publishes (phase, iter, round, level, a, b)
__device__ __forceinline__ void beacon(const Dev &d, int32_t phase, int32_t iter, int32_t round, int32_t lvl,
                                       int32_t a = 0, int32_t b = 0) {
  if (d.dbg && blockIdx.x == 0 && threadIdx.x == 0) {
    d.dbg[1] = iter; d.dbg[2] = round; d.dbg[3] = lvl; d.dbg[4] = a; d.dbg[5] = b;
    __threadfence_system();
    d.dbg[0] = phase;
  }
}

// ---------------------------------------------------------------- loads
__device__ __forceinline__ int32_t ldv(const int32_t *p) { return __ldcg(p); }
__device__ __forceinline__ long long ldv(const long long *p) { return __ldcg(p); }
__device__ __forceinline__ uint8_t ldv(const uint8_t *p) { return __ldcg(p); }
// L1-allocating load, for data that no thread of the grid changes in the current
// phase in a way the reader must observe (or whose stale values are harmless by
// construction).  Safe across phases: the grid barrier's ld.acquire.gpu + CTA
// barrier (cooperative_groups sync_grids_wait) orders the SM's later weak loads
// after every write made before the barrier, so no stale L1 line survives it.
#ifdef DMF_NO_L1
__device__ __forceinline__ int32_t ldl1(const int32_t *p) { return __ldcg(p); }
#else
__device__ __forceinline__ int32_t ldl1(const int32_t *p) { return __ldca(p); }
#endif
__device__ __forceinline__ uint32_t ldl1(const uint32_t *p) { return __ldca(p); }
__device__ __forceinline__ void atom_add(long long *p, long long x) {
  atomicAdd(reinterpret_cast<unsigned long long *>(p), static_cast<unsigned long long>(x));
}

// ---------------------------------------------------------------- groups
// One vertex is processed cooperatively by a group of 1 thread, 1 warp or 1 CTA.
// All members of a group call every collective below the same number of times.
struct ThreadG {
  static constexpr int size = 1;
  __device__ void sync() const {}
  __device__ int rank() const { return 0; }
  __device__ unsigned long long min(unsigned long long x) const { return x; }
  __device__ long long sum(long long x) const { return x; }
  __device__ long long bcast(long long x) const { return x; }
  __device__ long long exscan(long long x, long long &tot) const { tot = x; return 0; }
  __device__ bool any(bool p) const { return p; }
};

struct WarpG {
  static constexpr int size = 32;
  int lane;
  __device__ void sync() const { __syncwarp(); }
  __device__ int rank() const { return lane; }
  __device__ unsigned long long min(unsigned long long x) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long y = __shfl_xor_sync(0xffffffffu, x, o);
      x = y < x ? y : x;
    }
    return x;
  }
  __device__ long long sum(long long x) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
  }
  __device__ long long bcast(long long x) const { return __shfl_sync(0xffffffffu, x, 0); }
  __device__ bool any(bool p) const { return __any_sync(0xffffffffu, p); }
  __device__ long long exscan(long long x, long long &tot) const {
    long long inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    tot = __shfl_sync(0xffffffffu, inc, 31);
    return inc - x;
  }
};

// Sub-warp tile of W lanes (W = 8: four low-degree vertices per warp).  Tiles of a
// warp may diverge; every collective names only the tile's lanes.
template <int W>
struct TileG {
  static constexpr int size = W;
  int lane;          // lane within the warp
  unsigned mask;     // this tile's lanes
  __device__ TileG(int l) : lane(l), mask(((1u << W) - 1u) << (l & ~(W - 1))) {}
  __device__ void sync() const { __syncwarp(mask); }
  __device__ int rank() const { return lane & (W - 1); }
  __device__ unsigned long long min(unsigned long long x) const {
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
      unsigned long long y = __shfl_xor_sync(mask, x, o, W);
      x = y < x ? y : x;
    }
    return x;
  }
  __device__ long long sum(long long x) const {
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) x += __shfl_xor_sync(mask, x, o, W);
    return x;
  }
  __device__ long long bcast(long long x) const { return __shfl_sync(mask, x, 0, W); }
  __device__ bool any(bool p) const { return __any_sync(mask, p); }
};

// CTA group: needs WPB+1 long longs of shared scratch.
struct BlockG {
  static constexpr int size = NT;
  long long *sm;   // shared scratch
  __device__ void sync() const { __syncthreads(); }
  __device__ int rank() const { return threadIdx.x; }
  __device__ unsigned long long min(unsigned long long x) const {
    WarpG w{(int)(threadIdx.x & 31)};
    x = w.min(x);
    if (w.lane == 0) sm[threadIdx.x >> 5] = (long long)x;
    __syncthreads();
    unsigned long long r = ~0ull;
#pragma unroll 4
    for (int i = 0; i < WPB; i++) { unsigned long long y = (unsigned long long)sm[i]; r = y < r ? y : r; }
    __syncthreads();
    return r;
  }
  __device__ long long sum(long long x) const {
    WarpG w{(int)(threadIdx.x & 31)};
    x = w.sum(x);
    if (w.lane == 0) sm[threadIdx.x >> 5] = x;
    __syncthreads();
    long long r = 0;
#pragma unroll 4
    for (int i = 0; i < WPB; i++) r += sm[i];
    __syncthreads();
    return r;
  }
  __device__ bool any(bool p) const { return __syncthreads_or(p) != 0; }
  __device__ long long bcast(long long x) const {
    if (threadIdx.x == 0) sm[WPB] = x;
    __syncthreads();
    long long r = sm[WPB];
    __syncthreads();
    return r;
  }
  __device__ long long exscan(long long x, long long &tot) const {
    WarpG w{(int)(threadIdx.x & 31)};
    long long wt;
    long long ex = w.exscan(x, wt);
    if (w.lane == 0) sm[threadIdx.x >> 5] = wt;
    __syncthreads();
    long long before = 0, all = 0;
    const int me = threadIdx.x >> 5;
    for (int i = 0; i < WPB; i++) { long long y = sm[i]; if (i < me) before += y; all += y; }
    __syncthreads();
    tot = all;
    return before + ex;
  }
};

// Warp-aggregated append (ballot + popc + one leader atomic per warp).
// Must be called by all 32 lanes (convergent).
__device__ __forceinline__ void warp_append(bool pred, int32_t val, int32_t *list, int32_t *cnt) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (m == 0) return;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(cnt, __popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (pred) list[base + __popc(m & ((1u << lane) - 1u))] = val;
}

}  // namespace dmf
