// solve.cuh -- the persistent cooperative kernel of libdmf (sm_100a).
//
// One launch runs one API call to convergence entirely on the device (the paper's
// "entirely GPU-resident ... without CPU intervention"; termination "by
// checking if an active vertex exists"): phases are separated by grid-wide
// barriers instead of kernel boundaries, and the loop condition is evaluated on the
// device.  The phases follow the paper's algorithms:
//
//   batch      Updates Processing, Alg.5 P:393-407 (validated first, R11; O(k), R10)
//   source     saturate s's residual out-slots, Alg.1 l.9-13 / Alg.4 l.3-8 (R3)
//   S->T       saturate touched S->T slots, Alg.8 l.10-13 (R12: with excess deltas)
//   RESET      heights of the sink/source sets, Alg.1 l.15, Alg.4 l.9-16, Alg.8 l.16-24
//   BFS        BFS_Backward / forward BFS (global relabel),
//              level-synchronous, fused with the active-vertex worklist compaction
//               and the termination test (R9: a FRESH BFS decides)
//   DISCHARGE  PushRelabel (Alg.2) / PullRelabel (Alg.6, R7),
//              in ROUNDS: a vertex made active by a push (its excess crosses 0) is
//              queued for the next round without waiting for another global relabel
//              -- the "immediately process any new active vertices" property of the
//              topology-driven schedule on a data-driven worklist
//   RIE        RemoveInvalidEdges (Alg.3 P:217-231 / Alg.7) after every
//              round, relabelled vertices only (R13)
//
// Tracks.  The push track (h+, Alg.2/3) and the pull track (h-, Alg.6/7) are the
// same code with the roles of the residual array and its mirror swapped:
//   push: heights hp, discharge scans res[i]  = c_f(u,v), BFS scans rres[i] = c_f(v,u),
//         active e > 0, roots {t} u deficits, never claims s
//   pull: heights hm, discharge scans rres[i] = c_f(v,u), BFS scans res[i]  = c_f(u,v),
//         active e < 0, roots {s} u overflowing, never claims t
// A pull of d on in-slot (v,u) is exactly a push of d on out-slot (u,v) with
// (res, rres) exchanged and the excess sign flipped.
#pragma once

#include "dmf_device.cuh"

namespace dmf {

constexpr int MAX_ROUNDS = 4096;  // hard cap of discharge rounds per global relabel

// Block-staged appends (BFS): see stage_conv / stage_flush.
constexpr int SF = 1024;            // staged entries per frontier bin (bins 0, 1)
constexpr int SW = 256;             // staged entries per worklist bin (bins 0..3)

struct Stage {
  int32_t cnt[6];                   // 0,1: frontier bins 0,1; 2..5: worklist bins 0..3
  int32_t base[6];
  int32_t lv[2];                    // vertices labelled in this phase per track (local-gap level counts)
  int32_t f[2][SF];
  int32_t w[4][SW];
};

struct TileSm {
  int32_t cnt[8];
  int32_t base[8];
};

constexpr int32_t ADMCAP = 64;      // admissible slots listed per warp by a chunk scan (discharge_chunk)

struct Smem {
  long long red[WPB + 1];
  unsigned long long stat[ST_N];
  long long budget[4 * WPB + 1];   // push budgets: one per sub-warp tile / warp + one for the CTA
  unsigned long long work;         // discharge work of this CTA in the current round
  unsigned long long tprev;        // trace mode: this CTA's last barrier exit
  unsigned long long tclk;         // PhaseClock: block 0's last lap
  long long cv[8];                 // control words snapped once per CTA (cta_snap)
  int32_t acnt, rcnt;              // discharge: staged activations / relabelled vertices (in st.f / st.w)
  int32_t ccnt;                    // discharge: staged push heads (activation candidates)
  int32_t wcc[WPB];                // async discharge: per-warp candidate counts (warp w: cand[w*WCAP..])
  int32_t astop;                   // async discharge: this CTA has seen ctl->astop
  unsigned long long apoll;        // async discharge: last global poll of ctl->astop
  int32_t amode;                   // current discharge phase: 1 = asynchronous ring, 0 = rounds / topology
  int32_t topo;                    // current discharge phase is topology-driven
  int32_t tslot;                   // topology round r: activity flag ctl->tact[r % 3]
  int32_t lvcnt[2];                // BFS: vertices labelled by this CTA in the current level, per track
  int32_t cand[2048];
  int32_t adm_i[WPB * ADMCAP], adm_v[WPB * ADMCAP], adm_r[WPB * ADMCAP];   // chunk scan: admissible slots per warp
  Stage st;                    // block-staged appends (BFS)
  TileSm ts;                   // tiled compaction (dense top-down BFS levels)
};

// Phase clock (block 0, thread 0): time between consecutive grid barriers is
// charged to the phase that just ran.
// (Stateless: the timestamp lives in shared memory, so no thread keeps a clock
// object in local memory.)
struct PhaseClock {
  __device__ void start(Smem &sm) { if (blockIdx.x == 0 && threadIdx.x == 0) sm.tclk = gtimer(); }
  __device__ void lap(const Dev &d, Smem &sm, int which, int32_t it = 0, int32_t sub = 0, int32_t items = 0,
                      int32_t extra = 0);
};

struct Track {
  int32_t *hgt;
  int32_t *F;        // residual scanned by discharge (out-slot direction of the track)
  int32_t *R;        // its mirror
  const int32_t *B;  // residual scanned by BFS
  int32_t excl;      // vertex never claimed (s for push, t for pull)
  int32_t sign;      // +1 push, -1 pull
};

__device__ __forceinline__ Track make_track(const Dev &d, int tr) {
  Track k;
  if (tr == 0) { k.hgt = d.hp; k.F = d.res; k.R = d.rres; k.B = d.rres; k.excl = d.s; k.sign = 1; }
  else         { k.hgt = d.hm; k.F = d.rres; k.R = d.res; k.B = d.res; k.excl = d.t; k.sign = -1; }
  return k;
}

__device__ __forceinline__ void sstat_add(Smem &sm, int which, unsigned long long x) {
  if (x) atomicAdd(&sm.stat[which], x);
}

// ---------------------------------------------------------------------------
// Local gap (R14 form 2; the gap heuristic of P:114).  cnt[tr][h] counts the vertices
// of track tr's region at height h < GAPW: the BFS adds each labelled vertex to its
// level, a lift moves u from its old height to the new one.  When a lift empties a
// level g, no vertex above g can reach a root of the track any more (a residual path
// descends at most one level per edge under a valid labelling, so it would cross g),
// and every vertex above the lowest emptied level stops discharging for the rest of
// the phase WITHOUT writing its height: RIE and the next fresh BFS (R9) see the same
// state as without the heuristic.  A count that is transiently wrong under races can
// only stop a vertex that could still reach a root; it stays active and the fresh BFS
// re-collects it, so the heuristic never changes a result, only the work.
__device__ __forceinline__ int32_t gap_limit(const Dev &d, int tr) {
  if (!d.local_gap) return 0x7fffffff;
  const int32_t g = *(const volatile int32_t *)&d.ctl->gtop[tr];
  return g ? GAPW - g : 0x7fffffff;
}
// u of track tr moves from height `from` (< |V|) to `to` (<= |V|)
__device__ __forceinline__ void gap_move(const Dev &d, Smem &sm, int tr, int32_t from, int32_t to) {
  if (!d.local_gap) return;
  int32_t *c = d.cnt + tr * GAPW;
  if (to < GAPW && to < d.n) atomicAdd(c + to, 1);          // arrive first: u itself never leaves a false gap
  if (from < GAPW && atomicSub(c + from, 1) == 1 && from > 0) {
    atomicMax(&d.ctl->gtop[tr], GAPW - from);
    sstat_add(sm, ST_GAP_LEVELS, 1);
  }
}

__device__ void PhaseClock::lap(const Dev &d, Smem &sm, int which, int32_t it, int32_t sub, int32_t items,
                                int32_t extra) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long now = gtimer();
    const unsigned long long t = sm.tclk;
    sm.stat[which] += now - t;
    if (d.trace && d.ctl->ntrace < d.trace_cap) {       // per-phase trace record (DMF_TRACE)
      int32_t *rec = d.trace + 8 * d.ctl->ntrace++;
      rec[0] = which - ST_T_PRO; rec[1] = it; rec[2] = sub; rec[3] = items; rec[4] = extra; rec[5] = (int32_t)(now - t);
      const unsigned long long sl = d.ctl->slow;        // slowest discharge of the phase (if any)
      rec[6] = (int32_t)(sl >> 32); rec[7] = (int32_t)(sl & 0xffffffffu);
      d.ctl->slow = 0;
    }
    sm.tclk = now;
  }
}

// Grid barrier.  In trace mode every CTA records how long it was busy in the phase
// that ends here (load-balance / tail diagnostics, dmf_get_trace_cta).
__device__ __forceinline__ void gsync(const Dev &d, cg::grid_group &grid, Smem &sm) {
  if (d.trace_cta) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const int32_t rec = ldv(&d.ctl->ntrace);
      if (rec < d.trace_cap) d.trace_cta[(size_t)rec * gridDim.x + blockIdx.x] = (uint32_t)(gtimer() - sm.tprev);
    }
  }
  grid.sync();
  if (d.trace_cta && threadIdx.x == 0) sm.tprev = gtimer();
}

// Global warp index, CTA-major: with few items they land on different SMs (each SM's
// memory pipeline serves one dependent chain instead of sixteen).
__device__ __forceinline__ int32_t gwarp_spread() { return (int32_t)((threadIdx.x >> 5) * gridDim.x + blockIdx.x); }

__device__ __forceinline__ int bin_of(const Dev &d, int32_t v) {
  const int32_t deg = d.row[v + 1] - d.row[v];
  return deg <= BIN0_MAX ? 0 : (deg <= BIN1_MAX ? 1 : (deg <= BIN2_MAX ? 2 : 3));
}

// Binned list view: NB buffers (n entries each) and NB counters.  A CHUNKED list
// (BFS frontiers, relabelled lists: phases whose per-slot work is independent)
// stores every vertex of more than BIN1_MAX slots as ceil(deg/CH) (vertex, chunk)
// entries in `cq` (count in c[3]), so that one warp takes one CH-slot chunk and
// hub rows are spread over the whole grid (edge-balanced work units).
constexpr int32_t CH = 512;
// BFS frontier chunks of big rows: CH slots, or BCH (one warp-step each) in the small
// certificate BFS of a DYN_PP warm start, whose levels are bound by latency, not scans
constexpr int32_t BCH = 128;

// Discharge chunks of a big vertex: CH slots each, but at most dmaxch chunks per
// activation (then bigger chunks, multiples of 128 slots) when dmaxch > 0.  A hub
// re-activated many times then costs a bounded number of ring items per activation.
__device__ __forceinline__ int32_t dis_csize(const Dev &d, int32_t deg) {
  if (d.dmaxch <= 0) return CH;
  int32_t c = (deg + d.dmaxch - 1) / d.dmaxch;
  c = (c + 127) & ~127;
  return c < CH ? CH : c;
}
__device__ __forceinline__ int32_t dis_nch(const Dev &d, int32_t deg) {
  const int32_t c = dis_csize(d, deg);
  return (deg + c - 1) / c;
}

struct BL {
  int32_t *buf;   // bin b at buf + b*n
  int32_t *c;
  int32_t n;
  long long *cq;  // chunk queue (nullptr: not chunked)
  __device__ int32_t *bin(int b) const { return buf + (size_t)b * n; }
};

__device__ __forceinline__ long long chunk_entry(int32_t v, uint32_t tag, int32_t k) {
  return ((long long)k << 32) | (long long)((uint32_t)v | tag);
}

// append v (with track tag) to its degree bin; convergent (whole warp) or not
__device__ __forceinline__ void bl_append_conv(const Dev &d, const BL &bl, bool pred, int32_t v, uint32_t tag) {
  const int32_t deg = pred ? d.row[v + 1] - d.row[v] : 0;
  const int bin = !pred ? -1 : (deg <= BIN0_MAX ? 0 : (deg <= BIN1_MAX ? 1 : (deg <= BIN2_MAX ? 2 : 3)));
  warp_append(bin == 0, (int32_t)((uint32_t)v | tag), bl.bin(0), bl.c);
  warp_append(bin == 1, (int32_t)((uint32_t)v | tag), bl.bin(1), bl.c + 1);
  if (bl.cq) {
    const int32_t nch = bin >= 2 ? (deg + CH - 1) / CH : 0;
    if (__ballot_sync(0xffffffffu, nch > 0) == 0) return;
    WarpG g{(int)(threadIdx.x & 31)};
    long long tot;
    const int32_t ex = (int32_t)g.exscan(nch, tot);
    int32_t base = 0;
    if (g.lane == 0) base = atomicAdd(bl.c + 3, (int32_t)tot);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int32_t k = 0; k < nch; k++) bl.cq[base + ex + k] = chunk_entry(v, tag, k);
  } else {
    warp_append(bin == 2, (int32_t)((uint32_t)v | tag), bl.bin(2), bl.c + 2);
    warp_append(bin == 3, (int32_t)((uint32_t)v | tag), bl.bin(3), bl.c + 3);
  }
}
__device__ __forceinline__ void bl_append_one(const Dev &d, const BL &bl, int32_t v, uint32_t tag, bool dis = false) {
  const int32_t deg = d.row[v + 1] - d.row[v];
  const int bin = deg <= BIN0_MAX ? 0 : (deg <= BIN1_MAX ? 1 : (deg <= BIN2_MAX ? 2 : 3));
  if (bin >= 2 && bl.cq) {
    const int32_t nch = dis ? dis_nch(d, deg) : (deg + CH - 1) / CH;
    const int32_t pos = atomicAdd(bl.c + 3, nch);
    for (int32_t k = 0; k < nch; k++) bl.cq[pos + k] = chunk_entry(v, tag, k);
    return;
  }
  const int pos = atomicAdd(bl.c + bin, 1);
  bl.bin(bin)[pos] = (int32_t)((uint32_t)v | tag);
}

// Process a binned list: CTA per bin-3 / bin-2 entry, warp per bin-1 entry, thread
// per bin-0 entry.  fn(group, entry).
template <class Fn>
__device__ __forceinline__ void process_bl(const BL &bl, const int32_t c[NB], Smem &sm, Fn fn) {
  {
    BlockG g{sm.red};
    for (int b = 3; b >= 2; b--) {
      const int32_t *lst = bl.bin(b);
      for (int32_t x = blockIdx.x; x < c[b]; x += gridDim.x) fn(g, lst[x]);
    }
  }
  {
    WarpG g{(int)(threadIdx.x & 31)};
    const int32_t *b = bl.bin(1);
    const int32_t gw = gwarp_spread(), nw = gridDim.x * WPB;
    for (int32_t x = gw; x < c[1]; x += nw) fn(g, b[x]);
  }
  {
    TileG<8> g((int)(threadIdx.x & 31));
    const int32_t *b = bl.bin(0);
    const int32_t gt = (int32_t)((threadIdx.x >> 3) * gridDim.x + blockIdx.x), nt = (gridDim.x * NT) >> 3;
    for (int32_t x = gt; x < c[0]; x += nt) fn(g, b[x]);
  }
}

// Dynamic variant (discharge rounds): every CTA, warp and 8-lane tile takes its
// first item statically (group id) and the next ones from atomic claim counters
// `cl[0..2]` (zeroed by the caller's counter discipline), so a CTA busy with a big
// vertex takes nothing else and idle groups absorb the remaining items.  A group
// claims only after finishing an item: a near-empty round costs no claims (one
// single-address atomic per group would serialise ~19k tile claims at L2).
template <class Fn>
__device__ __forceinline__ void process_bl_dyn(const BL &bl, const int32_t c[NB], Smem &sm, int32_t *cl, Fn fn) {
  {
    BlockG g{sm.red};
    const int32_t nbig = c[3] + c[2];
    long long x = blockIdx.x;
    while (x < nbig) {
      fn(g, x < c[3] ? bl.bin(3)[x] : bl.bin(2)[x - c[3]]);
      if (threadIdx.x == 0) x = (long long)gridDim.x + atomicAdd(cl, 1);
      x = g.bcast(x);
    }
  }
  {
    WarpG g{(int)(threadIdx.x & 31)};
    const int32_t *b = bl.bin(1);
    const int32_t nw = gridDim.x * WPB;
    int32_t x = gwarp_spread();
    while (x < c[1]) {
      fn(g, b[x]);
      if (g.lane == 0) x = nw + atomicAdd(cl + 1, 1);
      x = __shfl_sync(0xffffffffu, x, 0);
    }
  }
  {
    TileG<8> g((int)(threadIdx.x & 31));
    const int32_t *b = bl.bin(0);
    const int32_t ntl = (gridDim.x * NT) >> 3;
    int32_t x = (int32_t)((threadIdx.x >> 3) * gridDim.x + blockIdx.x);
    while (x < c[0]) {
      fn(g, b[x]);
      if (g.rank() == 0) x = ntl + atomicAdd(cl + 2, 1);
      x = __shfl_sync(g.mask, x, 0, 8);
    }
  }
}

// Uniform control-word reads (counters published by the last grid barrier): ONE
// request per CTA, broadcast through shared memory.  If every warp read them, the
// same L2 line would take ~4.7k requests per word per phase, serialised in one L2
// slice: ~9 us of floor per phase on B200 (measured with dmf_get_trace_cta).
// fetch(k) is evaluated by thread k < K.
template <class F>
__device__ __forceinline__ void cta_snap(Smem &sm, int K, F fetch) {
  __syncthreads();
  if ((int)threadIdx.x < K) sm.cv[threadIdx.x] = fetch((int)threadIdx.x);
  __syncthreads();
}
__device__ __forceinline__ void cta_counts(Smem &sm, const int32_t *p, int32_t c[NB]) {
  cta_snap(sm, NB, [&](int k) { return (long long)ldv(p + k); });
#pragma unroll
  for (int b = 0; b < NB; b++) c[b] = (int32_t)sm.cv[b];
}
__device__ __forceinline__ long long cta_ld(Smem &sm, const long long *p) {
  cta_snap(sm, 1, [&](int) { return ldv(p); });
  return sm.cv[0];
}
__device__ __forceinline__ int32_t cta_ld(Smem &sm, const int32_t *p) {
  cta_snap(sm, 1, [&](int) { return (long long)ldv(p); });
  return (int32_t)sm.cv[0];
}

__device__ __forceinline__ void read_counts(const int32_t *p, int32_t c[NB]) {
#pragma unroll
  for (int b = 0; b < NB; b++) c[b] = ldv(p + b);
}
__device__ __forceinline__ int32_t total(const int32_t c[NB]) {
  int32_t t = 0;
#pragma unroll
  for (int b = 0; b < NB; b++) t += c[b];
  return t;
}

// Queue a vertex whose excess (track-signed) just crossed from <= 0 to > 0 for the
// next discharge round, at most once per round (inq flag).
// Discharge-phase appends are BLOCK-STAGED: the entry goes to a shared-memory list
// (activations in st.f, relabelled vertices in st.w) and vflush moves each CTA's list
// to the global binned list with one global atomic per bin at the end of the round
// (a single global counter per list took one L2 atomic per activation, serialised
// in one L2 slice).  Overflow goes straight to the global list.
constexpr int32_t ACAP = 2 * SF;     // staged activations per CTA
constexpr int32_t RCAP = 4 * SW;     // staged relabelled vertices per CTA
__device__ __forceinline__ int32_t *act_buf(Smem &sm);
__device__ __forceinline__ int32_t *rel_buf(Smem &sm);

#ifdef DMF_DEBUG_BUSY
__device__ __forceinline__ void dbg_rec(const Dev &d, int32_t kind, int32_t a, int32_t b, int32_t c, int32_t e5) {
  if (!d.trace) return;
  const int32_t r = atomicAdd(&d.ctl->ntrace, 1);
  if (r >= d.trace_cap) return;
  int32_t *p = d.trace + 8 * r;
  p[0] = kind; p[1] = a; p[2] = (int32_t)(blockIdx.x * WPB + (threadIdx.x >> 5)); p[3] = b; p[4] = c; p[5] = e5;
  p[6] = (int32_t)(gtimer() & 0x7fffffff); p[7] = 0;
}
#define DBG(...) dbg_rec(__VA_ARGS__)
#else
#define DBG(...)
#endif
// Asynchronous discharge: append v (every CH-slot chunk of a big row) to the ring.  One
// atomic reserves the ring positions AND counts the items as pending, so a consumer
// can never finish an item before it is counted.
// A big vertex (> BIN1_MAX slots) activated through the ring first gets ONE probe item:
// its current-arc chunk (the last chunk that pushed, d.arc).  Only if the probe leaves
// excess does it enqueue all its chunks (enqueue_full).  A hub drained again and again
// by its neighbours (pull track) is then re-served by one item, not by all its chunks.
constexpr uint32_t PROBE_BIT = 0x40000000u;
__device__ __forceinline__ void enqueue_items(const Dev &d, int32_t v, uint32_t tag, int32_t nch, uint32_t k0) {
  const unsigned long long old = atomicAdd(&d.ctl->aw, ((unsigned long long)nch << 32) | (unsigned long long)nch);
  const uint32_t pos = (uint32_t)(old >> 32);
  DBG(d, 202, v, (int32_t)pos, (int32_t)(uint32_t)old, nch);
  for (int32_t k = 0; k < nch; k++)
    *(volatile long long *)(d.aq + ((pos + (uint32_t)k) & (uint32_t)d.aq_mask)) = chunk_entry(v, tag, (int32_t)(k0 + k));
}
__device__ __forceinline__ void async_enqueue(const Dev &d, int32_t v, uint32_t tag) {
  const int32_t deg = d.row[v + 1] - d.row[v];
  if (deg > BIN1_MAX && d.arc) {
    const int32_t a = ldv(d.arc + v);
    const int32_t nch = dis_nch(d, deg);
    enqueue_items(d, v, tag, 1, PROBE_BIT | (uint32_t)(a < nch ? a : 0));
    return;
  }
  enqueue_items(d, v, tag, deg > BIN1_MAX ? dis_nch(d, deg) : 1, 0u);
}

__device__ __forceinline__ void activate(const Dev &d, const Track &k, const BL &nxt, int32_t v, uint32_t tag,
                                         Smem &sm, bool ring = true) {
  if (v == d.s || v == d.t) return;
  if (sm.topo) {                                    // topology-driven: the next sweep finds v itself
    sstat_add(sm, ST_ACTIVATIONS, 1);
    d.ctl->tact[sm.tslot] = 1;
    return;
  }
  if (atomicCAS(d.inq + v, 0, 1) != 0) return;     // (a vertex at height >= |V| exits at once)
  sstat_add(sm, ST_ACTIVATIONS, 1);
  if (sm.amode && ring) { async_enqueue(d, v, tag); return; }
  const int32_t pos = atomicAdd(&sm.acnt, 1);
  if (pos < ACAP) act_buf(sm)[pos] = (int32_t)((uint32_t)v | tag);
  else bl_append_one(d, nxt, v, tag, true);
}
// One push of d on slot i = (u,v) of track k (ri = rev[i]): the four residual updates and
// e(v) += d are fire-and-forget reductions; v is staged as an activation CANDIDATE that
// dis_flush checks once per round (e(v) > 0 after a fence: the last pusher into v sees
// every push), so no push waits for an atomic's return.  Candidate overflow falls back
// to the returning atomic and the 0-crossing test.
constexpr int32_t CCAP = 2048;
constexpr int32_t WCAP = CCAP / WPB;   // async: per-warp candidate slots
__device__ __forceinline__ void push_slot(const Dev &d, const Track &k, const BL &nxt, int32_t i, int32_t ri, int32_t v,
                                          int32_t take, uint32_t tag, Smem &sm);

__device__ __forceinline__ void stage_relabelled(const Dev &d, const BL &rl, int32_t u, uint32_t tag, Smem &sm) {
  const int32_t pos = atomicAdd(&sm.rcnt, 1);
  if (pos < RCAP) rel_buf(sm)[pos] = (int32_t)((uint32_t)u | tag);
  else bl_append_one(d, rl, u, tag);
}

__device__ __forceinline__ void push_slot(const Dev &d, const Track &k, const BL &nxt, int32_t i, int32_t ri, int32_t v,
                                          int32_t take, uint32_t tag, Smem &sm) {
  atomicSub(k.F + i, take);          // c_f(u,v) -= d
  atomicSub(k.R + ri, take);         //   mirror
  atomicAdd(k.F + ri, take);         // c_f(v,u) += d
  atomicAdd(k.R + i, take);          //   mirror
  if (sm.amode && d.imm_act) {
    // asynchronous phase: the returning atomic tells whether e(v) crossed 0, and v is
    // queued at once (the next warp sees e(v): the atomic is performed; a residual it
    // reads before this push's reductions land is only lower, so it never pushes twice)
    const long long eo = (long long)atomicAdd(reinterpret_cast<unsigned long long *>(d.e + v),
                                              (unsigned long long)((long long)take * k.sign)) * k.sign;
    if (eo <= 0 && eo + take > 0) activate(d, k, nxt, v, tag, sm);
    return;
  }
  // rounds: one list per CTA, checked at the round end; async: one list per warp,
  // checked after the warp's item (async_candidates)
  const int w = (int)(threadIdx.x >> 5);
  const int32_t pos = sm.amode ? atomicAdd(&sm.wcc[w], 1) : atomicAdd(&sm.ccnt, 1);
  if (pos < (sm.amode ? WCAP : CCAP)) {
    atom_add(d.e + v, (long long)take * k.sign);                           // e(v) += d
    sm.cand[sm.amode ? w * WCAP + pos : pos] = (int32_t)((uint32_t)v | tag);
  } else {
    const long long eo = (long long)atomicAdd(reinterpret_cast<unsigned long long *>(d.e + v),
                                              (unsigned long long)((long long)take * k.sign)) * k.sign;
    if (eo <= 0 && eo + take > 0) activate(d, k, nxt, v, tag, sm);
  }
}

// ---------------------------------------------------------------------------
// BFS (global relabel).  Level-synchronous; per level and per
// track either
//   top-down   the frontier's rows are scanned: a residual edge (v -> w) [push
//              track] / (w -> v) [pull track] from frontier vertex w labels v, or
//   bottom-up  every unlabelled vertex of the track's region looks for a residual
//              edge into the frontier and stops at the first (direction-optimising
//              BFS; chosen when the frontier's slots exceed 1/BU_ALPHA of the
//              unlabelled vertices' slots).
// Region encoding: RESET gives vertices outside a track's region the height |V|+1,
// so "unlabelled" (h == |V|) already means "in the region": one gather per slot.
// Top-down claims are atomicCAS(h, |V|, lvl+1) (unique claimer); bottom-up claims
// are plain stores (one examiner per vertex).  Claimed vertices are appended to the
// next frontier and, if active, to the worklist through BLOCK-STAGED appends:
// warp ballot + shared-memory reservation, flushed with one global atomic per list
// per CTA at the end of the phase (the paper's ballot worklist).
constexpr unsigned long long BU_ALPHA = 2;
constexpr unsigned long long DENSE_DIV = 64;      // top-down by stores + compaction iff frontier slots >= S/64
constexpr int TILE_ITEMS = 4;                     // vertices per thread per compaction tile

struct BfsCtx {
  int32_t lvl;
  int32_t tgt;                      // height the vertices labelled in this phase receive (lvl + 1; 0 in RESET)
  int32_t bch;                      // frontier chunk size (CH or BCH)
  bool collect;
  uint32_t bu;                      // bit tr: bottom-up this level on track tr
  uint32_t dense;                   // bit tr: top-down by idempotent stores + compaction
  BL next, wl;
  unsigned long long *fs_next;      // [2] slot counts of the next frontier per track
  __device__ bool isbu(int tr) const { return (bu >> tr) & 1u; }
  __device__ bool isdense(int tr) const { return (dense >> tr) & 1u; }
};

// Per-thread slot sums of the next frontier, per track (two registers: an array
// indexed by the track would live in local memory).
struct FS {
  long long a = 0, b = 0;
  __device__ void add(int tr, long long x) { if (tr) b += x; else a += x; }
};

// ---- block-staged appends (Stage is declared with Smem above) ----------------------

__device__ __forceinline__ int32_t *stage_buf(Stage &st, int k) { return k < 2 ? st.f[k] : st.w[k - 2]; }
__device__ __forceinline__ int32_t stage_cap(int k) { return k < 2 ? SF : SW; }
__device__ __forceinline__ void stage_target(const BL &next, const BL &wl, int k, int32_t *&list, int32_t *&cnt) {
  if (k < 2) { list = next.bin(k); cnt = next.c + k; } else { list = wl.bin(k - 2); cnt = wl.c + (k - 2); }
}

// warp-convergent append of `val` into stage k (overflow goes straight to global)
__device__ __forceinline__ void stage_conv(Stage &st, int k, int32_t *glist, int32_t *gcnt, bool pred, int32_t val) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (m == 0) return;
  const int lane = threadIdx.x & 31;
  const int lead = __ffs(m) - 1;
  int pos = 0;
  if (lane == lead) pos = atomicAdd(&st.cnt[k], __popc(m));
  pos = __shfl_sync(0xffffffffu, pos, lead) + __popc(m & ((1u << lane) - 1u));
  const bool in_sm = pred && pos < stage_cap(k);
  if (in_sm) stage_buf(st, k)[pos] = val;
  warp_append(pred && !in_sm, val, glist, gcnt);
}

__device__ __forceinline__ void stage_one(Stage &st, int k, int32_t *glist, int32_t *gcnt, int32_t val) {
  const int pos = atomicAdd(&st.cnt[k], 1);
  if (pos < stage_cap(k)) { stage_buf(st, k)[pos] = val; return; }
  glist[atomicAdd(gcnt, 1)] = val;
}

// block-wide: move the staged entries to their global lists (one atomic per list)
__device__ __forceinline__ void stage_flush(Stage &st, const BL &next, const BL &wl) {
  __syncthreads();
  if (threadIdx.x < 6) {
    const int k = threadIdx.x;
    const int32_t c = min(st.cnt[k], stage_cap(k));
    int32_t *list, *cnt;
    stage_target(next, wl, k, list, cnt);
    st.base[k] = c ? atomicAdd(cnt, c) : 0;
  }
  __syncthreads();
  for (int k = 0; k < 6; k++) {
    const int32_t c = min(st.cnt[k], stage_cap(k));
    if (c == 0) continue;
    int32_t *list, *cnt;
    stage_target(next, wl, k, list, cnt);
    const int32_t *b = stage_buf(st, k);
    for (int32_t i = threadIdx.x; i < c; i += NT) list[st.base[k] + i] = b[i];
  }
  __syncthreads();
  if (threadIdx.x < 6) st.cnt[threadIdx.x] = 0;
  __syncthreads();
}

__device__ __forceinline__ int front_bin(int32_t deg) { return deg <= BIN0_MAX ? 0 : (deg <= BIN1_MAX ? 1 : 2); }
__device__ __forceinline__ int wl_bin(int32_t deg) {
  return deg <= BIN0_MAX ? 0 : (deg <= BIN1_MAX ? 1 : (deg <= BIN2_MAX ? 2 : 3));
}

// warp-convergent: every lane with pred appends ceil(deg/CH) chunk entries of v to bl's
// chunk queue (count in bl.c[3]); one global atomic per warp
__device__ __forceinline__ void chunks_conv(const Dev &d, const BL &bl, bool pred, int32_t deg, int32_t v, uint32_t tag) {
  if (__ballot_sync(0xffffffffu, pred) == 0) return;
  const int32_t nch = pred ? dis_nch(d, deg) : 0;
  WarpG g{(int)(threadIdx.x & 31)};
  long long tot;
  const int32_t ex = (int32_t)g.exscan(nch, tot);
  int32_t base = 0;
  if (g.lane == 0) base = atomicAdd(bl.c + 3, (int32_t)tot);
  base = __shfl_sync(0xffffffffu, base, 0);
  for (int32_t k = 0; k < nch; k++) bl.cq[base + ex + k] = chunk_entry(v, tag, k);
}

// warp-convergent: claimed vertex -> next frontier (+ worklist if active); counts
// the claimed vertex's slots into fs[track]
__device__ __forceinline__ void claim_push_deg(const Dev &d, Stage &st, const BfsCtx &c, bool claimed, bool act,
                                               int32_t v, int tr, FS &fs, int32_t deg);
__device__ __forceinline__ void claim_push(const Dev &d, Stage &st, const BfsCtx &c, bool claimed, bool act, int32_t v,
                                           int tr, FS &fs) {
  claim_push_deg(d, st, c, claimed, act, v, tr, fs, claimed ? d.row[v + 1] - d.row[v] : 0);
}
// (deg = the claimed vertex's slot count, loaded by the caller)
__device__ __forceinline__ void claim_push_deg(const Dev &d, Stage &st, const BfsCtx &c, bool claimed, bool act,
                                               int32_t v, int tr, FS &fs, int32_t deg) {
  const int fb = claimed ? front_bin(deg) : -1;
  const int32_t val = (int32_t)((uint32_t)v | (tr ? TRACK_BIT : 0u));
  stage_conv(st, 0, c.next.bin(0), c.next.c, fb == 0, val);
  stage_conv(st, 1, c.next.bin(1), c.next.c + 1, fb == 1, val);
  if (__ballot_sync(0xffffffffu, fb == 2)) {          // big rows -> edge-balanced chunks
    const int32_t nch = fb == 2 ? (deg + c.bch - 1) / c.bch : 0;
    WarpG g{(int)(threadIdx.x & 31)};
    long long tot;
    const int32_t ex = (int32_t)g.exscan(nch, tot);
    int32_t base = 0;
    if (g.lane == 0) base = atomicAdd(c.next.c + 3, (int32_t)tot);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int32_t k = 0; k < nch; k++) c.next.cq[base + ex + k] = chunk_entry(v, tr ? TRACK_BIT : 0u, k);
  }
  if (c.collect) {                  // active: queued for discharge round 0 (inq: see activate)
    const int wb = act ? wl_bin(deg) : -1;
    if (act) d.inq[v] = 1;
    stage_conv(st, 2, c.wl.bin(0), c.wl.c, wb == 0, val);
    stage_conv(st, 3, c.wl.bin(1), c.wl.c + 1, wb == 1, val);
    chunks_conv(d, c.wl, wb >= 2, deg, v, tr ? TRACK_BIT : 0u);   // big rows: chunked discharge
  }
  if (claimed) fs.add(tr, deg);
  if (d.local_gap) {                // level counts of the local gap (R14 form 2)
    const unsigned m = __ballot_sync(0xffffffffu, claimed);
    if (m) {
      const unsigned m1 = __ballot_sync(0xffffffffu, claimed && tr);
      if ((threadIdx.x & 31) == 0) {
        if (m & ~m1) atomicAdd(&st.lv[0], __popc(m & ~m1));
        if (m1) atomicAdd(&st.lv[1], __popc(m1));
      }
    }
  }
}

// single-thread version (bottom-up pass B leaders)
__device__ __forceinline__ void claim_one(const Dev &d, Stage &st, const BfsCtx &c, bool act, int32_t v, int tr,
                                          FS &fs) {
  const int32_t deg = d.row[v + 1] - d.row[v];
  const int32_t val = (int32_t)((uint32_t)v | (tr ? TRACK_BIT : 0u));
  const int fb = front_bin(deg);
  if (fb < 2) stage_one(st, fb, c.next.bin(fb), c.next.c + fb, val);
  else {
    const int32_t nch = (deg + c.bch - 1) / c.bch;
    const int32_t pos = atomicAdd(c.next.c + 3, nch);
    for (int32_t k = 0; k < nch; k++) c.next.cq[pos + k] = chunk_entry(v, tr ? TRACK_BIT : 0u, k);
  }
  if (c.collect && act) {
    d.inq[v] = 1;
    const int wb = wl_bin(deg);
    if (wb < 2) stage_one(st, 2 + wb, c.wl.bin(wb), c.wl.c + wb, val);
    else {
      const int32_t nch = dis_nch(d, deg);
      const int32_t pos = atomicAdd(c.wl.c + 3, nch);
      for (int32_t k = 0; k < nch; k++) c.wl.cq[pos + k] = chunk_entry(v, tr ? TRACK_BIT : 0u, k);
    }
  }
  fs.add(tr, deg);
  if (d.local_gap) atomicAdd(&st.lv[tr], 1);
}

__device__ __forceinline__ bool activity(const Dev &d, bool collect, int tr, int32_t v) {
  if (!collect) return false;
  const long long ev = ldv(d.e + v);
  return tr ? (ev < 0) : (ev > 0);
}

// one scanned slot (rb = the track's BFS residual, v = head); warp-convergent
__device__ __forceinline__ void td_slot(const Dev &d, Stage &st, const BfsCtx &c, int tr, int32_t rb, int32_t v,
                                        FS &fs) {
  const Track k = make_track(d, tr);
  bool claimed = false, act = false;
  const bool ok = rb > 0 && v != k.excl && ldl1(k.hgt + v) == d.n;   // stale n: the CAS decides
  const bool dn = c.isdense(tr);          // many discoverers per vertex: a store, deduplicated by compaction
  if (dn && ok) k.hgt[v] = c.lvl + 1;
  if (!dn && ok) {
    claimed = atomicCAS(k.hgt + v, d.n, c.lvl + 1) == d.n;
    if (claimed) act = activity(d, c.collect, tr, v);
  }
  if (__ballot_sync(0xffffffffu, !dn) == 0) return;   // whole warp dense: nothing to append here
  claim_push(d, st, c, claimed, act, v, tr, fs);
}

// Four slots per lane (one warp-step of td_vertex_warp / td_chunk_warp): the height
// gathers, the claiming CASes, the activity and degree loads of the four are each
// issued together, so a step costs four dependent round trips instead of sixteen.
// (tr4[j]: the track of element j; dense tracks label by stores and append nothing)
__device__ __forceinline__ void td_slot4(const Dev &d, Stage &st, const BfsCtx &c, const int tr4[4],
                                         const int32_t rb[4], const int32_t vv[4], FS &fs) {
  bool ok[4], claimed[4], act[4], dn[4];
  int32_t old[4], deg[4];
  int32_t *hg[4];
  long long ev[4];
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const Track k = make_track(d, tr4[j]);
    hg[j] = k.hgt;
    dn[j] = c.isdense(tr4[j]);
    ok[j] = rb[j] > 0 && vv[j] != k.excl && ldl1(k.hgt + vv[j]) == d.n;   // stale n: the CAS decides
  }
#pragma unroll
  for (int j = 0; j < 4; j++) if (dn[j] && ok[j]) hg[j][vv[j]] = c.lvl + 1;
  if (__ballot_sync(0xffffffffu, !(dn[0] && dn[1] && dn[2] && dn[3])) == 0) return;   // all dense: compaction appends
#pragma unroll
  for (int j = 0; j < 4; j++) old[j] = (ok[j] && !dn[j]) ? atomicCAS(hg[j] + vv[j], d.n, c.lvl + 1) : -1;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    claimed[j] = ok[j] && !dn[j] && old[j] == d.n;
    ev[j] = claimed[j] && c.collect ? ldv(d.e + vv[j]) : 0;
    deg[j] = claimed[j] ? d.row[vv[j] + 1] - d.row[vv[j]] : 0;
  }
#pragma unroll
  for (int j = 0; j < 4; j++) {
    act[j] = claimed[j] && (tr4[j] ? ev[j] < 0 : ev[j] > 0);
    claim_push_deg(d, st, c, claimed[j], act[j], vv[j], tr4[j], fs, deg[j]);
  }
}

// warp per frontier vertex (bin 1): coalesced scan of its row, 4 slots per lane per step
__device__ __forceinline__ void td_vertex_warp(const Dev &d, Smem &sm, Stage &st, int32_t entry, const BfsCtx &c,
                                               FS &fs) {
  const int tr = ((uint32_t)entry & TRACK_BIT) ? 1 : 0;
  if (c.isbu(tr)) return;
  const int lane = threadIdx.x & 31;
  const int32_t w = (int32_t)((uint32_t)entry & ~TRACK_BIT);
  const int32_t beg = d.row[w], end = d.row[w + 1];
  const int32_t *B = make_track(d, tr).B;
  for (int32_t base = beg; base < end; base += 128) {
    int32_t rb[4], vv[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int32_t i = base + j * 32 + lane;
      rb[j] = i < end ? ldv(B + i) : 0;
      vv[j] = i < end ? d.dst[i] : 0;
    }
    const int tr4[4] = {tr, tr, tr, tr};
    td_slot4(d, st, c, tr4, rb, vv, fs);
  }
  if (lane == 0) {
    sstat_add(sm, ST_BFS_SLOTS, (unsigned long long)(end - beg));
    sstat_add(sm, ST_BFS_V, 1);
  }
}

// warp per CH-slot chunk of a big frontier row (edge-balanced)
__device__ __forceinline__ void td_chunk_warp(const Dev &d, Smem &sm, Stage &st, long long ce, const BfsCtx &c,
                                              FS &fs) {
  const uint32_t lo = (uint32_t)ce;
  const int tr = (lo & TRACK_BIT) ? 1 : 0;
  if (c.isbu(tr)) return;
  const int lane = threadIdx.x & 31;
  const int32_t w = (int32_t)(lo & ~TRACK_BIT);
  const unsigned long long t_start = d.trace ? gtimer() : 0;
  const int32_t rb0 = d.row[w] + (int32_t)(ce >> 32) * c.bch;
  const int32_t end = min(d.row[w + 1], rb0 + c.bch);
  const int32_t *B = make_track(d, tr).B;
  for (int32_t base = rb0; base < end; base += 128) {
    int32_t rb[4], vv[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int32_t i = base + j * 32 + lane;
      rb[j] = i < end ? ldv(B + i) : 0;
      vv[j] = i < end ? d.dst[i] : 0;
    }
    const int tr4[4] = {tr, tr, tr, tr};
    td_slot4(d, st, c, tr4, rb, vv, fs);
  }
  if (lane == 0) sstat_add(sm, ST_BFS_SLOTS, (unsigned long long)(end - rb0));
  if (d.trace && lane == 0) {           // slowest chunk of the level: (ns, vertex)
    const unsigned long long dt = gtimer() - t_start;
    atomicMax(&d.ctl->slow, (min(dt, 0xffffffffull) << 32) | (unsigned long long)(uint32_t)w);
  }
}

// warp over up to 32 low-degree frontier vertices (bin 0): their rows are
// concatenated and split evenly over the lanes (degree scan + shuffle search)
__device__ __forceinline__ void td_small_chunk(const Dev &d, Smem &sm, Stage &st, const int32_t *list, int32_t x0,
                                               int32_t cnt, const BfsCtx &c, FS &fs) {
  const int lane = threadIdx.x & 31;
  int32_t entry = 0, beg = 0, deg = 0;
  if (lane < cnt) {
    entry = list[x0 + lane];
    const int32_t w = (int32_t)((uint32_t)entry & ~TRACK_BIT);
    if (!c.isbu(((uint32_t)entry & TRACK_BIT) ? 1 : 0)) {
      beg = d.row[w];
      deg = d.row[w + 1] - beg;
    }
  }
  WarpG g{lane};
  long long tot;
  const int32_t off = (int32_t)g.exscan(deg, tot);
  const int32_t total = (int32_t)tot;
  for (int32_t t0 = 0; t0 < total; t0 += 128) {
    int tr4[4];
    int32_t rb[4], vv[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {               // slots t0 + q*32 + lane: locate, then load
      const int32_t k = t0 + q * 32 + lane;
      int j = 0;
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) {
        const int32_t o = __shfl_sync(0xffffffffu, off, j + s);
        if (o <= k) j += s;
      }
      const int32_t ej = __shfl_sync(0xffffffffu, entry, j);
      const int32_t bj = __shfl_sync(0xffffffffu, beg, j);
      const int32_t oj = __shfl_sync(0xffffffffu, off, j);
      tr4[q] = ((uint32_t)ej & TRACK_BIT) ? 1 : 0;
      const int32_t i = bj + (k - oj);
      rb[q] = k < total ? ldv(make_track(d, tr4[q]).B + i) : 0;
      vv[q] = k < total ? d.dst[i] : 0;
    }
    td_slot4(d, st, c, tr4, rb, vv, fs);
  }
  if (lane == 0) {
    sstat_add(sm, ST_BFS_SLOTS, (unsigned long long)total);
    sstat_add(sm, ST_BFS_V, (unsigned long long)cnt);
  }
}

// ---- bottom-up ----------------------------------------------------------------
// Pass A (thread per vertex) settles low-degree candidates and queues the others
// (degree-binned); pass B (after a grid barrier) scans the queued rows with a
// warp / a CTA per vertex and group-wide early exit.
constexpr int32_t BU_THREAD_MAX = 16;

__device__ __forceinline__ void bfs_bottom_up_a(const Dev &d, Smem &sm, Stage &st, const BfsCtx &c, int32_t *bul,
                                                int32_t *bulc, FS &fs) {
  const int32_t n = d.n;
  const int32_t nt = gridDim.x * NT;
  unsigned long long scanned = 0;
  for (int32_t b = blockIdx.x * NT + (threadIdx.x & ~31); b < n; b += nt) {
    const int32_t v = b + (threadIdx.x & 31);
    bool q1 = false, q2 = false, claimed = false, act = false;
    int tr = 0;
    if (v < n) {
      int cand = -1;
      if (c.isbu(0) && v != d.s && ldv(d.hp + v) == n) cand = 0;
      else if (c.isbu(1) && v != d.t && ldv(d.hm + v) == n) cand = 1;
      if (cand >= 0) {
        tr = cand;
        const int32_t beg = d.row[v], end = d.row[v + 1];
        if (end - beg > BU_THREAD_MAX) {
          q1 = end - beg <= BIN1_MAX;
          q2 = !q1;
        } else {
          const Track k = make_track(d, tr);
          for (int32_t i0 = beg; i0 < end && !claimed; i0 += 4) {
            int32_t r[4], w[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
              r[j] = i0 + j < end ? ldv(k.F + i0 + j) : 0;
              w[j] = i0 + j < end ? d.dst[i0 + j] : 0;
            }
#pragma unroll
            for (int j = 0; j < 4; j++)
              if (!claimed && r[j] > 0 && ldl1(k.hgt + w[j]) == c.lvl) claimed = true;   // level-lvl labels are frozen
            scanned += 4;
          }
          if (claimed) {
            k.hgt[v] = c.lvl + 1;
            act = activity(d, c.collect, tr, v);
          }
        }
      }
    }
    claim_push(d, st, c, claimed, act, v, tr, fs);
    const uint32_t tag = tr ? TRACK_BIT : 0u;
    warp_append(q1, (int32_t)((uint32_t)v | tag), bul, bulc);
    warp_append(q2, (int32_t)((uint32_t)v | tag), bul + n, bulc + 1);
  }
  sstat_add(sm, ST_BFS_SLOTS, scanned);
}

template <class G>
__device__ __forceinline__ void bfs_bottom_up_b(const Dev &d, const G &g, Smem &sm, Stage &st, const BfsCtx &c,
                                                int32_t entry, FS &fs) {
  const int tr = ((uint32_t)entry & TRACK_BIT) ? 1 : 0;
  const int32_t v = (int32_t)((uint32_t)entry & ~TRACK_BIT);
  const Track k = make_track(d, tr);
  const int32_t beg = d.row[v], end = d.row[v + 1];
  bool found = false;
  unsigned long long scanned = 0;
  for (int32_t base = beg; base < end; base += 4 * G::size) {
    int32_t r[4], w[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int32_t i = base + j * G::size + g.rank();
      r[j] = i < end ? ldv(k.F + i) : 0;
      w[j] = i < end ? d.dst[i] : 0;
    }
    bool hit = false;
#pragma unroll
    for (int j = 0; j < 4; j++)
      if (r[j] > 0 && ldl1(k.hgt + w[j]) == c.lvl) hit = true;
    scanned += 4 * G::size;
    if (g.any(hit)) { found = true; break; }
  }
  if (g.rank() == 0) {
    if (found) {
      k.hgt[v] = c.lvl + 1;
      claim_one(d, st, c, activity(d, c.collect, tr, v), v, tr, fs);
    }
    sstat_add(sm, ST_BFS_SLOTS, scanned);
  }
}

// ---- DENSE compaction ---------------------------------------------------------
// Tiled pass over the vertex domain (all n, or the P list): every thread classifies
// TILE_ITEMS vertices; per tile, warps reserve positions with shared-memory atomics
// and thread 0 reserves each list's global range with ONE atomic.  Categories:
// 0,1 = frontier bins 0/1, 2 = frontier chunks (several entries per vertex),
// 3,4 = worklist bins 0/1, 5 = worklist chunks (vertices of > BIN1_MAX slots).  `classify(v, tr, front, act)` decides for vertex v.
template <class Classify>
__device__ __forceinline__ void compact_domain(const Dev &d, TileSm &ts, int32_t N, const int32_t *dom,
                                               const BL &next, const BL &wl, bool collect, Classify classify,
                                               long long &fs0, long long &fs1, int32_t &nv0, int32_t &nv1,
                                               int32_t bch) {
  const int lane = threadIdx.x & 31;
  const int32_t tile_sz = TILE_ITEMS * NT;
  WarpG g{lane};
  for (int32_t t0 = blockIdx.x * tile_sz; t0 < N; t0 += gridDim.x * tile_sz) {
    if (threadIdx.x < 8) ts.cnt[threadIdx.x] = 0;
    __syncthreads();
    int32_t vv[TILE_ITEMS], fo[TILE_ITEMS], wo[TILE_ITEMS];
    int8_t fc[TILE_ITEMS], wc[TILE_ITEMS];
    uint32_t tg[TILE_ITEMS];
    int32_t nchv[TILE_ITEMS];
    // classification loads of every item first, then the degree loads, then the
    // appends (each stage's loads in flight together)
    int trj[TILE_ITEMS];
    bool frj[TILE_ITEMS], acj[TILE_ITEMS];
    int32_t dgj[TILE_ITEMS];
#pragma unroll
    for (int j = 0; j < TILE_ITEMS; j++) {
      const int32_t x = t0 + j * NT + threadIdx.x;
      vv[j] = -1; trj[j] = 0; frj[j] = false; acj[j] = false;
      if (x < N) {
        vv[j] = dom ? dom[x] : x;
        classify(vv[j], trj[j], frj[j], acj[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < TILE_ITEMS; j++)
      dgj[j] = (frj[j] || acj[j]) ? d.row[vv[j] + 1] - d.row[vv[j]] : 0;
#pragma unroll
    for (int j = 0; j < TILE_ITEMS; j++) {
      const int32_t v = vv[j];
      const int tr = trj[j];
      const bool front = frj[j], act = acj[j];
      const int32_t deg = dgj[j];
      const int fb = front ? (deg <= BIN0_MAX ? 0 : (deg <= BIN1_MAX ? 1 : 2)) : -1;
      const int wb = (collect && act) ? (deg <= BIN0_MAX ? 0 : (deg <= BIN1_MAX ? 1 : 2)) : -1;
      if (wb >= 0) d.inq[v] = 1;
      if (front) { if (tr) { fs1 += deg; nv1++; } else { fs0 += deg; nv0++; } }
      vv[j] = v; fc[j] = (int8_t)fb; wc[j] = (int8_t)wb; tg[j] = tr ? TRACK_BIT : 0u;
      fo[j] = 0; wo[j] = 0;
      // frontier bins 0/1: ballot per bin
#pragma unroll
      for (int b = 0; b < 2; b++) {
        const unsigned m = __ballot_sync(0xffffffffu, fb == b);
        if (m) {
          int bs = 0;
          if (lane == __ffs(m) - 1) bs = atomicAdd(&ts.cnt[b], __popc(m));
          bs = __shfl_sync(0xffffffffu, bs, __ffs(m) - 1);
          if (fb == b) fo[j] = bs + __popc(m & ((1u << lane) - 1u));
        }
      }
      // frontier chunks
      const int32_t nch = fb == 2 ? (deg + bch - 1) / bch : 0;
      nchv[j] = nch;
      if (__ballot_sync(0xffffffffu, nch > 0)) {
        long long tot;
        const int32_t ex = (int32_t)g.exscan(nch, tot);
        int bs = 0;
        if (lane == 0) bs = atomicAdd(&ts.cnt[2], (int32_t)tot);
        bs = __shfl_sync(0xffffffffu, bs, 0);
        if (fb == 2) fo[j] = bs + ex;
      }
      // worklist bins 0/1, chunks
      if (collect) {
#pragma unroll
        for (int b = 0; b < 2; b++) {
          const unsigned m = __ballot_sync(0xffffffffu, wb == b);
          if (m) {
            int bs = 0;
            if (lane == __ffs(m) - 1) bs = atomicAdd(&ts.cnt[3 + b], __popc(m));
            bs = __shfl_sync(0xffffffffu, bs, __ffs(m) - 1);
            if (wb == b) wo[j] = bs + __popc(m & ((1u << lane) - 1u));
          }
        }
        const int32_t wch = wb == 2 ? dis_nch(d, deg) : 0;
        if (__ballot_sync(0xffffffffu, wch > 0)) {
          long long tot;
          const int32_t ex = (int32_t)g.exscan(wch, tot);
          int bs = 0;
          if (lane == 0) bs = atomicAdd(&ts.cnt[5], (int32_t)tot);
          bs = __shfl_sync(0xffffffffu, bs, 0);
          if (wb == 2) wo[j] = bs + ex;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x < 6) {
      const int32_t cc = ts.cnt[threadIdx.x];
      const int k = threadIdx.x;     // categories -> global counters
      int32_t *gc = k == 0 ? next.c : k == 1 ? next.c + 1 : k == 2 ? next.c + 3 : k == 5 ? wl.c + 3 : wl.c + (k - 3);
      ts.base[threadIdx.x] = cc ? atomicAdd(gc, cc) : 0;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < TILE_ITEMS; j++) {
      const int32_t e = (int32_t)((uint32_t)vv[j] | tg[j]);
      if (fc[j] == 0 || fc[j] == 1) next.bin(fc[j])[ts.base[fc[j]] + fo[j]] = e;
      else if (fc[j] == 2)
        for (int32_t k = 0; k < nchv[j]; k++) next.cq[ts.base[2] + fo[j] + k] = chunk_entry(vv[j], tg[j], k);
      if (wc[j] == 0 || wc[j] == 1) wl.bin(wc[j])[ts.base[3 + wc[j]] + wo[j]] = e;
      else if (wc[j] == 2) {
        const int32_t deg = d.row[vv[j] + 1] - d.row[vv[j]];
        for (int32_t k = 0; k < dis_nch(d, deg); k++) wl.cq[ts.base[5] + wo[j] + k] = chunk_entry(vv[j], tg[j], k);
      }
    }
    __syncthreads();
  }
}

__device__ __forceinline__ int32_t *act_buf(Smem &sm) { return &sm.st.f[0][0]; }
__device__ __forceinline__ int32_t *rel_buf(Smem &sm) { return &sm.st.w[0][0]; }

// block-wide: move `cnt` staged entries (vertex | track tag) into the binned list bl
// (bins 0/1, chunk entries for bigger rows when bl is chunked, else bins 2/3): one
// global atomic per category per CTA.  Uses sm.ts; callers pass a block-uniform cnt.
__device__ __forceinline__ void vflush(const Dev &d, TileSm &ts, const int32_t *buf, int32_t cnt, const BL &bl,
                                       bool dis) {
  for (int32_t t0 = 0; t0 < cnt; t0 += NT) {
    if (threadIdx.x < 4) ts.cnt[threadIdx.x] = 0;
    __syncthreads();
    const int32_t x = t0 + threadIdx.x;
    int32_t e = 0, cat = -1, nch = 0, off = 0;
    if (x < cnt) {
      e = buf[x];
      const int32_t v = (int32_t)((uint32_t)e & ~TRACK_BIT);
      const int32_t deg = d.row[v + 1] - d.row[v];
      cat = deg <= BIN0_MAX ? 0 : (deg <= BIN1_MAX ? 1 : (deg <= BIN2_MAX ? 2 : 3));
      if (cat >= 2 && bl.cq) { cat = 3; nch = dis ? dis_nch(d, deg) : (deg + CH - 1) / CH; }
      off = atomicAdd(&ts.cnt[cat], nch ? nch : 1);
    }
    __syncthreads();
    if (threadIdx.x < 4) ts.base[threadIdx.x] = ts.cnt[threadIdx.x] ? atomicAdd(bl.c + threadIdx.x, ts.cnt[threadIdx.x]) : 0;
    __syncthreads();
    if (cat >= 0) {
      if (nch) {
        const int32_t v = (int32_t)((uint32_t)e & ~TRACK_BIT);
        for (int32_t k = 0; k < nch; k++) bl.cq[ts.base[3] + off + k] = chunk_entry(v, (uint32_t)e & TRACK_BIT, k);
      } else {
        bl.bin(cat)[ts.base[cat] + off] = e;
      }
    }
    __syncthreads();
  }
}

// block-wide, end of a discharge round: flush the staged activations / relabels
__device__ __forceinline__ void dis_flush(const Dev &d, Smem &sm, const BL &nxt, const BL &rl) {
  // activation candidates: every thread's reductions are performed before any check
  __threadfence();
  __syncthreads();
  {
    const int32_t c = min(sm.ccnt, CCAP);
    for (int32_t x = threadIdx.x; x < c; x += NT) {
      const uint32_t e = (uint32_t)sm.cand[x];
      const int tr = (e & TRACK_BIT) ? 1 : 0;
      const int32_t v = (int32_t)(e & ~TRACK_BIT);
      const Track k = make_track(d, tr);
      if (ldv(d.e + v) * k.sign > 0) activate(d, k, nxt, v, e & TRACK_BIT, sm);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) sm.ccnt = 0;
  const int32_t a = min(sm.acnt, ACAP), r = min(sm.rcnt, RCAP);
  __syncthreads();
  if (threadIdx.x == 0) { sm.acnt = 0; sm.rcnt = 0; }
  vflush(d, sm.ts, act_buf(sm), a, nxt, true);
  vflush(d, sm.ts, rel_buf(sm), r, rl, false);
}

// block-wide: flush the stages and publish the per-CTA frontier slot sums and the
// level counts of the vertices labelled in this phase
__device__ __forceinline__ void bfs_flush(const Dev &d, Smem &sm, Stage &st, const BfsCtx &c, FS &fs) {
  stage_flush(st, c.next, c.wl);
  BlockG bg{sm.red};
  const long long f0 = bg.sum(fs.a), f1 = bg.sum(fs.b);
  if (threadIdx.x == 0) {
    if (f0) atomicAdd(c.fs_next, (unsigned long long)f0);
    if (f1) atomicAdd(c.fs_next + 1, (unsigned long long)f1);
    if (c.tgt < GAPW && c.tgt < d.n) {
      if (st.lv[0]) atomicAdd(d.cnt + c.tgt, st.lv[0]);
      if (st.lv[1]) atomicAdd(d.cnt + GAPW + c.tgt, st.lv[1]);
    }
    st.lv[0] = 0; st.lv[1] = 0;
  }
}

// One BFS level.  Ends after its grid barrier(s).
__device__ __forceinline__ void bfs_expand_level(const Dev &d, cg::grid_group &grid, Smem &sm, Stage &st,
                                                 PhaseClock &clk, int32_t it, const BL &cur, const int32_t c[NB],
                                                 const BfsCtx &ctx, int32_t *bul, int32_t *bulc) {
  const bool bu = ctx.bu != 0;
  FS fs;
  if (bu) bfs_bottom_up_a(d, sm, st, ctx, bul, bulc, fs);
  if (ctx.bu != 3u) {
    // one index space over the level's items (chunks of big rows, bin-1 rows, groups of
    // 32 bin-0 rows), so that no warp takes an item of each kind while others idle
    const int32_t gw = gwarp_spread(), nw = gridDim.x * WPB;
    const int32_t c31 = c[3] + c[1], tot = c31 + (c[0] + 31) / 32;
    const int32_t *b0 = cur.bin(0);
    for (int32_t x = gw; x < tot; x += nw) {
      if (x < c[3]) td_chunk_warp(d, sm, st, cur.cq[x], ctx, fs);
      else if (x < c31) td_vertex_warp(d, sm, st, cur.bin(1)[x - c[3]], ctx, fs);
      else {
        const int32_t x0 = (x - c31) * 32;
        td_small_chunk(d, sm, st, b0, x0, min(32, c[0] - x0), ctx, fs);
      }
    }
  }
  bfs_flush(d, sm, st, ctx, fs);
  gsync(d, grid, sm);
  clk.lap(d, sm, ST_T_BFS, it, ctx.lvl, total(c), (int32_t)ctx.bu | (c[3] << 3));
  if (bu) {
    cta_snap(sm, 2, [&](int k) { return (long long)ldv(bulc + k); });
    const int32_t q1 = (int32_t)sm.cv[0], q2 = (int32_t)sm.cv[1];
    if (q1 + q2 > 0) {
      fs = FS();
      {
        BlockG g{sm.red};
        for (int32_t x = blockIdx.x; x < q2; x += gridDim.x) bfs_bottom_up_b(d, g, sm, st, ctx, bul[d.n + x], fs);
      }
      {
        WarpG g{(int)(threadIdx.x & 31)};
        const int32_t gw = gwarp_spread(), nw = gridDim.x * WPB;
        for (int32_t x = gw; x < q1; x += nw) bfs_bottom_up_b(d, g, sm, st, ctx, bul[x], fs);
      }
      bfs_flush(d, sm, st, ctx, fs);
      gsync(d, grid, sm);
      clk.lap(d, sm, ST_T_BFS_BU, it, ctx.lvl, q1 + q2, q2);
    }
  }
}

// ---------------------------------------------------------------------------
// Discharge of one active vertex (Alg.2 / Alg.6), up to KERNELCYCLES cycles.  A
// cycle is ONE pass over u's residual slots:
//  * push to every admissible slot (h(v) < h(u)) until the excess is gone.  With the
//    exact BFS labels every admissible slot has h(v) = h(u)-1 = h^, the lowest
//    residual neighbour, so this is the run of Alg.2 pushes to v^ (l.15-19) in one
//    pass; the excess is a budget the lanes claim with
//    shared-memory atomics (any order among equal heights, R6);
//  * the same pass records the lowest height among slots left residual, so if excess
//    remains (all admissible slots saturated) the lift (l.21) goes straight to that
//    minimum + 1 (clamped to |V|, R4/R5) and the next cycle pushes again.
// A vertex whose excess is drained stops; a later push into it re-queues it (the
// excess crosses 0).  A vertex that spends all KERNELCYCLES while active re-queues
// itself for the next round.
template <class G>
__device__ __forceinline__ void discharge(const Dev &d, const G &g, Smem &sm, int32_t entry, const BL &rl,
                                          const BL &nxt, unsigned long long *workc) {
  const int tr = ((uint32_t)entry & TRACK_BIT) ? 1 : 0;
  const uint32_t tag = tr ? TRACK_BIT : 0u;
  const int32_t u = (int32_t)((uint32_t)entry & ~TRACK_BIT);
  const Track k = make_track(d, tr);
  const int32_t n = d.n;
  const int32_t beg = d.row[u], end = d.row[u + 1];
  // rounds: clear the queued flag first, so a push into u during this discharge queues
  // u for the next round.  async: u keeps the flag while it is being discharged (no
  // second warp may take u concurrently: both would push the same residual) and the
  // epilogue below clears it and re-checks e(u).
  if (!sm.amode && g.rank() == 0) { d.inq[u] = 0; __threadfence(); }
  const unsigned long long t_start = d.trace ? gtimer() : 0;
#ifdef DMF_DEBUG_BUSY
  if (g.rank() == 0 && atomicExch(d.dcnt + u, 1) != 0) atomicCAS(&d.ctl->pad, 0, u + 1);
#endif
  int32_t hu = ldv(k.hgt + u);
  if (g.rank() == 0) DBG(d, 200, u, (int32_t)ldv(d.e + u), hu, ldv(d.inq + u));
  bool relabelled = false;
  unsigned long long scanned = 0, pushes = 0, lifts = 0;
  long long eu = 0;
  int32_t glim = 0x7fffffff;          // local gap: heights above this stop (R14 form 2)
  if (g.rank() == 0) { eu = ldv(d.e + u) * k.sign; glim = gap_limit(d, tr); }
  eu = g.bcast(eu);
  glim = (int32_t)g.bcast(glim);
  const bool gapped = hu < n && hu > glim && eu > 0;
  if (gapped) eu = 0;                 // above an emptied level: cannot reach a root this phase
  int cyc = 0;
  long long *bud = G::size == 1 ? nullptr
                  : (G::size == NT ? &sm.budget[4 * WPB]
                                   : &sm.budget[4 * (threadIdx.x >> 5) + (G::size < 32 ? (int)((threadIdx.x & 31) / G::size) : 0)]);
  for (; cyc < d.kc && hu < n && eu > 0; ++cyc) {
    long long remaining = eu;
    unsigned long long nmin = ~0ull;     // lowest height among slots left residual
    if (G::size > 1) {
      if (g.rank() == 0) *bud = eu;
      g.sync();
    }
    for (int32_t i0 = beg + g.rank(); i0 < end; i0 += 4 * G::size) {
      if (G::size == 1 ? remaining <= 0 : *((volatile long long *)bud) <= 0) break;
      int32_t r[4], v[4], h[4], ri[4];
#pragma unroll
      for (int j = 0; j < 4; j++) {     // independent loads first (ILP), then the gathers
        const int32_t i = i0 + j * G::size;
        r[j] = i < end ? ldv(k.F + i) : 0;
        v[j] = i < end ? d.dst[i] : 0;
      }
#pragma unroll
      for (int j = 0; j < 4; j++) {     // neighbour height + the reverse slot, in the same wave
        h[j] = r[j] > 0 ? ldv(k.hgt + v[j]) : 0;
        ri[j] = r[j] > 0 ? d.rev[i0 + j * G::size] : 0;
      }
      long long take[4];
#pragma unroll
      for (int j = 0; j < 4; j++) {       // budget claims
        take[j] = 0;
        if (r[j] > 0 && h[j] < hu) {
          long long old;
          if (G::size == 1) { old = remaining; remaining -= r[j]; }
          else old = (long long)atomicAdd(reinterpret_cast<unsigned long long *>(bud),
                                          (unsigned long long)(-(long long)r[j]));
          take[j] = old < 0 ? 0 : (old < r[j] ? old : r[j]);
        }
        if (r[j] > 0 && take[j] < r[j])
          nmin = (unsigned long long)(uint32_t)h[j] < nmin ? (unsigned long long)(uint32_t)h[j] : nmin;
      }
#pragma unroll
      for (int j = 0; j < 4; j++) {       // pushes: fire-and-forget
        if (take[j] > 0) {
          push_slot(d, k, nxt, i0 + j * G::size, ri[j], v[j], (int32_t)take[j], tag, sm);
          pushes++;
        }
      }
    }
    scanned += (unsigned long long)(end - beg);
    if (G::size > 1) {
      g.sync();
      remaining = *bud;
      g.sync();
    }
    const long long done = eu - (remaining > 0 ? remaining : 0);
    long long left = 0;                      // exact excess after our pushes (others may have added)
    if (g.rank() == 0) {
      if (done > 0) {
        const long long old = (long long)atomicAdd(reinterpret_cast<unsigned long long *>(d.e + u),
                                                   (unsigned long long)(-done * k.sign));   // e(u) -= d
        left = old * k.sign - done;
      } else {
        left = ldv(d.e + u) * k.sign;
      }
    }
    left = g.bcast(left);
    eu = left;
    if (left <= 0) break;                    // drained
    if (remaining <= 0) continue;            // excess arrived meanwhile: push again at the same height
    nmin = g.min(nmin);                      // every admissible slot saturated: lift
    const int32_t nh = nmin == ~0ull ? n : (int32_t)min((unsigned long long)n, nmin + 1);
    if (nh > hu) {
      if (g.rank() == 0) {
        k.hgt[u] = nh;
        gap_move(d, sm, tr, hu, nh);
        glim = gap_limit(d, tr);
      }
      hu = nh;
      relabelled = true;
      lifts++;
      glim = (int32_t)g.bcast(glim);
      if (hu < n && hu > glim) { eu = 0; break; }   // lifted above an emptied level: stop
    }
  }
  if (sm.amode) {                       // every member's pushes land before u is released
    if (pushes > 0) __threadfence();
    g.sync();
  }
  if (g.rank() == 0) {
    if (d.trace) {                      // slowest discharge of the round: (ns, degree, cycles)
      const unsigned long long dt = gtimer() - t_start;
      const unsigned long long key = (min(dt, 0xffffffffull) << 32) |
                                     ((unsigned long long)min(end - beg, 0xffffff) << 8) | (unsigned long long)min(cyc, 255);
      atomicMax(&d.ctl->slow, key);
    }
#ifdef DMF_DEBUG_BUSY
    DBG(d, 201, u, (int32_t)ldv(d.e + u), hu, pushes);
    if (atomicExch(d.dcnt + u, 0) != 1) atomicCAS(&d.ctl->pad, 0, -(u + 1));
    __threadfence();
#endif
    const bool stopped = gapped || (hu < n && hu > glim);   // local gap: not re-queued this phase
    if (stopped) sstat_add(sm, ST_GAP_SKIPS, 1);
    if (sm.amode) {
      atomicExch(d.inq + u, 0);
      __threadfence();
      if (!stopped && hu < n && ldv(d.e + u) * k.sign > 0) activate(d, k, nxt, u, tag, sm);
    } else if (!stopped && cyc == d.kc && hu < n && eu > 0) {
      activate(d, k, nxt, u, tag, sm);  // KERNELCYCLES spent
    }
    if (relabelled && d.rlf[u] == 0) { d.rlf[u] = 1; stage_relabelled(d, rl, u, tag, sm); }
    atomicAdd(&sm.work, scanned + 16ull * lifts + 16ull);
    sstat_add(sm, ST_DIS_V, 1);
    sstat_add(sm, ST_DIS_SLOTS, scanned);
    sstat_add(sm, ST_RELABELS, lifts);
  }
  sstat_add(sm, ST_PUSHES, pushes);
}

// ---------------------------------------------------------------------------
// Chunked discharge of a big vertex u (> BIN1_MAX slots): one cycle of Alg.2 / Alg.6
// per round, its row split into CH-slot chunks that warps anywhere on the grid take
// in parallel (a hub no longer serialises a round behind one CTA).
//  * The chunks claim u's excess directly from e(u): one warp-aggregated atomic per
//    step takes the admissible residual of the step; whatever e(u) could not cover is
//    refunded at once, and the chunk is then "dry" (stops scanning: excess gone).
//  * Each chunk folds the lowest height among its slots left residual into dmin[u]
//    (0 when dry: an admissible slot may remain) and counts itself in dcnt[u].
//  * The LAST chunk to finish decides, as Alg.2 l.20-22 does after the pushes: if u
//    still has excess and every residual slot is at height >= h(u), lift u to
//    min(dmin + 1, |V|) (R4/R5); if excess remains below |V|, re-queue u.  It resets
//    dcnt / dmin / inq for the next round and re-reads e(u) after clearing inq, so an
//    activation that lost to the stale flag is not lost.
// Heights of u are read once per round; stale neighbour heights cost work only (RIE
// and the fresh BFS of R9 repair them), exactly as in the one-group discharge.
__device__ __forceinline__ void discharge_chunk(const Dev &d, Smem &sm, long long ce, const BL &rl, const BL &nxt) {
  const int lane = threadIdx.x & 31;
  const uint32_t lo = (uint32_t)ce;
  const int tr = (lo & TRACK_BIT) ? 1 : 0;
  const uint32_t tag = tr ? TRACK_BIT : 0u;
  const int32_t u = (int32_t)(lo & ~TRACK_BIT);
  const Track k = make_track(d, tr);
  const int32_t n = d.n;
  const int32_t rbeg = d.row[u], rend = d.row[u + 1];
  const int32_t csz = dis_csize(d, rend - rbeg);
  const uint32_t kraw = (uint32_t)(ce >> 32);
  const bool probe = (kraw & PROBE_BIT) != 0;
  const int32_t kc = (int32_t)(kraw & ~PROBE_BIT);
  const int32_t beg = rbeg + kc * csz;
  const int32_t end = min(rend, beg + csz);
  const int32_t nch = (rend - rbeg + csz - 1) / csz;
  const unsigned long long t_start = d.trace ? gtimer() : 0;
  const int32_t hu = ldv(k.hgt + u);
  if (lane == 0) DBG(d, 204, u, (int32_t)(ce >> 32), rend - rbeg, 0);
  uint32_t nmin = 0xffffffffu;           // lowest height among slots left residual
  unsigned long long pushes = 0, scanned = 0;
  bool dry = false;
  WarpG g{lane};
  // excess already claimed by the other chunks (or drained): nothing to push here,
  // and an admissible slot may remain -> no lift (dry); skips the slot loads
  int32_t glim = 0x7fffffff;             // local gap (R14 form 2)
  if (hu < n) {
    long long e0 = 0;
    if (lane == 0) { e0 = ldv(d.e + u) * k.sign; glim = gap_limit(d, tr); }
    glim = (int32_t)g.bcast(glim);
    dry = g.bcast(e0) <= 0 || hu > glim;  // above an emptied level: no pushes, and no lift below
  }
  if (hu < n && !dry && d.scan2) {
    // Two passes: (1) a read-only scan of the whole chunk, 8 slots per lane per step
    // with every load of a step issued before the first use, that records the
    // admissible slots (h(v) < h(u)) in a per-warp shared list and the lowest height
    // among the residual non-admissible ones; (2) ONE claim of the listed residual
    // from e(u) and the pushes from the list.  A chunk with nothing admissible (most
    // chunks of a hub's row) costs the scan only.  The slots of u's row in this track
    // are pushed only by u's discharger, so a residual can only grow between the
    // passes and every take stays <= the residual it was read as.
    int32_t *ai = sm.adm_i + (threadIdx.x >> 5) * ADMCAP;
    int32_t *av = sm.adm_v + (threadIdx.x >> 5) * ADMCAP;
    int32_t *ar = sm.adm_r + (threadIdx.x >> 5) * ADMCAP;
    const unsigned lt = (1u << lane) - 1u;
    int32_t nadm = 0;                      // warp-uniform: admissible slots found
    long long lsum = 0;                    // this lane's listed admissible residual
    bool complete = true;                  // every slot of the chunk was examined
    long long e0 = 0;
    if (lane == 0) e0 = ldv(d.e + u) * k.sign;
    e0 = g.bcast(e0);
    for (int32_t b0 = beg; b0 < end; b0 += 256) {
      int32_t r[8], v[8], h[8];
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const int32_t i = b0 + lane + 32 * j;
        r[j] = i < end ? ldv(k.F + i) : 0;
        v[j] = i < end ? d.dst[i] : 0;
      }
#pragma unroll
      for (int j = 0; j < 8; j++) h[j] = r[j] > 0 ? ldv(k.hgt + v[j]) : 0;
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const bool adm = r[j] > 0 && h[j] < hu;
        if (r[j] > 0 && !adm) nmin = (uint32_t)h[j] < nmin ? (uint32_t)h[j] : nmin;
        const unsigned m = __ballot_sync(0xffffffffu, adm);
        if (m) {
          const int32_t pos = nadm + __popc(m & lt);
          if (adm && pos < ADMCAP) { ai[pos] = b0 + lane + 32 * j; av[pos] = v[j]; ar[pos] = r[j]; lsum += r[j]; }
          nadm += __popc(m);
        }
      }
      scanned += 256;
      if (nadm >= ADMCAP || (b0 + 256 < end && g.sum(lsum) >= e0)) {   // list full / excess covered
        complete = b0 + 256 >= end;
        break;
      }
    }
    const long long tot = g.sum(lsum);
    long long got = 0;
    if (tot > 0) {                         // claim the listed residual from e(u)
      if (lane == 0) {
        const long long old = (long long)atomicAdd(reinterpret_cast<unsigned long long *>(d.e + u),
                                                   (unsigned long long)(-tot * k.sign)) * k.sign;
        got = old <= 0 ? 0 : (old < tot ? old : tot);
        if (got < tot) atom_add(d.e + u, (tot - got) * k.sign);   // refund what e(u) did not cover
      }
      got = g.bcast(got);
    }
    __syncwarp();
    const int32_t nl = nadm < ADMCAP ? nadm : ADMCAP;
    long long before = 0;                  // listed residual of earlier list entries
    for (int32_t x0 = 0; x0 < nl && before < got; x0 += 32) {
      const int32_t x = x0 + lane;
      const int32_t r = x < nl ? ar[x] : 0;
      long long t32;
      const long long pre = before + g.exscan(r, t32);
      long long take = got - pre;
      take = take < 0 ? 0 : (take > r ? r : take);
      if (take > 0) {
        const int32_t i = ai[x];
        push_slot(d, k, nxt, i, d.rev[i], av[x], (int32_t)take, tag, sm);
        pushes++;
      }
      before += t32;
    }
    __syncwarp();
    // dry: u's excess is gone, an admissible slot may remain, or part of the chunk was
    // not examined -- no lift decided by this chunk
    if (got < tot || nadm > ADMCAP || !complete) dry = true;
  } else if (hu < n && !dry) {
    for (int32_t b0 = beg; b0 < end; b0 += 128) {   // warp-uniform trip count (collectives inside)
      const int32_t i0 = b0 + lane;
      int32_t r[4], v[4], h[4], ri[4];
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int32_t i = i0 + j * 32;
        r[j] = i < end ? ldv(k.F + i) : 0;
        v[j] = i < end ? d.dst[i] : 0;
      }
#pragma unroll
      for (int j = 0; j < 4; j++) {
        h[j] = r[j] > 0 ? ldv(k.hgt + v[j]) : 0;
        ri[j] = r[j] > 0 ? d.rev[i0 + j * 32] : 0;
      }
      long long asum = 0;
#pragma unroll
      for (int j = 0; j < 4; j++) asum += (r[j] > 0 && h[j] < hu) ? r[j] : 0;
      long long tot;
      const long long pre = g.exscan(asum, tot);
      long long got = 0;
      if (tot > 0) {                       // claim the step's admissible residual from e(u)
        if (lane == 0) {
          const long long old = (long long)atomicAdd(reinterpret_cast<unsigned long long *>(d.e + u),
                                                     (unsigned long long)(-tot * k.sign)) * k.sign;
          got = old <= 0 ? 0 : (old < tot ? old : tot);
          if (got < tot) atom_add(d.e + u, (tot - got) * k.sign);   // refund what e(u) did not cover
        }
        got = g.bcast(got);
      }
      long long mine = got - pre;          // this lane's share, lane order
      mine = mine < 0 ? 0 : (mine > asum ? asum : mine);
      long long take[4];
#pragma unroll
      for (int j = 0; j < 4; j++) {
        take[j] = 0;
        if (r[j] > 0 && h[j] < hu) { take[j] = mine < r[j] ? mine : r[j]; mine -= take[j]; }
        if (r[j] > 0 && take[j] < r[j]) nmin = (uint32_t)h[j] < nmin ? (uint32_t)h[j] : nmin;
      }
#pragma unroll
      for (int j = 0; j < 4; j++) {
        if (take[j] > 0) {
          push_slot(d, k, nxt, i0 + j * 32, ri[j], v[j], (int32_t)take[j], tag, sm);
          pushes++;
        }
      }
      scanned += 128;
      if (got < tot) { dry = true; break; }   // u's excess is gone (warp-uniform)
    }
  }
  nmin = (uint32_t)g.min(dry ? 0ull : (unsigned long long)nmin);
  const bool pushed = g.any(pushes > 0);
  if (pushed) __threadfence();              // every lane's pushes land before u can be taken again
  __syncwarp();
  if (probe) {                              // current-arc probe (async ring only)
    if (lane == 0) {
      if (pushed && ldv(d.arc + u) != kc) d.arc[u] = kc;
      const long long eu = ldv(d.e + u) * k.sign;
      if (eu > 0 && hu < n && hu <= glim) {
        enqueue_items(d, u, tag, nch, 0u);  // excess left: every chunk (u stays queued; their last one releases it)
      } else {
        atomicExch(d.inq + u, 0);
        __threadfence();
        if (hu < n && hu > glim) sstat_add(sm, ST_GAP_SKIPS, 1);
        else if (hu < n && ldv(d.e + u) * k.sign > 0) activate(d, k, nxt, u, tag, sm);
        sstat_add(sm, ST_DIS_V, 1);
      }
      DBG(d, 205, u, (int32_t)kc, (int32_t)pushes, 0);
      atomicAdd(&sm.work, scanned + 16ull);
      sstat_add(sm, ST_DIS_SLOTS, scanned);
    }
    sstat_add(sm, ST_PUSHES, pushes);
    return;
  }
  if (lane == 0) {
    if (pushes > 0 && d.arc && ldv(d.arc + u) != kc) d.arc[u] = kc;
    if (nmin < (uint32_t)DMIN_NONE) atomicMin(d.dmin + u, (int32_t)nmin);
    __threadfence();
    const int32_t done = atomicAdd(d.dcnt + u, 1);
    unsigned long long lifts = 0;
    if (done == nch - 1) {                 // last chunk of u this round
      __threadfence();
      const int32_t mn = atomicExch(d.dmin + u, DMIN_NONE);
      d.dcnt[u] = 0;
      atomicExch(d.inq + u, 0);
      __threadfence();
      const long long eu = ldv(d.e + u) * k.sign;
      if (eu > 0 && hu < n && hu > glim) {
        sstat_add(sm, ST_GAP_SKIPS, 1);      // above an emptied level: parked until the fresh BFS
      } else if (eu > 0 && hu < n) {
        int32_t nh = hu;
        if (mn >= hu) nh = mn >= n ? n : mn + 1;   // every residual slot at >= h(u): lift
        if (nh > hu) {
          k.hgt[u] = nh;
          gap_move(d, sm, tr, hu, nh);
          lifts = 1;
          if (d.rlf[u] == 0) { d.rlf[u] = 1; stage_relabelled(d, rl, u, tag, sm); }
        }
        if (nh < n && nh <= gap_limit(d, tr)) activate(d, k, nxt, u, tag, sm);
        else if (nh < n) sstat_add(sm, ST_GAP_SKIPS, 1);
      }
      sstat_add(sm, ST_DIS_V, 1);
      sstat_add(sm, ST_RELABELS, lifts);
    }
    DBG(d, 205, u, (int32_t)(ce >> 32), (int32_t)pushes, (int32_t)lifts);
    if (d.trace) {
      const unsigned long long dt = gtimer() - t_start;
      const unsigned long long key = (min(dt, 0xffffffffull) << 32) |
                                     ((unsigned long long)min(rend - rbeg, 0xffffff) << 8) | 1ull;
      atomicMax(&d.ctl->slow, key);
    }
    atomicAdd(&sm.work, scanned + 16ull * lifts + 16ull);
    sstat_add(sm, ST_DIS_SLOTS, scanned);
  }
  sstat_add(sm, ST_PUSHES, pushes);
}

// Discharge round: warps take worklist chunks (big vertices) and bin-1 vertices from
// one index space, 8-lane tiles take bin-0 vertices; the first item of every group is
// static (group id), later ones are claimed from cl[1] / cl[2] (see process_bl_dyn).
template <class FnC, class FnW, class FnT>
__device__ __forceinline__ void process_dis(const BL &bl, const int32_t c[NB], int32_t *cl, FnC chunk, FnW warp1,
                                            FnT tile0) {
  {
    WarpG g{(int)(threadIdx.x & 31)};
    const int32_t nwi = c[3] + c[1];
    const int32_t nw = gridDim.x * WPB;
    int32_t x = gwarp_spread();
    while (x < nwi) {
      if (x < c[3]) chunk(bl.cq[x]);
      else warp1(g, bl.bin(1)[x - c[3]]);
      if (g.lane == 0) x = nw + atomicAdd(cl + 1, 1);
      x = __shfl_sync(0xffffffffu, x, 0);
    }
  }
  {
    TileG<8> g((int)(threadIdx.x & 31));
    const int32_t *b = bl.bin(0);
    const int32_t ntl = (gridDim.x * NT) >> 3;
    int32_t x = (int32_t)((threadIdx.x >> 3) * gridDim.x + blockIdx.x);
    while (x < c[0]) {
      tile0(g, b[x]);
      if (g.rank() == 0) x = ntl + atomicAdd(cl + 2, 1);
      x = __shfl_sync(g.mask, x, 0, 8);
    }
  }
}

// ---------------------------------------------------------------------------
// RemoveInvalidEdges (Alg.3 / Alg.7) on one relabelled vertex u: saturate every
// residual slot made steep by u's lift.  Push track: out-slots (u,v) with
// h+(u) > h+(v)+1.  Pull track: in-slots (v,u) with h-(u) > h-(v)+1 (the head is
// the relabelled end, R13).  Heights are frozen in this phase and each residual
// pair has one writer, so the slot stores need no atomics.
// slots [i0, end) step `step` of relabelled vertex u (one thread's share)
__device__ __forceinline__ void rie_slots(const Dev &d, const Track &k, int32_t u, int32_t hu, int32_t i0, int32_t end,
                                          int32_t step, uint32_t tag, const BL &nxt, Smem &sm, long long &moved,
                                          unsigned long long &sat) {
  (void)nxt;                             // the next global relabel finds newly active vertices
  for (int32_t b = i0; b < end; b += 4 * step) {
    int32_t r[4], v[4], h[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {        // independent loads first (ILP), then the gathers
      const int32_t i = b + j * step;
      r[j] = i < end ? ldv(k.F + i) : 0;
      v[j] = i < end ? d.dst[i] : 0;
    }
#pragma unroll
    for (int j = 0; j < 4; j++) h[j] = r[j] > 0 ? ldl1(k.hgt + v[j]) : 0x3fffffff;   // heights are frozen in RIE
#pragma unroll
    for (int j = 0; j < 4; j++) {
      if (r[j] > 0 && hu > h[j] + 1) {
        const int32_t i = b + j * step;
        const int32_t ri = d.rev[i];
        k.F[i] = 0;
        k.R[ri] = 0;
        atomicAdd(k.F + ri, r[j]);
        atomicAdd(k.R + i, r[j]);
        atom_add(d.e + v[j], (long long)r[j] * k.sign);
        moved += r[j];
        sat++;
      }
    }
  }
}

template <class G>
__device__ __forceinline__ void rie(const Dev &d, const G &g, Smem &sm, int32_t entry, const BL &nxt,
                                    unsigned long long *workc) {
  const int tr = ((uint32_t)entry & TRACK_BIT) ? 1 : 0;
  const uint32_t tag = tr ? TRACK_BIT : 0u;
  const int32_t u = (int32_t)((uint32_t)entry & ~TRACK_BIT);
  const Track k = make_track(d, tr);
  const int32_t beg = d.row[u], end = d.row[u + 1];
  const int32_t hu = ldv(k.hgt + u);
  if (g.rank() == 0) d.rlf[u] = 0;
  long long moved = 0;
  unsigned long long sat = 0;
  rie_slots(d, k, u, hu, beg + g.rank(), end, G::size, tag, nxt, sm, moved, sat);
  moved = g.sum(moved);
  if (g.rank() == 0) {
    if (moved) atom_add(d.e + u, -moved * k.sign);
    sstat_add(sm, ST_RIE_SLOTS, (unsigned long long)(end - beg));
  }
  sstat_add(sm, ST_RIE_SAT, sat);
}

// RIE of chunked relabelled entries: one warp per CH-slot piece of a big row.
__device__ __forceinline__ void rie_chunks(const Dev &d, Smem &sm, const long long *cq, int32_t cnt, const BL &nxt,
                                           unsigned long long *workc) {
  const int lane = threadIdx.x & 31;
  const int32_t gw = gwarp_spread(), nw = gridDim.x * WPB;
  WarpG g{lane};
  for (int32_t x = gw; x < cnt; x += nw) {
    const long long ce = cq[x];
    const uint32_t lo = (uint32_t)ce;
    const int tr = (lo & TRACK_BIT) ? 1 : 0;
    const uint32_t tag = tr ? TRACK_BIT : 0u;
    const int32_t u = (int32_t)(lo & ~TRACK_BIT);
    const Track k = make_track(d, tr);
    const int32_t beg = d.row[u] + (int32_t)(ce >> 32) * CH;
    const int32_t end = min(d.row[u + 1], beg + CH);
    const int32_t hu = ldv(k.hgt + u);
    if (lane == 0) d.rlf[u] = 0;
    long long moved = 0;
    unsigned long long sat = 0;
    rie_slots(d, k, u, hu, beg + lane, end, 32, tag, nxt, sm, moved, sat);
    moved = g.sum(moved);
    if (lane == 0) {
      if (moved) atom_add(d.e + u, -moved * k.sign);
      sstat_add(sm, ST_RIE_SLOTS, (unsigned long long)(end - beg));
    }
    sstat_add(sm, ST_RIE_SAT, sat);
  }
}

// ---------------------------------------------------------------------------
// ASYNCHRONOUS discharge phase (replaces the barrier-separated rounds; DMF_ASYNC=0
// restores them).  Every warp repeatedly claims the next item index: first the
// worklist the BFS (or the warm start) collected, then the ring into which activate()
// appends newly active vertices at once, so excess moves on without waiting for a grid
// barrier per hop.  An item is a vertex of <= BIN1_MAX slots (discharge by the warp,
// up to KERNELCYCLES cycles) or one chunk of a bigger row (discharge_chunk).
// Termination: aw's low word counts items queued or in progress (set to the initial
// worklist size before the phase; every enqueue adds before publishing, every item
// subtracts after its own enqueues), so it reaches 0 only when no item exists or can
// appear; the warp that takes it to 0, or one that spends the work budget, raises
// astop.  Waiting warps poll their ring slot and, at most once per ~1 us per CTA, the
// flag (through shared memory).  Items left behind by a budget stop are swept (their
// inq flags cleared) by async_sweep; the next fresh BFS re-collects them (R9).
constexpr uint32_t TAIL_PEND = 64;       // async: "tail" = at most this many items pending
__device__ __forceinline__ long long ldvol(const long long *p) { return *(const volatile long long *)p; }
__device__ __forceinline__ int32_t ldvol(const int32_t *p) { return *(const volatile int32_t *)p; }

// (the CTA's cached stop flag and poll time are shared by its consumer warps: read and
// written with shared-memory atomics)
__device__ __forceinline__ bool async_stopped(const Dev &d, Smem &sm) {
  if (atomicAdd(&sm.astop, 0)) return true;
  const unsigned long long now = gtimer();
  if (now - atomicAdd(&sm.apoll, 0ull) > 1000) {   // one global poll per CTA per microsecond
    atomicExch(&sm.apoll, now);
    if (ldvol(&d.ctl->astop)) { atomicExch(&sm.astop, 1); return true; }
  }
  return false;
}

// warp-wide, after an item whose members fenced their pushes: activate the staged heads
// that hold excess (same rule as dis_flush)
__device__ __forceinline__ void async_candidates(const Dev &d, Smem &sm, const BL &nxt) {
  const int w = (int)(threadIdx.x >> 5), lane = threadIdx.x & 31;
  __syncwarp();
  const int32_t c = min(sm.wcc[w], WCAP);
  for (int32_t x = lane; x < c; x += 32) {
    const uint32_t e = (uint32_t)sm.cand[w * WCAP + x];
    const int tr = (e & TRACK_BIT) ? 1 : 0;
    const int32_t v = (int32_t)(e & ~TRACK_BIT);
    const Track k = make_track(d, tr);
    if (ldv(d.e + v) * k.sign > 0) activate(d, k, nxt, v, e & TRACK_BIT, sm);
  }
  __syncwarp();
  if (lane == 0) sm.wcc[w] = 0;
  __syncwarp();
}

__device__ __forceinline__ void async_phase(const Dev &d, Smem &sm, const BL &init, const int32_t c[NB], const BL &rl,
                                            const BL &nxt) {
  const int lane = threadIdx.x & 31;
  WarpG g{lane};
  Ctl *ctl = d.ctl;
  const int32_t c3 = c[3], c31 = c[3] + c[1], total = c[3] + c[1] + c[0];
  if ((int)(threadIdx.x >> 5) >= d.async_warps) return;   // consumer warps per CTA (fewer pollers)
  for (;;) {
    int32_t idx = -1;
    if (lane == 0 && !async_stopped(d, sm)) idx = atomicAdd(&ctl->ahead, 1);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx < 0) break;
    long long e = AQ_EMPTY;
    if (idx < total) {
      e = idx < c3 ? init.cq[idx] : (long long)(uint32_t)(idx < c31 ? init.bin(1)[idx - c3] : init.bin(0)[idx - c31]);
    } else if (lane == 0) {
      long long *slot = d.aq + ((uint32_t)(idx - total) & (uint32_t)d.aq_mask);
      for (int spin = 0;; spin++) {
        e = ldvol(slot);
        if (e != AQ_EMPTY) { *(volatile long long *)slot = AQ_EMPTY; break; }
        if (async_stopped(d, sm)) break;
        __nanosleep(spin < 4 ? 64 : d.async_sleep_ns);
      }
    }
    e = __shfl_sync(0xffffffffu, e, 0);
    if (e == AQ_EMPTY) break;
    if (lane == 0) DBG(d, 203, (int32_t)((uint32_t)e & ~TRACK_BIT), idx, total, (int32_t)(e >> 32));
    const int32_t v = (int32_t)((uint32_t)e & ~TRACK_BIT);
    if (d.row[v + 1] - d.row[v] > BIN1_MAX) discharge_chunk(d, sm, e, rl, nxt);
    else discharge(d, g, sm, (int32_t)(uint32_t)e, rl, nxt, nullptr);
    async_candidates(d, sm, nxt);
    if (lane == 0) {
      const unsigned long long old = atomicAdd(&ctl->aw, ~0ull);        // item done (after its enqueues)
      bool stop = (uint32_t)old == 1u;                                    // nothing left anywhere
      // progress stop: a long low-parallelism tail means excess creeping up one lift at a
      // time on stale heights (a ping-pong the rounds bound by charging every round); one
      // global relabel fixes every height at once.  Counted in items, not time, so the
      // work done does not depend on the clock or the box.
      if (!stop && d.tail_items > 0 && (uint32_t)old <= (uint32_t)TAIL_PEND &&
          atomicAdd(&ctl->atail, 1) + 1 >= d.tail_items) {
        stop = true;
        sstat_add(sm, ST_TAIL_STOPS, 1);
      }
      if (!stop && *(volatile unsigned long long *)&sm.work > 32768ull) {  // budget: flushed in 32K-slot units
        const unsigned long long w = atomicExch(&sm.work, 0ull);
        stop = (long long)(atomicAdd(&ctl->awork, w) + w) > d.work_budget;
      }
      if (stop) { if (!ldvol(&ctl->astop)) atomicExch(&ctl->astop, 1); atomicExch(&sm.astop, 1); }
    }
  }
}

// A queued item dropped by a budget stop: clear the vertex's queued flag and, for a
// chunked vertex (some of whose chunks may already have counted themselves), its
// chunk protocol state -- none of its chunks runs after the phase's barrier.
__device__ __forceinline__ void async_unqueue(const Dev &d, long long e) {
  const int32_t v = (int32_t)((uint32_t)e & ~TRACK_BIT);
  d.inq[v] = 0;
  if (d.row[v + 1] - d.row[v] > BIN1_MAX) { d.dcnt[v] = 0; d.dmin[v] = DMIN_NONE; }
}

// After the phase's barrier: clear the inq flags of items a budget stop left queued.
__device__ __forceinline__ bool async_sweep(const Dev &d, Smem &sm, const BL &init, const int32_t c[NB]) {
  const long long w = cta_ld(sm, reinterpret_cast<const long long *>(&d.ctl->aw));
  const int32_t head = cta_ld(sm, &d.ctl->ahead);
  if ((uint32_t)w == 0) return false;      // terminated normally: every item was consumed
  const int32_t c3 = c[3], c31 = c[3] + c[1], total = c[3] + c[1] + c[0];
  const int32_t gt = blockIdx.x * NT + threadIdx.x, nt = gridDim.x * NT;
  for (int32_t x = min(head, total) + gt; x < total; x += nt) {
    const long long e = x < c3 ? init.cq[x] : (long long)(uint32_t)(x < c31 ? init.bin(1)[x - c3] : init.bin(0)[x - c31]);
    async_unqueue(d, e);
  }
  const long long tail = (long long)((unsigned long long)w >> 32);
  const long long cap = (long long)d.aq_mask + 1;
  for (long long x = gt; x < (tail < cap ? tail : cap); x += nt) {
    const long long e = d.aq[x];
    if (e != AQ_EMPTY) { async_unqueue(d, e); d.aq[x] = AQ_EMPTY; }
  }
  return true;
}

// ---------------------------------------------------------------------------
// Roots of a global relabel.
enum ResetKind : int { RK_PUSH = 0, RK_PP = 1, RK_STAGE2 = 2, RK_MINCUT = 3, RK_MAXCUT = 4, RK_MINCUT_P = 5,
                       RK_RETURN_S = 6,   // stage (ii): push track, roots {s}: excess flows back to s (Lemma 4)
                       RK_FILL_T = 7 };   // stage (ii): pull track, roots {t}: deficits are filled from t

struct Lists {      // (members, not arrays: a dynamically indexed array would live in local memory)
  int32_t *q0, *q1;       // frontier ping-pong, [NB bins][n] each
  long long *qc0, *qc1;   // their chunk queues
  int32_t *wl0, *wl1;     // worklist ping-pong, [NB bins][n] each
  int32_t *rl;            // relabelled, [NB bins][n]
  long long *rlc;         // its chunk queue
  long long *cw0, *cw1;   // worklist chunk queues (ping-pong with wl0 / wl1)
  __device__ int32_t *q(int i) const { return i ? q1 : q0; }
  __device__ long long *qc(int i) const { return i ? qc1 : qc0; }
  __device__ int32_t *wl(int i) const { return i ? wl1 : wl0; }
  __device__ long long *cw(int i) const { return i ? cw1 : cw0; }
};


// Topology-driven sweep: every vertex of the domain is tested
// (thread per vertex, "idle when inactive") and an active one is discharged in place:
// by its own thread (<= BIN0_MAX slots), by its warp (<= BIN1_MAX), or queued as
// CH-slot chunks for the grid after the sweep.  No worklist is built: the next sweep
// finds the vertices that became active (activate() only raises ctl->tact).
__device__ __forceinline__ void topology_sweep(const Dev &d, Smem &sm, const int32_t *dom, int32_t N, bool use0,
                                               bool use1, const BL &rl, const BL &tch) {
  const int lane = threadIdx.x & 31;
  const int32_t nt = gridDim.x * NT, n = d.n;
  WarpG wg{lane};
  for (int32_t b = blockIdx.x * NT + (threadIdx.x & ~31); b < N; b += nt) {
    const int32_t x = b + lane;
    int32_t v = 0, deg = 0, entry = 0;
    bool act = false;
    if (x < N) {
      v = dom ? dom[x] : x;
      if (ldv(d.inq + v)) d.inq[v] = 0;        // worklist flag of the BFS collection: unused here
      if (v != d.s && v != d.t) {
        const long long ev = ldv(d.e + v);
        int tr = -1;
        if (use0 && ev > 0 && ldv(d.hp + v) < n) tr = 0;
        else if (use1 && ev < 0 && ldv(d.hm + v) < n) tr = 1;
        if (tr >= 0) {
          deg = d.row[v + 1] - d.row[v];
          act = deg > 0;
          entry = (int32_t)((uint32_t)v | (tr ? TRACK_BIT : 0u));
        }
      }
    }
    chunks_conv(d, tch, act && deg > BIN1_MAX, deg, v, (uint32_t)entry & TRACK_BIT);
    if (act && deg <= BIN0_MAX) discharge(d, ThreadG{}, sm, entry, rl, tch, nullptr);
    __syncwarp();
    unsigned m = __ballot_sync(0xffffffffu, act && deg > BIN0_MAX && deg <= BIN1_MAX);
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      discharge(d, wg, sm, __shfl_sync(0xffffffffu, entry, j), rl, tch, nullptr);
    }
  }
}

// The device loop: repeat { RESET; BFS levels (+ worklist); if no active: stop;
//                           rounds of { DISCHARGE; RIE } until no vertex is queued }.
// Counter discipline (each counter is zeroed by block 0 in a phase where nobody
// else reads or appends it, then published by the next grid barrier):
//   qc/fs[l%3]  appended at level l-1 (RESET for l=0), read at level l, zeroed at
//               level l+1; [1] zeroed in RESET; [0] zeroed in every RIE phase (or by
//               the caller before the loop)
//   wlc[r%3]    read in DISCHARGE of round r, appended in round r-1 (the BFS for r=0),
//               zeroed in round r+1 (as wlc[(r+3-1)%3]) and all of them in the RIE phase
//   rlc         appended in every DISCHARGE round of an iteration (once per vertex,
//               rlf flag), read in the iteration's RIE phase, zeroed in RESET
//   bulc[l&1]   appended in pass A of level l, read in pass B; [(l+1)&1] zeroed at l
//   mu          accumulated in RESET, read at level 0; zeroed with qc[0]
// Requires qc[0], fs[0], mu == 0 and wlc == 0 on entry.
// Returns 0 when the loop ended normally.  `lazy` (DYN_PP warm start, DESIGN.md
// "certificate"): after the warm iteration the termination test is the universal one of
// R9 -- a fresh backward BFS from {t} u {all deficits} over the whole graph (kind
// RK_PUSH) that reaches no excess vertex, and s reaching none of its labelled vertices;
// then the loop returns 1 (converged; the partition is that BFS's reach, R15).  If the
// test fails it returns -1 with its queued flags dropped and the counters zeroed, and
// the caller continues with the full Alg.8 stage 1.
__device__ int device_loop(const Dev &d, cg::grid_group &grid, Smem &sm, PhaseClock &clk, int kind0,
                           bool collect, bool stage2, bool warm = false, bool lazy = false) {
  const size_t nb = (size_t)NB * d.n;
  const Lists L{d.q0, d.q1, d.cq0, d.cq1, d.wl, d.wl + nb, d.rl, d.cqr, d.cw0, d.cw1};
  const int32_t n = d.n;
  Ctl *ctl = d.ctl;
  int32_t *qc = ctl->qc, *wlc = ctl->wlc, *rlc = ctl->rlc;
  const int32_t nt = gridDim.x * NT;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  for (int iter = 0;; ++iter) {
   if (lazy && iter >= 1 && d.split) return 2;   // the certificate runs in k_reach<true> (reach.cuh)
   const bool certify = lazy && iter >= 1;       // the universal certificate pass
   const int kind = certify ? (int)RK_PUSH : kind0;
   const bool use0 = kind != RK_MINCUT && kind != RK_MINCUT_P && kind != RK_FILL_T;
   const bool use1 = kind == RK_PP || kind == RK_MINCUT || kind == RK_MINCUT_P || kind == RK_FILL_T;
   const bool on_plist = kind == RK_STAGE2 || kind == RK_MINCUT_P;
   // warm start (DYN_PP after DYN_PP): iteration 0 discharges the worklist seeded by
   // the batch prologue on the previous call's final labels; the fresh BFS of
   // iteration 1 still decides termination (R9), so stale labels cost work only
   if (!(warm && iter == 0)) {
    // ---------------- RESET: heights of the domain, roots -> frontier level 0
    if (blockIdx.x == 0 && threadIdx.x < NB) {
      if (threadIdx.x == 0) { ctl->aw = 0; ctl->ahead = 0; ctl->astop = 0; ctl->awork = 0; ctl->atail = 0; }
      rlc[threadIdx.x] = 0;
      qc[NB + threadIdx.x] = 0;
      if (threadIdx.x < 3) { ctl->work[threadIdx.x] = 0; ctl->tact[threadIdx.x] = 0; }
      if (threadIdx.x < 2) { ctl->fs[2 + threadIdx.x] = 0; ctl->bulc[threadIdx.x] = 0; }
    }
    const int32_t N = on_plist ? cta_ld(sm, &ctl->pcnt) : n;
    {
      // heights: 0 for roots, |V| for the rest of the track's region, |V|+1 outside it
      FS fs;
      long long mu0 = 0, mu1 = 0;
      const BfsCtx c0{0, 0, certify ? BCH : CH, false, 0u, 0u, BL{L.q0, qc, n, L.qc0},
                      BL{L.wl0, wlc, n, L.cw0}, ctl->fs};
      // RU vertices per thread per step, every load of the step issued before the first
      // use (the sweep is bound by dependent round trips, not bytes)
      constexpr int RU = 4;
      for (int32_t t0 = blockIdx.x * NT * RU; t0 < N; t0 += nt * RU) {
        int32_t v[RU], deg[RU];
        long long ev[RU];
        uint8_t p[RU];
        bool ok[RU];
#pragma unroll
        for (int j = 0; j < RU; j++) {
          const int32_t x = t0 + j * NT + threadIdx.x;
          ok[j] = x < N;
          v[j] = ok[j] ? (on_plist ? d.plist[x] : x) : 0;
        }
#pragma unroll
        for (int j = 0; j < RU; j++) {
          ev[j] = ok[j] ? ldv(d.e + v[j]) : 0;
          p[j] = (ok[j] && kind == RK_PP) ? ldv(d.part + v[j]) : (uint8_t)0;
          deg[j] = ok[j] ? d.row[v[j] + 1] - d.row[v[j]] : 0;
        }
#pragma unroll
        for (int j = 0; j < RU; j++) {
          bool r0 = false, r1 = false, in0 = false, in1 = false;
          if (ok[j]) {
            const int32_t x = v[j];
            if (kind == RK_PUSH || kind == RK_MAXCUT) {
              r0 = x == d.t || (x != d.s && ev[j] < 0);
              in0 = x != d.s;
              d.hp[x] = r0 ? 0 : n;
            } else if (kind == RK_PP) {
              in0 = p[j] == PART_T && x != d.s;
              in1 = p[j] == PART_S && x != d.t;
              r0 = in0 && (x == d.t || ev[j] < 0);
              r1 = in1 && (x == d.s || ev[j] > 0);
              d.hp[x] = r0 ? 0 : (in0 ? n : n + 1);
              d.hm[x] = r1 ? 0 : (in1 ? n : n + 1);
            } else if (kind == RK_STAGE2) {       // P only; outside P heights stay >= |V| or
              r0 = ev[j] < 0;                     // belong to T\P, which no P vertex reaches
              in0 = true;
              d.hp[x] = r0 ? 0 : n;
            } else if (kind == RK_RETURN_S) {     // t is outside the region: its excess is F
              r0 = x == d.s;
              in0 = x != d.t;
              d.hp[x] = r0 ? 0 : (in0 ? n : n + 1);
            } else if (kind == RK_FILL_T) {       // s is outside the region
              r1 = x == d.t;
              in1 = x != d.s;
              d.hm[x] = r1 ? 0 : (in1 ? n : n + 1);
            } else if (kind == RK_MINCUT_P) {     // forward reach of the excess left in P
              r1 = ev[j] > 0;
              in1 = true;
              d.hm[x] = r1 ? 0 : n;
            } else {  // RK_MINCUT
              r1 = x == d.s || (x != d.t && ev[j] > 0);
              in1 = x != d.t;
              d.hm[x] = r1 ? 0 : n;
            }
            if (in0 && !r0) mu0 += deg[j];
            else if (in1 && !r1) mu1 += deg[j];
          }
          claim_push_deg(d, sm.st, c0, r0 || r1, false, v[j], r1 ? 1 : 0, fs, deg[j]);
        }
      }
      bfs_flush(d, sm, sm.st, c0, fs);
      BlockG bg{sm.red};
      mu0 = bg.sum(mu0); mu1 = bg.sum(mu1);
      if (threadIdx.x == 0) {
        if (mu0) atomicAdd(ctl->mu, (unsigned long long)mu0);
        if (mu1) atomicAdd(ctl->mu + 1, (unsigned long long)mu1);
      }
      if (lead) sstat_add(sm, ST_RESET_V, (unsigned long long)N);
    }
    beacon(d, 10 + kind, iter, 0, 0);
    gsync(d, grid, sm);
    clk.lap(d, sm, ST_T_RESET, iter, kind, N);
    // ---------------- BFS levels (fused worklist compaction + termination test)
    cta_snap(sm, 2, [&](int k) { return ldv(reinterpret_cast<const long long *>(ctl->mu + k)); });
    long long mu[2] = {use0 ? sm.cv[0] : 0, use1 ? sm.cv[1] : 0};
    int32_t lvl = 0;
    for (;; ++lvl) {
      int32_t *cur_c = qc + NB * (lvl % 3);
      int32_t c[NB];
      unsigned long long *fsl = ctl->fs + 2 * (lvl % 3);
      cta_snap(sm, NB + 2, [&](int k) {
        return k < NB ? (long long)ldv(cur_c + k) : ldv(reinterpret_cast<const long long *>(fsl + (k - NB)));
      });
#pragma unroll
      for (int b = 0; b < NB; b++) c[b] = (int32_t)sm.cv[b];
      const long long f0 = sm.cv[NB], f1 = sm.cv[NB + 1];
      beacon(d, 20 + kind, iter, 0, lvl, total(c), c[3]);
      if (total(c) == 0) break;
      if (lvl > 0) { mu[0] -= f0; mu[1] -= f1; }
      if (blockIdx.x == 0 && threadIdx.x < NB) {
        qc[NB * ((lvl + 2) % 3) + threadIdx.x] = 0;
        if (threadIdx.x < 2) {
          ctl->fs[2 * ((lvl + 2) % 3) + threadIdx.x] = 0;
          ctl->bulc[2 * ((lvl + 1) & 1) + threadIdx.x] = 0;
        }
      }
      const bool bu0 = f0 > 0 && (unsigned long long)f0 * d.bu_alpha > (unsigned long long)(mu[0] > 0 ? mu[0] : 0);
      const bool bu1 = f1 > 0 && (unsigned long long)f1 * d.bu_alpha > (unsigned long long)(mu[1] > 0 ? mu[1] : 0);
      const bool dn0 = !bu0 && f0 > 0 && (unsigned long long)f0 * d.dense_div >= (unsigned long long)d.S;
      const bool dn1 = !bu1 && f1 > 0 && (unsigned long long)f1 * d.dense_div >= (unsigned long long)d.S;
      const BfsCtx ctx{lvl, lvl + 1, certify ? BCH : CH, collect, (bu0 ? 1u : 0u) | (bu1 ? 2u : 0u),
                       (dn0 ? 1u : 0u) | (dn1 ? 2u : 0u),
                       BL{L.q((lvl + 1) & 1), qc + NB * ((lvl + 1) % 3), n, L.qc((lvl + 1) & 1)},
                       BL{L.wl0, wlc, n, L.cw0}, ctl->fs + 2 * ((lvl + 1) % 3)};
      if (lead && (bu0 || bu1)) sstat_add(sm, ST_BU_LEVELS, 1);
      bfs_expand_level(d, grid, sm, sm.st, clk, iter, BL{L.q(lvl & 1), cur_c, n, L.qc(lvl & 1)}, c, ctx, d.bul,
                       ctl->bulc + 2 * (lvl & 1));
      if (dn0 || dn1) {                             // dense top-down tracks: build lvl+1 by compaction
        long long g0 = 0, g1 = 0;
        int32_t v0 = 0, v1 = 0;
        compact_domain(d, sm.ts, N, on_plist ? d.plist : nullptr, ctx.next, ctx.wl, collect,
          [&](int32_t v, int &tr, bool &front, bool &act) {
            if (dn0 && ldv(d.hp + v) == lvl + 1) { tr = 0; front = true; }
            else if (dn1 && ldv(d.hm + v) == lvl + 1) { tr = 1; front = true; }
            if (front) act = activity(d, collect, tr, v);
          }, g0, g1, v0, v1, ctx.bch);
        BlockG bg{sm.red};
        g0 = bg.sum(g0); g1 = bg.sum(g1);
        const long long nv0 = bg.sum(v0), nv1 = bg.sum(v1);
        if (threadIdx.x == 0) {
          if (g0) atomicAdd(ctx.fs_next, (unsigned long long)g0);
          if (g1) atomicAdd(ctx.fs_next + 1, (unsigned long long)g1);
          if (d.local_gap && lvl + 1 < GAPW && lvl + 1 < n) {     // dense levels: counted here, once per vertex
            if (nv0) atomicAdd(d.cnt + lvl + 1, (int32_t)nv0);
            if (nv1) atomicAdd(d.cnt + GAPW + lvl + 1, (int32_t)nv1);
          }
        }
        gsync(d, grid, sm);
        clk.lap(d, sm, ST_T_BFS_CMP, iter, lvl, N);
      }
    }
    if (lead) sstat_add(sm, ST_LEVELS, (unsigned long long)lvl);
    {
      int32_t w0[NB];
      cta_counts(sm, wlc, w0);
      if (certify) {
        // s is never labelled by the backward BFS (h+(s) = |V|, R1) and DYN_PP does not
        // re-saturate s (R16): s must reach no labelled vertex either
        if (total(w0) == 0) {
          const int32_t sb = d.row[d.s], se = d.row[d.s + 1];
          bool hit = false;
          for (int32_t i = sb + blockIdx.x * NT + threadIdx.x; i < se; i += nt)
            hit |= ldv(d.res + i) > 0 && ldv(d.hp + d.dst[i]) < n;
          if (__syncthreads_or(hit) && threadIdx.x == 0) atomicExch(&ctl->sreach, 1);
          gsync(d, grid, sm);
          if (cta_ld(sm, &ctl->sreach) == 0) return 1;     // converged (R9)
        }
        // not certified: drop the queued flags of the collected worklist, clear the
        // counters device_loop expects zero, and hand back to the full stage 1
        for (int32_t x = blockIdx.x * NT + threadIdx.x; x < w0[0] + w0[1]; x += nt)
          d.inq[(uint32_t)(x < w0[0] ? L.wl0[x] : L.wl0[(size_t)d.n + x - w0[0]]) & ~TRACK_BIT] = 0;
        for (int32_t x = blockIdx.x * NT + threadIdx.x; x < w0[3]; x += nt)
          d.inq[(uint32_t)L.cw0[x] & ~TRACK_BIT] = 0;
        if (blockIdx.x == 0 && threadIdx.x < NB) {
          for (int q = 0; q < 3; q++) { wlc[NB * q + threadIdx.x] = 0; qc[NB * q + threadIdx.x] = 0; }
          rlc[threadIdx.x] = 0;
          if (threadIdx.x < 6) ctl->fs[threadIdx.x] = 0;
          if (threadIdx.x < 2) { ctl->mu[threadIdx.x] = 0; ctl->gtop[threadIdx.x] = 0; }
        }
        if (blockIdx.x == 0 && d.local_gap)
          for (int i = threadIdx.x; i < 2 * GAPW; i += NT) d.cnt[i] = 0;
        gsync(d, grid, sm);
        return -1;
      }
      if (total(w0) == 0) break;                  // no active vertex: converged (R9)
    }
   }
    if (lead) {
      sstat_add(sm, ST_ITERS, 1);
      if (stage2) sstat_add(sm, ST_S2_ITERS, 1);
    }
    if (iter + 1 >= d.max_iters) {
      if (lead) ctl->status = -8;                // DMF_ENOCONV
      break;
    }
    // ---------------- DISCHARGE (push || pull tracks), then RIE once
    // (Alg.1 l.168-169: PushRelabel, then RemoveInvalidEdges, then the next BFS).
    // Schedule of the phase: topology-driven sweeps when many vertices are
    // active (the auto-switch of P:923), else the data-driven worklist as an
    // asynchronous ring or as barrier-separated rounds.
    unsigned long long spent = 0;                 // work since the global relabel (same in every thread)
    const BL rl{L.rl, rlc, n, L.rlc};
    int32_t w_async[NB];
    cta_counts(sm, wlc, w_async);
    const int32_t ndom = on_plist ? cta_ld(sm, &ctl->pcnt) : n;
    const bool topo = d.topo_div > 0 && (long long)total(w_async) * d.topo_div > (long long)ndom;
    if (threadIdx.x == 0) { sm.amode = d.async && !topo; sm.topo = topo; }
    __syncthreads();
    if (topo) {
      for (int r = 0;; ++r) {
        // rings of 3 (round r uses slot r % 3, zeroes slot (r+1) % 3, last read in
        // round r-2): activity flag, work and the chunk-list count of the sweep.  (Not
        // wlc: other CTAs may still be reading the BFS worklist counts in slot 0.)
        const int cur = r % 3, nx = (r + 1) % 3;
        if (threadIdx.x == 0) sm.tslot = cur;
        if (blockIdx.x == 0 && threadIdx.x < NB) {
          ctl->tcq[NB * nx + threadIdx.x] = 0;
          if (threadIdx.x == 0) { ctl->tact[nx] = 0; ctl->work[nx] = 0; }
        }
        __syncthreads();
        const BL tch{L.wl1, ctl->tcq + NB * cur, n, L.cw1};   // chunks of the big active vertices of this sweep
        topology_sweep(d, sm, on_plist ? d.plist : nullptr, ndom, use0, use1, rl, tch);
        dis_flush(d, sm, tch, rl);
        gsync(d, grid, sm);
        {
          const int32_t nc = cta_ld(sm, ctl->tcq + NB * cur + 3);
          const int32_t gw = gwarp_spread(), nw = gridDim.x * WPB;
          for (int32_t x = gw; x < nc; x += nw) discharge_chunk(d, sm, tch.cq[x], rl, tch);
          dis_flush(d, sm, tch, rl);
        }
        __syncthreads();                          // every warp's work is in sm.work
        if (threadIdx.x == 0) { const unsigned long long w_ = atomicExch(&sm.work, 0ull); if (w_) atomicAdd(ctl->work + cur, w_); }
        if (lead) { sstat_add(sm, ST_ROUNDS, 1); sstat_add(sm, ST_TOPO_ROUNDS, 1); }
        gsync(d, grid, sm);
        clk.lap(d, sm, ST_T_DIS, iter, r, ndom, 0);
        cta_snap(sm, 2, [&](int k) {
          return k == 0 ? (long long)ldv(ctl->tact + cur) : ldv(reinterpret_cast<const long long *>(ctl->work + cur));
        });
        spent += (unsigned long long)sm.cv[1] + (unsigned long long)(d.S >> 4);
        if (sm.cv[0] == 0) break;                 // no vertex became or stayed active
        if (r + 1 >= MAX_ROUNDS || (long long)spent > d.work_budget) {
          if (lead) sstat_add(sm, ST_BUDGET_STOPS, 1);
          break;
        }
      }
      if (threadIdx.x == 0) sm.topo = 0;
    } else if (d.async && total(w_async) > 0) {
      const int32_t *w = w_async;
      if (lead) ctl->aw = (unsigned long long)total(w);   // (tail 0) published by the barrier below
      if (threadIdx.x == 0) { sm.astop = 0; sm.apoll = 0; }
      gsync(d, grid, sm);
      const BL init{L.wl0, wlc, n, L.cw0};
      async_phase(d, sm, init, w, rl, BL{L.wl1, wlc + NB, n, L.cw1});
      dis_flush(d, sm, BL{L.wl1, wlc + NB, n, L.cw1}, rl);
      __syncthreads();
      if (threadIdx.x == 0) { const unsigned long long w_ = atomicExch(&sm.work, 0ull); if (w_) atomicAdd(&ctl->awork, w_); }
      if (lead) sstat_add(sm, ST_ROUNDS, 1);
      gsync(d, grid, sm);
      clk.lap(d, sm, ST_T_DIS, iter, 0, total(w), w[3]);
      const bool stopped = async_sweep(d, sm, init, w);
      if (lead && stopped) sstat_add(sm, ST_BUDGET_STOPS, 1);
    }
    for (int r = 0; !d.async && !topo; ++r) {
      // wlc / work rings of 3: round r reads [r%3], fills [(r+1)%3]; a slot is zeroed
      // only when every block has passed the barrier after its last read
      const int cur = r % 3, nx = (r + 1) % 3, nn = (r + 2) % 3;
      int32_t w[NB];
      cta_counts(sm, wlc + NB * cur, w);
      beacon(d, 30 + kind, iter, r, 0, total(w), w[3]);
      if (blockIdx.x == 0 && threadIdx.x < NB) {
        wlc[NB * nn + threadIdx.x] = 0;           // last read in round r-1 (before its barrier)
        if (threadIdx.x < 3) ctl->claim[3 * nn + threadIdx.x] = 0;   // claimed in round r-1
        if (threadIdx.x == 0) ctl->work[nx] = 0;  // last read at the end of round r-2; filled in round r+1
      }
      const BL nxt{L.wl((r + 1) & 1), wlc + NB * nx, n, L.cw((r + 1) & 1)};
      process_dis(BL{L.wl(r & 1), wlc + NB * cur, n, L.cw(r & 1)}, w, ctl->claim + 3 * cur,
                  [&](long long ce) { discharge_chunk(d, sm, ce, rl, nxt); },
                  [&](const WarpG &g, int32_t entry) { discharge(d, g, sm, entry, rl, nxt, ctl->work + cur); },
                  [&](const TileG<8> &g, int32_t entry) { discharge(d, g, sm, entry, rl, nxt, ctl->work + cur); });
      dis_flush(d, sm, nxt, rl);
      __syncthreads();
      if (threadIdx.x == 0) { const unsigned long long w_ = atomicExch(&sm.work, 0ull); if (w_) atomicAdd(ctl->work + cur, w_); }
      if (lead) sstat_add(sm, ST_ROUNDS, 1);
      gsync(d, grid, sm);
      clk.lap(d, sm, ST_T_DIS, iter, r, total(w), w[3]);
      int32_t wn[NB];
      cta_snap(sm, NB + 1, [&](int k) {
        return k < NB ? (long long)ldv(wlc + NB * nx + k) : ldv(reinterpret_cast<const long long *>(ctl->work + cur));
      });
#pragma unroll
      for (int b = 0; b < NB; b++) wn[b] = (int32_t)sm.cv[b];
      // a round's barrier + latency floor is charged like S/16 scanned slots, so that
      // long tails of near-empty rounds (excess creeping up one lift at a time) hand
      // over to a global relabel, which lifts unreachable vertices to |V| at once
      spent += (unsigned long long)sm.cv[NB] + (unsigned long long)(d.S >> 4);
      if (total(wn) == 0) break;
      if (r + 1 >= MAX_ROUNDS || (long long)spent > d.work_budget) {   // hand the rest to a global relabel
        if (lead) sstat_add(sm, ST_BUDGET_STOPS, 1);
        for (int b = 0; b < 2; b++) {
          const int32_t *lst = nxt.bin(b);
          for (int32_t x = blockIdx.x * NT + threadIdx.x; x < wn[b]; x += nt)
            d.inq[(uint32_t)lst[x] & ~TRACK_BIT] = 0;
        }
        for (int32_t x = blockIdx.x * NT + threadIdx.x; x < wn[3]; x += nt)
          d.inq[(uint32_t)nxt.cq[x] & ~TRACK_BIT] = 0;
        break;                                    // (the RIE barrier below publishes the flags)
      }
    }
    // ---------------- RIE over the vertices relabelled in this iteration
    if (blockIdx.x == 0 && threadIdx.x < NB) {
      for (int q = 0; q < 3; q++) { wlc[NB * q + threadIdx.x] = 0; ctl->tcq[NB * q + threadIdx.x] = 0; }
      if (threadIdx.x < 3) for (int q = 0; q < 3; q++) ctl->claim[3 * q + threadIdx.x] = 0;
      qc[threadIdx.x] = 0;                        // for the next RESET
      if (threadIdx.x < 2) { ctl->fs[threadIdx.x] = 0; ctl->mu[threadIdx.x] = 0; ctl->gtop[threadIdx.x] = 0; }
    }
    if (blockIdx.x == 0 && d.local_gap)           // level counts: rebuilt by the next RESET + BFS
      for (int i = threadIdx.x; i < 2 * GAPW; i += NT) d.cnt[i] = 0;
    {
      int32_t rc[NB];
      cta_counts(sm, rlc, rc);
      beacon(d, 40 + kind, iter, 0, 0, total(rc), rc[3]);
      rie_chunks(d, sm, rl.cq, rc[3], rl, ctl->work);
      const int32_t rc2[NB] = {rc[0], rc[1], 0, 0};
      process_bl(rl, rc2, sm, [&](auto &g, int32_t entry) { rie(d, g, sm, entry, rl, ctl->work); });
      gsync(d, grid, sm);
      clk.lap(d, sm, ST_T_RIE, iter, 0, total(rc), rc[3]);
    }
  }
  return 0;
}

// Slot of (u,v), -1 if absent: open-addressing (u,v) -> slot table built by
// dmf_create (linear probing, load <= 1/2); an entry {v, slot} matches when its slot
// lies in u's row.  One 8-byte load per probe, probes of a run share a sector.
__device__ __forceinline__ uint32_t slot_hash(int32_t u, int32_t v) {
  unsigned long long k = ((unsigned long long)(uint32_t)u << 32) | (uint32_t)v;
  k ^= k >> 33; k *= 0xff51afd7ed558ccdull; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ull; k ^= k >> 33;
  return (uint32_t)k;
}
__device__ __forceinline__ int32_t find_slot(const Dev &d, int32_t u, int32_t v) {
  for (uint32_t h = slot_hash(u, v) & (uint32_t)d.hmask;; h = (h + 1) & (uint32_t)d.hmask) {
    const int4 e = __ldg(d.htab + h);
    if (e.x == u && e.y == v) return e.z;
    if (e.x < 0) return -1;
  }
}

__device__ __forceinline__ void set_status(const Dev &d, int32_t code, int32_t entry) {
  if (atomicCAS(&d.ctl->status, 0, code) == 0) d.ctl->err_entry = entry;
}

// saturate slot i (res -> 0, all of it moved to the reverse and to e(head))
__device__ __forceinline__ long long saturate_slot(const Dev &d, int32_t i) {
  const int32_t r = ldv(d.res + i);
  if (r <= 0) return 0;
  const int32_t ri = d.rev[i];
  d.res[i] = 0;
  d.rres[ri] = 0;
  atomicAdd(d.res + ri, r);
  atomicAdd(d.rres + i, r);
  atom_add(d.e + d.dst[i], r);
  return r;
}

// Grid-stride sweep over the vertices [0, n), RU per thread per step: load(v) of all RU
// vertices first (independent loads in flight together), then apply(v, x, ok) for each,
// called by every lane (ok = v < n) so that apply may use warp collectives.
template <class T, int RU = 4, class Load, class Apply>
__device__ __forceinline__ void vsweep(int32_t n, Load load, Apply apply) {
  const int32_t nt = gridDim.x * NT;
  for (int32_t t0 = blockIdx.x * NT * RU; t0 < n; t0 += nt * RU) {
    T x[RU];
#pragma unroll
    for (int j = 0; j < RU; j++) {
      const int32_t v = t0 + j * NT + threadIdx.x;
      x[j] = v < n ? load(v) : T{};
    }
#pragma unroll
    for (int j = 0; j < RU; j++) {
      const int32_t v = t0 + j * NT + threadIdx.x;
      apply(v, x[j], v < n);
    }
  }
}

// warp-convergent histogram increment: lanes with the same bin add once (heights of a
// BFS labelling take a handful of values, so per-lane shared atomics would serialise)
__device__ __forceinline__ void hist_add(int32_t *hist, bool pred, int32_t idx) {
  const unsigned act = __ballot_sync(0xffffffffu, pred);
  if (!pred) return;
  const unsigned grp = __match_any_sync(act, idx);
  if ((int)(threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(hist + idx, __popc(grp));
}

struct VX { long long e; int32_t hp, hm; };

template <int NTHREADS>
__global__ void __launch_bounds__(NTHREADS, MIN_BLOCKS) k_solve(const __grid_constant__ Dev d, int32_t mode) {
  cg::grid_group grid = cg::this_grid();
  __shared__ Smem sm;
  // the continuation of a DYN_PP whose k_reach certificate held has nothing to do
  if (mode == MODE_PP_CONT && *(const volatile int32_t *)&d.ctl->lazy_ok) return;
  for (int i = threadIdx.x; i < ST_N; i += NTHREADS) sm.stat[i] = 0;
  if (threadIdx.x < 6) sm.st.cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) { sm.work = 0; sm.tprev = gtimer(); sm.acnt = 0; sm.rcnt = 0; sm.ccnt = 0; sm.astop = 0; sm.apoll = 0;
                          sm.amode = 0; sm.topo = 0; sm.tslot = 0; sm.st.lv[0] = 0; sm.st.lv[1] = 0; }
  if (threadIdx.x < WPB) sm.wcc[threadIdx.x] = 0;
  if (blockIdx.x == 0 && d.local_gap) {
    // level counts of the local gap: a DYN_PP warm start keeps the previous call's
    // (the final labels' histogram, see the PP epilogue); every other call rebuilds
    // them from its first RESET.  Published by the first grid barrier.
    if (!(mode == MODE_PP && d.warm)) for (int i = threadIdx.x; i < 2 * GAPW; i += NTHREADS) d.cnt[i] = 0;
    if (mode == MODE_PP || mode == MODE_PP_CONT || mode == MODE_MINCUT)
      for (int i = threadIdx.x; i < 2 * GAPW; i += NTHREADS) d.cnt_next[i] = 0;
  }
  __syncthreads();
  const int32_t n = d.n;
  const int32_t gt = blockIdx.x * NTHREADS + threadIdx.x, nt = gridDim.x * NTHREADS;
  Ctl *ctl = d.ctl;
  BlockG bg{sm.red};
  PhaseClock clk;
  clk.start(sm);

  if (mode == MODE_STATIC) {
    // Alg.1 l.1-8: e = 0, c_f = c  (and the mirror)
    for (int64_t i = gt; i < d.S; i += nt) { d.res[i] = d.cap[i]; d.rres[i] = d.cap[d.rev[i]]; }
    for (int32_t v = gt; v < n; v += nt) d.e[v] = 0;
    gsync(d, grid, sm);
  } else if (mode == MODE_PR || mode == MODE_PP) {
    // ---- Updates Processing (Alg.5), all-or-nothing (R11), in ONE pass per entry:
    // validate (ids, capacity, slot lookup in the (u,v) hash table, duplicate stamp)
    // and apply optimistically, recording what was added.  Every update below is a
    // commutative atomic add, so if any entry of the batch is invalid a second pass
    // subtracts exactly what the first added and the state is byte-identical again.
    // Alg.5 l.1-3 (c_f += c' - c) and l.4-11 (a negative slot returns its excess flow:
    // e(u) += d, e(v) -= d, R10) are fused per entry: the clamp of slot i depends only
    // on c_f(i) + delta_i (the entry of the reverse slot never changes c_f(i) unless it
    // is the negative one, and a pair has at most one: their sum c'_i + c'_ri >= 0).
    // DYN_PP also saturates a touched S->T slot here (Alg.8 l.10-13, R12): at a
    // converged cut a T->S slot can never go negative, so nothing else changes it.
    // e(s) / e(t) deltas are summed per CTA: batches are biased toward s-out and t-in
    // slots (R20), so per-entry atomics would serialise on those two addresses.
    long long ds = 0, dt = 0;
    auto eadd = [&](int32_t x, long long delta) {
      if (x == d.s) ds += delta; else if (x == d.t) dt += delta; else atom_add(d.e + x, delta);
    };
    // Two entries per thread per step, every independent load of both issued before the
    // first dependent use (the pass is bound by dependent random accesses).
    constexpr int EU = 2;
    for (int64_t j0 = gt; j0 < d.k; j0 += (int64_t)EU * nt) {
      int32_t u[EU], v[EU], c[EU], i[EU], st[EU], ri[EU], cap0[EU];
      uint8_t pu[EU], pv[EU];
      bool ok[EU];
      int4 e0[EU];
      uint32_t h0[EU];
#pragma unroll
      for (int q = 0; q < EU; q++) {               // entry, parts, first probe
        const int64_t j = j0 + (int64_t)q * nt;
        ok[q] = j < d.k;
        u[q] = ok[q] ? d.bu[j] : 0; v[q] = ok[q] ? d.bv[j] : 0; c[q] = ok[q] ? d.bc[j] : 0;
        if (ok[q] && (u[q] < 0 || u[q] >= n || v[q] < 0 || v[q] >= n)) { set_status(d, -1, (int32_t)j); ok[q] = false; }
        else if (ok[q] && (c[q] < 0 || c[q] > 1073741823)) { set_status(d, -7, (int32_t)j); ok[q] = false; }
        pu[q] = (ok[q] && mode == MODE_PP) ? ldv(d.part + u[q]) : (uint8_t)0;
        pv[q] = (ok[q] && mode == MODE_PP) ? ldv(d.part + v[q]) : (uint8_t)0;
        h0[q] = ok[q] ? slot_hash(u[q], v[q]) & (uint32_t)d.hmask : 0u;
        e0[q] = ok[q] ? __ldg(d.htab + h0[q]) : make_int4(-1, -1, -1, -1);
      }
#pragma unroll
      for (int q = 0; q < EU; q++) {               // resolve slot and reverse slot (rarely a second probe)
        i[q] = -1; ri[q] = 0;
        if (!ok[q]) continue;
        if (e0[q].x == u[q] && e0[q].y == v[q]) { i[q] = e0[q].z; ri[q] = e0[q].w; }
        else if (e0[q].x >= 0) {
          for (uint32_t h = (h0[q] + 1) & (uint32_t)d.hmask;; h = (h + 1) & (uint32_t)d.hmask) {
            const int4 e = __ldg(d.htab + h);
            if (e.x == u[q] && e.y == v[q]) { i[q] = e.z; ri[q] = e.w; break; }
            if (e.x < 0) break;
          }
        }
        if (i[q] < 0) { set_status(d, -2, (int32_t)(j0 + (int64_t)q * nt)); ok[q] = false; }
      }
#pragma unroll
      for (int q = 0; q < EU; q++) {               // duplicate stamp; new capacity in, old one out
        const int64_t j = j0 + (int64_t)q * nt;
        if (j < d.k) d.bslot[j] = ok[q] ? i[q] : -1;
        st[q] = ok[q] ? atomicExch(d.stamp + i[q], d.batch_id) : 0;
        cap0[q] = ok[q] ? atomicExch(d.cap + i[q], c[q]) : 0;   // (entries naming one slot chain: their deltas add up)
      }
#pragma unroll
      for (int q = 0; q < EU; q++) {
        if (!ok[q]) continue;
        const int64_t j = j0 + (int64_t)q * nt;
        const int32_t delta = c[q] - cap0[q];
        int32_t r = atomicAdd(d.res + i[q], delta) + delta;
        atomicAdd(d.rres + ri[q], delta);
        int32_t dd = 0, sat = 0;
        if (r < 0) {                               // flow on (u,v) above the new capacity
          dd = -r;
          atomicAdd(d.res + i[q], dd);
          atomicAdd(d.rres + ri[q], dd);
          atomicAdd(d.res + ri[q], -dd);
          atomicAdd(d.rres + i[q], -dd);
          eadd(u[q], (long long)dd);
          eadd(v[q], -(long long)dd);
          r = 0;
        }
        if (mode == MODE_PP && r > 0 && pu[q] == PART_S && pv[q] == PART_T) {
          sat = r;                                 // saturate the touched S->T slot
          atomicAdd(d.res + i[q], -r);
          atomicAdd(d.rres + ri[q], -r);
          atomicAdd(d.res + ri[q], r);
          atomicAdd(d.rres + i[q], r);
          eadd(v[q], (long long)r);
          eadd(u[q], -(long long)r);
        }
        d.brec[3 * j] = delta; d.brec[3 * j + 1] = dd; d.brec[3 * j + 2] = sat;
        if (st[q] == d.batch_id) set_status(d, -3, (int32_t)j);   // a second entry for this slot
      }
    }
    auto flush_st = [&]() {
      const long long a = bg.sum(ds), b = bg.sum(dt);
      if (threadIdx.x == 0) {
        if (a) atom_add(d.e + d.s, a);
        if (b) atom_add(d.e + d.t, b);
      }
      ds = 0; dt = 0;
    };
    flush_st();
    gsync(d, grid, sm);
    clk.lap(d, sm, ST_T_PRO, 0, 1, (int32_t)d.k);
    if (cta_ld(sm, &ctl->status) != 0) {           // an invalid entry: undo every applied one
      mode = -1;
      for (int64_t j = gt; j < d.k; j += nt) {
        const int32_t i = d.bslot[j];
        if (i < 0) continue;
        const int32_t ri = d.rev[i];
        const int32_t u = d.bu[j], v = d.bv[j];
        const int32_t delta = d.brec[3 * j], dd = d.brec[3 * j + 1], sat = d.brec[3 * j + 2];
        if (sat) {
          atomicAdd(d.res + i, sat); atomicAdd(d.rres + ri, sat); atomicAdd(d.res + ri, -sat); atomicAdd(d.rres + i, -sat);
          eadd(v, -(long long)sat); eadd(u, (long long)sat);
        }
        if (dd) {
          atomicAdd(d.res + i, -dd); atomicAdd(d.rres + ri, -dd); atomicAdd(d.res + ri, dd); atomicAdd(d.rres + i, dd);
          eadd(u, -(long long)dd); eadd(v, (long long)dd);
        }
        atomicAdd(d.res + i, -delta); atomicAdd(d.rres + ri, -delta); atomicAdd(d.cap + i, -delta);
      }
      flush_st();
      gsync(d, grid, sm);
    }
    if (mode == MODE_PP && d.warm) {
      // Warm start of Alg.8 stage 1: only batch endpoints changed excess, so the
      // new roots (T-deficits for h+, S-excess for h-, Alg.8 l.16-24) drop to 0 and
      // the active ones seed round 0's worklist (ring slot 0, deduplicated by inq)
      const BL wl0{d.wl, ctl->wlc, n, d.cw0};
      constexpr int EW = 4;                        // endpoints per thread per step (loads first)
      for (int64_t j0 = gt; j0 < 2 * d.k; j0 += (int64_t)EW * nt) {
        int32_t x[EW], hx[EW];
        uint8_t p[EW];
        long long ev[EW];
#pragma unroll
        for (int q = 0; q < EW; q++) {
          const int64_t j = j0 + (int64_t)q * nt;
          x[q] = j < 2 * d.k ? ((j & 1) ? d.bv[j >> 1] : d.bu[j >> 1]) : d.s;
        }
#pragma unroll
        for (int q = 0; q < EW; q++) {
          const bool live = x[q] != d.s && x[q] != d.t;
          p[q] = live ? ldv(d.part + x[q]) : (uint8_t)PART_NONE;
          ev[q] = live ? ldv(d.e + x[q]) : 0;
        }
#pragma unroll
        for (int q = 0; q < EW; q++)
          hx[q] = p[q] == PART_T ? ldv(d.hp + x[q]) : (p[q] == PART_S ? ldv(d.hm + x[q]) : 0);
#pragma unroll
        for (int q = 0; q < EW; q++) {
          if (p[q] == PART_T) {
            if (ev[q] < 0) {
              if (hx[q] != 0) {
                const int32_t old = atomicExch(d.hp + x[q], 0);      // (x may be named by several entries)
                if (old != 0 && old < n) gap_move(d, sm, 0, old, 0);
              }
            } else if (ev[q] > 0 && hx[q] < n) activate(d, make_track(d, 0), wl0, x[q], 0u, sm, false);
          } else if (p[q] == PART_S) {
            if (ev[q] > 0) {
              if (hx[q] != 0) {
                const int32_t old = atomicExch(d.hm + x[q], 0);
                if (old != 0 && old < n) gap_move(d, sm, 1, old, 0);
              }
            } else if (ev[q] < 0 && hx[q] < n) activate(d, make_track(d, 1), wl0, x[q], TRACK_BIT, sm, false);
          }
        }
      }
      {
        const BL none{d.rl, ctl->rlc, n, d.cqr};    // (no relabels staged here)
        dis_flush(d, sm, wl0, none);
      }
      gsync(d, grid, sm);
      clk.lap(d, sm, ST_T_PRO, 0, 3, (int32_t)d.k);
    }
  }
  if (mode == MODE_STATIC || mode == MODE_PR) {
    // Alg.1 l.9-13 / Alg.4 l.3-8 (R3): saturate every residual out-slot of s
    const int32_t beg = d.row[d.s], end = d.row[d.s + 1];
    long long tot = 0;
    for (int32_t i = beg + gt; i < end; i += nt) tot += saturate_slot(d, i);
    tot = bg.sum(tot);
    if (threadIdx.x == 0 && tot) atom_add(d.e + d.s, -tot);
    if (mode == MODE_STATIC && d.static_pp) {
      // static push-pull: also saturate every residual in-edge (v,t); the
      // deficient tails are secondary sinks -- roots of the global relabel (R2)
      const int32_t tb = d.row[d.t], te = d.row[d.t + 1];
      long long into = 0;
      for (int32_t i = tb + gt; i < te; i += nt) {     // slot i = (t,v), rev[i] = (v,t)
        if (d.dst[i] == d.s) continue;                 // (s,t) was saturated with s's row
        const int32_t j = d.rev[i];
        const int32_t r = ldv(d.res + j);
        if (r <= 0) continue;
        d.res[j] = 0;
        d.rres[i] = 0;
        atomicAdd(d.res + i, r);
        atomicAdd(d.rres + j, r);
        atom_add(d.e + d.dst[i], -(long long)r);
        into += r;
      }
      into = bg.sum(into);
      if (threadIdx.x == 0 && into) atom_add(d.e + d.t, into);
    }
    gsync(d, grid, sm);
    clk.lap(d, sm, ST_T_PRO);
    device_loop(d, grid, sm, clk, RK_PUSH, true, false);
    // part from the final fresh BFS (S = unreached = S_max, R15) + flow (R8)
    long long f = 0;
    vsweep<VX>(n, [&](int32_t v) { return VX{ldv(d.e + v), ldv(d.hp + v), 0}; },
               [&](int32_t v, const VX &x, bool ok) {
                 if (!ok) return;
                 d.part[v] = x.hp < n ? PART_T : PART_S;
                 f += v == d.t ? x.e : (v != d.s && x.e < 0 ? x.e : 0);
               });
    f = bg.sum(f);
    if (threadIdx.x == 0 && f) atomicAdd(reinterpret_cast<unsigned long long *>(&ctl->flow), (unsigned long long)f);
  } else if (mode == MODE_PP || mode == MODE_PP_CONT) {
    // ---- stage 1: push on T || pull on S (Alg.8 l.15-28)
    clk.lap(d, sm, ST_T_PRO);
    // Warm start: discharge on the previous labels, then the universal certificate
    // (R9).  When it holds, the state is converged and Alg.8's remaining work (the
    // two-track BFS, P, stage 2) has nothing to change; the partition is the
    // certificate's reach (R15) and S_min is left to dmf_min_cut_source_side.
    // With d.split the certificate runs in k_reach<true> (lz = 2: nothing more here) and a
    // MODE_PP_CONT launch continues below (lz = -1) only if it failed.
    const int lz = mode == MODE_PP_CONT ? -1
                 : (d.warm && d.lazy) ? device_loop(d, grid, sm, clk, RK_PP, true, false, true, true) : 0;
    if (lz == 2) {
      // (handed to k_reach<true>)
    } else if (lz == 1) {
      long long f = 0;
      int32_t *hist = sm.cand;
      const bool want_hist = d.local_gap && d.cnt_next;
      if (want_hist) {
        for (int i = threadIdx.x; i < 2 * GAPW; i += NTHREADS) hist[i] = 0;
        __syncthreads();
      }
      vsweep<VX>(n, [&](int32_t v) { return VX{ldv(d.e + v), ldv(d.hp + v), ldv(d.hm + v)}; },
                 [&](int32_t v, const VX &x, bool ok) {
        int32_t hmv = x.hm;
        if (ok) {
          f += v == d.t ? x.e : (v != d.s && x.e < 0 ? x.e : 0);
          const bool tside = x.hp < n;             // reaches t or a deficit: T' (R15)
          d.part[v] = tside ? PART_T : PART_S;
          if (tside) { d.hm[v] = n + 1; hmv = n + 1; }
          else {
            d.hp[v] = n + 1;
            if (hmv > n) { d.hm[v] = n; hmv = n; }  // (T -> S': in the pull region, unreached)
          }
        }
        if (want_hist) {
          hist_add(hist, ok && x.hp < n && x.hp < GAPW, x.hp);
          hist_add(hist + GAPW, ok && hmv < n && hmv < GAPW, hmv);
        }
      });
      f = bg.sum(f);
      if (threadIdx.x == 0 && f) atomicAdd(reinterpret_cast<unsigned long long *>(&ctl->flow), (unsigned long long)f);
      if (blockIdx.x == 0 && threadIdx.x == 0) ctl->lazy_ok = 1;
      if (want_hist) {
        __syncthreads();
        for (int i = threadIdx.x; i < 2 * GAPW; i += NTHREADS)
          if (hist[i]) atomicAdd(d.cnt_next + i, hist[i]);
      }
    } else {
    // (certificate failed after the warm iteration: the full stage 1 from fresh labels)
    device_loop(d, grid, sm, clk, RK_PP, true, false, d.warm != 0 && lz == 0);
    // ---- P = {h+ = |V| and h- = |V|} (Alg.8 l.29-33), vertices with slots only
    if (blockIdx.x == 0 && threadIdx.x < NB) {
      ctl->qc[threadIdx.x] = 0;
      if (threadIdx.x < 2) { ctl->fs[threadIdx.x] = 0; ctl->mu[threadIdx.x] = 0; ctl->gtop[threadIdx.x] = 0; }
    }
    if (blockIdx.x == 0 && d.local_gap)            // stage 2 rebuilds the level counts of P
      for (int i = threadIdx.x; i < 2 * GAPW; i += NTHREADS) d.cnt[i] = 0;
    long long pdef = 0, pexc = 0;                  // deficits / excess vertices in P
    for (int32_t v = gt; v < n; v += nt) {         // block-staged appends (one global atomic per CTA)
      if (d.row[v + 1] > d.row[v] && ldv(d.hp + v) >= n && ldv(d.hm + v) >= n) {
        d.part[v] = PART_P;
        const long long ev = ldv(d.e + v);
        pdef += ev < 0;
        pexc += ev > 0;
        const int32_t pos = atomicAdd(&sm.acnt, 1);
        if (pos < ACAP) act_buf(sm)[pos] = v;
        else d.plist[atomicAdd(&ctl->pcnt, 1)] = v;
      }
    }
    pdef = bg.sum(pdef);
    pexc = bg.sum(pexc);
    if (threadIdx.x == 0) {
      if (pdef) atomicAdd(&ctl->pdef, (int32_t)pdef);
      if (pexc) atomicAdd(&ctl->pexc, (int32_t)pexc);
    }
    __syncthreads();
    {
      if (threadIdx.x == 0) {
        const int32_t c0 = min(sm.acnt, ACAP);
        sm.ts.cnt[0] = c0;
        sm.ts.base[0] = c0 ? atomicAdd(&ctl->pcnt, c0) : 0;
        sm.acnt = 0;
      }
      __syncthreads();
      const int32_t c = sm.ts.cnt[0];
      for (int32_t x = threadIdx.x; x < c; x += NTHREADS) d.plist[sm.ts.base[0] + x] = act_buf(sm)[x];
      __syncthreads();
    }
    gsync(d, grid, sm);
    const int32_t pc = cta_ld(sm, &ctl->pcnt);
    cta_snap(sm, 2, [&](int k) { return (long long)ldv(k ? &ctl->pexc : &ctl->pdef); });
    const bool has_def = sm.cv[0] > 0, has_exc = sm.cv[1] > 0;
    if (threadIdx.x == 0 && blockIdx.x == 0) sstat_add(sm, ST_S2_V, (unsigned long long)pc);
    // ---- stage 2: Dynamic Push-Relabel restricted to P (Alg.8 l.34).  Its roots are
    //      P's deficits: without any, its first global relabel ends the loop at once and
    //      reaches no P vertex (all of P goes to S'), so it is skipped.  With deficits
    //      but no excess it still runs: its final BFS decides which P vertices go to T'.
    clk.lap(d, sm, ST_T_EPI);
    if (pc > 0 && has_def) device_loop(d, grid, sm, clk, RK_STAGE2, true, true);
    else if (pc > 0 && blockIdx.x == 0 && threadIdx.x == 0) sstat_add(sm, ST_S2_SKIP, 1);
    if (pc > 0 && has_exc) {
      // ---- S_min (R19) = stage 1's final forward reach from {s} u Exc_S (h- < |V|)
      //      united with the forward reach, inside P, of the excess left in P: no
      //      residual edge enters P from S\P or leaves P towards T\P.
      //      (Stage 2 moves excess only inside P and never creates any where P had none.)
      if (blockIdx.x == 0 && threadIdx.x < NB) {
        ctl->qc[threadIdx.x] = 0;
        if (threadIdx.x < 2) { ctl->fs[threadIdx.x] = 0; ctl->mu[threadIdx.x] = 0; }
      }
      gsync(d, grid, sm);
      device_loop(d, grid, sm, clk, RK_MINCUT_P, false, false);
    } else if (pc > 0 && blockIdx.x == 0 && threadIdx.x == 0) {
      sstat_add(sm, ST_S2_SKIP, 1);              // no excess in P: its forward reach is empty
    }
    // ---- relabel partitions (Alg.8 l.35-49) and F (= sum over T' of e, R8)
    for (int32_t x = gt; x < pc; x += nt) {     // (+ the region encoding of the next warm start:
      const int32_t v = d.plist[x];              //  h+ = |V|+1 on S', h- = |V|+1 on T')
      const bool tside = ldv(d.hp + v) < n;
      d.part[v] = tside ? PART_T : PART_S;
      if (tside) d.hm[v] = n + 1;
      else { d.hp[v] = n + 1; if (ldv(d.hm + v) > n) d.hm[v] = n; }   // (n: in S', unreached)
    }
    long long f = 0;
    int32_t *hist = sm.cand;                     // final labels' histogram (warm start of the next call)
    const bool want_hist = d.local_gap && d.cnt_next;
    if (want_hist) {
      for (int i = threadIdx.x; i < 2 * GAPW; i += NTHREADS) hist[i] = 0;
      __syncthreads();
    }
    vsweep<VX>(n, [&](int32_t v) { return VX{ldv(d.e + v), want_hist ? ldv(d.hp + v) : 0, ldv(d.hm + v)}; },
               [&](int32_t v, const VX &x, bool ok) {
      if (ok) {
        f += v == d.t ? x.e : (v != d.s && x.e < 0 ? x.e : 0);
        d.mask[v] = x.hm < n ? 1 : 0;            // S_min, cached for dmf_min_cut_source_side
      }
      if (want_hist) {
        hist_add(hist, ok && x.hp < n && x.hp < GAPW, x.hp);
        hist_add(hist + GAPW, ok && x.hm < n && x.hm < GAPW, x.hm);
      }
    });
    f = bg.sum(f);
    if (threadIdx.x == 0 && f) atomicAdd(reinterpret_cast<unsigned long long *>(&ctl->flow), (unsigned long long)f);
    if (want_hist) {
      __syncthreads();
      for (int i = threadIdx.x; i < 2 * GAPW; i += NTHREADS)
        if (hist[i]) atomicAdd(d.cnt_next + i, hist[i]);
    }
    }   // full stage 1
  } else if (mode == MODE_FLOW) {
    // Stage (ii): turn the converged pseudoflow into a
    // true maximum flow.  Every vertex with excess reaches s in the residual graph
    // (Lemma 4) and every deficient vertex is reached from t;
    // neither can reach the other side at convergence, so F is unchanged.  The same
    // engine runs twice: push track with roots {s}, then pull track with roots {t}.
    gsync(d, grid, sm);                              // (publishes the zeroed level counts)
    device_loop(d, grid, sm, clk, RK_RETURN_S, true, false);
    if (blockIdx.x == 0 && threadIdx.x < NB) {
      ctl->qc[threadIdx.x] = 0;
      if (threadIdx.x < 2) { ctl->fs[threadIdx.x] = 0; ctl->mu[threadIdx.x] = 0; }
    }
    gsync(d, grid, sm);
    device_loop(d, grid, sm, clk, RK_FILL_T, true, false);
    long long f = 0;
    for (int32_t v = gt; v < n; v += nt) {
      const long long ev = ldv(d.e + v);
      f += v == d.t ? ev : (v != d.s && ev < 0 ? ev : 0);
      if (v != d.s && v != d.t && ev != 0) set_status(d, -8, v);   // not a flow: DMF_ENOCONV
    }
    f = bg.sum(f);
    if (threadIdx.x == 0 && f) atomicAdd(reinterpret_cast<unsigned long long *>(&ctl->flow), (unsigned long long)f);
  } else if (mode == MODE_MINCUT || mode == MODE_MAXCUT) {
    device_loop(d, grid, sm, clk, mode == MODE_MINCUT ? RK_MINCUT : RK_MAXCUT, false, false);
    // MINCUT rewrites h- with the exact forward distances from {s} u Exc: the pull
    // labels of a following DYN_PP warm start, with their level histogram
    int32_t *hist = sm.cand;
    const bool want_hist = mode == MODE_MINCUT && d.local_gap && d.cnt_next;
    if (want_hist) {
      for (int i = threadIdx.x; i < 2 * GAPW; i += NTHREADS) hist[i] = 0;
      __syncthreads();
    }
    vsweep<VX>(n, [&](int32_t v) { return VX{0, ldv(d.hp + v), ldv(d.hm + v)}; },
               [&](int32_t v, const VX &x, bool ok) {
      if (ok) d.mask[v] = mode == MODE_MINCUT ? (x.hm < n ? 1 : 0) : (x.hp < n ? 0 : 1);
      if (want_hist) {
        hist_add(hist, ok && x.hp < n && x.hp < GAPW, x.hp);
        hist_add(hist + GAPW, ok && x.hm < n && x.hm < GAPW, x.hm);
      }
    });
    if (want_hist) {
      __syncthreads();
      for (int i = threadIdx.x; i < 2 * GAPW; i += NTHREADS)
        if (hist[i]) atomicAdd(d.cnt_next + i, hist[i]);
    }
  }
  clk.lap(d, sm, ST_T_EPI);
  __syncthreads();
  for (int i = threadIdx.x; i < ST_N; i += NTHREADS)
    if (sm.stat[i]) atomicAdd(&ctl->stat[i], sm.stat[i]);
}

}  // namespace dmf
