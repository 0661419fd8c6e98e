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

struct Smem {
  long long red[WPB + 1];
  unsigned long long stat[ST_N];
};

// Phase clock (block 0, thread 0): time between consecutive grid barriers is
// charged to the phase that just ran.
struct PhaseClock {
  unsigned long long t;
  __device__ void start() { if (blockIdx.x == 0 && threadIdx.x == 0) t = gtimer(); }
  __device__ void lap(Smem &sm, int which);
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

__device__ void PhaseClock::lap(Smem &sm, int which) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long now = gtimer();
    sm.stat[which] += now - t;
    t = now;
  }
}

__device__ __forceinline__ int bin_of(const Dev &d, int32_t v) {
  const int32_t deg = d.row[v + 1] - d.row[v];
  return deg <= BIN0_MAX ? 0 : (deg <= BIN1_MAX ? 1 : 2);
}

// Binned list view: three buffers (n entries each) and three counters.
struct BL {
  int32_t *buf;   // bin b at buf + b*n
  int32_t *c;
  int32_t n;
  __device__ int32_t *bin(int b) const { return buf + (size_t)b * n; }
};

// append v (with track tag) to its degree bin; convergent (whole warp) or not
__device__ __forceinline__ void bl_append_conv(const Dev &d, const BL &bl, bool pred, int32_t v, uint32_t tag) {
  const int bin = pred ? bin_of(d, v) : -1;
#pragma unroll
  for (int b = 0; b < 3; b++) warp_append(pred && bin == b, (int32_t)((uint32_t)v | tag), bl.bin(b), bl.c + b);
}
__device__ __forceinline__ void bl_append_one(const Dev &d, const BL &bl, int32_t v, uint32_t tag) {
  const int bin = bin_of(d, v);
  const int pos = atomicAdd(bl.c + bin, 1);
  bl.bin(bin)[pos] = (int32_t)((uint32_t)v | tag);
}

// Process a binned list: CTA per bin-2 entry, warp per bin-1 entry, thread per
// bin-0 entry.  fn(group, entry).
template <class Fn>
__device__ __forceinline__ void process_bl(const BL &bl, const int32_t c[3], Smem &sm, Fn fn) {
  {
    BlockG g{sm.red};
    const int32_t *b = bl.bin(2);
    for (int32_t x = blockIdx.x; x < c[2]; x += gridDim.x) fn(g, b[x]);
  }
  {
    WarpG g{(int)(threadIdx.x & 31)};
    const int32_t *b = bl.bin(1);
    const int32_t gw = blockIdx.x * WPB + (threadIdx.x >> 5), nw = gridDim.x * WPB;
    for (int32_t x = gw; x < c[1]; x += nw) fn(g, b[x]);
  }
  {
    ThreadG g;
    const int32_t *b = bl.bin(0);
    const int32_t gt = blockIdx.x * NT + threadIdx.x, nt = gridDim.x * NT;
    for (int32_t x = gt; x < c[0]; x += nt) fn(g, b[x]);
  }
}

// Queue a vertex whose excess (track-signed) just crossed from <= 0 to > 0 for the
// next discharge round, at most once per round (inq flag).
__device__ __forceinline__ void activate(const Dev &d, const Track &k, const BL &nxt, int32_t v, uint32_t tag,
                                         Smem &sm) {
  if (v == d.s || v == d.t) return;
  if (ldv(k.hgt + v) >= d.n) return;
  if (atomicCAS(d.inq + v, 0, 1) != 0) return;
  bl_append_one(d, nxt, v, tag);
  sstat_add(sm, ST_ACTIVATIONS, 1);
}

// ---------------------------------------------------------------------------
// BFS: one residual slot i scanned from frontier vertex w at level lvl.  A residual
// edge (v -> w) [push track] / (w -> v) [pull track] lets v be labelled lvl+1.
struct BfsCtx {
  int32_t lvl;
  uint8_t reg0, reg1;
  bool collect;
  BL next, wl;
};

__device__ __forceinline__ void bfs_slot(const Dev &d, const BfsCtx &c, int tr, int32_t i, bool valid,
                                         bool &claimed, bool &act, int32_t &v) {
  claimed = false; act = false; v = -1;
  if (!valid) return;
  const Track k = make_track(d, tr);
  const int32_t rb = ldv(k.B + i);
  const int32_t vv = d.dst[i];
  if (rb <= 0) return;
  v = vv;
  const uint8_t reg = tr ? c.reg1 : c.reg0;
  if (v == k.excl || ldv(k.hgt + v) != d.n) return;
  if (reg != 0 && ldv(d.part + v) != reg) return;
  claimed = atomicCAS(k.hgt + v, d.n, c.lvl + 1) == d.n;
  if (claimed && c.collect) {
    const long long ev = ldv(d.e + v);
    act = tr ? (ev < 0) : (ev > 0);
  }
}

// warp (or CTA) per frontier vertex: coalesced scan of its row
template <class G>
__device__ __forceinline__ void bfs_expand_group(const Dev &d, const G &g, Smem &sm, int32_t entry, const BfsCtx &c) {
  const int tr = ((uint32_t)entry & TRACK_BIT) ? 1 : 0;
  const int32_t w = (int32_t)((uint32_t)entry & ~TRACK_BIT);
  const uint32_t tag = tr ? TRACK_BIT : 0u;
  const int32_t beg = d.row[w], end = d.row[w + 1];
  for (int32_t base = beg; base < end; base += G::size) {
    const int32_t i = base + g.rank();
    bool claimed, act;
    int32_t v;
    bfs_slot(d, c, tr, i, i < end, claimed, act, v);
    bl_append_conv(d, c.next, claimed, v, tag);
    if (c.collect) bl_append_conv(d, c.wl, act, v, tag);
  }
  if (g.rank() == 0) {
    sstat_add(sm, ST_BFS_SLOTS, (unsigned long long)(end - beg));
    sstat_add(sm, ST_BFS_V, 1);
  }
}

// warp over a chunk of up to 32 low-degree frontier vertices: the concatenation of
// their rows is split evenly over the lanes (degree exclusive scan + shuffle search)
__device__ __forceinline__ void bfs_expand_chunk(const Dev &d, Smem &sm, const int32_t *list, int32_t x0,
                                                 int32_t cnt, const BfsCtx &c) {
  const int lane = threadIdx.x & 31;
  int32_t entry = 0, beg = 0, deg = 0;
  if (lane < cnt) {
    entry = list[x0 + lane];
    const int32_t w = (int32_t)((uint32_t)entry & ~TRACK_BIT);
    beg = d.row[w];
    deg = d.row[w + 1] - beg;
  }
  WarpG g{lane};
  long long tot;
  const int32_t off = (int32_t)g.exscan(deg, tot);
  const int32_t total = (int32_t)tot;
  for (int32_t t0 = 0; t0 < total; t0 += 32) {
    const int32_t k = t0 + lane;
    int j = 0;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const int32_t o = __shfl_sync(0xffffffffu, off, j + s);
      if (o <= k) j += s;
    }
    const int32_t ej = __shfl_sync(0xffffffffu, entry, j);
    const int32_t bj = __shfl_sync(0xffffffffu, beg, j);
    const int32_t oj = __shfl_sync(0xffffffffu, off, j);
    const int tr = ((uint32_t)ej & TRACK_BIT) ? 1 : 0;
    bool claimed, act;
    int32_t v;
    bfs_slot(d, c, tr, bj + (k - oj), k < total, claimed, act, v);
    // tracks may differ between lanes: append per tag
    bl_append_conv(d, c.next, claimed && tr == 0, v, 0u);
    bl_append_conv(d, c.next, claimed && tr == 1, v, TRACK_BIT);
    if (c.collect) {
      bl_append_conv(d, c.wl, act && tr == 0, v, 0u);
      bl_append_conv(d, c.wl, act && tr == 1, v, TRACK_BIT);
    }
  }
  if (lane == 0) {
    sstat_add(sm, ST_BFS_SLOTS, (unsigned long long)total);
    sstat_add(sm, ST_BFS_V, (unsigned long long)cnt);
  }
}

__device__ __forceinline__ void bfs_level(const Dev &d, Smem &sm, const BL &cur, const int32_t c[3], const BfsCtx &ctx) {
  {
    BlockG g{sm.red};
    const int32_t *b = cur.bin(2);
    for (int32_t x = blockIdx.x; x < c[2]; x += gridDim.x) bfs_expand_group(d, g, sm, b[x], ctx);
  }
  const int32_t gw = blockIdx.x * WPB + (threadIdx.x >> 5), nw = gridDim.x * WPB;
  {
    WarpG g{(int)(threadIdx.x & 31)};
    const int32_t *b = cur.bin(1);
    for (int32_t x = gw; x < c[1]; x += nw) bfs_expand_group(d, g, sm, b[x], ctx);
  }
  {
    const int32_t *b = cur.bin(0);
    for (int32_t x = gw * 32; x < c[0]; x += nw * 32) bfs_expand_chunk(d, sm, b, x, min(32, c[0] - x), ctx);
  }
}

// ---------------------------------------------------------------------------
// Discharge of one active vertex (Alg.2 / Alg.6): up to KERNELCYCLES cycles of
// "scan residual out-slots for the lowest neighbour (h, slot); push if h(u) > h^,
// else lift h(u) = h^+1" (clamped to n, R4/R5; ties by slot index, R6).  A push
// cycle pushes to the successive lowest neighbours at height h^ in slot order until
// the excess is gone -- exactly the run of Alg.2 cycles that would follow with the
// heights as read.
template <class G>
__device__ __forceinline__ void discharge(const Dev &d, const G &g, Smem &sm, int32_t entry, const BL &rl,
                                          const BL &nxt, unsigned long long *workc) {
  const int tr = ((uint32_t)entry & TRACK_BIT) ? 1 : 0;
  const uint32_t tag = tr ? TRACK_BIT : 0u;
  const int32_t u = (int32_t)((uint32_t)entry & ~TRACK_BIT);
  const Track k = make_track(d, tr);
  const int32_t n = d.n;
  const int32_t beg = d.row[u], end = d.row[u + 1];
  if (g.rank() == 0) { d.inq[u] = 0; __threadfence(); }
  int32_t hu = ldv(k.hgt + u);
  bool relabelled = false;
  unsigned long long scanned = 0, pushes = 0, lifts = 0;
  long long eu = 0;
  int cyc = 0;
  for (; cyc < d.kc; ++cyc) {
    if (g.rank() == 0) eu = ldv(d.e + u) * k.sign;
    eu = g.bcast(eu);
    if (hu >= n || eu <= 0) break;
    unsigned long long best = ~0ull;
    for (int32_t i0 = beg + g.rank(); i0 < end; i0 += 4 * G::size) {
      int32_t r[4], v[4];
#pragma unroll
      for (int j = 0; j < 4; j++) {             // independent loads first (ILP), then the gathers
        const int32_t i = i0 + j * G::size;
        r[j] = i < end ? ldv(k.F + i) : 0;
        v[j] = i < end ? d.dst[i] : 0;
      }
#pragma unroll
      for (int j = 0; j < 4; j++) {
        if (r[j] > 0) {
          const int32_t h = ldv(k.hgt + v[j]);
          const unsigned long long key = ((unsigned long long)(uint32_t)h << 32) | (uint32_t)(i0 + j * G::size - beg);
          best = key < best ? key : best;
        }
      }
    }
    scanned += (unsigned long long)(end - beg);
    best = g.min(best);
    if (best == ~0ull) {                 // no residual out-edge: h^ = inf -> |V| (R4)
      hu = n;
      if (g.rank() == 0) k.hgt[u] = n;
      relabelled = true;
      lifts++;
      break;
    }
    const int32_t hhat = (int32_t)(best >> 32);
    if (hu > hhat) {                     // push(u, v^) applicable (Alg.2 l.15-19)
      long long remaining = eu;
      const int32_t start = beg + (int32_t)(best & 0xffffffffu);
      for (int32_t base = start; base < end && remaining > 0; base += G::size) {
        const int32_t i = base + g.rank();
        long long amt = 0;
        int32_t v = -1;
        if (i < end) {
          const int32_t r = ldv(k.F + i);
          if (r > 0) {
            v = d.dst[i];
            if (ldv(k.hgt + v) == hhat) amt = r;
          }
        }
        long long tot;
        const long long ex = g.exscan(amt, tot);
        long long take = remaining - ex;
        take = take < 0 ? 0 : (take > amt ? amt : take);
        if (take > 0) {
          const int32_t ri = d.rev[i];
          atomicSub(k.F + i, (int32_t)take);       // c_f(u,v^) -= d
          atomicSub(k.R + ri, (int32_t)take);      //   mirror
          atomicAdd(k.F + ri, (int32_t)take);      // c_f(v^,u) += d
          atomicAdd(k.R + i, (int32_t)take);       //   mirror
          const long long old = (long long)atomicAdd(reinterpret_cast<unsigned long long *>(d.e + v),
                                                     (unsigned long long)(take * k.sign));   // e(v^) += d
          const long long eo = old * k.sign;
          if (eo <= 0 && eo + take > 0) activate(d, k, nxt, v, tag, sm);
          pushes++;
        }
        remaining -= tot;
        scanned += (unsigned long long)G::size;
      }
      const long long done = eu - (remaining > 0 ? remaining : 0);
      if (g.rank() == 0 && done > 0) atom_add(d.e + u, -done * k.sign);   // e(u) -= d
    } else {                             // lift(u) (Alg.2 l.21), clamped to |V| (R5)
      hu = hhat + 1 < n ? hhat + 1 : n;
      if (g.rank() == 0) k.hgt[u] = hu;
      relabelled = true;
      lifts++;
    }
  }
  if (g.rank() == 0) {
    if (cyc == d.kc && hu < n && ldv(d.e + u) * k.sign > 0) activate(d, k, nxt, u, tag, sm);  // KC spent
    if (relabelled) bl_append_one(d, rl, u, tag);
    atomicAdd(workc, scanned + 16ull * lifts + 16ull);
    sstat_add(sm, ST_DIS_V, 1);
    sstat_add(sm, ST_DIS_SLOTS, scanned);
    sstat_add(sm, ST_RELABELS, lifts);
  }
  sstat_add(sm, ST_PUSHES, pushes);
}

// ---------------------------------------------------------------------------
// RemoveInvalidEdges (Alg.3 / Alg.7) on one relabelled vertex u: saturate every
// residual slot made steep by u's lift.  Push track: out-slots (u,v) with
// h+(u) > h+(v)+1.  Pull track: in-slots (v,u) with h-(u) > h-(v)+1 (the head is
// the relabelled end, R13).  Heights are frozen in this phase and each residual
// pair has one writer, so the slot stores need no atomics.
template <class G>
__device__ __forceinline__ void rie(const Dev &d, const G &g, Smem &sm, int32_t entry, const BL &nxt,
                                    unsigned long long *workc) {
  const int tr = ((uint32_t)entry & TRACK_BIT) ? 1 : 0;
  const uint32_t tag = tr ? TRACK_BIT : 0u;
  const int32_t u = (int32_t)((uint32_t)entry & ~TRACK_BIT);
  const Track k = make_track(d, tr);
  const int32_t beg = d.row[u], end = d.row[u + 1];
  const int32_t hu = ldv(k.hgt + u);
  long long moved = 0;
  unsigned long long sat = 0;
  for (int32_t i = beg + g.rank(); i < end; i += G::size) {
    const int32_t r = ldv(k.F + i);
    if (r > 0) {
      const int32_t v = d.dst[i];
      if (hu > ldv(k.hgt + v) + 1) {
        const int32_t ri = d.rev[i];
        k.F[i] = 0;
        k.R[ri] = 0;
        atomicAdd(k.F + ri, r);
        atomicAdd(k.R + i, r);
        const long long old = (long long)atomicAdd(reinterpret_cast<unsigned long long *>(d.e + v),
                                                   (unsigned long long)((long long)r * k.sign));
        const long long eo = old * k.sign;
        if (eo <= 0 && eo + r > 0) activate(d, k, nxt, v, tag, sm);
        moved += r;
        sat++;
      }
    }
  }
  moved = g.sum(moved);
  if (g.rank() == 0) {
    if (moved) atom_add(d.e + u, -moved * k.sign);
    atomicAdd(workc, (unsigned long long)(end - beg));
    sstat_add(sm, ST_RIE_SLOTS, (unsigned long long)(end - beg));
  }
  sstat_add(sm, ST_RIE_SAT, sat);
}

// ---------------------------------------------------------------------------
// Roots of a global relabel.
enum ResetKind : int { RK_PUSH = 0, RK_PP = 1, RK_STAGE2 = 2, RK_MINCUT = 3, RK_MAXCUT = 4 };

struct Lists {
  int32_t *q[2];    // frontier ping-pong, [3 bins][n] each
  int32_t *wl[2];   // worklist ping-pong, [3 bins][n] each
  int32_t *rl;      // relabelled, [3 bins][n]
};

// The device loop: repeat { RESET; BFS levels (+ worklist); if no active: stop;
//                           rounds of { DISCHARGE; RIE } until no vertex is queued }.
// Counter discipline (each counter is zeroed by block 0 in a phase where nobody
// else reads or appends it, then published by the next grid barrier):
//   qc[l%3]   appended at level l-1 (RESET for l=0), read at level l,
//             zeroed at level l+1 (as qc[(l+3-1)%3]); qc[1] zeroed in RESET,
//             qc[0] zeroed after the last round (or by the caller before the loop)
//   wlc[r&1]  read in DISCHARGE of round r, appended in round r-1, zeroed in RIE r
//   rlc[r&1]  appended in DISCHARGE r, read in RIE r; rlc[(r+1)&1] zeroed in RIE r
// Requires qc[0][*] == 0 and wlc[*] == 0 on entry.
__device__ void device_loop(const Dev &d, cg::grid_group &grid, Smem &sm, PhaseClock &clk, int kind,
                            const Lists &L, bool collect, bool stage2) {
  const int32_t n = d.n;
  Ctl *ctl = d.ctl;
  int32_t *qc = ctl->qc, *wlc = ctl->wlc, *rlc = ctl->rlc;
  const int32_t nt = gridDim.x * NT;
  const uint8_t reg0 = kind == RK_PP ? PART_T : (kind == RK_STAGE2 ? PART_P : 0);
  const uint8_t reg1 = kind == RK_PP ? PART_S : 0;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  for (int iter = 0;; ++iter) {
    // ---------------- RESET: heights of the domain, roots -> frontier level 0
    if (blockIdx.x == 0 && threadIdx.x < 6) {
      rlc[threadIdx.x] = 0;
      if (threadIdx.x < 3) qc[3 + threadIdx.x] = 0;
      if (threadIdx.x < 2) ctl->work[threadIdx.x] = 0;
    }
    {
      BL f0{L.q[0], qc, n};
      const int32_t N = kind == RK_STAGE2 ? ldv(&ctl->pcnt) : n;
      const int32_t wbase = blockIdx.x * NT + (threadIdx.x & ~31);
      for (int32_t b = wbase; b < N; b += nt) {
        const int32_t x = b + (threadIdx.x & 31);
        bool r0 = false, r1 = false;
        int32_t v = x;
        if (x < N) {
          if (kind == RK_STAGE2) v = d.plist[x];
          const long long ev = ldv(d.e + v);
          if (kind == RK_PUSH || kind == RK_MAXCUT) {
            r0 = v == d.t || (v != d.s && ev < 0);
            d.hp[v] = r0 ? 0 : n;
          } else if (kind == RK_PP) {
            const uint8_t p = ldv(d.part + v);
            r0 = p == PART_T && (v == d.t || (v != d.s && ev < 0));
            r1 = p == PART_S && (v == d.s || (v != d.t && ev > 0));
            d.hp[v] = r0 ? 0 : n;
            d.hm[v] = r1 ? 0 : n;
          } else if (kind == RK_STAGE2) {
            r0 = ev < 0;
            d.hp[v] = r0 ? 0 : n;
          } else {  // RK_MINCUT
            r1 = v == d.s || (v != d.t && ev > 0);
            d.hm[v] = r1 ? 0 : n;
          }
        }
        bl_append_conv(d, f0, r0, v, 0u);
        bl_append_conv(d, f0, r1, v, TRACK_BIT);
      }
      if (lead) sstat_add(sm, ST_RESET_V, (unsigned long long)N);
    }
    beacon(d, 10 + kind, iter, 0, 0);
    grid.sync();
    clk.lap(sm, ST_T_RESET);
    // ---------------- BFS levels (fused worklist compaction + termination test)
    int32_t lvl = 0;
    for (;; ++lvl) {
      int32_t *cur_c = qc + 3 * (lvl % 3);
      const int32_t c[3] = {ldv(cur_c), ldv(cur_c + 1), ldv(cur_c + 2)};
      beacon(d, 20 + kind, iter, 0, lvl, c[0] + c[1] + c[2], c[2]);
      if (c[0] + c[1] + c[2] == 0) break;
      if (blockIdx.x == 0 && threadIdx.x < 3) qc[3 * ((lvl + 2) % 3) + threadIdx.x] = 0;
      BfsCtx ctx{lvl, reg0, reg1, collect, BL{L.q[(lvl + 1) & 1], qc + 3 * ((lvl + 1) % 3), n}, BL{L.wl[0], wlc, n}};
      bfs_level(d, sm, BL{L.q[lvl & 1], cur_c, n}, c, ctx);
      grid.sync();
      clk.lap(sm, ST_T_BFS);
    }
    if (lead) sstat_add(sm, ST_LEVELS, (unsigned long long)lvl);
    {
      const int32_t w0 = ldv(wlc) + ldv(wlc + 1) + ldv(wlc + 2);
      if (w0 == 0) break;                         // no active vertex: converged (R9)
    }
    if (lead) {
      sstat_add(sm, ST_ITERS, 1);
      if (stage2) sstat_add(sm, ST_S2_ITERS, 1);
    }
    if (iter + 1 >= d.max_iters) {
      if (lead) ctl->status = -8;                // DMF_ENOCONV
      break;
    }
    // ---------------- rounds of DISCHARGE (push || pull tracks) + RIE
    unsigned long long spent = 0;                 // work since the global relabel (same in every thread)
    for (int r = 0;; ++r) {
      const int cur = r & 1, nx = cur ^ 1;
      const int32_t w[3] = {ldv(wlc + 3 * cur), ldv(wlc + 3 * cur + 1), ldv(wlc + 3 * cur + 2)};
      beacon(d, 30 + kind, iter, r, 0, w[0] + w[1] + w[2], w[2]);
      BL nxt{L.wl[nx], wlc + 3 * nx, n};
      BL rl{L.rl, rlc + 3 * cur, n};
      process_bl(BL{L.wl[cur], wlc + 3 * cur, n}, w, sm,
                 [&](auto &g, int32_t entry) { discharge(d, g, sm, entry, rl, nxt, ctl->work + cur); });
      grid.sync();
      clk.lap(sm, ST_T_DIS);
      if (blockIdx.x == 0 && threadIdx.x < 3) {
        wlc[3 * cur + threadIdx.x] = 0;
        rlc[3 * nx + threadIdx.x] = 0;
        qc[threadIdx.x] = 0;                      // for the next RESET
        if (threadIdx.x == 0) ctl->work[nx] = 0;  // read at the end of round r-1
      }
      {
        const int32_t rc[3] = {ldv(rlc + 3 * cur), ldv(rlc + 3 * cur + 1), ldv(rlc + 3 * cur + 2)};
        beacon(d, 40 + kind, iter, r, 0, rc[0] + rc[1] + rc[2], rc[2]);
        process_bl(rl, rc, sm, [&](auto &g, int32_t entry) { rie(d, g, sm, entry, nxt, ctl->work + cur); });
      }
      if (lead) sstat_add(sm, ST_ROUNDS, 1);
      grid.sync();
      clk.lap(sm, ST_T_RIE);
      const int32_t wn[3] = {ldv(wlc + 3 * nx), ldv(wlc + 3 * nx + 1), ldv(wlc + 3 * nx + 2)};
      spent += (unsigned long long)ldv(reinterpret_cast<const long long *>(ctl->work + cur));
      if (wn[0] + wn[1] + wn[2] == 0) break;
      if (r + 1 >= MAX_ROUNDS || (long long)spent > d.work_budget) {   // hand the rest to a global relabel
        if (lead) sstat_add(sm, ST_BUDGET_STOPS, 1);
        for (int b = 0; b < 3; b++) {
          const int32_t *lst = nxt.bin(b);
          for (int32_t x = blockIdx.x * NT + threadIdx.x; x < wn[b]; x += nt)
            d.inq[(uint32_t)lst[x] & ~TRACK_BIT] = 0;
        }
        grid.sync();                              // everyone has read wn before this
        clk.lap(sm, ST_T_DIS);
        if (blockIdx.x == 0 && threadIdx.x < 3) wlc[3 * nx + threadIdx.x] = 0;
        break;
      }
    }
  }
}

// Binary search of v in the sorted row of u; -1 if absent.
__device__ __forceinline__ int32_t find_slot(const Dev &d, int32_t u, int32_t v) {
  int32_t lo = d.row[u], hi = d.row[u + 1];
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    const int32_t x = d.dst[mid];
    if (x < v) lo = mid + 1; else hi = mid;
  }
  return (lo < d.row[u + 1] && d.dst[lo] == v) ? lo : -1;
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

template <int NTHREADS>
__global__ void __launch_bounds__(NTHREADS, MIN_BLOCKS) k_solve(Dev d, int32_t mode) {
  cg::grid_group grid = cg::this_grid();
  __shared__ Smem sm;
  for (int i = threadIdx.x; i < ST_N; i += NTHREADS) sm.stat[i] = 0;
  __syncthreads();
  const int32_t n = d.n;
  const int32_t gt = blockIdx.x * NTHREADS + threadIdx.x, nt = gridDim.x * NTHREADS;
  Ctl *ctl = d.ctl;
  const size_t n3 = 3 * (size_t)n;
  const Lists L{{d.q0, d.q1}, {d.wl, d.wl + n3}, d.rl};
  BlockG bg{sm.red};
  PhaseClock clk;
  clk.start();

  if (mode == MODE_STATIC) {
    // Alg.1 l.1-8: e = 0, c_f = c  (and the mirror)
    for (int64_t i = gt; i < d.S; i += nt) { const int32_t c = d.cap[i]; d.res[i] = c; d.rres[d.rev[i]] = c; }
    for (int32_t v = gt; v < n; v += nt) d.e[v] = 0;
    grid.sync();
  } else if (mode == MODE_PR || mode == MODE_PP) {
    // ---- Updates Processing (Alg.5), validated first (R11)
    for (int64_t j = gt; j < d.k; j += nt) {
      const int32_t u = d.bu[j], v = d.bv[j], c = d.bc[j];
      int32_t slot = -1;
      if (u < 0 || u >= n || v < 0 || v >= n) set_status(d, -1, (int32_t)j);
      else if (c < 0 || c > 1073741823) set_status(d, -7, (int32_t)j);
      else if ((slot = find_slot(d, u, v)) < 0) set_status(d, -2, (int32_t)j);
      else if (atomicExch(d.stamp + slot, d.batch_id) == d.batch_id) set_status(d, -3, (int32_t)j);
      d.bslot[j] = slot;
    }
    grid.sync();
    if (ldv(&ctl->status) != 0) mode = -1;       // all-or-nothing: state untouched
    for (int64_t j = gt; mode >= 0 && j < d.k; j += nt) {   // Alg.5 l.1-3: c_f += c' - c
      const int32_t i = d.bslot[j];
      const int32_t delta = d.bc[j] - d.cap[i];
      d.res[i] += delta;
      d.rres[d.rev[i]] += delta;
      d.cap[i] = d.bc[j];
    }
    if (mode >= 0) grid.sync();
    for (int64_t j = gt; mode >= 0 && j < d.k; j += nt) {   // Alg.5 l.4-11 on touched slots only (R10)
      const int32_t i = d.bslot[j];
      const int32_t r = ldv(d.res + i);
      if (r < 0) {
        const int32_t ri = d.rev[i];
        d.res[i] = 0;
        d.rres[ri] = 0;
        atomicAdd(d.res + ri, r);                 // c_f(v,u) += c_f(u,v)  (r < 0)
        atomicAdd(d.rres + i, r);
        atom_add(d.e + d.bu[j], -(long long)r);   // flow on (u,v) drops by -r: e(u) += -r
        atom_add(d.e + d.bv[j], (long long)r);    //                           e(v) -= -r
      }
    }
    if (mode >= 0) grid.sync();
    if (mode == MODE_PP) {                        // Alg.8 l.10-13 on touched slots (R12)
      for (int64_t j = gt; j < d.k; j += nt) {
        const int32_t i = d.bslot[j];
        const int32_t u = d.bu[j], v = d.bv[j];
        if (d.part[u] == PART_S && d.part[v] == PART_T) {
          const long long r = saturate_slot(d, i);
          if (r) atom_add(d.e + u, -r);
        }
      }
      grid.sync();
    }
  }
  if (mode == MODE_STATIC || mode == MODE_PR) {
    // Alg.1 l.9-13 / Alg.4 l.3-8 (R3): saturate every residual out-slot of s
    const int32_t beg = d.row[d.s], end = d.row[d.s + 1];
    long long tot = 0;
    for (int32_t i = beg + gt; i < end; i += nt) tot += saturate_slot(d, i);
    tot = bg.sum(tot);
    if (threadIdx.x == 0 && tot) atom_add(d.e + d.s, -tot);
    grid.sync();
    clk.lap(sm, ST_T_PRO);
    device_loop(d, grid, sm, clk, RK_PUSH, L, true, false);
    // part from the final fresh BFS (S = unreached = S_max, R15) + flow (R8)
    long long f = 0;
    for (int32_t v = gt; v < n; v += nt) {
      d.part[v] = ldv(d.hp + v) < n ? PART_T : PART_S;
      const long long ev = ldv(d.e + v);
      f += v == d.t ? ev : (v != d.s && ev < 0 ? ev : 0);
    }
    f = bg.sum(f);
    if (threadIdx.x == 0 && f) atomicAdd(reinterpret_cast<unsigned long long *>(&ctl->flow), (unsigned long long)f);
  } else if (mode == MODE_PP) {
    // ---- stage 1: push on T || pull on S (Alg.8 l.15-28)
    clk.lap(sm, ST_T_PRO);
    device_loop(d, grid, sm, clk, RK_PP, L, true, false);
    // ---- P = {h+ = |V| and h- = |V|} (Alg.8 l.29-33), vertices with slots only
    if (blockIdx.x == 0 && threadIdx.x < 3) ctl->qc[threadIdx.x] = 0;
    for (int32_t b = blockIdx.x * NTHREADS + (threadIdx.x & ~31); b < n; b += nt) {
      const int32_t v = b + (threadIdx.x & 31);
      bool inP = false;
      if (v < n) {
        inP = d.row[v + 1] > d.row[v] && ldv(d.hp + v) == n && ldv(d.hm + v) == n;
        if (inP) d.part[v] = PART_P;
      }
      warp_append(inP, v, d.plist, &ctl->pcnt);
    }
    grid.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) sstat_add(sm, ST_S2_V, (unsigned long long)ldv(&ctl->pcnt));
    // ---- stage 2: Dynamic Push-Relabel restricted to P (Alg.8 l.34)
    clk.lap(sm, ST_T_EPI);
    if (ldv(&ctl->pcnt) > 0) device_loop(d, grid, sm, clk, RK_STAGE2, L, true, true);
    // ---- relabel partitions (Alg.8 l.35-49) and F (= sum over T' of e, R8)
    const int32_t pc = ldv(&ctl->pcnt);
    for (int32_t x = gt; x < pc; x += nt) {
      const int32_t v = d.plist[x];
      d.part[v] = ldv(d.hp + v) < n ? PART_T : PART_S;
    }
    long long f = 0;
    for (int32_t v = gt; v < n; v += nt) {
      const long long ev = ldv(d.e + v);
      f += v == d.t ? ev : (v != d.s && ev < 0 ? ev : 0);
    }
    f = bg.sum(f);
    if (threadIdx.x == 0 && f) atomicAdd(reinterpret_cast<unsigned long long *>(&ctl->flow), (unsigned long long)f);
  } else if (mode == MODE_MINCUT || mode == MODE_MAXCUT) {
    device_loop(d, grid, sm, clk, mode == MODE_MINCUT ? RK_MINCUT : RK_MAXCUT, L, false, false);
    for (int32_t v = gt; v < n; v += nt)
      d.mask[v] = mode == MODE_MINCUT ? (ldv(d.hm + v) < n ? 1 : 0) : (ldv(d.hp + v) < n ? 0 : 1);
  }
  clk.lap(sm, ST_T_EPI);
  __syncthreads();
  for (int i = threadIdx.x; i < ST_N; i += NTHREADS)
    if (sm.stat[i]) atomicAdd(&ctl->stat[i], sm.stat[i]);
}

}  // namespace dmf
