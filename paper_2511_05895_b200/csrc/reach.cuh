// reach.cuh -- k_reach, the two pure-BFS jobs of the engine:
//  * k_reach<false>: the S_min query (dmf_min_cut_source_side, reading
//    R19): S_min is the set of vertices reachable from {s} u {v != t : e(v) > 0} in the
//    residual graph of the converged state (c_f(u,v) = res[slot (u,v)] > 0).  It
//    is the intersection of all minimum cuts' source sides, unique, and it does not
//    depend on which maximum (pre)flow the engine holds.
//  * k_reach<true>: the universal certificate of a DYN_PP warm start (reading R9, H8):
//    a fresh backward BFS from {t} u {v != s : e(v) < 0} on h+ must label no excess
//    vertex, and s must reach no labelled vertex; then the state is converged, the
//    partition is the labelled set (T', R15) and the epilogue writes it, F (R8) and the
//    label histogram of the next warm start.  Otherwise it writes nothing and the
//    MODE_PP_CONT launch of k_solve that follows runs the full Alg.8 stage 1.
//
// A lean level-synchronous, direction-optimising BFS in its OWN persistent cooperative
// kernel: 256 threads and <= 40 registers per thread, i.e. 48 resident warps per SM --
// 1.5x the warps k_solve can keep resident -- because a BFS level is a chain of
// dependent loads (row -> slot -> neighbour height) whose throughput is set by how
// many such chains are in flight.  It writes
//   * hm[v] = the exact BFS distance from the roots (|V| if unreached): the pull-track
//     labels a following DYN_PP warm start discharges on (as k_solve's MINCUT did),
//   * mask[v] = hm[v] < |V|,
//   * the level histogram of the warm start's local gap (R14 form 2) into cnt_next
//     (hm half = the level sizes; hp half copied from cnt: hp is unchanged here).
// Top-down levels claim by atomicCAS(hm, |V|, L+1) over frontier items, slot ranges of
// <= RCH slots (hub rows split, so that no warp serialises a level; no row lookup per
// item), or by idempotent stores and a sweep for the next frontier when the frontier is
// dense; bottom-up levels (frontier
// slots x RALPHA > slots still unvisited) let every unvisited vertex look for an
// in-neighbour at level L with residual towards it, thread-serial for short rows, a warp
// with early exit for longer ones.
#pragma once

#include "dmf_device.cuh"

namespace dmf {

constexpr int RNT = 256;                    // threads per CTA
#ifndef DMF_RMINB
#define DMF_RMINB 6
#endif
constexpr int RMINB = DMF_RMINB;            // resident CTAs per SM (6: <= 40 registers, 48 warps)
constexpr int RWPB = RNT / 32;
#ifndef DMF_RCH
#define DMF_RCH 256
#endif
#ifndef DMF_RALPHA
#define DMF_RALPHA 2
#endif
constexpr int32_t RCH = DMF_RCH;            // top-down: slots per frontier item
constexpr int32_t RBU_T = 24;               // bottom-up: rows of more slots go to the warp pass
constexpr unsigned long long RALPHA = DMF_RALPHA;   // bottom-up iff frontier slots x RALPHA > unvisited slots
constexpr unsigned long long RDENSE_DIV = 64;   // dense top-down iff frontier slots x RDENSE_DIV >= S

constexpr int32_t RSTG = 1024;              // frontier items staged per CTA (flushed once per phase)
constexpr int32_t RQSTG = 256;              // bottom-up warp-pass candidates staged per CTA

struct RSm {
  long long red[RWPB];
  unsigned long long tclk;
  long long it[RSTG];                       // staged frontier items
  int32_t q[RQSTG];                         // staged bottom-up warp-pass candidates
  int32_t icnt, qcnt, ibase, qbase;
  int32_t hist[2 * GAPW];                   // certificate epilogue: per-CTA label histogram
};

__device__ __forceinline__ long long r_bsum(RSm &sm, long long x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sm.red[threadIdx.x >> 5] = x;
  __syncthreads();
  long long r = 0;
#pragma unroll
  for (int i = 0; i < RWPB; i++) r += sm.red[i];
  return r;
}

// block 0 / thread 0: charge the time since the last lap to stat `which` (and write a
// phase trace record when tracing, same layout as k_solve's PhaseClock)
__device__ __forceinline__ void r_lap(const Dev &d, RSm &sm, int which, int32_t sub = 0, int32_t items = 0,
                                      int32_t extra = 0) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long now = gtimer();
    d.ctl->stat[which] += now - sm.tclk;
    if (d.trace && d.ctl->ntrace < d.trace_cap) {
      int32_t *rec = d.trace + 8 * d.ctl->ntrace++;
      rec[0] = which - ST_T_PRO; rec[1] = 0; rec[2] = sub; rec[3] = items; rec[4] = extra;
      rec[5] = (int32_t)(now - sm.tclk); rec[6] = 0; rec[7] = 0;
    }
    sm.tclk = now;
  }
}

// Certificate refuted during level L: the global flag decides after the final barrier;
// the early exit at the top of level L+1 reads the level's own slot rfl[(L+1) % 3],
// which no thread writes during level L+1 (a single flag read there would race with
// writers of level L+1: CTAs would leave the level loop at different levels and
// their grid barriers would no longer pair up).
__device__ __forceinline__ void r_refute(Ctl *ctl, int nx) {
  ctl->rfl[nx] = 1;
  ctl->rfail = 1;
}

// warp-convergent: lanes with pred append the row [rb, rb + deg) of a labelled vertex as
// ceil(deg / RCH) frontier items, each a slot range (end << 32 | begin): a top-down
// level then needs no row lookup per item.  Items are
// staged in shared memory (a returning global atomic per warp on ONE counter serialises
// every appending warp of the grid in one L2 slice); overflow goes to the global list
__device__ __forceinline__ void r_append(RSm &sm, long long *list, int32_t *cnt, bool pred, int32_t rb, int32_t deg) {
  const int32_t nit = pred ? (deg + RCH - 1) / RCH : 0;
  if (__ballot_sync(0xffffffffu, nit > 0) == 0) return;
  const int lane = threadIdx.x & 31;
  int32_t inc = nit;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  // positions base.. of the CTA's stage; those at >= RSTG go to a global range of the
  // overflow's size (so that the first RSTG stage positions are always all written)
  int32_t base = 0, gb = 0;
  if (lane == 31) {
    base = atomicAdd(&sm.icnt, inc);
    const int32_t over = base + inc - max(base, RSTG);
    if (over > 0) gb = atomicAdd(cnt, over) - max(base, RSTG);
  }
  base = __shfl_sync(0xffffffffu, base, 31) + inc - nit;
  gb = __shfl_sync(0xffffffffu, gb, 31);
  for (int32_t k = 0; k < nit; k++) {
    const int32_t b = rb + k * RCH;
    const long long e = ((long long)min(rb + deg, b + RCH) << 32) | (long long)(uint32_t)b;
    if (base + k < RSTG) sm.it[base + k] = e;
    else list[gb + base + k] = e;
  }
}
// warp-convergent: stage a bottom-up warp-pass candidate
__device__ __forceinline__ void r_queue(RSm &sm, int32_t *q, int32_t *qc, bool pred, int32_t v) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (m == 0) return;
  const int lane = threadIdx.x & 31, lead = __ffs(m) - 1;
  int32_t base = 0, gb = 0;
  if (lane == lead) {
    base = atomicAdd(&sm.qcnt, __popc(m));
    const int32_t over = base + __popc(m) - max(base, RQSTG);
    if (over > 0) gb = atomicAdd(qc, over) - max(base, RQSTG);
  }
  gb = __shfl_sync(0xffffffffu, gb, lead);
  base = __shfl_sync(0xffffffffu, base, lead) + __popc(m & ((1u << lane) - 1u));
  if (pred) { if (base < RQSTG) sm.q[base] = v; else q[gb + base] = v; }
}
// block-wide: move the staged items / candidates to the global lists (one atomic each)
__device__ __forceinline__ void r_flush(RSm &sm, long long *list, int32_t *cnt, int32_t *q, int32_t *qc) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const int32_t a = min(sm.icnt, RSTG), b = min(sm.qcnt, RQSTG);
    sm.icnt = a; sm.qcnt = b;
    sm.ibase = a ? atomicAdd(cnt, a) : 0;
    sm.qbase = b ? atomicAdd(qc, b) : 0;
  }
  __syncthreads();
  for (int32_t x = threadIdx.x; x < sm.icnt; x += RNT) list[sm.ibase + x] = sm.it[x];
  for (int32_t x = threadIdx.x; x < sm.qcnt; x += RNT) q[sm.qbase + x] = sm.q[x];
  __syncthreads();
  if (threadIdx.x == 0) { sm.icnt = 0; sm.qcnt = 0; }
  __syncthreads();
}

template <bool BACK>
__global__ void __launch_bounds__(RNT, RMINB) k_reach(const __grid_constant__ Dev d) {
  cg::grid_group grid = cg::this_grid();
  __shared__ RSm sm;
  Ctl *ctl = d.ctl;
  const int32_t n = d.n;
  const int lane = threadIdx.x & 31;
  const int32_t nt = gridDim.x * RNT;
  const int32_t gw = (int32_t)((threadIdx.x >> 5) * gridDim.x + blockIdx.x), nw = gridDim.x * RWPB;
  const bool want_hist = d.local_gap && d.cnt_next;
  // forward (S_min): labels h-, roots {s} u Exc, t never labelled, a top-down scan reads
  // c_f(u,v) = res of u's slot; backward (certificate): labels h+, roots {t} u Def, s never
  // labelled, the residual read is the mirror (c_f(v,u) of u's slot (u,v) = rres)
  int32_t *const H = BACK ? d.hp : d.hm;
  const int32_t *const RTD = BACK ? d.rres : d.res;    // top-down: frontier u's slot (u,v) -> v
  const int32_t *const RBU = BACK ? d.res : d.rres;    // bottom-up: v's slot (v,u), u in the frontier
  const int32_t xv = BACK ? d.s : d.t;                 // never labelled
  if (threadIdx.x == 0) { sm.tclk = gtimer(); sm.icnt = 0; sm.qcnt = 0; }
  __syncthreads();
  if (blockIdx.x == 0 && want_hist)
    for (int i = threadIdx.x; i < GAPW; i += RNT) { d.cnt_next[i] = BACK ? 0 : d.cnt[i]; d.cnt_next[GAPW + i] = 0; }

  // ---- roots: level 0 = {s} u {v != t : e(v) > 0}; everything else |V|
  {
    long long fdeg = 0, udeg = 0, nroot = 0;
    for (int32_t t0 = blockIdx.x * RNT * 4; t0 < n; t0 += nt * 4) {
      long long ev[4];
      int32_t rb[4], dg[4];
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int32_t v = t0 + j * RNT + threadIdx.x;
        ev[j] = v < n ? ldv(d.e + v) : 0;
        rb[j] = v < n ? d.row[v] : 0;
        dg[j] = v < n ? d.row[v + 1] - rb[j] : 0;
      }
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int32_t v = t0 + j * RNT + threadIdx.x;
        const bool root = v < n && (BACK ? (v == d.t || (v != d.s && ev[j] < 0)) : (v == d.s || (v != d.t && ev[j] > 0)));
        if (v < n) H[v] = root ? 0 : n;
        if (root) { fdeg += dg[j]; nroot++; }
        else if (v < n && v != xv) udeg += dg[j];
        r_append(sm, d.cq0, &ctl->rcnt[0], root, rb[j], dg[j]);
      }
    }
    r_flush(sm, d.cq0, &ctl->rcnt[0], d.bul, &ctl->rbq[0]);
    fdeg = r_bsum(sm, fdeg); udeg = r_bsum(sm, udeg); nroot = r_bsum(sm, nroot);
    if (threadIdx.x == 0) {
      if (fdeg) atomicAdd(&ctl->rfs[0], (unsigned long long)fdeg);
      if (udeg) atomicAdd(&ctl->rmu, (unsigned long long)udeg);
      if (nroot) atomicAdd(&ctl->rnv[0], (int32_t)nroot);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) d.ctl->stat[ST_RESET_V] += (unsigned long long)n;
  }
  grid.sync();
  r_lap(d, sm, ST_T_RESET, 0, n);

  unsigned long long mu = ldv(reinterpret_cast<const long long *>(&ctl->rmu));
  // The item list of level L exists only if level L-1 was a sparse top-down level (its
  // claims append) or L = 0; after a dense or bottom-up level it is built by a sweep
  // only if level L goes top-down (usually the level after those goes bottom-up).
  bool built = true;
  for (int32_t L = 0;; ++L) {
    const int cur = L % 3, nx = (L + 1) % 3, nn = (L + 2) % 3;
    const int32_t nv = ldv(&ctl->rnv[cur]);
    if (nv == 0) break;                            // nothing labelled at level L: done
    if (BACK && ldv(&ctl->rfl[cur])) break;        // certificate refuted at level L-1: stop here
    int32_t cnt = ldv(&ctl->rcnt[cur]);
    const unsigned long long f = (unsigned long long)ldv(reinterpret_cast<const long long *>(&ctl->rfs[cur]));
    if (L > 0) mu = mu > f ? mu - f : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {    // slot nn was last read in level L-1
      ctl->rcnt[nn] = 0; ctl->rfs[nn] = 0; ctl->rnv[nn] = 0; ctl->rbq[nn] = 0; ctl->rfl[nn] = 0;
      if (!BACK && want_hist && L < GAPW) d.cnt_next[GAPW + L] = nv;
      ctl->stat[ST_LEVELS] += 1;
      ctl->stat[ST_BFS_V] += (unsigned long long)nv;
    }
    long long *cl = (L & 1) ? d.cq1 : d.cq0;
    long long *nl = (L & 1) ? d.cq0 : d.cq1;
    long long fdeg = 0, nlab = 0, slots = 0;      // (slots: scanned, for the stats)
    const bool bu = f * RALPHA > mu;
    if (!bu && !built) {                           // the level's items: {v : hm[v] = L}
      for (int32_t t0 = blockIdx.x * RNT * 4; t0 < n; t0 += nt * 4) {
        int32_t h[4], rb[4], dg[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int32_t v = t0 + j * RNT + threadIdx.x;
          h[j] = v < n ? ldv(H + v) : n;
        }
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int32_t v = t0 + j * RNT + threadIdx.x;
          rb[j] = h[j] == L ? d.row[v] : 0;
          dg[j] = h[j] == L ? d.row[v + 1] - rb[j] : 0;
        }
#pragma unroll
        for (int j = 0; j < 4; j++) r_append(sm, cl, &ctl->rcnt[cur], h[j] == L, rb[j], dg[j]);
      }
      r_flush(sm, cl, &ctl->rcnt[cur], d.bul, &ctl->rbq[cur]);
      grid.sync();
      cnt = ldv(&ctl->rcnt[cur]);
    }
    // dense top-down: a frontier of >= S / RDENSE_DIV slots discovers most vertices many
    // times over -- label by idempotent stores, then build the next frontier by a sweep
    const bool dense = !bu && f * RDENSE_DIV >= (unsigned long long)d.S;
    if (!bu) {
      // ---- top-down: warp per frontier item, 4 slots per lane per step
      if (dense) {
        // labels by stores only: a whole item (<= 256 slots, 8 per lane) per step, every
        // load of the step in flight together
        long long itn = gw < cnt ? cl[gw] : 0;
        for (int32_t x = gw; x < cnt; x += nw) {
          const long long it = itn;
          itn = x + nw < cnt ? cl[x + nw] : 0;
          const int32_t beg = (int32_t)(uint32_t)it, end = (int32_t)(it >> 32);
          if (lane == 0) slots += end - beg;
          for (int32_t b = beg; b < end; b += 256) {
            int32_t r[8], w[8];
#pragma unroll
            for (int j = 0; j < 8; j++) {
              const int32_t i = b + j * 32 + lane;
              r[j] = i < end ? ldv(RTD + i) : 0;
              w[j] = i < end ? d.dst[i] : 0;
            }
#pragma unroll
            for (int j = 0; j < 8; j++) r[j] = r[j] > 0 && w[j] != xv && ldl1(H + w[j]) == n;
#pragma unroll
            for (int j = 0; j < 8; j++) if (r[j]) H[w[j]] = L + 1;
          }
        }
      }
      long long itn = !dense && gw < cnt ? cl[gw] : 0;     // next item, loaded one item ahead
      for (int32_t x = dense ? cnt : gw; x < cnt; x += nw) {
        const long long it = itn;
        itn = x + nw < cnt ? cl[x + nw] : 0;
        const int32_t beg = (int32_t)(uint32_t)it, end = (int32_t)(it >> 32);
        if (lane == 0) slots += end - beg;
        for (int32_t b = beg; b < end; b += 128) {
          int32_t r[4], w[4];
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const int32_t i = b + j * 32 + lane;
            r[j] = i < end ? ldv(RTD + i) : 0;
            w[j] = i < end ? d.dst[i] : 0;
          }
#pragma unroll
          for (int j = 0; j < 4; j++)          // stale |V| is harmless: the CAS decides
            r[j] = (r[j] > 0 && w[j] != xv && ldl1(H + w[j]) == n) ? 1 : 0;
#pragma unroll
          for (int j = 0; j < 4; j++) r[j] = r[j] && atomicCAS(H + w[j], n, L + 1) == n;
          int32_t rb[4], dg[4];
#pragma unroll
          for (int j = 0; j < 4; j++) {
            rb[j] = r[j] ? d.row[w[j]] : 0;
            dg[j] = r[j] ? d.row[w[j] + 1] - rb[j] : 0;
            if (BACK && r[j] && ldv(d.e + w[j]) > 0) r_refute(ctl, nx);   // an excess vertex reaches a sink
          }
#pragma unroll
          for (int j = 0; j < 4; j++) {
            if (r[j]) { fdeg += dg[j]; nlab++; }
            r_append(sm, nl, &ctl->rcnt[nx], r[j] != 0, rb[j], dg[j]);
          }
        }
      }
      if (dense) {
        grid.sync();
        r_lap(d, sm, ST_T_BFS, L, nv, 4 | (cnt << 3));
        // ---- size of the next frontier {v : hm[v] = L+1} (its items: built if needed)
        for (int32_t t0 = blockIdx.x * RNT * 4; t0 < n; t0 += nt * 4) {
          int32_t h[4], rb[4], dg[4];
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const int32_t v = t0 + j * RNT + threadIdx.x;
            h[j] = v < n ? ldv(H + v) : n;
          }
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const int32_t v = t0 + j * RNT + threadIdx.x;
            rb[j] = h[j] == L + 1 ? d.row[v] : 0;
            dg[j] = h[j] == L + 1 ? d.row[v + 1] - rb[j] : 0;
            if (BACK && h[j] == L + 1 && ldv(d.e + v) > 0) r_refute(ctl, nx);
          }
#pragma unroll
          for (int j = 0; j < 4; j++)
            if (h[j] == L + 1) { fdeg += dg[j]; nlab++; }
        }
      }
    } else {
      if (blockIdx.x == 0 && threadIdx.x == 0) ctl->stat[ST_BU_LEVELS] += 1;
      // ---- bottom-up pass A: thread per unvisited vertex with a short row
      // (the next vertex's label and row bounds are loaded one iteration ahead)
      int32_t v = blockIdx.x * RNT + threadIdx.x;
      int32_t hN = v < n ? ldv(H + v) : 0, rbN = v < n ? d.row[v] : 0, reN = v < n ? d.row[v + 1] : 0;
      for (; v - (int32_t)threadIdx.x < n; v += nt) {
        const bool in = v < n;
        const int32_t h = hN, rb = rbN, re = reN;
        {
          const int32_t vn = v + nt;
          hN = vn < n ? ldv(H + vn) : 0;
          rbN = vn < n ? d.row[vn] : 0;
          reN = vn < n ? d.row[vn + 1] : 0;
        }
        const bool cand = in && h == n && v != xv;
        const bool big = cand && re - rb > RBU_T;
        bool found = false;
        if (cand && !big) {
          for (int32_t i0 = rb; i0 < re && !found; i0 += 4) {
            slots += min(4, re - i0);
            int32_t r[4], w[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {      // in-slot (v,u): rres = c_f(u,v)
              r[j] = i0 + j < re ? ldv(RBU + i0 + j) : 0;
              w[j] = i0 + j < re ? d.dst[i0 + j] : 0;
            }
#pragma unroll
            for (int j = 0; j < 4; j++) found |= r[j] > 0 && ldl1(H + w[j]) == L;   // level-L labels are frozen
          }
          if (found) {
            H[v] = L + 1; fdeg += re - rb; nlab++;
            if (BACK && ldv(d.e + v) > 0) r_refute(ctl, nx);
          }
        }
        r_queue(sm, d.bul, &ctl->rbq[cur], big, v);
      }
      r_flush(sm, nl, &ctl->rcnt[nx], d.bul, &ctl->rbq[cur]);
      grid.sync();
      // ---- pass B: warp per queued vertex, early exit on the first in-neighbour at L
      const int32_t q = ldv(&ctl->rbq[cur]);
      for (int32_t x = gw; x < q; x += nw) {
        const int32_t v = d.bul[x];
        const int32_t rb = d.row[v], re = d.row[v + 1];
        bool found = false;
        for (int32_t b = rb; b < re; b += 128) {
          if (lane == 0) slots += min(128, re - b);
          int32_t r[4], w[4];
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const int32_t i = b + j * 32 + lane;
            r[j] = i < re ? ldv(RBU + i) : 0;
            w[j] = i < re ? d.dst[i] : 0;
          }
          bool hit = false;
#pragma unroll
          for (int j = 0; j < 4; j++) hit |= r[j] > 0 && ldl1(H + w[j]) == L;
          if (__any_sync(0xffffffffu, hit)) { found = true; break; }
        }
        if (found && lane == 0) {
          H[v] = L + 1; fdeg += re - rb; nlab++;
          if (BACK && ldv(d.e + v) > 0) r_refute(ctl, nx);
        }
      }
    }
    r_flush(sm, nl, &ctl->rcnt[nx], d.bul, &ctl->rbq[cur]);
    built = !bu && !dense;
    fdeg = r_bsum(sm, fdeg); nlab = r_bsum(sm, nlab); slots = r_bsum(sm, slots);
    if (threadIdx.x == 0) {
      if (slots) atomicAdd(&ctl->stat[ST_BFS_SLOTS], (unsigned long long)slots);
      if (fdeg) atomicAdd(&ctl->rfs[nx], (unsigned long long)fdeg);
      if (nlab) atomicAdd(&ctl->rnv[nx], (int32_t)nlab);
    }
    grid.sync();
    r_lap(d, sm, dense ? ST_T_BFS_CMP : ST_T_BFS, L, nv, (bu ? 2 : 0) | (dense ? 4 : 0) | (cnt << 3));
  }

  if (BACK) {
    // ---- the certificate (R9): no excess vertex was labelled (checked at labelling) and
    //      s reaches no labelled vertex (DYN_PP does not re-saturate s, R16)
    const int32_t sb = d.row[d.s], se = d.row[d.s + 1];
    bool hit = false;
    for (int32_t i = sb + blockIdx.x * RNT + (int32_t)threadIdx.x; i < se; i += nt)
      hit |= ldv(d.res + i) > 0 && ldv(d.hp + d.dst[i]) < n;
    if (hit) ctl->rfail = 1;
    grid.sync();
    if (ldv(&ctl->rfail)) { r_lap(d, sm, ST_T_EPI); return; }   // MODE_PP_CONT takes over
    // ---- converged: partition = the certificate's reach (T' = labelled, R15), region
    //      encoding of the next warm start, F (R8), the final labels' histogram
    long long f = 0;
    if (want_hist) {
      for (int i = threadIdx.x; i < 2 * GAPW; i += RNT) sm.hist[i] = 0;
      __syncthreads();
    }
    for (int32_t t0 = blockIdx.x * RNT * 2; t0 < n; t0 += nt * 2) {
      long long ev[2];
      int32_t hp[2], hm[2];
#pragma unroll
      for (int j = 0; j < 2; j++) {
        const int32_t v = t0 + j * RNT + threadIdx.x;
        ev[j] = v < n ? ldv(d.e + v) : 0;
        hp[j] = v < n ? ldv(d.hp + v) : n;
        hm[j] = v < n ? ldv(d.hm + v) : n;
      }
#pragma unroll
      for (int j = 0; j < 2; j++) {
        const int32_t v = t0 + j * RNT + threadIdx.x;
        const bool ok = v < n;
        int32_t hmv = hm[j];
        if (ok) {
          f += v == d.t ? ev[j] : (v != d.s && ev[j] < 0 ? ev[j] : 0);
          const bool tside = hp[j] < n;
          d.part[v] = tside ? PART_T : PART_S;
          if (tside) { d.hm[v] = n + 1; hmv = n + 1; }
          else {
            d.hp[v] = n + 1;
            if (hmv > n) { d.hm[v] = n; hmv = n; }
          }
        }
        if (want_hist) {
          hist_add(sm.hist, ok && hp[j] < n && hp[j] < GAPW, hp[j]);
          hist_add(sm.hist + GAPW, ok && hmv < n && hmv < GAPW, hmv);
        }
      }
    }
    if (want_hist) {                               // one global add per non-zero bin per CTA
      __syncthreads();
      for (int i = threadIdx.x; i < 2 * GAPW; i += RNT)
        if (sm.hist[i]) atomicAdd(d.cnt_next + i, sm.hist[i]);
    }
    f = r_bsum(sm, f);
    if (threadIdx.x == 0 && f) atomicAdd(reinterpret_cast<unsigned long long *>(&ctl->flow), (unsigned long long)f);
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->lazy_ok = 1;
  } else {
    // ---- the S_min mask
    for (int32_t t0 = blockIdx.x * RNT * 4; t0 < n; t0 += nt * 4) {
      int32_t h[4];
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int32_t v = t0 + j * RNT + threadIdx.x;
        h[j] = v < n ? ldv(d.hm + v) : n;
      }
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int32_t v = t0 + j * RNT + threadIdx.x;
        if (v < n) d.mask[v] = h[j] < n ? 1 : 0;
      }
    }
  }
  r_lap(d, sm, ST_T_EPI);
}

}  // namespace dmf
