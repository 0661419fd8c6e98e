// dmf.cu -- libdmf.so: C ABI (include/dmf.h) + the one-time Bi-CSR builder.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared
//        -Xcompiler -fPIC -I include -o paper_2511_05895_b200/libdmf.so dmf.cu
//
// Every step of the hot path runs in kernels of this file / solve.cuh.  CUB is used
// only by dmf_create (the one-time Bi-CSR build: sort + run-length merge), never
// on the per-batch path.
#include "dmf.h"
#include "dmf_device.cuh"
#include "solve.cuh"
#include "reach.cuh"

#include <cub/cub.cuh>

#include <chrono>
#include <cstdlib>
#include <thread>
#include <unistd.h>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

using namespace dmf;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CK(call)                                                                             \
  do {                                                                                       \
    cudaError_t err__ = (call);                                                              \
    if (err__ != cudaSuccess) return fail(DMF_ECUDA, "%s: %s (%s:%d)", #call,                \
                                          cudaGetErrorString(err__), __FILE__, __LINE__);    \
  } while (0)

bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

struct dmf_graph {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  dmf_options opt{};
  int32_t n = 0, s = 0, t = 0, kc = 1;
  int64_t S = 0, m = 0;
  int32_t *row = nullptr, *dst = nullptr, *rev = nullptr, *cap = nullptr, *res = nullptr, *rres = nullptr;
  int32_t *hp = nullptr, *hm = nullptr, *q0 = nullptr, *q1 = nullptr, *wl = nullptr, *rl = nullptr;
  int32_t *plist = nullptr, *stamp = nullptr, *inq = nullptr, *bul = nullptr;
  long long *cq0 = nullptr, *cq1 = nullptr, *cqr = nullptr, *cw0 = nullptr, *cw1 = nullptr;
  int32_t *dcnt = nullptr, *dmin = nullptr, *arc = nullptr;
  bool probes = true;        // DMF_PROBE=0: big vertices always enqueue all their chunks
  long long *aq = nullptr;
  int32_t aq_mask = 0;
  // engine knobs, resolved from dmf_options (+ DMF_* environment overrides) in dmf_create
  bool async = true;         // repairs (DYN_PR / DYN_PP): asynchronous discharge (else rounds)
  bool async_static = false; // static solve from zero flow: rounds (massively parallel work)
  int32_t async_warps = 8;
  int32_t bu_alpha = (int32_t)BU_ALPHA, dense_div = (int32_t)DENSE_DIV;
  int32_t async_sleep_ns = 128;
  int32_t tail_items = 2048;
  int32_t local_gap = 1;
  int32_t topo_div = 0;
  int32_t check_level = 0;
  int32_t lazy = 1;          // DYN_PP warm start certified by the universal backward BFS
  int32_t dmaxch = 0;
  int32_t scan2 = 1;         // DMF_SCAN2=0: chunk discharge claims and pushes per 128-slot step
  int32_t imm_act = 1;       // DMF_IMM_ACT=0: stage pushed heads and check them after the item        // DMF_DMAXCH: chunk items per big-vertex discharge activation (0: CH slots each)
  long long budget_mul = 1;
  int32_t *cnt = nullptr, *cnt_next = nullptr;   // local-gap level counts (this call / next warm call)
  int32_t *chk = nullptr;                          // invariant check scratch (64 bytes)
  long long *e = nullptr;
  uint8_t *part = nullptr, *mask = nullptr, *rlf = nullptr;
  int32_t *bbuf = nullptr;   // batch staging: u, v, c, slot, 3 undo records  (7 * bcap)
  int4 *htab = nullptr;      // (u,v) -> slot table
  int32_t hmask = 0;
  int64_t bcap = 0;
  Ctl *ctl = nullptr;
  Ctl *hctl = nullptr;       // pinned mirror
  int32_t *hdbg = nullptr;   // mapped pinned beacon (host view)
  int32_t *trace = nullptr;  // device trace ring (DMF_TRACE / dmf_set_trace)
  uint32_t *trace_cta = nullptr;  // per-record per-CTA busy times (dmf_set_trace)
  int32_t trace_cap = 0;
  int32_t *ddbg = nullptr;   // device view
  int grid_blocks = 0;
  int reach_blocks = 0;      // cooperative grid of k_reach (S_min query)
  int32_t cert_skip = 0;     // DYN_PP calls left that skip the certificate (after a failed one)
  int32_t cert_backoff = 0;  // current back-off length: 0, 1, 3, 7, 15, 16
  bool reach = true;         // DMF_REACH=0: the S_min query runs k_solve's MINCUT mode and the DYN_PP
                             // certificate runs inside k_solve instead of k_reach
  double watchdog_s = 0;
  int32_t batch_id = 0;
  bool solved = false;
  bool smin_valid = false;   // g->mask holds S_min of the current state
  bool warm = false;         // hp/hm/part hold the final labels of the last DYN_PP repair
  bool no_warm = false;      // options.warm < 0: always run stage 1's initial global relabel
  int64_t launches = 0;      // kernels launched by solve / apply / cut calls since create
  int64_t flow = 0;
  dmf_stats stats{};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<std::pair<void *, size_t>> allocs;

  void *alloc(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes == 0) bytes = 256;
    void *p = nullptr;
    if (opt.alloc) p = opt.alloc(bytes, opt.alloc_ctx);
    else if (cudaMalloc(&p, bytes) != cudaSuccess) { cudaGetLastError(); p = nullptr; }
    if (p) allocs.emplace_back(p, bytes);
    return p;
  }
  void release(void *p) {
    for (size_t i = 0; i < allocs.size(); i++)
      if (allocs[i].first == p) {
        if (opt.free) opt.free(p, allocs[i].second, opt.alloc_ctx); else cudaFree(p);
        allocs.erase(allocs.begin() + (long)i);
        return;
      }
  }
  void release_all() {
    for (auto &a : allocs) { if (opt.free) opt.free(a.first, a.second, opt.alloc_ctx); else cudaFree(a.first); }
    allocs.clear();
  }
};

// ============================================================================ build kernels
namespace {

__global__ void k_expand_edges(int32_t n, int64_t m, const int64_t *rp, const int32_t *col, const int32_t *cap,
                               unsigned long long *key, int32_t *val, int32_t *err) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
    int32_t lo = 0, hi = n;             // u = last row with rp[u] <= j
    while (lo < hi) {
      const int32_t mid = (lo + hi + 1) >> 1;
      if (rp[mid] <= j) lo = mid; else hi = mid - 1;
    }
    const int32_t u = lo, v = col[j], c = cap[j];
    if (v < 0 || v >= n || v == u) { atomicCAS(err, 0, DMF_EINVAL); continue; }
    if (c < 0) { atomicCAS(err, 0, DMF_EINVAL); continue; }
    if (c > DMF_CAP_MAX) { atomicCAS(err, 0, DMF_EOVERFLOW); continue; }
    key[2 * j] = (unsigned long long)u * (unsigned long long)n + (unsigned long long)v;
    val[2 * j] = c;
    key[2 * j + 1] = (unsigned long long)v * (unsigned long long)n + (unsigned long long)u;
    val[2 * j + 1] = -1;                // materialised reverse (zero capacity)
  }
}

__global__ void k_run_heads(int64_t N, const unsigned long long *key, int32_t *head) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < N; p += (int64_t)gridDim.x * blockDim.x)
    head[p] = (p == 0 || key[p] != key[p - 1]) ? 1 : 0;
}

// scan[p] = inclusive count of run heads -> slot = scan[p] - 1
__global__ void k_merge_runs(int64_t N, const unsigned long long *key, const int32_t *val, const int32_t *scan,
                             unsigned long long *ukey, long long *capsum, int32_t *isinput) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < N; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t slot = scan[p] - 1;
    if (p == 0 || key[p] != key[p - 1]) ukey[slot] = key[p];
    if (val[p] >= 0) {
      atomicAdd(reinterpret_cast<unsigned long long *>(capsum + slot), (unsigned long long)val[p]);
      isinput[slot] = 1;
    }
  }
}

__device__ int64_t lower_bound_u64(const unsigned long long *a, int64_t N, unsigned long long x) {
  int64_t lo = 0, hi = N;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_rows(int32_t n, int64_t S, const unsigned long long *ukey, int32_t *row) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u <= n; u += (int64_t)gridDim.x * blockDim.x)
    row[u] = (int32_t)(u == n ? S : lower_bound_u64(ukey, S, (unsigned long long)u * (unsigned long long)n));
}

__global__ void k_slots(int32_t n, int64_t S, const unsigned long long *ukey, const long long *capsum,
                        int32_t *dst, int32_t *rev, int32_t *cap, int32_t *err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = ukey[i];
    const unsigned long long u = k / (unsigned long long)n, v = k % (unsigned long long)n;
    dst[i] = (int32_t)v;
    rev[i] = (int32_t)lower_bound_u64(ukey, S, v * (unsigned long long)n + u);
    const long long c = capsum[i];
    if (c > DMF_CAP_MAX) atomicCAS(err, 0, DMF_EOVERFLOW);
    cap[i] = (int32_t)(c > DMF_CAP_MAX ? DMF_CAP_MAX : c);
  }
}

// (u,v) -> slot table for O(1) batch lookups (linear probing; 16-byte entry
// {u, v, slot, rev[slot]}: one probe gives both slots of the pair, no row lookup).
// The key half is claimed by a 64-bit CAS, the value half stored after it (the table
// is read only by later launches).
__global__ void k_hash_insert(int64_t S, int32_t n, const unsigned long long *ukey, const int32_t *rev, int4 *htab,
                              uint32_t hmask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = ukey[i];
    const int32_t u = (int32_t)(k / (unsigned long long)n), v = (int32_t)(k % (unsigned long long)n);
    const unsigned long long key = ((unsigned long long)(uint32_t)v << 32) | (uint32_t)u;   // {x = u, y = v}
    for (uint32_t h = slot_hash(u, v) & hmask;; h = (h + 1) & hmask)
      if (atomicCAS(reinterpret_cast<unsigned long long *>(htab + h), ~0ull, key) == ~0ull) {
        reinterpret_cast<int2 *>(htab + h)[1] = make_int2((int32_t)i, rev[i]);
        break;
      }
  }
}

__global__ void k_init_state(int64_t S, int32_t n, const int32_t *rev, const int32_t *cap, int32_t *res,
                             int32_t *rres, int32_t *stamp, long long *e, uint8_t *part, int32_t *hp, int32_t *hm) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S; i += st) {
    res[i] = cap[i];
    rres[i] = cap[rev[i]];
    stamp[i] = 0;
  }
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += st) {
    e[v] = 0; part[v] = PART_NONE; hp[v] = n; hm[v] = n;
  }
}

__global__ void k_sum_i32(int64_t N, const int32_t *a, unsigned long long *out) {
  unsigned long long s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) s += a[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// Invariant check (check_level 1, dmf_check_state, dmf_import_state): writes the first
// violated check code and a witness index to out[0..1].
//   1: 0 <= res[i] <= cap[i] + cap[rev[i]]        (capacity)
//   2: res[i] + res[rev[i]] == cap[i] + cap[rev[i]] (pair sum)
//   3: rres[i] == res[rev[i]]                    (mirror; skipped when rres is NULL)
//   4: e(v) == sum over the slots j of v of (res[j] - cap[j])   (net inflow)
// and accumulates sum(e) into *esum (check 5 on the host: sum of e == 0).
__device__ void chk_report(int32_t *out, int32_t code, long long at) {
  if (atomicCAS(out, 0, code) == 0) out[1] = (int32_t)at;
}
__global__ void k_check(int32_t n, int64_t S, const int32_t *row, const int32_t *rev, const int32_t *cap,
                        const int32_t *res, const int32_t *rres, const long long *e, int32_t *out,
                        unsigned long long *esum) {
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = gt; i < S; i += nt) {
    const int32_t ri = rev[i];
    const long long c = (long long)cap[i] + cap[ri], r = res[i];
    if (r < 0 || r > c) chk_report(out, 1, i);
    if (r + res[ri] != c) chk_report(out, 2, i);
    if (rres && rres[i] != res[ri]) chk_report(out, 3, i);
  }
  const int lane = threadIdx.x & 31;
  for (int64_t v = gt >> 5; v < n; v += nt >> 5) {      // warp per vertex
    long long sum = 0;
    for (int32_t j = row[v] + lane; j < row[v + 1]; j += 32) sum += (long long)res[j] - cap[j];
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) {
      if (sum != e[v]) chk_report(out, 4, v);
      atomicAdd(esum, (unsigned long long)e[v]);
    }
  }
}

__global__ void k_mirror(int64_t S, const int32_t *rev, const int32_t *res, int32_t *rres) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S; i += (int64_t)gridDim.x * blockDim.x)
    rres[i] = res[rev[i]];
}

int bits_for(unsigned long long x) {
  int b = 1;
  while (b < 64 && (x >> b)) b++;
  return b;
}

}  // namespace

// ============================================================================ helpers

static Dev make_dev(dmf_graph *g) {
  Dev d{};
  d.n = g->n; d.s = g->s; d.t = g->t; d.kc = g->kc;
  d.max_iters = g->opt.max_iters > 0 ? g->opt.max_iters : (int32_t)(4LL * g->n + 64 > 0x3fffffff ? 0x3fffffff : 4LL * g->n + 64);
  d.batch_id = g->batch_id;
  d.warm = g->warm ? 1 : 0;
  // ~ the cost of one whole-graph global relabel, times budget_mul (or divided by -budget_mul)
  d.work_budget = g->budget_mul > 0 ? (g->S + 6LL * g->n) * g->budget_mul : (g->S + 6LL * g->n) / -g->budget_mul;
  d.S = g->S; d.k = 0;
  d.row = g->row; d.dst = g->dst; d.rev = g->rev; d.cap = g->cap; d.res = g->res; d.rres = g->rres;
  d.e = g->e; d.hp = g->hp; d.hm = g->hm; d.part = g->part;
  d.q0 = g->q0; d.q1 = g->q1;
  d.wl = g->wl; d.rl = g->rl; d.inq = g->inq; d.bul = g->bul; d.rlf = g->rlf;
  d.cq0 = g->cq0; d.cq1 = g->cq1; d.cqr = g->cqr; d.cw0 = g->cw0; d.cw1 = g->cw1;
  d.dcnt = g->dcnt; d.dmin = g->dmin; d.arc = g->probes ? g->arc : nullptr;
  d.aq = g->aq; d.aq_mask = g->aq_mask; d.async = g->async ? 1 : 0;
  d.async_warps = g->async_warps;
  d.bu_alpha = g->bu_alpha; d.dense_div = g->dense_div;
  d.async_sleep_ns = g->async_sleep_ns;
  d.cnt = g->cnt; d.cnt_next = g->cnt_next;
  d.local_gap = g->local_gap; d.topo_div = g->topo_div; d.tail_items = g->tail_items;
  d.check_level = g->check_level;
  d.lazy = g->lazy;
  d.dmaxch = g->dmaxch;
  d.imm_act = g->imm_act;
  d.scan2 = g->scan2;
  d.plist = g->plist; d.stamp = g->stamp;
  d.htab = g->htab; d.hmask = g->hmask;
  d.mask = g->mask; d.ctl = g->ctl;
  d.dbg = g->ddbg;
  d.trace = g->trace;
  d.trace_cta = g->trace_cta;
  d.trace_cap = g->trace_cap;
  return d;
}

static const char *check_name(int32_t code) {
  switch (code) {
    case 1: return "capacity: res outside [0, cap + cap_rev] at slot";
    case 2: return "pair sum: res + res_rev != cap + cap_rev at slot";
    case 3: return "mirror: rres != res[rev] at slot";
    case 4: return "excess: e(v) != net inflow at vertex";
    case 5: return "excess: sum of e != 0";
    default: return "invariant";
  }
}

// Device invariant check of (cap, res, rres, e); DMF_OK or DMF_ECHECK.
static int check_arrays(dmf_graph *g, const int32_t *cap, const int32_t *res, const int32_t *rres, const long long *e) {
  CK(cudaMemsetAsync(g->chk, 0, 64, g->stream));
  const int blocks = g->grid_blocks > 0 ? g->grid_blocks : 296;
  k_check<<<blocks, 512, 0, g->stream>>>(g->n, g->S, g->row, g->rev, cap, res, rres, e, g->chk,
                                          reinterpret_cast<unsigned long long *>(g->chk + 8));
  CK(cudaGetLastError());
  int32_t h[16];
  CK(cudaMemcpyAsync(h, g->chk, 64, cudaMemcpyDeviceToHost, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  long long esum = 0;
  memcpy(&esum, h + 8, 8);
  if (h[0]) return fail(DMF_ECHECK, "%s %d", check_name(h[0]), h[1]);
  if (esum != 0) return fail(DMF_ECHECK, "%s (%lld)", check_name(5), esum);
  return DMF_OK;
}
static int check_state(dmf_graph *g) { return check_arrays(g, g->cap, g->res, g->rres, g->e); }

static int run_solve(dmf_graph *g, int32_t mode, const Dev &dv) {
  Dev d = dv;
  const bool smin_before = g->smin_valid;
  if (mode != MODE_MINCUT) g->smin_valid = false;  // the state (or the mask buffer) is about to change
  const bool warm_before = g->warm;
  g->warm = false;                                  // every launch rewrites hp or hm
  CK(cudaMemsetAsync(g->ctl, 0, sizeof(Ctl), g->stream));
  CK(cudaEventRecord(g->ev0, g->stream));
  d.async = (mode == MODE_STATIC ? g->async_static : g->async) ? 1 : 0;
  int32_t md = mode;
  void *args[] = {&d, &md};
  bool attempted = false;           // a certificate attempt (k_reach<true>) was made
  if (mode == MODE_MINCUT && g->reach) {
    void *rargs[] = {&d};
    CK(cudaLaunchCooperativeKernel((const void *)k_reach<false>, dim3(g->reach_blocks), dim3(RNT), rargs, 0, g->stream));
  } else if (mode == MODE_PP && d.warm && d.lazy && g->cert_skip > 0) {
    // the last certificate attempt failed: run the full stage 1 from the warm labels
    // for a while (exponential back-off), without the certificate's extra BFS
    g->cert_skip--;
    d.lazy = 0;
    CK(cudaLaunchCooperativeKernel((const void *)k_solve<NT>, dim3(g->grid_blocks), dim3(NT), args, 0, g->stream));
  } else if (mode == MODE_PP && d.warm && d.lazy && g->reach) {
    attempted = true;
    // DYN_PP warm start: batch + warm discharge iteration (k_solve), the universal
    // certificate (k_reach<true>), and -- only if it failed, decided on the device --
    // the full Alg.8 stage 1 / P / stage 2 (k_solve MODE_PP_CONT, a no-op otherwise)
    d.split = 1;
    CK(cudaLaunchCooperativeKernel((const void *)k_solve<NT>, dim3(g->grid_blocks), dim3(NT), args, 0, g->stream));
    void *rargs[] = {&d};
    CK(cudaLaunchCooperativeKernel((const void *)k_reach<true>, dim3(g->reach_blocks), dim3(RNT), rargs, 0, g->stream));
    int32_t mc = MODE_PP_CONT;
    void *cargs[] = {&d, &mc};
    CK(cudaLaunchCooperativeKernel((const void *)k_solve<NT>, dim3(g->grid_blocks), dim3(NT), cargs, 0, g->stream));
    g->launches += 2;
  } else {
    CK(cudaLaunchCooperativeKernel((const void *)k_solve<NT>, dim3(g->grid_blocks), dim3(NT), args, 0, g->stream));
  }
  g->launches++;
  CK(cudaEventRecord(g->ev1, g->stream));
  CK(cudaMemcpyAsync(g->hctl, g->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, g->stream));
  if (g->watchdog_s > 0) {             // debug watchdog: poll instead of blocking
    auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      cudaError_t q = cudaStreamQuery(g->stream);
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) CK(q);
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > g->watchdog_s) {
        fprintf(stderr, "[dmf watchdog] mode %d stuck %.1fs: phase=%d iter=%d round=%d lvl=%d a=%d b=%d\n", mode, el,
                g->hdbg[0], g->hdbg[1], g->hdbg[2], g->hdbg[3], g->hdbg[4], g->hdbg[5]);
        fflush(stderr);
        _exit(3);
      }
      std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
  }
  CK(cudaStreamSynchronize(g->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, g->ev0, g->ev1);
  const Ctl &c = *g->hctl;
  dmf_stats &st = g->stats;
  st.iterations = (int64_t)c.stat[ST_ITERS];
  st.bfs_levels = (int64_t)c.stat[ST_LEVELS];
  st.bfs_vertices = (int64_t)c.stat[ST_BFS_V];
  st.bfs_slots = (int64_t)c.stat[ST_BFS_SLOTS];
  st.discharge_vertices = (int64_t)c.stat[ST_DIS_V];
  st.discharge_slots = (int64_t)c.stat[ST_DIS_SLOTS];
  st.pushes = (int64_t)c.stat[ST_PUSHES];
  st.relabels = (int64_t)c.stat[ST_RELABELS];
  st.rie_slots = (int64_t)c.stat[ST_RIE_SLOTS];
  st.rie_saturations = (int64_t)c.stat[ST_RIE_SAT];
  st.stage2_vertices = (int64_t)c.stat[ST_S2_V];
  st.stage2_iterations = (int64_t)c.stat[ST_S2_ITERS];
  st.rounds = (int64_t)c.stat[ST_ROUNDS];
  st.activations = (int64_t)c.stat[ST_ACTIVATIONS];
  st.reset_vertices = (int64_t)c.stat[ST_RESET_V];
  st.budget_stops = (int64_t)c.stat[ST_BUDGET_STOPS];
  st.bottom_up_levels = (int64_t)c.stat[ST_BU_LEVELS];
  st.t_prologue_us = c.stat[ST_T_PRO] * 1e-3f;
  st.t_reset_us = c.stat[ST_T_RESET] * 1e-3f;
  st.t_bfs_us = (c.stat[ST_T_BFS] + c.stat[ST_T_BFS_BU] + c.stat[ST_T_BFS_CMP]) * 1e-3f;
  st.t_discharge_us = c.stat[ST_T_DIS] * 1e-3f;
  st.t_rie_us = c.stat[ST_T_RIE] * 1e-3f;
  st.t_epilogue_us = c.stat[ST_T_EPI] * 1e-3f;
  st.gap_levels = (int64_t)c.stat[ST_GAP_LEVELS];
  st.gap_skips = (int64_t)c.stat[ST_GAP_SKIPS];
  st.topology_rounds = (int64_t)c.stat[ST_TOPO_ROUNDS];
  st.tail_stops = (int64_t)c.stat[ST_TAIL_STOPS];
  st.stage2_skipped = (int64_t)c.stat[ST_S2_SKIP];
  st.certified = c.lazy_ok;
  if (attempted && c.status == 0) {     // back-off of the certificate after a failed attempt
    g->cert_backoff = c.lazy_ok ? 0 : (g->cert_backoff * 2 + 1 < 16 ? g->cert_backoff * 2 + 1 : 16);
    g->cert_skip = g->cert_backoff;
  }
  st.batch_entries = dv.k;
  st.device_ms = ms;
  if (c.pad != 0) fprintf(stderr, "[dmf debug] vertex %d discharged concurrently\n", c.pad - 1);
  if (c.status != 0) {
    const char *what = c.status == DMF_ENOSLOT ? "no slot for (u,v)"
                     : c.status == DMF_EDUP ? "duplicate (u,v) in batch"
                     : c.status == DMF_EINVAL ? "vertex id out of range"
                     : c.status == DMF_EOVERFLOW ? "capacity outside [0, DMF_CAP_MAX]"
                     : c.status == DMF_ENOCONV ? "iteration cap reached" : "error";
    if (c.status != DMF_ENOCONV) {                  // rejected before any mutation: state unchanged
      g->warm = warm_before;
      g->smin_valid = smin_before;
    } else {                                        // a partial repair: no converged state any more
      g->solved = false;
      g->smin_valid = false;
      // the loop stopped after a global relabel had queued its worklist: drop the
      // queued flags so that the next call starts clean
      CK(cudaMemsetAsync(g->inq, 0, (size_t)g->n * 4, g->stream));
      CK(cudaMemsetAsync(g->rlf, 0, (size_t)g->n, g->stream));
      CK(cudaStreamSynchronize(g->stream));
    }
    return fail(c.status, "%s (batch entry %d)", what, c.err_entry);
  }
  if (mode == MODE_FLOW && c.flow != g->flow) {
    g->solved = false;
    return fail(DMF_ENOCONV, "stage (ii) changed F (%lld -> %lld)", (long long)g->flow, (long long)c.flow);
  }
  if (mode == MODE_STATIC || mode == MODE_PR || mode == MODE_PP) {
    g->flow = c.flow;
    g->solved = true;
  }
  // MAXCUT / STATIC / PR leave no S_min; FLOW keeps it (stage (ii) moves flow only
  // inside S_max and inside T, and S_min of a maximum flow is unique)
  g->smin_valid = (mode == MODE_PP && !c.lazy_ok) || mode == MODE_MINCUT || (mode == MODE_FLOW && smin_before);
  // DYN_PP leaves its final labels for the next DYN_PP; MINCUT refreshes h- (exact
  // forward distances) and keeps a warm start warm; every other launch ends it
  g->warm = (mode == MODE_PP && !g->no_warm) || (mode == MODE_MINCUT && warm_before);
  if (g->warm && g->local_gap) std::swap(g->cnt, g->cnt_next);   // the final labels' histogram
  if (g->check_level > 0 && mode != MODE_MINCUT && mode != MODE_MAXCUT) {
    const int rc = check_state(g);
    if (rc != DMF_OK) { g->solved = false; g->smin_valid = false; g->warm = false; return rc; }
  }
  return DMF_OK;
}

// ============================================================================ C ABI

extern "C" {

void dmf_default_options(dmf_options *opt) {
  if (!opt) return;
  memset(opt, 0, sizeof(*opt));
  opt->algo = DMF_DYN_PP;
}

const char *dmf_last_error(void) { return g_last_error.c_str(); }

int dmf_create(int32_t n, const int64_t *row_ptr, const int32_t *col, const int32_t *cap, int32_t s, int32_t t,
               const dmf_options *opt, dmf_graph **out) {
  g_last_error.clear();
  if (!out) return fail(DMF_EINVAL, "out is NULL");
  *out = nullptr;
  if (n < 2 || !row_ptr) return fail(DMF_EINVAL, "n must be >= 2 and row_ptr non-NULL");
  if (s < 0 || s >= n || t < 0 || t >= n || s == t) return fail(DMF_EINVAL, "bad source/sink (%d, %d)", s, t);
  dmf_graph *g = new dmf_graph();
  if (opt) g->opt = *opt; else dmf_default_options(&g->opt);
  g->n = n; g->s = s; g->t = t;
  auto bail = [&](int code) { g->release_all(); if (g->own_stream && g->stream) cudaStreamDestroy(g->stream);
                              if (g->hctl) cudaFreeHost(g->hctl); delete g; return code; };
#define CKB(call) do { cudaError_t e__ = (call); if (e__ != cudaSuccess) { \
      fail(DMF_ECUDA, "%s: %s", #call, cudaGetErrorString(e__)); return bail(DMF_ECUDA); } } while (0)
  CKB(cudaGetDevice(&g->device));
  if (g->opt.stream) g->stream = (cudaStream_t)g->opt.stream;
  else { CKB(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking)); g->own_stream = true; }
  cudaStream_t st = g->stream;
  // ---- input to the device
  int64_t m = 0;
  const bool rp_dev = is_device_ptr(row_ptr);
  if (rp_dev) CKB(cudaMemcpy(&m, row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost));
  else {
    m = row_ptr[n];
    if (row_ptr[0] != 0) { fail(DMF_EINVAL, "row_ptr[0] != 0"); return bail(DMF_EINVAL); }
    for (int32_t u = 0; u < n; u++)
      if (row_ptr[u + 1] < row_ptr[u]) { fail(DMF_EINVAL, "row_ptr decreasing at %d", u); return bail(DMF_EINVAL); }
  }
  if (m < 0) { fail(DMF_EINVAL, "negative edge count"); return bail(DMF_EINVAL); }
  if (2 * m >= (int64_t)0x7fffffff) { fail(DMF_EOVERFLOW, "too many edges (%lld)", (long long)m); return bail(DMF_EOVERFLOW); }
  const int64_t N2 = 2 * m;
  int64_t *d_rp = (int64_t *)g->alloc((n + 1) * sizeof(int64_t));
  int32_t *d_col = (int32_t *)g->alloc((m ? m : 1) * sizeof(int32_t));
  int32_t *d_cap = (int32_t *)g->alloc((m ? m : 1) * sizeof(int32_t));
  unsigned long long *k0 = (unsigned long long *)g->alloc((N2 ? N2 : 1) * 8);
  unsigned long long *k1 = (unsigned long long *)g->alloc((N2 ? N2 : 1) * 8);
  int32_t *v0 = (int32_t *)g->alloc((N2 ? N2 : 1) * 4);
  int32_t *v1 = (int32_t *)g->alloc((N2 ? N2 : 1) * 4);
  int32_t *scan = (int32_t *)g->alloc((N2 ? N2 : 1) * 4);
  int32_t *err = (int32_t *)g->alloc(64);
  if (!d_rp || !d_col || !d_cap || !k0 || !k1 || !v0 || !v1 || !scan || !err) { fail(DMF_ENOMEM, "device allocation failed (input staging)"); return bail(DMF_ENOMEM); }
  CKB(cudaMemcpyAsync(d_rp, row_ptr, (n + 1) * sizeof(int64_t), cudaMemcpyDefault, st));
  if (m) {
    CKB(cudaMemcpyAsync(d_col, col, m * sizeof(int32_t), cudaMemcpyDefault, st));
    CKB(cudaMemcpyAsync(d_cap, cap, m * sizeof(int32_t), cudaMemcpyDefault, st));
  }
  CKB(cudaMemsetAsync(err, 0, 64, st));
  const int TB = 256;
  auto blocks = [](int64_t N) { int64_t b = (N + 255) / 256; return (int)(b < 1 ? 1 : (b > 148 * 64 ? 148 * 64 : b)); };
  int64_t S = 0;
  unsigned long long *ukey = nullptr;
  long long *capsum = nullptr;
  int32_t *isinput = nullptr;
  if (m) {
    k_expand_edges<<<blocks(m), TB, 0, st>>>(n, m, d_rp, d_col, d_cap, k0, v0, err);
    CKB(cudaGetLastError());
    int32_t herr = 0;
    CKB(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st));
    CKB(cudaStreamSynchronize(st));
    if (herr) { fail(herr, herr == DMF_EOVERFLOW ? "input capacity above DMF_CAP_MAX" : "invalid input edge (self-loop, id out of range or negative capacity)"); return bail(herr); }
    const int endbit = bits_for((unsigned long long)n * (unsigned long long)n);
    size_t tb = 0;
    CKB(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, v1, (int)N2, 0, endbit, st));
    size_t tb2 = 0;
    CKB(cub::DeviceScan::InclusiveSum(nullptr, tb2, scan, scan, (int)N2, st));
    void *tmp = g->alloc(tb > tb2 ? tb : tb2);
    if (!tmp) { fail(DMF_ENOMEM, "device allocation failed (sort)"); return bail(DMF_ENOMEM); }
    CKB(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, (int)N2, 0, endbit, st));
    k_run_heads<<<blocks(N2), TB, 0, st>>>(N2, k1, scan);
    CKB(cub::DeviceScan::InclusiveSum(tmp, tb2, scan, scan, (int)N2, st));
    int32_t hS = 0;
    CKB(cudaMemcpyAsync(&hS, scan + N2 - 1, 4, cudaMemcpyDeviceToHost, st));
    CKB(cudaStreamSynchronize(st));
    S = hS;
    ukey = k0;                       // reuse
    capsum = (long long *)g->alloc(S * 8);
    isinput = v0;                    // reuse (N2 >= S)
    if (!capsum) { fail(DMF_ENOMEM, "device allocation failed (merge)"); return bail(DMF_ENOMEM); }
    CKB(cudaMemsetAsync(capsum, 0, S * 8, st));
    CKB(cudaMemsetAsync(isinput, 0, S * 4, st));
    k_merge_runs<<<blocks(N2), TB, 0, st>>>(N2, k1, v1, scan, ukey, capsum, isinput);
    CKB(cudaGetLastError());
    g->release(tmp);
  }
  g->S = S;
  // ---- persistent arrays
  const size_t nn = (size_t)n;
  g->row = (int32_t *)g->alloc((nn + 1) * 4);
  g->dst = (int32_t *)g->alloc(S * 4);
  g->rev = (int32_t *)g->alloc(S * 4);
  g->cap = (int32_t *)g->alloc(S * 4);
  g->res = (int32_t *)g->alloc(S * 4);
  g->rres = (int32_t *)g->alloc(S * 4);
  g->stamp = (int32_t *)g->alloc(S * 4);
  g->e = (long long *)g->alloc(nn * 8);
  g->hp = (int32_t *)g->alloc(nn * 4);
  g->hm = (int32_t *)g->alloc(nn * 4);
  g->part = (uint8_t *)g->alloc(nn);
  g->mask = (uint8_t *)g->alloc(nn);
  g->q0 = (int32_t *)g->alloc(NB * nn * 4);
  g->q1 = (int32_t *)g->alloc(NB * nn * 4);
  g->wl = (int32_t *)g->alloc(2 * NB * nn * 4);
  g->inq = (int32_t *)g->alloc(nn * 4);
  g->rlf = (uint8_t *)g->alloc(nn);
  g->bul = (int32_t *)g->alloc(2 * nn * 4);
  const size_t cqn = (size_t)(S / CH) + nn + 64;   // >= sum over vertices of ceil(deg / CH)
  const size_t fqn = (size_t)(S / BCH) + nn + 64;  // >= sum over vertices of ceil(deg / BCH) (BFS frontier chunks)
  g->cq0 = (long long *)g->alloc(fqn * 8);
  g->cq1 = (long long *)g->alloc(fqn * 8);
  g->cqr = (long long *)g->alloc(cqn * 8);
  g->cw0 = (long long *)g->alloc(cqn * 8);
  g->cw1 = (long long *)g->alloc(cqn * 8);
  g->dcnt = (int32_t *)g->alloc(nn * 4);
  g->dmin = (int32_t *)g->alloc(nn * 4);
  g->arc = (int32_t *)g->alloc(nn * 4);
  {
    // live ring window <= queued items (<= n + S/CH, inq-deduplicated) + one outstanding
    // claim per warp of the grid (idle warps claim ahead of the tail): no index aliases
    size_t cap = 1024;
    while (cap < 2 * cqn + 65536) cap <<= 1;
    g->aq = (long long *)g->alloc(cap * 8);
    g->aq_mask = (int32_t)(cap - 1);
  }
  g->rl = (int32_t *)g->alloc(NB * nn * 4);
  g->plist = (int32_t *)g->alloc(nn * 4);
  g->ctl = (Ctl *)g->alloc(sizeof(Ctl));
  if (!g->row || !g->dst || !g->rev || !g->cap || !g->res || !g->rres || !g->stamp || !g->e || !g->hp || !g->hm ||
      !g->part || !g->mask || !g->q0 || !g->q1 || !g->wl || !g->rl || !g->plist || !g->ctl || !g->inq || !g->rlf || !g->bul || !g->cq0 || !g->cq1 || !g->cqr ||
      !g->cw0 || !g->cw1 || !g->dcnt || !g->dmin || !g->arc || !g->aq) {
    fail(DMF_ENOMEM, "device allocation failed (state, S=%lld)", (long long)S);
    return bail(DMF_ENOMEM);
  }
  CKB(cudaMallocHost((void **)&g->hctl, sizeof(Ctl)));
  {
    // engine knobs: dmf_options fields (0 = default), each overridable by its DMF_*
    // environment variable (process-wide; for experiments)
    const dmf_options &o = g->opt;
    auto knob = [](int32_t field, const char *env) -> int32_t {
      const char *e = getenv(env);
      return e ? (int32_t)atoi(e) : field;
    };
    const int32_t sched = knob(o.schedule, "DMF_SCHED");
    if (sched < 0 || sched > DMF_SCHED_TOPOLOGY) { fail(DMF_EINVAL, "unknown schedule %d", sched); return bail(DMF_EINVAL); }
    g->async = sched == DMF_SCHED_AUTO || sched == DMF_SCHED_ASYNC;
    g->async_static = sched == DMF_SCHED_ASYNC;
    if (const char *as = getenv("DMF_ASYNC")) g->async = atoi(as) != 0;          // legacy switches
    if (const char *ss = getenv("DMF_ASYNC_STATIC")) g->async_static = atoi(ss) != 0;
    const int32_t aw = knob(o.async_warps, "DMF_ASYNC_WARPS");
    g->async_warps = aw > 0 ? (aw < WPB ? aw : WPB) : 8;
    const int32_t bm = knob(o.budget_mul, "DMF_BUDGET_MUL");
    g->budget_mul = bm == 0 ? 1 : bm;
    const int32_t ti = knob(o.tail_items, "DMF_TAIL_ITEMS");
    g->tail_items = ti == 0 ? 2048 : (ti < 0 ? 0 : ti);
    g->local_gap = knob(o.local_gap, "DMF_LOCAL_GAP") < 0 ? 0 : 1;
    g->no_warm = knob(o.warm, "DMF_WARM") < 0;
    if (const char *nw = getenv("DMF_NO_WARM")) g->no_warm = atoi(nw) != 0;
    const int32_t td = knob(o.topo_div, "DMF_TOPO_DIV");
    // the auto-switch is off by default: on B200 the worklist (its compaction fused into
    // the BFS) beat every topology-driven variant measured (tools/ab_topology.py)
    g->topo_div = sched == DMF_SCHED_TOPOLOGY ? 0x3fffffff : (td <= 0 ? 0 : td);
    g->lazy = knob(o.certify, "DMF_CERTIFY") < 0 ? 0 : 1;
    if (const char *mc = getenv("DMF_DMAXCH")) g->dmaxch = atoi(mc) > 0 ? atoi(mc) : 0;
    if (const char *pb = getenv("DMF_PROBE")) g->probes = atoi(pb) != 0;
    if (const char *ia = getenv("DMF_IMM_ACT")) g->imm_act = atoi(ia) != 0;
    if (const char *s2 = getenv("DMF_SCAN2")) g->scan2 = atoi(s2) != 0;
    g->check_level = knob(o.check_level, "DMF_CHECK_LEVEL");
    if (const char *ba = getenv("DMF_BU_ALPHA")) g->bu_alpha = atoi(ba) >= 0 ? atoi(ba) : g->bu_alpha;   // 0: never bottom-up
    if (const char *dd = getenv("DMF_DENSE_DIV")) g->dense_div = atoi(dd) > 0 ? atoi(dd) : g->dense_div;
    if (const char *sl = getenv("DMF_ASYNC_SLEEP_NS")) g->async_sleep_ns = atoi(sl) > 0 ? atoi(sl) : 128;
    for (int i = 0; i < 7; i++)
      if (o.reserved[i]) { fail(DMF_EINVAL, "dmf_options.reserved must be zero"); return bail(DMF_EINVAL); }
  }
  g->chk = (int32_t *)g->alloc(64);
  g->cnt = (int32_t *)g->alloc(2 * GAPW * sizeof(int32_t));
  g->cnt_next = (int32_t *)g->alloc(2 * GAPW * sizeof(int32_t));
  if (!g->cnt || !g->cnt_next || !g->chk) { fail(DMF_ENOMEM, "device allocation failed (level counts)"); return bail(DMF_ENOMEM); }
  CKB(cudaMemsetAsync(g->cnt, 0, 2 * GAPW * sizeof(int32_t), st));
  CKB(cudaMemsetAsync(g->cnt_next, 0, 2 * GAPW * sizeof(int32_t), st));
  if (const char *wd = getenv("DMF_WATCHDOG_S")) {
    g->watchdog_s = atof(wd);
    CKB(cudaHostAlloc((void **)&g->hdbg, 64, cudaHostAllocMapped));
    memset(g->hdbg, 0, 64);
    CKB(cudaHostGetDevicePointer((void **)&g->ddbg, g->hdbg, 0));
  }
  CKB(cudaMemsetAsync(g->inq, 0, nn * 4, st));
  CKB(cudaMemsetAsync(g->rlf, 0, nn, st));
  CKB(cudaMemsetAsync(g->dcnt, 0, nn * 4, st));
  CKB(cudaMemsetAsync(g->dmin, 0x7f, nn * 4, st));   // DMIN_NONE
  CKB(cudaMemsetAsync(g->arc, 0, nn * 4, st));
  CKB(cudaMemsetAsync(g->aq, 0xff, ((size_t)g->aq_mask + 1) * 8, st));   // AQ_EMPTY
  {
    if (S > (1LL << 30)) { fail(DMF_EOVERFLOW, "too many slots for the slot table (%lld > 2^30)", (long long)S); return bail(DMF_EOVERFLOW); }
    size_t T = 1024;
    while (T < 2 * (size_t)S) T <<= 1;
    g->htab = (int4 *)g->alloc(T * sizeof(int4));
    if (!g->htab) { fail(DMF_ENOMEM, "device allocation failed (slot table)"); return bail(DMF_ENOMEM); }
    g->hmask = (int32_t)(T - 1);
    CKB(cudaMemsetAsync(g->htab, 0xff, T * sizeof(int4), st));
  }
  if (S) {
    CKB(cudaMemsetAsync(err, 0, 64, st));
    k_rows<<<blocks(nn + 1), TB, 0, st>>>(n, S, ukey, g->row);
    k_slots<<<blocks(S), TB, 0, st>>>(n, S, ukey, capsum, g->dst, g->rev, g->cap, err);
    k_hash_insert<<<blocks(S), TB, 0, st>>>(S, n, ukey, g->rev, g->htab, (uint32_t)g->hmask);
    unsigned long long *msum = (unsigned long long *)(err + 8);
    k_sum_i32<<<blocks(S), TB, 0, st>>>(S, isinput, msum);
    CKB(cudaGetLastError());
    int32_t hbuf[16];
    CKB(cudaMemcpyAsync(hbuf, err, 64, cudaMemcpyDeviceToHost, st));
    CKB(cudaStreamSynchronize(st));
    if (hbuf[0]) { fail(DMF_EOVERFLOW, "merged capacity of a pair exceeds DMF_CAP_MAX"); return bail(DMF_EOVERFLOW); }
    unsigned long long hm_ = 0;
    memcpy(&hm_, hbuf + 8, 8);
    g->m = (int64_t)hm_;
  } else {
    CKB(cudaMemsetAsync(g->row, 0, (nn + 1) * 4, st));
  }
  k_init_state<<<blocks(S > (int64_t)nn ? S : (int64_t)nn), TB, 0, st>>>(S, n, g->rev, g->cap, g->res, g->rres, g->stamp,
                                                                      g->e, g->part, g->hp, g->hm);
  CKB(cudaGetLastError());
  CKB(cudaStreamSynchronize(st));
  // free staging
  for (void *p : {(void *)d_rp, (void *)d_col, (void *)d_cap, (void *)k0, (void *)k1, (void *)v0, (void *)v1,
                  (void *)scan, (void *)capsum})
    if (p) g->release(p);
  // KERNELCYCLES = max(1, floor(m/n)) (R17)
  g->kc = g->opt.kernel_cycles > 0 ? g->opt.kernel_cycles : (int32_t)(g->m / n > 0 ? g->m / n : 1);
  // cooperative grid
  int per_sm = 0, sms = 0;
  CKB(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve<NT>, NT, 0));
  CKB(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device));
  if (per_sm < 1) { fail(DMF_ECUDA, "solve kernel cannot be resident (occupancy 0)"); return bail(DMF_ECUDA); }
  g->grid_blocks = per_sm * sms;
  if (g->opt.grid_blocks > 0 && g->opt.grid_blocks < g->grid_blocks) g->grid_blocks = g->opt.grid_blocks;
  {
    int rper = 0;
    int rper2 = 0;
    CKB(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rper, k_reach<false>, RNT, 0));
    CKB(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rper2, k_reach<true>, RNT, 0));
    rper = rper2 < rper ? rper2 : rper;
    if (rper < 1) { fail(DMF_ECUDA, "reach kernel cannot be resident (occupancy 0)"); return bail(DMF_ECUDA); }
    g->reach_blocks = rper * sms;
    if (const char *rc = getenv("DMF_REACH")) g->reach = atoi(rc) != 0;
  }
  CKB(cudaEventCreate(&g->ev0));
  CKB(cudaEventCreate(&g->ev1));
  g->stats.n = n; g->stats.m = g->m; g->stats.S = S; g->stats.kernel_cycles = g->kc;
  g->stats.grid_blocks = g->grid_blocks; g->stats.block_threads = NT;
  *out = g;
#undef CKB
  return DMF_OK;
}

int dmf_static_solve(dmf_graph *g) {
  g_last_error.clear();
  if (!g) return fail(DMF_EINVAL, "NULL handle");
  Dev d = make_dev(g);
  return run_solve(g, MODE_STATIC, d);
}

int dmf_static_solve_pp(dmf_graph *g) {
  g_last_error.clear();
  if (!g) return fail(DMF_EINVAL, "NULL handle");
  Dev d = make_dev(g);
  d.static_pp = 1;
  return run_solve(g, MODE_STATIC, d);
}

int dmf_apply_batch(dmf_graph *g, int64_t k, const int32_t *u, const int32_t *v, const int32_t *new_cap, int32_t algo) {
  g_last_error.clear();
  if (!g) return fail(DMF_EINVAL, "NULL handle");
  if (k < 0 || (k > 0 && (!u || !v || !new_cap))) return fail(DMF_EINVAL, "bad batch arrays");
  if (k >= 0x7fffffff) return fail(DMF_EINVAL, "batch too large");
  if (algo < 0) algo = g->opt.algo;
  if (algo != DMF_DYN_PR && algo != DMF_DYN_PP) return fail(DMF_EINVAL, "unknown algo %d", algo);
  if (algo == DMF_DYN_PP && !g->solved) return fail(DMF_ESTATE, "DMF_DYN_PP needs a previous converged solve");
  Dev d = make_dev(g);
  if (k > 0) {
    const bool dev_in = is_device_ptr(u) && is_device_ptr(v) && is_device_ptr(new_cap);
    if (k > g->bcap) {
      if (g->bbuf) g->release(g->bbuf);
      g->bcap = k + k / 4 + 1024;
      g->bbuf = (int32_t *)g->alloc(7 * g->bcap * sizeof(int32_t));
      if (!g->bbuf) { g->bcap = 0; return fail(DMF_ENOMEM, "batch buffer allocation failed"); }
    }
    if (dev_in) { d.bu = u; d.bv = v; d.bc = new_cap; }
    else {
      CK(cudaMemcpyAsync(g->bbuf, u, k * 4, cudaMemcpyDefault, g->stream));
      CK(cudaMemcpyAsync(g->bbuf + g->bcap, v, k * 4, cudaMemcpyDefault, g->stream));
      CK(cudaMemcpyAsync(g->bbuf + 2 * g->bcap, new_cap, k * 4, cudaMemcpyDefault, g->stream));
      d.bu = g->bbuf; d.bv = g->bbuf + g->bcap; d.bc = g->bbuf + 2 * g->bcap;
    }
    d.bslot = g->bbuf + 3 * g->bcap;
    d.brec = g->bbuf + 4 * g->bcap;
  }
  d.k = k;
  d.batch_id = ++g->batch_id;
  if (g->batch_id >= 0x7ffffff0) {   // stamp wrap-around: clear the stamps
    CK(cudaMemsetAsync(g->stamp, 0, g->S * 4, g->stream));
    g->batch_id = 1;
    d.batch_id = 1;
  }
  return run_solve(g, algo == DMF_DYN_PP ? MODE_PP : MODE_PR, d);
}

int dmf_flow_value(const dmf_graph *g, int64_t *out) {
  g_last_error.clear();
  if (!g || !out) return fail(DMF_EINVAL, "NULL argument");
  if (!g->solved) return fail(DMF_ESTATE, "no converged solve yet");
  *out = g->flow;
  return DMF_OK;
}

static int cut_query(dmf_graph *g, uint8_t *mask, int32_t mode) {
  g_last_error.clear();
  if (!g || !mask) return fail(DMF_EINVAL, "NULL argument");
  if (!g->solved) return fail(DMF_ESTATE, "no converged solve yet");
  if (!(mode == MODE_MINCUT && g->smin_valid)) {   // a DYN_PP repair already produced S_min
    dmf_stats keep = g->stats;
    Dev d = make_dev(g);
    int rc = run_solve(g, mode, d);
    keep.query_ms = g->stats.device_ms;
    keep.query_bfs_vertices = g->stats.bfs_vertices;
    keep.query_bfs_slots = g->stats.bfs_slots;
    g->stats = keep;
    if (rc) return rc;
  } else {
    g->stats.query_ms = 0.f;
    g->stats.query_bfs_vertices = 0;
    g->stats.query_bfs_slots = 0;
  }
  CK(cudaMemcpyAsync(mask, g->mask, (size_t)g->n, cudaMemcpyDefault, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  return DMF_OK;
}

int dmf_min_cut_source_side(dmf_graph *g, uint8_t *mask) { return cut_query(g, mask, MODE_MINCUT); }

int dmf_to_flow(dmf_graph *g) {
  g_last_error.clear();
  if (!g) return fail(DMF_EINVAL, "NULL handle");
  if (!g->solved) return fail(DMF_ESTATE, "no converged solve yet");
  dmf_stats keep = g->stats;
  Dev d = make_dev(g);
  const int rc = run_solve(g, MODE_FLOW, d);
  g->stats = keep;
  return rc;
}

namespace {
__global__ void k_edge_flow(int64_t S, const int32_t *cap, const int32_t *res, int32_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t x = cap[i] - res[i];      // net flow on the pair, seen from this slot
    out[i] = x > 0 ? x : 0;
  }
}
}  // namespace

int dmf_edge_flow(dmf_graph *g, int32_t *flow) {
  g_last_error.clear();
  if (!g || !flow) return fail(DMF_EINVAL, "NULL argument");
  if (!g->solved) return fail(DMF_ESTATE, "no converged solve yet");
  int32_t *dst = flow;
  const bool dev = is_device_ptr(flow);
  if (!dev) {
    dst = (int32_t *)g->alloc((size_t)g->S * 4);
    if (!dst) return fail(DMF_ENOMEM, "device allocation failed (edge flow)");
  }
  if (g->S) k_edge_flow<<<(int)(g->S < 148LL * 256 * 16 ? (g->S + 255) / 256 : 148LL * 16), 256, 0, g->stream>>>(g->S, g->cap, g->res, dst);
  g->launches++;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && !dev) e = cudaMemcpyAsync(flow, dst, (size_t)g->S * 4, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (!dev) g->release(dst);
  if (e != cudaSuccess) return fail(DMF_ECUDA, "edge flow: %s", cudaGetErrorString(e));
  return DMF_OK;
}
int dmf_max_cut_source_side(dmf_graph *g, uint8_t *mask) { return cut_query(g, mask, MODE_MAXCUT); }

int dmf_set_trace(dmf_graph *g, int32_t capacity) {
  g_last_error.clear();
  if (!g || capacity < 0) return fail(DMF_EINVAL, "bad arguments");
  if (g->trace) { g->release(g->trace); g->trace = nullptr; g->trace_cap = 0; }
  if (g->trace_cta) { g->release(g->trace_cta); g->trace_cta = nullptr; }
  if (capacity > 0) {
    g->trace = (int32_t *)g->alloc((size_t)capacity * 8 * sizeof(int32_t));
    g->trace_cta = (uint32_t *)g->alloc((size_t)capacity * g->grid_blocks * sizeof(uint32_t));
    if (!g->trace || !g->trace_cta) return fail(DMF_ENOMEM, "trace buffer allocation failed");
    g->trace_cap = capacity;
  }
  return DMF_OK;
}

int dmf_get_trace(const dmf_graph *g, int32_t *records, int32_t capacity, int32_t *count) {
  g_last_error.clear();
  if (!g || !count) return fail(DMF_EINVAL, "bad arguments");
  const int32_t nrec = g->trace ? (g->hctl->ntrace < g->trace_cap ? g->hctl->ntrace : g->trace_cap) : 0;
  *count = nrec;
  if (records && nrec) {
    const int32_t c = nrec < capacity ? nrec : capacity;
    CK(cudaMemcpy(records, g->trace, (size_t)c * 8 * sizeof(int32_t), cudaMemcpyDefault));
  }
  return DMF_OK;
}

int dmf_get_trace_cta(const dmf_graph *g, uint32_t *busy_ns, int32_t capacity, int32_t *grid) {
  g_last_error.clear();
  if (!g || !grid) return fail(DMF_EINVAL, "bad arguments");
  *grid = g->grid_blocks;
  const int32_t nrec = g->trace ? (g->hctl->ntrace < g->trace_cap ? g->hctl->ntrace : g->trace_cap) : 0;
  if (busy_ns && nrec) {
    const int32_t c = nrec < capacity ? nrec : capacity;
    CK(cudaMemcpy(busy_ns, g->trace_cta, (size_t)c * g->grid_blocks * sizeof(uint32_t), cudaMemcpyDefault));
  }
  return DMF_OK;
}

int dmf_get_stats(const dmf_graph *g, dmf_stats *out) {
  if (!g || !out) return fail(DMF_EINVAL, "NULL argument");
  *out = g->stats;
  out->kernel_launches = g->launches;
  return DMF_OK;
}

int dmf_sizes(const dmf_graph *g, int32_t *n, int64_t *S, int64_t *m) {
  if (!g) return fail(DMF_EINVAL, "NULL handle");
  if (n) *n = g->n;
  if (S) *S = g->S;
  if (m) *m = g->m;
  return DMF_OK;
}

int dmf_export_state(const dmf_graph *g, int64_t *row_ptr, int32_t *dst, int32_t *rev, int32_t *cap, int32_t *res,
                     int64_t *excess) {
  g_last_error.clear();
  if (!g) return fail(DMF_EINVAL, "NULL handle");
  cudaStream_t st = g->stream;
  if (row_ptr) {
    std::vector<int32_t> r(g->n + 1);
    CK(cudaMemcpyAsync(r.data(), g->row, (g->n + 1) * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<int64_t> r64(r.begin(), r.end());
    CK(cudaMemcpyAsync(row_ptr, r64.data(), (g->n + 1) * 8, cudaMemcpyDefault, st));
    CK(cudaStreamSynchronize(st));
  }
  if (dst) CK(cudaMemcpyAsync(dst, g->dst, g->S * 4, cudaMemcpyDefault, st));
  if (rev) CK(cudaMemcpyAsync(rev, g->rev, g->S * 4, cudaMemcpyDefault, st));
  if (cap) CK(cudaMemcpyAsync(cap, g->cap, g->S * 4, cudaMemcpyDefault, st));
  if (res) CK(cudaMemcpyAsync(res, g->res, g->S * 4, cudaMemcpyDefault, st));
  if (excess) CK(cudaMemcpyAsync(excess, g->e, (size_t)g->n * 8, cudaMemcpyDefault, st));
  CK(cudaStreamSynchronize(st));
  return DMF_OK;
}

int dmf_check_state(dmf_graph *g) {
  g_last_error.clear();
  if (!g) return fail(DMF_EINVAL, "NULL handle");
  return check_state(g);
}

int dmf_import_state(dmf_graph *g, const int32_t *cap, const int32_t *res, const int64_t *excess) {
  g_last_error.clear();
  if (!g || !cap || !res || !excess) return fail(DMF_EINVAL, "NULL argument");
  cudaStream_t st = g->stream;
  const size_t S4 = (size_t)g->S * 4, n8 = (size_t)g->n * 8;
  int32_t *tcap = (int32_t *)g->alloc(S4 ? S4 : 4), *tres = (int32_t *)g->alloc(S4 ? S4 : 4);
  long long *te = (long long *)g->alloc(n8);
  int rc = DMF_OK;
  if (!tcap || !tres || !te) rc = fail(DMF_ENOMEM, "device allocation failed (import)");
  if (rc == DMF_OK) {
    cudaError_t e = cudaMemcpyAsync(tcap, cap, S4, cudaMemcpyDefault, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(tres, res, S4, cudaMemcpyDefault, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(te, excess, n8, cudaMemcpyDefault, st);
    if (e != cudaSuccess) rc = fail(DMF_ECUDA, "import copy: %s", cudaGetErrorString(e));
  }
  if (rc == DMF_OK) {
    // capacities of the import: the pair sum 2 needs cap_rev from the same array
    rc = check_arrays(g, tcap, tres, nullptr, te);
    if (rc == DMF_ECHECK) { std::string m = g_last_error; rc = fail(DMF_EINVAL, "import rejected: %s", m.c_str()); }
  }
  if (rc == DMF_OK) {
    cudaError_t e = cudaMemcpyAsync(g->cap, tcap, S4, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(g->res, tres, S4, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(g->e, te, n8, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess && g->S) {
      k_mirror<<<g->grid_blocks > 0 ? g->grid_blocks : 296, 512, 0, st>>>(g->S, g->rev, g->res, g->rres);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = fail(DMF_ECUDA, "import commit: %s", cudaGetErrorString(e));
    g->solved = false;       // a valid pseudoflow, not known to be converged
    g->smin_valid = false;
    g->warm = false;
  }
  if (tcap) g->release(tcap);
  if (tres) g->release(tres);
  if (te) g->release(te);
  return rc;
}

int dmf_export_labels(const dmf_graph *g, int32_t *hp, int32_t *hm, uint8_t *part, int32_t *rres) {
  g_last_error.clear();
  if (!g) return fail(DMF_EINVAL, "NULL handle");
  cudaStream_t st = g->stream;
  if (hp) CK(cudaMemcpyAsync(hp, g->hp, (size_t)g->n * 4, cudaMemcpyDefault, st));
  if (hm) CK(cudaMemcpyAsync(hm, g->hm, (size_t)g->n * 4, cudaMemcpyDefault, st));
  if (part) CK(cudaMemcpyAsync(part, g->part, (size_t)g->n, cudaMemcpyDefault, st));
  if (rres) CK(cudaMemcpyAsync(rres, g->rres, (size_t)g->S * 4, cudaMemcpyDefault, st));
  CK(cudaStreamSynchronize(st));
  return DMF_OK;
}

void dmf_destroy(dmf_graph *g) {
  if (!g) return;
  if (g->stream) cudaStreamSynchronize(g->stream);
  g->release_all();
  if (g->hctl) cudaFreeHost(g->hctl);
  if (g->hdbg) cudaFreeHost(g->hdbg);
  if (g->ev0) cudaEventDestroy(g->ev0);
  if (g->ev1) cudaEventDestroy(g->ev1);
  if (g->own_stream && g->stream) cudaStreamDestroy(g->stream);
  delete g;
}

}  // extern "C"
