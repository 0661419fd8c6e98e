/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU
 * max-flow / min-cut oracle for arXiv 2511.05895 ("Efficient Dynamic MaxFlow
 * Computation on GPUs").  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or helper with the CUDA path (paper_2511_05895_b200/csrc).
 *
 * What the method computes has a plain definition:
 *   F     = max{|f| : 0 <= f <= c, conservation on V\{s,t}}
 *   S_min = {v : s ~> v in G_{f*}} for any maximum flow f*      (intersection of all
 *           minimum-cut source sides; unique)
 *   S_max = V \ {v : v ~> t in G_{f*}}                          (union of all minimum-cut
 *           source sides; the paper's {h = |V|} certificate)
 * so the oracle is that definition computed by textbook algorithms:
 *   O1 Edmonds-Karp            orc_maxflow(ORC_EK, ...)
 *   O1' Dinitz blocking flows  orc_maxflow(ORC_DINIC, ...)
 *   O2 two-phase FIFO push-relabel (Goldberg-Tarjan) with global relabel
 *      and gap; phase 2 returns the stuck excess to s so a TRUE flow results
 *                                      orc_maxflow(ORC_FIFO_PR, ...)
 *   O4 Hopcroft-Karp maximum bipartite matching   orc_hopcroft_karp
 * plus a CHECKER of a solver state exported by any implementation
 * (orc_check_state): capacity, pair-sum, excess consistency, no augmenting path,
 * conversion of the pseudoflow to a true flow (Lemma 4 P:276-304 and Lemma
 * route excess back to s, fill deficits from t), conservation of the
 * converted flow, and S_min / cut-capacity certificate (Thm 3).
 *
 * Residual network representation (the oracle's own): every input edge j becomes
 * the arc pair (2j: u->v, residual cap c_j) and (2j+1: v->u, residual 0);
 * parallel edges are NOT merged (max-flow is indifferent to that); self-loops are
 * skipped (they carry no s-t flow).  Arcs are bucketed by tail (CSR).
 * All capacities / flows are int64.
 *
 * Build: gcc -O2 -shared -fPIC -o liboracle.so oracle.c
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>

enum { ORC_EK = 0, ORC_DINIC = 1, ORC_FIFO_PR = 2 };

typedef struct {
    int32_t n;
    int64_t na;
    int64_t *first;   /* n+1 */
    int32_t *head;    /* na */
    int64_t *res;     /* na */
    int64_t *pair;    /* na */
    int64_t *orig;    /* na: index of the arc in the caller's arc list */
} net_t;

static void net_free(net_t *g) {
    free(g->first); free(g->head); free(g->res); free(g->pair); free(g->orig);
    memset(g, 0, sizeof(*g));
}

/* Build a CSR network from an arc list (tail, head, res, pair-in-list). */
static int net_from_arcs(net_t *g, int32_t n, int64_t na, const int32_t *tail,
                         const int32_t *head, const int64_t *res, const int64_t *pair) {
    g->n = n; g->na = na;
    g->first = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    g->head = (int32_t *)malloc((size_t)(na ? na : 1) * sizeof(int32_t));
    g->res = (int64_t *)malloc((size_t)(na ? na : 1) * sizeof(int64_t));
    g->pair = (int64_t *)malloc((size_t)(na ? na : 1) * sizeof(int64_t));
    g->orig = (int64_t *)malloc((size_t)(na ? na : 1) * sizeof(int64_t));
    int64_t *pos = (int64_t *)malloc((size_t)(na ? na : 1) * sizeof(int64_t));
    int64_t *fill = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    if (!g->first || !g->head || !g->res || !g->pair || !g->orig || !pos || !fill) {
        free(pos); free(fill); net_free(g); return -1;
    }
    for (int64_t a = 0; a < na; a++) g->first[tail[a] + 1]++;
    for (int32_t v = 0; v < n; v++) g->first[v + 1] += g->first[v];
    memcpy(fill, g->first, ((size_t)n + 1) * sizeof(int64_t));
    for (int64_t a = 0; a < na; a++) pos[a] = fill[tail[a]]++;
    for (int64_t a = 0; a < na; a++) {
        int64_t p = pos[a];
        g->head[p] = head[a];
        g->res[p] = res[a];
        g->pair[p] = pos[pair[a]];
        g->orig[p] = a;
    }
    free(pos); free(fill);
    return 0;
}

/* Input edge list -> network with arc pairs (2j, 2j+1). */
static int net_from_edges(net_t *g, int32_t n, int64_t m, const int32_t *u, const int32_t *v,
                          const int32_t *cap, int64_t *edge_arc /* m, nullable: position of arc 2j */) {
    int64_t na = 0;
    for (int64_t j = 0; j < m; j++) if (u[j] != v[j]) na += 2;
    int32_t *tl = (int32_t *)malloc((size_t)(na ? na : 1) * sizeof(int32_t));
    int32_t *hd = (int32_t *)malloc((size_t)(na ? na : 1) * sizeof(int32_t));
    int64_t *rs = (int64_t *)malloc((size_t)(na ? na : 1) * sizeof(int64_t));
    int64_t *pr = (int64_t *)malloc((size_t)(na ? na : 1) * sizeof(int64_t));
    int64_t *which = (int64_t *)malloc((size_t)(m ? m : 1) * sizeof(int64_t));
    if (!tl || !hd || !rs || !pr || !which) { free(tl); free(hd); free(rs); free(pr); free(which); return -1; }
    int64_t a = 0;
    for (int64_t j = 0; j < m; j++) {
        if (u[j] == v[j]) { which[j] = -1; continue; }
        which[j] = a;
        tl[a] = u[j]; hd[a] = v[j]; rs[a] = cap[j]; pr[a] = a + 1;
        tl[a + 1] = v[j]; hd[a + 1] = u[j]; rs[a + 1] = 0; pr[a + 1] = a;
        a += 2;
    }
    int rc = net_from_arcs(g, n, na, tl, hd, rs, pr);
    if (rc == 0 && edge_arc) {
        /* position of each list arc after bucketing */
        int64_t *inv = (int64_t *)malloc((size_t)(na ? na : 1) * sizeof(int64_t));
        for (int64_t p = 0; p < na; p++) inv[g->orig[p]] = p;
        for (int64_t j = 0; j < m; j++) edge_arc[j] = which[j] < 0 ? -1 : inv[which[j]];
        free(inv);
    }
    free(tl); free(hd); free(rs); free(pr); free(which);
    return rc;
}

static inline int32_t arc_tail(const net_t *g, int64_t a) { return g->head[g->pair[a]]; }

/* ---------------------------------------------------------------- reachability */

/* forward reach over residual arcs from every v with roots[v] != 0 */
static void reach_forward(const net_t *g, const uint8_t *roots, uint8_t *mark) {
    int32_t *q = (int32_t *)malloc((size_t)g->n * sizeof(int32_t) + 4);
    int64_t qh = 0, qt = 0;
    for (int32_t v = 0; v < g->n; v++) { mark[v] = roots[v] ? 1 : 0; if (roots[v]) q[qt++] = v; }
    while (qh < qt) {
        int32_t x = q[qh++];
        for (int64_t a = g->first[x]; a < g->first[x + 1]; a++)
            if (g->res[a] > 0 && !mark[g->head[a]]) { mark[g->head[a]] = 1; q[qt++] = g->head[a]; }
    }
    free(q);
}

/* backward reach: every w that has a residual path into some root */
static void reach_backward(const net_t *g, const uint8_t *roots, uint8_t *mark) {
    int32_t *q = (int32_t *)malloc((size_t)g->n * sizeof(int32_t) + 4);
    int64_t qh = 0, qt = 0;
    for (int32_t v = 0; v < g->n; v++) { mark[v] = roots[v] ? 1 : 0; if (roots[v]) q[qt++] = v; }
    while (qh < qt) {
        int32_t x = q[qh++];
        for (int64_t a = g->first[x]; a < g->first[x + 1]; a++) {
            int32_t w = g->head[a];
            if (!mark[w] && g->res[g->pair[a]] > 0) { mark[w] = 1; q[qt++] = w; }
        }
    }
    free(q);
}

/* S_min = reach_{G_f}(s), S_max = V \ coreach_{G_f}(t), for a (true) max flow f */
static void cuts_of_flow(const net_t *g, int32_t s, int32_t t, uint8_t *smin, uint8_t *smax) {
    uint8_t *roots = (uint8_t *)calloc((size_t)g->n, 1);
    if (smin) { roots[s] = 1; reach_forward(g, roots, smin); roots[s] = 0; }
    if (smax) {
        roots[t] = 1;
        reach_backward(g, roots, smax);
        for (int32_t v = 0; v < g->n; v++) smax[v] = !smax[v];
    }
    free(roots);
}

/* ---------------------------------------------------------------- Edmonds-Karp */
/* Textbook: repeatedly augment along a shortest s-t path found by BFS. */
static int64_t maxflow_ek(net_t *g, int32_t s, int32_t t) {
    int64_t flow = 0;
    int64_t *par = (int64_t *)malloc((size_t)g->n * sizeof(int64_t));
    int32_t *q = (int32_t *)malloc((size_t)g->n * sizeof(int32_t));
    for (;;) {
        for (int32_t v = 0; v < g->n; v++) par[v] = -2;
        par[s] = -1;
        int64_t qh = 0, qt = 0;
        q[qt++] = s;
        while (qh < qt && par[t] == -2) {
            int32_t x = q[qh++];
            for (int64_t a = g->first[x]; a < g->first[x + 1]; a++) {
                int32_t y = g->head[a];
                if (g->res[a] > 0 && par[y] == -2) { par[y] = a; q[qt++] = y; }
            }
        }
        if (par[t] == -2) break;
        int64_t b = INT64_MAX;
        for (int32_t y = t; y != s; y = arc_tail(g, par[y])) if (g->res[par[y]] < b) b = g->res[par[y]];
        for (int32_t y = t; y != s; y = arc_tail(g, par[y])) { g->res[par[y]] -= b; g->res[g->pair[par[y]]] += b; }
        flow += b;
    }
    free(par); free(q);
    return flow;
}

/* ---------------------------------------------------------------- Dinitz */
/* Layered residual graph + blocking flow with current-arc pointers. */
static int64_t maxflow_dinic(net_t *g, int32_t s, int32_t t) {
    int32_t n = g->n;
    int64_t flow = 0;
    int32_t *lvl = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *q = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int64_t *cur = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int64_t *stk = (int64_t *)malloc(((size_t)n + 1) * sizeof(int64_t));
    if (s == t) goto done;
    for (;;) {
        for (int32_t v = 0; v < n; v++) lvl[v] = -1;
        lvl[s] = 0;
        int64_t qh = 0, qt = 0;
        q[qt++] = s;
        while (qh < qt) {
            int32_t x = q[qh++];
            for (int64_t a = g->first[x]; a < g->first[x + 1]; a++) {
                int32_t y = g->head[a];
                if (g->res[a] > 0 && lvl[y] < 0) { lvl[y] = lvl[x] + 1; q[qt++] = y; }
            }
        }
        if (lvl[t] < 0) break;
        for (int32_t v = 0; v < n; v++) cur[v] = g->first[v];
        int64_t sp = 0;      /* stack of arcs on the current path */
        int32_t x = s;
        for (;;) {
            if (x == t) {
                int64_t b = INT64_MAX, cut = 0;
                for (int64_t i = 0; i < sp; i++) if (g->res[stk[i]] < b) { b = g->res[stk[i]]; cut = i; }
                for (int64_t i = 0; i < sp; i++) { g->res[stk[i]] -= b; g->res[g->pair[stk[i]]] += b; }
                flow += b;
                sp = cut;                       /* retreat to the tail of the first saturated arc */
                x = arc_tail(g, stk[cut]);
                continue;
            }
            int64_t a = cur[x];
            for (; a < g->first[x + 1]; a++)
                if (g->res[a] > 0 && lvl[g->head[a]] == lvl[x] + 1) break;
            cur[x] = a;
            if (a < g->first[x + 1]) { stk[sp++] = a; x = g->head[a]; continue; }
            lvl[x] = -1;                        /* dead end: remove from the level graph */
            if (sp == 0) break;
            sp--;
            x = arc_tail(g, stk[sp]);
            cur[x]++;
        }
    }
done:
    free(lvl); free(q); free(cur); free(stk);
    return flow;
}

/* ---------------------------------------------------------------- FIFO push-relabel */
/* Sequential Goldberg-Tarjan with FIFO selection, current arcs, periodic
 * global relabel (backward BFS from the sink) and the gap heuristic.
 * `sink` receives flow; `blocked` is never active and never admissible
 * (height n).  Heights are capped at n (n = dead).  Used twice: phase 1 (sink t,
 * blocked s) computes a maximum preflow; phase 2 (sink s, blocked t) returns every
 * stuck excess to s (possible by Lemma 4), leaving a true max flow. */
static void pr_global_relabel(net_t *g, int32_t sink, int32_t blocked, int32_t *h, int64_t *cnt, int32_t *q) {
    int32_t n = g->n;
    for (int32_t v = 0; v <= n; v++) cnt[v] = 0;
    for (int32_t v = 0; v < n; v++) h[v] = n;
    int64_t qh = 0, qt = 0;
    h[sink] = 0; q[qt++] = sink;
    while (qh < qt) {
        int32_t x = q[qh++];
        for (int64_t a = g->first[x]; a < g->first[x + 1]; a++) {
            int32_t w = g->head[a];
            if (w != blocked && h[w] == n && g->res[g->pair[a]] > 0) { h[w] = h[x] + 1; q[qt++] = w; }
        }
    }
    for (int32_t v = 0; v < n; v++) cnt[h[v]]++;
}

static void pr_phase(net_t *g, int32_t sink, int32_t blocked, int64_t *e, int64_t *stats) {
    int32_t n = g->n;
    int32_t *h = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int64_t *cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    int64_t *cur = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int32_t *q = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *fifo = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    uint8_t *inq = (uint8_t *)calloc((size_t)n, 1);
    int64_t fh = 0, fcount = 0;
    int64_t work_since_gr = 0, gr_period = 6 * (int64_t)n + g->na / 2;
    pr_global_relabel(g, sink, blocked, h, cnt, q);
    for (int32_t v = 0; v < n; v++) cur[v] = g->first[v];
#define PUSHQ(v) do { fifo[(fh + fcount) % n] = (v); fcount++; inq[v] = 1; } while (0)
    for (int32_t v = 0; v < n; v++)
        if (v != sink && v != blocked && e[v] > 0 && h[v] < n) PUSHQ(v);
    while (fcount > 0) {
        int32_t x = fifo[fh]; fh = (fh + 1) % n; fcount--; inq[x] = 0;
        if (h[x] >= n) continue;
        while (e[x] > 0) {
            int64_t a = cur[x];
            if (a == g->first[x + 1]) {
                /* relabel */
                int32_t old = h[x], mh = n;
                for (int64_t b = g->first[x]; b < g->first[x + 1]; b++)
                    if (g->res[b] > 0 && h[g->head[b]] < mh) mh = h[g->head[b]];
                int32_t nh = mh + 1 < n ? mh + 1 : n;
                cnt[old]--; h[x] = nh; cnt[nh]++;
                cur[x] = g->first[x];
                if (stats) stats[1]++;
                work_since_gr += 12 + (g->first[x + 1] - g->first[x]);
                if (cnt[old] == 0 && old < n) {           /* gap: nobody above `old` reaches the sink */
                    for (int32_t v = 0; v < n; v++)
                        if (h[v] > old && h[v] < n) { cnt[h[v]]--; h[v] = n; cnt[n]++; }
                    if (stats) stats[2]++;
                }
                if (h[x] >= n) break;
                continue;
            }
            int32_t y = g->head[a];
            if (g->res[a] > 0 && h[x] == h[y] + 1) {
                int64_t d = e[x] < g->res[a] ? e[x] : g->res[a];
                g->res[a] -= d; g->res[g->pair[a]] += d;
                e[x] -= d; e[y] += d;
                if (stats) stats[0]++;
                if (y != sink && y != blocked && !inq[y] && h[y] < n) PUSHQ(y);
            } else {
                cur[x]++;
            }
        }
        if (work_since_gr > gr_period) {
            pr_global_relabel(g, sink, blocked, h, cnt, q);
            for (int32_t v = 0; v < n; v++) cur[v] = g->first[v];
            work_since_gr = 0;
            if (stats) stats[3]++;
            /* re-seed the queue: heights changed wholesale */
            fh = 0; fcount = 0;
            for (int32_t v = 0; v < n; v++) inq[v] = 0;
            for (int32_t v = 0; v < n; v++)
                if (v != sink && v != blocked && e[v] > 0 && h[v] < n) PUSHQ(v);
        }
    }
#undef PUSHQ
    free(h); free(cnt); free(cur); free(q); free(fifo); free(inq);
}

static int64_t maxflow_fifo_pr(net_t *g, int32_t s, int32_t t, int64_t *stats) {
    int32_t n = g->n;
    int64_t *e = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    for (int64_t a = g->first[s]; a < g->first[s + 1]; a++) {      /* saturate s's arcs */
        int64_t r = g->res[a];
        if (r > 0 && g->head[a] != s) { g->res[a] = 0; g->res[g->pair[a]] += r; e[g->head[a]] += r; e[s] -= r; }
    }
    pr_phase(g, t, s, e, stats);            /* phase 1: maximum preflow */
    pr_phase(g, s, t, e, stats);            /* phase 2: stuck excess back to s */
    int64_t F = e[t];
    for (int32_t v = 0; v < n; v++)
        if (v != s && v != t && e[v] != 0) { F = INT64_MIN; break; }   /* must be a true flow */
    free(e);
    return F;
}

/* ---------------------------------------------------------------- public: max flow */

/* algo: ORC_EK / ORC_DINIC / ORC_FIFO_PR.  Outputs (nullable): smin[n], smax[n]
 * (1 = in the source side), flow[m] = flow on input edge j (0 for self-loops),
 * stats[4] = {pushes, relabels, gaps, global relabels} (FIFO_PR only).
 * Returns F >= 0, or a negative value on error. */
int64_t orc_maxflow(int32_t algo, int32_t n, int64_t m, const int32_t *u, const int32_t *v,
                    const int32_t *cap, int32_t s, int32_t t, uint8_t *smin, uint8_t *smax,
                    int64_t *flow, int64_t *stats) {
    if (n <= 0 || s < 0 || t < 0 || s >= n || t >= n || s == t) return -1;
    for (int64_t j = 0; j < m; j++)
        if (u[j] < 0 || u[j] >= n || v[j] < 0 || v[j] >= n || cap[j] < 0) return -1;
    net_t g;
    int64_t *earc = flow ? (int64_t *)malloc((size_t)(m ? m : 1) * sizeof(int64_t)) : NULL;
    if (net_from_edges(&g, n, m, u, v, cap, earc) != 0) { free(earc); return -2; }
    int64_t F;
    if (algo == ORC_EK) F = maxflow_ek(&g, s, t);
    else if (algo == ORC_DINIC) F = maxflow_dinic(&g, s, t);
    else if (algo == ORC_FIFO_PR) F = maxflow_fifo_pr(&g, s, t, stats);
    else { net_free(&g); free(earc); return -1; }
    if (F >= 0) {
        cuts_of_flow(&g, s, t, smin, smax);
        if (flow) for (int64_t j = 0; j < m; j++) flow[j] = earc[j] < 0 ? 0 : (int64_t)cap[j] - g.res[earc[j]];
    }
    net_free(&g); free(earc);
    return F;
}

/* ---------------------------------------------------------------- Hopcroft-Karp */
/* Maximum matching in a bipartite graph (left 0..nl-1, right 0..nr-1), edges
 * (l[j], r[j]).  Textbook phases: BFS layering from free left vertices, then
 * vertex-disjoint shortest augmenting paths by DFS (iterative). */
int64_t orc_hopcroft_karp(int32_t nl, int32_t nr, int64_t m, const int32_t *l, const int32_t *r) {
    int64_t *first = (int64_t *)calloc((size_t)nl + 1, sizeof(int64_t));
    int32_t *adj = (int32_t *)malloc((size_t)(m ? m : 1) * sizeof(int32_t));
    for (int64_t j = 0; j < m; j++) first[l[j] + 1]++;
    for (int32_t x = 0; x < nl; x++) first[x + 1] += first[x];
    int64_t *fill = (int64_t *)malloc(((size_t)nl + 1) * sizeof(int64_t));
    memcpy(fill, first, ((size_t)nl + 1) * sizeof(int64_t));
    for (int64_t j = 0; j < m; j++) adj[fill[l[j]]++] = r[j];
    free(fill);
    int32_t *ml = (int32_t *)malloc((size_t)nl * sizeof(int32_t));
    int32_t *mr = (int32_t *)malloc((size_t)nr * sizeof(int32_t));
    int32_t *dist = (int32_t *)malloc((size_t)nl * sizeof(int32_t));
    int32_t *q = (int32_t *)malloc((size_t)nl * sizeof(int32_t));
    int64_t *it = (int64_t *)malloc((size_t)nl * sizeof(int64_t));
    int32_t *stk = (int32_t *)malloc(((size_t)nl + 1) * sizeof(int32_t));
    for (int32_t x = 0; x < nl; x++) ml[x] = -1;
    for (int32_t y = 0; y < nr; y++) mr[y] = -1;
    int64_t matching = 0;
    const int32_t INF = INT32_MAX;
    for (;;) {
        int64_t qh = 0, qt = 0;
        int32_t found = INF;
        for (int32_t x = 0; x < nl; x++) { if (ml[x] < 0) { dist[x] = 0; q[qt++] = x; } else dist[x] = INF; }
        while (qh < qt) {
            int32_t x = q[qh++];
            if (dist[x] >= found) continue;
            for (int64_t a = first[x]; a < first[x + 1]; a++) {
                int32_t y = adj[a], x2 = mr[y];
                if (x2 < 0) { if (found == INF) found = dist[x] + 1; }
                else if (dist[x2] == INF) { dist[x2] = dist[x] + 1; q[qt++] = x2; }
            }
        }
        if (found == INF) break;
        for (int32_t x = 0; x < nl; x++) it[x] = first[x];
        for (int32_t x0 = 0; x0 < nl; x0++) {
            if (ml[x0] >= 0) continue;
            int64_t sp = 0;
            stk[sp++] = x0;
            int done = 0;
            while (sp > 0 && !done) {
                int32_t x = stk[sp - 1];
                int advanced = 0;
                for (; it[x] < first[x + 1]; it[x]++) {
                    int32_t y = adj[it[x]], x2 = mr[y];
                    if (x2 < 0) {
                        if (dist[x] + 1 == found) {          /* augment along the stack */
                            for (int64_t i = sp - 1; i >= 0; i--) {
                                int32_t xi = stk[i];
                                int32_t yi = adj[it[xi]];
                                int32_t prev = ml[xi];
                                ml[xi] = yi; mr[yi] = xi;
                                (void)prev;
                            }
                            matching++;
                            done = 1;
                            break;
                        }
                    } else if (dist[x2] == dist[x] + 1) {
                        stk[sp++] = x2; advanced = 1; break;
                    }
                }
                if (done) break;
                if (!advanced) { dist[x] = INF; sp--; if (sp > 0) it[stk[sp - 1]]++; }
            }
        }
    }
    free(first); free(adj); free(ml); free(mr); free(dist); free(q); free(it); free(stk);
    return matching;
}

/* ---------------------------------------------------------------- state checker */
/* Checks a solver state given in "slot" form (any implementation's export):
 * row_ptr[n+1] (int64), dst[S], rev[S], cap[S], res[S] (int32), e[n] (int64),
 * claimed flow value F and claimed minimal source side smin[n] (nullable).
 * Returns 0 if every check passes, else a positive check id; msg gets a line.
 *   1 structure: rev involution, endpoints consistent, no self-loop slots
 *   2 capacity: 0 <= res[i] <= cap[i] + cap[rev i]
 *   3 pair-sum: res[i] + res[rev i] == cap[i] + cap[rev i]
 *   4 excess consistency: e(v) == sum over slots i into v of (cap[i]-res[i]); sum e == 0
 *   5 no augmenting path: no residual path from {s} u Exc to {t} u Def
 *   6 conversion to a true flow failed (excess cannot all return to s, or deficits
 *     cannot all be filled from t)
 *   7 converted flow violates capacity / conservation, or its value != F
 *   8 smin != reach from s in the converted (true, maximum) flow's residual graph
 *   9 cut capacity of smin != F
 * `out_flow` (nullable, S) receives the converted flow's residuals. */
int orc_check_state(int32_t n, int64_t S, const int64_t *row_ptr, const int32_t *dst, const int32_t *rev,
                    const int32_t *cap, const int32_t *res, const int64_t *e, int32_t s, int32_t t,
                    int64_t F, const uint8_t *smin, char *msg, int32_t msglen, int32_t *out_res) {
    int rc = 0;
#define FAIL(code, ...) do { rc = (code); if (msg && msglen > 0) snprintf(msg, (size_t)msglen, __VA_ARGS__); goto out; } while (0)
    int32_t *owner = (int32_t *)malloc((size_t)(S ? S : 1) * sizeof(int32_t));
    uint8_t *roots = (uint8_t *)calloc((size_t)n + 2, 1);
    uint8_t *mark = (uint8_t *)calloc((size_t)n + 2, 1);
    int64_t *ecalc = (int64_t *)calloc((size_t)n, sizeof(int64_t));
    int32_t *tl = NULL, *hd = NULL; int64_t *rs = NULL, *pr = NULL;
    net_t g; memset(&g, 0, sizeof(g));
    if (row_ptr[0] != 0 || row_ptr[n] != S) FAIL(1, "row_ptr ends %lld..%lld, S=%lld", (long long)row_ptr[0], (long long)row_ptr[n], (long long)S);
    for (int32_t x = 0; x < n; x++) {
        if (row_ptr[x + 1] < row_ptr[x]) FAIL(1, "row_ptr decreasing at %d", x);
        for (int64_t i = row_ptr[x]; i < row_ptr[x + 1]; i++) owner[i] = x;
    }
    for (int64_t i = 0; i < S; i++) {
        if (dst[i] < 0 || dst[i] >= n || rev[i] < 0 || rev[i] >= S) FAIL(1, "slot %lld out of range", (long long)i);
        if (rev[rev[i]] != i) FAIL(1, "rev not an involution at %lld", (long long)i);
        if (dst[rev[i]] != owner[i] || owner[rev[i]] != dst[i]) FAIL(1, "rev endpoints wrong at %lld", (long long)i);
        if (dst[i] == owner[i]) FAIL(1, "self-loop slot %lld", (long long)i);
    }
    for (int64_t i = 0; i < S; i++) {
        int64_t pc = (int64_t)cap[i] + cap[rev[i]];
        if (res[i] < 0 || res[i] > pc) FAIL(2, "res[%lld]=%d outside [0,%lld]", (long long)i, res[i], (long long)pc);
        if ((int64_t)res[i] + res[rev[i]] != pc) FAIL(3, "pair-sum broken at slot %lld", (long long)i);
    }
    for (int64_t i = 0; i < S; i++) ecalc[dst[i]] += (int64_t)cap[i] - res[i];
    {
        int64_t tot = 0;
        for (int32_t x = 0; x < n; x++) {
            if (ecalc[x] != e[x]) FAIL(4, "e[%d]=%lld but net inflow %lld", x, (long long)e[x], (long long)ecalc[x]);
            tot += e[x];
        }
        if (tot != 0) FAIL(4, "sum of excess %lld != 0", (long long)tot);
    }
    /* network on the slots: arc i = slot i, residual res[i], pair rev[i]; plus a
     * super node n (sigma / tau) and its arcs, appended later. */
    int64_t nexc = 0, ndef = 0;
    for (int32_t x = 0; x < n; x++) if (x != s && x != t) { if (e[x] > 0) nexc++; else if (e[x] < 0) ndef++; }
    int64_t na = S + 2 * (nexc + ndef);
    tl = (int32_t *)malloc((size_t)(na ? na : 1) * sizeof(int32_t));
    hd = (int32_t *)malloc((size_t)(na ? na : 1) * sizeof(int32_t));
    rs = (int64_t *)malloc((size_t)(na ? na : 1) * sizeof(int64_t));
    pr = (int64_t *)malloc((size_t)(na ? na : 1) * sizeof(int64_t));
    for (int64_t i = 0; i < S; i++) { tl[i] = owner[i]; hd[i] = dst[i]; rs[i] = res[i]; pr[i] = rev[i]; }
    /* check 5 on the plain residual graph (super arcs added with zero capacity) */
    int64_t a = S;
    int32_t SUP = n;
    for (int32_t x = 0; x < n; x++) {
        if (x == s || x == t || e[x] == 0) continue;
        if (e[x] > 0) { tl[a] = SUP; hd[a] = x; }   /* sigma -> excess vertex */
        else { tl[a] = x; hd[a] = SUP; }            /* deficit vertex -> tau */
        rs[a] = 0; pr[a] = a + 1;
        tl[a + 1] = hd[a]; hd[a + 1] = tl[a]; rs[a + 1] = 0; pr[a + 1] = a;
        a += 2;
    }
    if (net_from_arcs(&g, n + 1, na, tl, hd, rs, pr) != 0) FAIL(6, "out of memory");
    for (int32_t x = 0; x < n; x++) roots[x] = (x == s) || (x != t && e[x] > 0);
    roots[n] = 0;
    reach_forward(&g, roots, mark);
    if (mark[t]) FAIL(5, "augmenting path from {s}+excess to t");
    for (int32_t x = 0; x < n; x++)
        if (x != s && x != t && e[x] < 0 && mark[x]) FAIL(5, "augmenting path from {s}+excess to deficit %d", x);
    /* conversion (1): route each excess back to s.  sigma->x arcs get capacity e(x). */
    {
        int64_t want = 0;
        for (int64_t p = 0; p < g.na; p++) {
            int64_t o = g.orig[p];
            if (o >= S && ((o - S) & 1) == 0 && tl[o] == SUP) { g.res[p] = e[hd[o]]; want += e[hd[o]]; }
        }
        int64_t got = maxflow_dinic(&g, SUP, s);
        if (got != want) FAIL(6, "only %lld of %lld excess returns to s", (long long)got, (long long)want);
        for (int64_t p = 0; p < g.na; p++) if (g.orig[p] >= S) g.res[p] = 0;  /* retire sigma arcs */
    }
    /* conversion (2): fill each deficit from t.  x->tau arcs get capacity -e(x). */
    {
        int64_t want = 0;
        for (int64_t p = 0; p < g.na; p++) {
            int64_t o = g.orig[p];
            if (o >= S && ((o - S) & 1) == 0 && hd[o] == SUP) { g.res[p] = -e[tl[o]]; want += -e[tl[o]]; }
        }
        int64_t got = maxflow_dinic(&g, t, SUP);
        if (got != want) FAIL(6, "only %lld of %lld deficit is filled from t", (long long)got, (long long)want);
        for (int64_t p = 0; p < g.na; p++) if (g.orig[p] >= S) g.res[p] = 0;
    }
    /* converted flow: residual per slot */
    int32_t *r2 = (int32_t *)malloc((size_t)(S ? S : 1) * sizeof(int32_t));
    for (int64_t p = 0; p < g.na; p++) if (g.orig[p] < S) r2[g.orig[p]] = (int32_t)g.res[p];
    memset(ecalc, 0, (size_t)n * sizeof(int64_t));
    for (int64_t i = 0; i < S; i++) {
        int64_t pc = (int64_t)cap[i] + cap[rev[i]];
        if (r2[i] < 0 || r2[i] > pc || (int64_t)r2[i] + r2[rev[i]] != pc) { free(r2); FAIL(7, "converted flow violates capacity at slot %lld", (long long)i); }
        ecalc[dst[i]] += (int64_t)cap[i] - r2[i];
    }
    for (int32_t x = 0; x < n; x++)
        if (x != s && x != t && ecalc[x] != 0) { free(r2); FAIL(7, "converted flow not conserved at %d (%lld)", x, (long long)ecalc[x]); }
    if (ecalc[t] != F || ecalc[s] != -F) { free(r2); FAIL(7, "converted flow value %lld != F %lld", (long long)ecalc[t], (long long)F); }
    if (out_res) memcpy(out_res, r2, (size_t)S * sizeof(int32_t));
    /* S_min of the true maximum flow */
    for (int64_t p = 0; p < g.na; p++) g.res[p] = g.orig[p] < S ? r2[g.orig[p]] : 0;
    free(r2);
    memset(roots, 0, (size_t)n + 1);
    roots[s] = 1;
    reach_forward(&g, roots, mark);
    if (smin) {
        for (int32_t x = 0; x < n; x++)
            if ((smin[x] != 0) != (mark[x] != 0)) FAIL(8, "smin[%d]=%d but reach-from-s says %d", x, smin[x], mark[x]);
        int64_t cc = 0;
        for (int64_t i = 0; i < S; i++) if (smin[owner[i]] && !smin[dst[i]]) cc += cap[i];
        if (cc != F) FAIL(9, "cut capacity of smin %lld != F %lld", (long long)cc, (long long)F);
    }
out:
    free(owner); free(roots); free(mark); free(ecalc); free(tl); free(hd); free(rs); free(pr);
    net_free(&g);
    return rc;
#undef FAIL
}
