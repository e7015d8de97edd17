/*
 * oracle.c -- CPU restatement of the reference rcpsp_tabu hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links or calls
 * this file; only tests/, __graft_entry__.smoke() and bench.py's CPU legs
 * (`cpu_baseline`, `--impl reference`) load it, as the checker / the timed
 * CPU arm.  It restates, function by function, the numba kernels and the
 * host-side search loop of the reference package (`/root/reference/pkg/src/
 * rcpsp_tabu/`, cited below as kernels.py:L, search.py:L, ...).  Parity is
 * pinned by tests/test_oracle.py against golden vectors generated from the
 * reference itself (tests/golden/make_golden.py).
 *
 * Conventions follow the reference: int32 arrays, activity ids 0..N-1,
 * demands row-major [N][M], mode 0 = CAPACITY, 1 = TIME (kernels.py:22-23).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define MODE_CAPACITY 0
#define MODE_TIME 1

/* ------------------------------------------------------------------------ */
/* numpy Generator(PCG64) replica (numpy 2.x: pcg64.h, distributions.c).    */

typedef unsigned __int128 u128;
typedef struct {
    u128 state, inc;
    int has32;
    uint32_t u32;
} pcg64_t;

static const u128 PCG_MULT =
    (((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL;

static uint64_t pcg_next64(pcg64_t *g) {
    g->state = g->state * PCG_MULT + g->inc;
    uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
    unsigned rot = (unsigned)(g->state >> 122);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

static uint32_t pcg_next32(pcg64_t *g) {
    if (g->has32) {
        g->has32 = 0;
        return g->u32;
    }
    uint64_t v = pcg_next64(g);
    g->has32 = 1;
    g->u32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
}

/* Generator.integers(n) for 1 <= n <= 2^32 (Lemire, bitgen next_uint32). */
static int64_t pcg_integers(pcg64_t *g, int64_t n) {
    uint32_t rng = (uint32_t)(n - 1);
    if (rng == 0) return 0;
    uint32_t excl = rng + 1u;
    uint64_t m = (uint64_t)pcg_next32(g) * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
        uint32_t thr = (0xFFFFFFFFu - rng) % excl;
        while (left < thr) {
            m = (uint64_t)pcg_next32(g) * excl;
            left = (uint32_t)m;
        }
    }
    return (int64_t)(m >> 32);
}

/* random_interval(max) used by Generator.shuffle / permutation. */
static uint32_t pcg_interval(pcg64_t *g, uint32_t mx) {
    if (mx == 0) return 0;
    uint32_t mask = mx;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16;
    uint32_t v;
    while ((v = (pcg_next32(g) & mask)) > mx) {
    }
    return v;
}

static void pcg_permute(pcg64_t *g, int32_t *a, int n) {
    for (int i = n - 1; i >= 1; --i) {
        uint32_t j = pcg_interval(g, (uint32_t)i);
        int32_t t = a[i]; a[i] = a[j]; a[j] = t;
    }
}

static void pcg_load(pcg64_t *g, const uint64_t *s) {
    /* s = {state_hi, state_lo, inc_hi, inc_lo, has32, u32} */
    g->state = (((u128)s[0]) << 64) | (u128)s[1];
    g->inc = (((u128)s[2]) << 64) | (u128)s[3];
    g->has32 = (int)s[4];
    g->u32 = (uint32_t)s[5];
}

static void pcg_store(const pcg64_t *g, uint64_t *s) {
    s[0] = (uint64_t)(g->state >> 64); s[1] = (uint64_t)g->state;
    s[2] = (uint64_t)(g->inc >> 64); s[3] = (uint64_t)g->inc;
    s[4] = (uint64_t)g->has32; s[5] = g->u32;
}

/* exported for the RNG parity test */
int64_t oracle_pcg_integers(uint64_t *s, int64_t n) {
    pcg64_t g; pcg_load(&g, s);
    int64_t r = pcg_integers(&g, n);
    pcg_store(&g, s);
    return r;
}

void oracle_pcg_permute(uint64_t *s, int32_t *a, int n) {
    pcg64_t g; pcg_load(&g, s);
    pcg_permute(&g, a, n);
    pcg_store(&g, s);
}

/* ------------------------------------------------------------------------ */
/* Resource states and serial SGS (kernels.py:68-194).                      */

/* kernels.py:68-78 */
int oracle_cap_earliest_start(const int32_t *cap_state, int r_max, const int32_t *caps, int m,
                              const int32_t *dem, int act) {
    int es = 0;
    for (int k = 0; k < m; ++k) {
        int req = dem[act * m + k];
        if (req > 0) {
            int t = cap_state[k * r_max + caps[k] - req];
            if (t > es) es = t;
        }
    }
    return es;
}

/* kernels.py:81-110 (Alg. 4 shifted copy, quirks preserved) */
void oracle_cap_update(int32_t *cap_state, int r_max, const int32_t *caps, int m,
                       const int32_t *dem, int32_t *copy_buf, int act, int start, int dur) {
    for (int k = 0; k < m; ++k) {
        int req = dem[act * m + k];
        int effort = req * dur;
        if (effort > 0) {
            int32_t *c = cap_state + k * r_max;
            int res_idx = 0, copy_idx = 0;
            int new_time = start + dur;
            while (effort > 0 && res_idx < caps[k]) {
                if (c[res_idx] < new_time) {
                    if (copy_idx >= req) new_time = copy_buf[copy_idx - req];
                    int floor_ = c[res_idx];
                    if (floor_ < start) floor_ = start;
                    int diff = new_time - floor_;
                    if (effort - diff > 0) {
                        effort -= diff;
                        copy_buf[copy_idx] = c[res_idx];
                        copy_idx += 1;
                        c[res_idx] = new_time;
                    } else {
                        c[res_idx] = floor_ + effort;
                        effort = 0;
                    }
                }
                res_idx += 1;
            }
        }
    }
}

/* kernels.py:117-136 ; tau is [m][horizon+1] */
int oracle_time_earliest_start(const int32_t *tau, int hp1, int m, const int32_t *dem, int act,
                               int es_prec, int dur, int horizon) {
    int load = 0, t = es_prec;
    while (t < horizon && load < dur) {
        int enough = 1;
        for (int k = 0; k < m; ++k)
            if (tau[k * hp1 + t] < dem[act * m + k]) { load = 0; enough = 0; }
        if (enough) load += 1;
        t += 1;
    }
    return t - load;
}

/* kernels.py:139-146 */
void oracle_time_update(int32_t *tau, int hp1, int m, const int32_t *dem, int act, int start,
                        int dur) {
    for (int k = 0; k < m; ++k) {
        int req = dem[act * m + k];
        if (req > 0)
            for (int t = start; t < start + dur; ++t) tau[k * hp1 + t] -= req;
    }
}

typedef struct {
    int n, m, horizon, r_max;
    const int32_t *dur, *dem, *cap, *pred_ptr, *pred_dat, *succ_ptr, *succ_dat;
    const uint8_t *adj; /* n*n, adj[i*n+j] = edge i->j */
    const int32_t *lvl_ptr, *lvl_dat;
    int n_levels;
    int cpm;
} oinst_t;

typedef struct {
    int32_t *starts, *cap_state, *copy_buf, *tau;
    long evaluations;
} oscratch_t;

/* kernels.py:152-194 */
static int evaluate_order_raw(const int32_t *order, const oinst_t *I, const int32_t *pred_ptr,
                              const int32_t *pred_dat, int mode, oscratch_t *S, int reset_upto) {
    int n = I->n, m = I->m, hp1 = I->horizon + 1;
    if (mode == MODE_CAPACITY) {
        memset(S->cap_state, 0, sizeof(int32_t) * (size_t)m * I->r_max);
    } else {
        int top = reset_upto < I->horizon ? reset_upto : I->horizon;
        for (int k = 0; k < m; ++k)
            for (int t = 0; t <= top; ++t) S->tau[k * hp1 + t] = I->cap[k];
    }
    int cmax = 0;
    for (int pos = 0; pos < n; ++pos) {
        int act = order[pos];
        int dur = I->dur[act];
        int es_prec = 0;
        for (int e = pred_ptr[act]; e < pred_ptr[act + 1]; ++e) {
            int p = pred_dat[e];
            int fin = S->starts[p] + I->dur[p];
            if (fin > es_prec) es_prec = fin;
        }
        int start;
        if (mode == MODE_CAPACITY) {
            int es_res = oracle_cap_earliest_start(S->cap_state, I->r_max, I->cap, m, I->dem, act);
            start = es_prec > es_res ? es_prec : es_res;
            oracle_cap_update(S->cap_state, I->r_max, I->cap, m, I->dem, S->copy_buf, act, start,
                              dur);
        } else {
            start = oracle_time_earliest_start(S->tau, hp1, m, I->dem, act, es_prec, dur,
                                               I->horizon);
            oracle_time_update(S->tau, hp1, m, I->dem, act, start, dur);
        }
        S->starts[act] = start;
        int fin = start + dur;
        if (fin > cmax) cmax = fin;
    }
    return cmax;
}

static int scratch_alloc(oscratch_t *S, const oinst_t *I) {
    S->starts = calloc((size_t)I->n, sizeof(int32_t));
    S->cap_state = calloc((size_t)I->m * (I->r_max > 0 ? I->r_max : 1), sizeof(int32_t));
    S->copy_buf = calloc((size_t)(I->r_max > 0 ? I->r_max : 1), sizeof(int32_t));
    S->tau = calloc((size_t)I->m * (I->horizon + 1), sizeof(int32_t));
    S->evaluations = 0;
    return (S->starts && S->cap_state && S->copy_buf && S->tau) ? 0 : -1;
}

static void scratch_free(oscratch_t *S) {
    free(S->starts); free(S->cap_state); free(S->copy_buf); free(S->tau);
}

static void inst_fill(oinst_t *I, int n, int m, int horizon, const int32_t *dur, const int32_t *dem,
                      const int32_t *cap, const int32_t *pred_ptr, const int32_t *pred_dat,
                      const int32_t *succ_ptr, const int32_t *succ_dat) {
    memset(I, 0, sizeof(*I));
    I->n = n; I->m = m; I->horizon = horizon;
    I->dur = dur; I->dem = dem; I->cap = cap;
    I->pred_ptr = pred_ptr; I->pred_dat = pred_dat; I->succ_ptr = succ_ptr; I->succ_dat = succ_dat;
    int r = 1;
    for (int k = 0; k < m; ++k) if (cap[k] > r) r = cap[k];
    I->r_max = r;
}

/* Batch evaluation: B orders (B x n) -> cmax[B] (+ starts B x n if non-NULL).
 * `use_succ` evaluates on the reversed project (preds = successor lists), as
 * forward_backward_improve's eval_backward does (evaluator.py:234-242). */
int oracle_evaluate_batch(int n, int m, int horizon, const int32_t *dur, const int32_t *dem,
                          const int32_t *cap, const int32_t *pred_ptr, const int32_t *pred_dat,
                          const int32_t *succ_ptr, const int32_t *succ_dat, const int32_t *orders,
                          int B, int mode, int use_succ, int32_t *cmax, int32_t *starts) {
    oinst_t I;
    inst_fill(&I, n, m, horizon, dur, dem, cap, pred_ptr, pred_dat, succ_ptr, succ_dat);
    oscratch_t S;
    if (scratch_alloc(&S, &I)) return -1;
    for (int b = 0; b < B; ++b) {
        cmax[b] = evaluate_order_raw(orders + (size_t)b * n, &I, use_succ ? succ_ptr : pred_ptr,
                                     use_succ ? succ_dat : pred_dat, mode, &S, horizon);
        if (starts) memcpy(starts + (size_t)b * n, S.starts, sizeof(int32_t) * n);
    }
    scratch_free(&S);
    return 0;
}

/* Touch counter of one evaluation (BASELINE.md sec. 2.7 / SURVEY 8d):
 * instance loads N(1+M) + order reads/starts writes 2N + 2 per pred edge;
 * TIME: M per scanned step + 2*d per resource with r>0 + M*(top+1) reset;
 * CAP: 1 per resource with r>0 for es; per visited c-entry 1 read (+1 copy
 * read when copy_idx >= r) and 2 writes (1 on the final entry); M*R_max reset.
 * Returns W (element touches) for the order. */
long oracle_touches(int n, int m, int horizon, const int32_t *dur, const int32_t *dem,
                    const int32_t *cap, const int32_t *pred_ptr, const int32_t *pred_dat,
                    const int32_t *order, int mode, int reset_upto, long *scan_steps) {
    oinst_t I;
    inst_fill(&I, n, m, horizon, dur, dem, cap, pred_ptr, pred_dat, pred_ptr, pred_dat);
    oscratch_t S;
    if (scratch_alloc(&S, &I)) return -1;
    int hp1 = horizon + 1;
    long w = (long)n * (1 + m) + 2L * n + 2L * pred_ptr[n];
    long steps = 0;
    if (mode == MODE_CAPACITY) {
        w += (long)m * I.r_max;
    } else {
        int top = reset_upto < horizon ? reset_upto : horizon;
        w += (long)m * (top + 1);
        for (int k = 0; k < m; ++k)
            for (int t = 0; t < hp1; ++t) S.tau[k * hp1 + t] = cap[k];
    }
    for (int pos = 0; pos < n; ++pos) {
        int act = order[pos], d = dur[act], es_prec = 0;
        for (int e = pred_ptr[act]; e < pred_ptr[act + 1]; ++e) {
            int p = pred_dat[e];
            int fin = S.starts[p] + dur[p];
            if (fin > es_prec) es_prec = fin;
        }
        int start;
        if (mode == MODE_CAPACITY) {
            int es_res = 0;
            for (int k = 0; k < m; ++k) {
                int req = dem[act * m + k];
                if (req > 0) {
                    w += 1;
                    int t = S.cap_state[k * I.r_max + cap[k] - req];
                    if (t > es_res) es_res = t;
                }
            }
            start = es_prec > es_res ? es_prec : es_res;
            for (int k = 0; k < m; ++k) {
                int req = dem[act * m + k], effort = req * d;
                if (effort <= 0) continue;
                int32_t *c = S.cap_state + k * I.r_max;
                int res_idx = 0, copy_idx = 0, new_time = start + d;
                while (effort > 0 && res_idx < cap[k]) {
                    w += 1;
                    if (c[res_idx] < new_time) {
                        if (copy_idx >= req) { new_time = S.copy_buf[copy_idx - req]; w += 1; }
                        int fl = c[res_idx] < start ? start : c[res_idx];
                        int diff = new_time - fl;
                        if (effort - diff > 0) {
                            effort -= diff; S.copy_buf[copy_idx++] = c[res_idx]; c[res_idx] = new_time;
                            w += 2;
                        } else {
                            c[res_idx] = fl + effort; effort = 0; w += 1;
                        }
                    }
                    res_idx += 1;
                }
            }
        } else {
            int load = 0, t = es_prec;
            while (t < horizon && load < d) {
                int enough = 1;
                for (int k = 0; k < m; ++k)
                    if (S.tau[k * hp1 + t] < dem[act * m + k]) { load = 0; enough = 0; }
                w += m; steps += 1;
                if (enough) load += 1;
                t += 1;
            }
            start = t - load;
            for (int k = 0; k < m; ++k) {
                int req = dem[act * m + k];
                if (req > 0) {
                    for (int tt = start; tt < start + d; ++tt) S.tau[k * hp1 + tt] -= req;
                    w += 2L * d;
                }
            }
        }
        S.starts[act] = start;
    }
    if (scan_steps) *scan_steps = steps;
    scratch_free(&S);
    return w;
}

/* ------------------------------------------------------------------------ */
/* Moves, tabu, selection (kernels.py:200-309).                             */

/* kernels.py:218-255 (two-phase stable compaction) */
static int filter_moves_raw(const uint8_t *adj, int n, const int32_t *order, const int32_t *moves,
                            int n_moves, int32_t *out) {
    int kept = 0;
    for (int idx = 0; idx < n_moves; ++idx) {
        int u = moves[2 * idx], v = moves[2 * idx + 1];
        int wu = order[u], ok = 1;
        for (int x = u + 1; x <= v; ++x)
            if (adj[wu * n + order[x]]) { ok = 0; break; }
        if (ok) { out[2 * kept] = u; out[2 * kept + 1] = v; kept++; }
    }
    int fin = 0;
    for (int idx = 0; idx < kept; ++idx) {
        int u = out[2 * idx], v = out[2 * idx + 1];
        int wv = order[v], ok = 1;
        for (int x = u; x < v; ++x)
            if (adj[order[x] * n + wv]) { ok = 0; break; }
        if (ok) { out[2 * fin] = u; out[2 * fin + 1] = v; fin++; }
    }
    return fin;
}

int oracle_filter_moves(const uint8_t *adj, int n, const int32_t *order, const int32_t *moves,
                        int n_moves, int32_t *out) {
    return filter_moves_raw(adj, n, order, moves, n_moves, out);
}

/* kernels.py:263-277 ; counts is n x n */
static int tabu_add_raw(int32_t *list, int T, int32_t *counts, int n, int head, int u, int v) {
    int ou = list[2 * head], ov = list[2 * head + 1];
    if (ou != 0 || ov != 0) counts[ou * n + ov] -= 1;
    list[2 * head] = u; list[2 * head + 1] = v;
    counts[u * n + v] += 1;
    return (head + 1) % T;
}

int oracle_tabu_add(int32_t *list, int T, int32_t *counts, int n, int head, int u, int v) {
    return tabu_add_raw(list, T, counts, n, head, u, v);
}

/* kernels.py:280-297 */
static int select_move_raw(const int32_t *moves, int n_moves, const int32_t *cmax,
                           const int32_t *counts, int n, int asp) {
    int best_idx = -1, best_c = 0;
    for (int idx = 0; idx < n_moves; ++idx) {
        int c = cmax[idx];
        if (counts[moves[2 * idx] * n + moves[2 * idx + 1]] > 0 && c >= asp) continue;
        if (best_idx < 0 || c < best_c) { best_idx = idx; best_c = c; }
    }
    return best_idx;
}

int oracle_select_move(const int32_t *moves, int n_moves, const int32_t *cmax,
                       const int32_t *counts, int n, int asp) {
    return select_move_raw(moves, n_moves, cmax, counts, n, asp);
}

/* kernels.py:300-309 */
static int select_min_raw(int n_moves, const int32_t *cmax) {
    int best_idx = -1, best_c = 0;
    for (int idx = 0; idx < n_moves; ++idx)
        if (best_idx < 0 || cmax[idx] < best_c) { best_idx = idx; best_c = cmax[idx]; }
    return best_idx;
}

int oracle_select_min(int n_moves, const int32_t *cmax) { return select_min_raw(n_moves, cmax); }

/* moves.py:60-72: all (u, v), 1 <= u < v <= n-2, v-u <= delta, lex sorted */
static int32_t *gen_neighborhood(int n, int delta, int *count) {
    int c = 0;
    for (int u = 1; u < n - 2; ++u)
        for (int v = u + 1; v <= (u + delta < n - 2 ? u + delta : n - 2); ++v) c++;
    int32_t *mv = malloc(sizeof(int32_t) * 2 * (size_t)(c > 0 ? c : 1));
    int i = 0;
    for (int u = 1; u < n - 2; ++u)
        for (int v = u + 1; v <= (u + delta < n - 2 ? u + delta : n - 2); ++v) {
            mv[2 * i] = u; mv[2 * i + 1] = v; i++;
        }
    *count = c;
    return mv;
}

/* kernels.py:316-385 ; returns the 7-tuple in out7 */
static void run_chunk_raw(int32_t *order, const oinst_t *I, const int32_t *moves_all, int n_all,
                          int mode, int32_t *tabu_list, int T, int32_t *tabu_count, int *tabu_head,
                          int budget, int adopted_cmax, int start_cmax, int best_known_cmax,
                          int floor_cmax, int32_t *best_order, oscratch_t *S, int32_t *moves_buf,
                          int32_t *cmax_buf, int32_t *trace, long out7[7]) {
    int n = I->n;
    int local_best = start_cmax, cur = start_cmax;
    long iters = 0, evals = 0, forced = 0;
    int touched = I->horizon;
    int head = *tabu_head;
    for (int it = 0; it < budget; ++it) {
        int n_feas = filter_moves_raw(I->adj, n, order, moves_all, n_all, moves_buf);
        iters += 1;
        if (n_feas == 0) { trace[iters - 1] = cur; break; }
        for (int idx = 0; idx < n_feas; ++idx) {
            int u = moves_buf[2 * idx], v = moves_buf[2 * idx + 1];
            int32_t t = order[u]; order[u] = order[v]; order[v] = t;
            cmax_buf[idx] = evaluate_order_raw(order, I, I->pred_ptr, I->pred_dat, mode, S, touched);
            touched = cmax_buf[idx];
            t = order[u]; order[u] = order[v]; order[v] = t;
        }
        evals += n_feas;
        int asp = best_known_cmax < local_best ? best_known_cmax : local_best;
        int pick = select_move_raw(moves_buf, n_feas, cmax_buf, tabu_count, n, asp);
        if (pick < 0) { pick = select_min_raw(n_feas, cmax_buf); forced += 1; }
        int u = moves_buf[2 * pick], v = moves_buf[2 * pick + 1];
        int32_t t = order[u]; order[u] = order[v]; order[v] = t;
        head = tabu_add_raw(tabu_list, T, tabu_count, n, head, u, v);
        cur = cmax_buf[pick];
        trace[iters - 1] = cur;
        if (cur < local_best) {
            local_best = cur;
            memcpy(best_order, order, sizeof(int32_t) * n);
        }
        if (local_best < adopted_cmax) break;
        if (local_best <= floor_cmax) break;
    }
    *tabu_head = head;
    out7[0] = iters; out7[1] = evals; out7[2] = local_best < adopted_cmax ? 1 : 0;
    out7[3] = local_best; out7[4] = cur; out7[5] = head; out7[6] = forced;
}

static uint8_t *build_adj(int n, const int32_t *succ_ptr, const int32_t *succ_dat) {
    uint8_t *adj = calloc((size_t)n * n, 1);
    for (int i = 0; i < n; ++i)
        for (int e = succ_ptr[i]; e < succ_ptr[i + 1]; ++e) adj[i * n + succ_dat[e]] = 1;
    return adj;
}

/* Stand-alone run_chunk (the kernels.run_chunk drop-in parity oracle). */
int oracle_run_chunk(int n, int m, int horizon, const int32_t *dur, const int32_t *dem,
                     const int32_t *cap, const int32_t *pred_ptr, const int32_t *pred_dat,
                     const int32_t *succ_ptr, const int32_t *succ_dat, int delta, int mode,
                     int32_t *order, int32_t *tabu_list, int T, int32_t *tabu_count,
                     int tabu_head, int budget, int adopted_cmax, int start_cmax,
                     int best_known_cmax, int floor_cmax, int32_t *best_order, int32_t *trace,
                     long *out7) {
    oinst_t I;
    inst_fill(&I, n, m, horizon, dur, dem, cap, pred_ptr, pred_dat, succ_ptr, succ_dat);
    uint8_t *adj = build_adj(n, succ_ptr, succ_dat);
    I.adj = adj;
    int n_all;
    int32_t *moves_all = gen_neighborhood(n, delta, &n_all);
    int32_t *moves_buf = malloc(sizeof(int32_t) * 2 * (size_t)(n_all > 0 ? n_all : 1));
    int32_t *cmax_buf = malloc(sizeof(int32_t) * (size_t)(n_all > 0 ? n_all : 1));
    oscratch_t S;
    scratch_alloc(&S, &I);
    int head = tabu_head;
    run_chunk_raw(order, &I, moves_all, n_all, mode, tabu_list, T, tabu_count, &head, budget,
                  adopted_cmax, start_cmax, best_known_cmax, floor_cmax, best_order, &S, moves_buf,
                  cmax_buf, trace, out7);
    scratch_free(&S);
    free(adj); free(moves_all); free(moves_buf); free(cmax_buf);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Forward-backward improvement (evaluator.py:187-266).                      */

/* evaluator.py:187-205: topological order preferring small key, ties by id.
 * key2[i] is the primary key; (key2[i], i) is unique so a selection scan is
 * equivalent to the reference's heap.  The graph is given as CSR `nxt` (the
 * "successors" in the traversal direction) and in-degree array indeg0. */
static int priority_topo(int n, const int32_t *nxt_ptr, const int32_t *nxt_dat,
                         const int32_t *indeg0, const int64_t *key, int32_t *out, int32_t *indeg,
                         uint8_t *ready) {
    for (int i = 0; i < n; ++i) { indeg[i] = indeg0[i]; ready[i] = indeg[i] == 0; }
    int filled = 0;
    for (;;) {
        int best = -1;
        for (int i = 0; i < n; ++i)
            if (ready[i] && (best < 0 || key[i] < key[best])) best = i; /* ties: smaller id */
        if (best < 0) break;
        ready[best] = 0;
        out[filled++] = best;
        for (int e = nxt_ptr[best]; e < nxt_ptr[best + 1]; ++e) {
            int j = nxt_dat[e];
            if (--indeg[j] == 0) ready[j] = 1;
        }
    }
    return filled == n ? 0 : -1;
}

/* evaluator.py:207-266 ; writes final order and starts, returns cmax */
static int fbi_raw(const oinst_t *I, const int32_t *order_in, int mode, oscratch_t *S,
                   int32_t *final_order, int32_t *final_starts) {
    int n = I->n;
    int32_t *starts = malloc(sizeof(int32_t) * n), *bstarts = malloc(sizeof(int32_t) * n);
    int32_t *border = malloc(sizeof(int32_t) * n), *forder = malloc(sizeof(int32_t) * n);
    int32_t *indeg_p = malloc(sizeof(int32_t) * n), *indeg_s = malloc(sizeof(int32_t) * n);
    int32_t *tmp = malloc(sizeof(int32_t) * n);
    uint8_t *ready = malloc((size_t)n);
    int64_t *key = malloc(sizeof(int64_t) * n);
    for (int i = 0; i < n; ++i) {
        indeg_p[i] = I->pred_ptr[i + 1] - I->pred_ptr[i];
        indeg_s[i] = I->succ_ptr[i + 1] - I->succ_ptr[i];
    }
    int cmax = evaluate_order_raw(order_in, I, I->pred_ptr, I->pred_dat, mode, S, I->horizon);
    S->evaluations++;
    memcpy(starts, S->starts, sizeof(int32_t) * n);
    for (;;) {
        /* back_order: graph reversed (succ_of = preds), indeg = #succ, key -finish */
        for (int i = 0; i < n; ++i) key[i] = -(int64_t)(starts[i] + I->dur[i]);
        priority_topo(n, I->pred_ptr, I->pred_dat, indeg_s, key, border, tmp, ready);
        evaluate_order_raw(border, I, I->succ_ptr, I->succ_dat, mode, S, I->horizon);
        S->evaluations++;
        memcpy(bstarts, S->starts, sizeof(int32_t) * n);
        for (int i = 0; i < n; ++i) key[i] = -(int64_t)(bstarts[i] + I->dur[i]);
        priority_topo(n, I->succ_ptr, I->succ_dat, indeg_p, key, forder, tmp, ready);
        int new_cmax = evaluate_order_raw(forder, I, I->pred_ptr, I->pred_dat, mode, S, I->horizon);
        S->evaluations++;
        if (new_cmax < cmax) {
            memcpy(starts, S->starts, sizeof(int32_t) * n);
            cmax = new_cmax;
        } else {
            break;
        }
    }
    for (int i = 0; i < n; ++i) key[i] = starts[i];
    priority_topo(n, I->succ_ptr, I->succ_dat, indeg_p, key, final_order, tmp, ready);
    if (final_starts) memcpy(final_starts, starts, sizeof(int32_t) * n);
    free(starts); free(bstarts); free(border); free(forder); free(indeg_p); free(indeg_s);
    free(tmp); free(ready); free(key);
    return cmax;
}

int oracle_fbi(int n, int m, int horizon, const int32_t *dur, const int32_t *dem,
               const int32_t *cap, const int32_t *pred_ptr, const int32_t *pred_dat,
               const int32_t *succ_ptr, const int32_t *succ_dat, const int32_t *order, int mode,
               int32_t *final_order, int32_t *final_starts, long *evaluations) {
    oinst_t I;
    inst_fill(&I, n, m, horizon, dur, dem, cap, pred_ptr, pred_dat, succ_ptr, succ_dat);
    oscratch_t S;
    scratch_alloc(&S, &I);
    int c = fbi_raw(&I, order, mode, &S, final_order, final_starts);
    if (evaluations) *evaluations = S.evaluations;
    scratch_free(&S);
    return c;
}

/* ------------------------------------------------------------------------ */
/* Cooperation: working set, exchange, orchestrate (cooperation.py, search.py) */

typedef struct {
    int32_t *order;
    int cmax;
    int32_t *tabu; /* T x 2 */
    int head;
    long ic;
    long reads;
    int mode;
} oentry_t;

typedef struct {
    oentry_t *entries;
    int F;
    pthread_mutex_t lock;
    long cursor, total, planned, consumed;
    int floor_cmax, stop;
    int best_cmax, best_mode;
    int32_t *best_order;
} ows_t;

typedef struct {
    int n, T, delta, phi_steps, phi_max, mode, collect_trace;
    long total_iters, block_iters;
} oparams_t;

typedef struct {
    const oinst_t *I;
    const oparams_t *P;
    ows_t *ws;
    int index;
    pcg64_t rng;
    int32_t *tabu_list, *tabu_count;
    int tabu_head;
    oscratch_t S;
    const int32_t *moves_all;
    int n_all;
    int32_t *moves_buf, *cmax_buf, *best_order, *order, *trace_buf;
    /* stats */
    long iterations, evaluations, exchanges, diversifications, forced;
    /* exchange fields */
    int entry_index, adopted_cmax, improved, local_best;
    long granted, used;
    /* traces: concatenated, with chunk lengths */
    int32_t *trace_all;
    long trace_len, trace_cap;
    long *chunk_len;
    long n_chunks, chunk_cap;
} oworker_t;

/* cooperation.py:39-49 (Eq. 8, quantity term read as I_block/5) */
long oracle_assigned_iterations(int cmax, long ic, long block_iters, int best_cmax) {
    double quality = 0.8 * exp(-100.0 * ((double)cmax / (double)best_cmax - 1.0));
    double intact = 0.2 * exp(-4.0 * ((double)ic / (double)block_iters));
    return (long)floor(((double)block_iters / 5.0) * (quality + intact));
}

/* tabu.py:52-60 */
static void tabu_load(oworker_t *w, const int32_t *entries, int head) {
    int n = w->I->n, T = w->P->T;
    memcpy(w->tabu_list, entries, sizeof(int32_t) * 2 * T);
    memset(w->tabu_count, 0, sizeof(int32_t) * (size_t)n * n);
    for (int i = 0; i < T; ++i) {
        int u = entries[2 * i], v = entries[2 * i + 1];
        if (u != 0 || v != 0) w->tabu_count[u * n + v] += 1;
    }
    w->tabu_head = head % T;
}

/* cooperation.py:82-135 ; returns 1 with an adoption, 0 when the run is over */
static int exchange(oworker_t *w, ows_t *ws, long *grant_out, int *best_known, int *needs_div) {
    int n = w->I->n, T = w->P->T;
    pthread_mutex_lock(&ws->lock);
    if (w->entry_index >= 0) {
        long unused = w->granted - w->used;
        ws->planned -= unused > 0 ? unused : 0;
        ws->consumed += w->used;
        oentry_t *e = &ws->entries[w->entry_index];
        if (w->improved) {
            memcpy(e->order, w->best_order, sizeof(int32_t) * n);
            e->cmax = w->local_best;
            memcpy(e->tabu, w->tabu_list, sizeof(int32_t) * 2 * T);
            e->head = w->tabu_head;
            e->ic += w->used;
            e->reads = 0;
            e->mode = w->P->mode;
            if (w->local_best < ws->best_cmax) {
                ws->best_cmax = w->local_best;
                memcpy(ws->best_order, w->best_order, sizeof(int32_t) * n);
                ws->best_mode = w->P->mode;
            }
        } else {
            e->ic += w->used;
        }
        w->improved = 0;
        w->entry_index = -1;
    }
    if (ws->best_cmax <= ws->floor_cmax) ws->stop = 1;
    if (ws->stop || ws->planned >= ws->total) {
        pthread_mutex_unlock(&ws->lock);
        return 0;
    }
    long index = ws->cursor % ws->F;
    ws->cursor += 1;
    oentry_t *e = &ws->entries[index];
    e->reads += 1;
    *needs_div = e->reads > w->P->phi_max;
    long grant = oracle_assigned_iterations(e->cmax, e->ic, w->P->block_iters, ws->best_cmax);
    if (grant < 1) grant = 1;
    if (grant > ws->total - ws->planned) grant = ws->total - ws->planned;
    ws->planned += grant;
    w->entry_index = (int)index;
    w->adopted_cmax = e->cmax;
    w->granted = grant;
    w->used = 0;
    tabu_load(w, e->tabu, e->head);
    memcpy(w->order, e->order, sizeof(int32_t) * n);
    *grant_out = grant;
    *best_known = ws->best_cmax;
    pthread_mutex_unlock(&ws->lock);
    return 1;
}

/* search.py:77-94 ; work is modified in place */
static void diversify(oworker_t *w, int32_t *work) {
    const oinst_t *I = w->I;
    int n = I->n;
    if (w->P->phi_steps <= 0) return;
    int n_all;
    int32_t *all_moves = gen_neighborhood(n, n, &n_all);
    int32_t *feas = malloc(sizeof(int32_t) * 2 * (size_t)(n_all > 0 ? n_all : 1));
    for (int s = 0; s < w->P->phi_steps; ++s) {
        int k = filter_moves_raw(I->adj, n, work, all_moves, n_all, feas);
        if (k == 0) continue;
        int64_t pick = pcg_integers(&w->rng, k);
        int u = feas[2 * pick], v = feas[2 * pick + 1];
        int32_t t = work[u]; work[u] = work[v]; work[v] = t;
    }
    free(all_moves); free(feas);
}

static void trace_append(oworker_t *w, const int32_t *tr, long len) {
    if (w->trace_len + len > w->trace_cap) {
        long cap = (w->trace_cap + len) * 2 + 16;
        w->trace_all = realloc(w->trace_all, sizeof(int32_t) * cap);
        w->trace_cap = cap;
    }
    memcpy(w->trace_all + w->trace_len, tr, sizeof(int32_t) * len);
    w->trace_len += len;
    if (w->n_chunks + 1 > w->chunk_cap) {
        long cap = w->chunk_cap * 2 + 16;
        w->chunk_len = realloc(w->chunk_len, sizeof(long) * cap);
        w->chunk_cap = cap;
    }
    w->chunk_len[w->n_chunks++] = len;
}

/* search.py:176-194 with run_adopted (144-173) inlined */
static void *run_worker(void *arg) {
    oworker_t *w = arg;
    const oinst_t *I = w->I;
    int n = I->n;
    for (;;) {
        long grant;
        int best_known, needs_div;
        if (!exchange(w, w->ws, &grant, &best_known, &needs_div)) return NULL;
        if (needs_div) {
            diversify(w, w->order);
            w->diversifications++;
        }
        w->exchanges++;
        /* run_adopted */
        int start_cmax =
            evaluate_order_raw(w->order, I, I->pred_ptr, I->pred_dat, w->P->mode, &w->S, I->horizon);
        w->evaluations++;
        memcpy(w->best_order, w->order, sizeof(int32_t) * n);
        if (grant > w->P->total_iters + 1) grant = w->P->total_iters + 1;
        long out7[7];
        run_chunk_raw(w->order, I, w->moves_all, w->n_all, w->P->mode, w->tabu_list, w->P->T,
                      w->tabu_count, &w->tabu_head, (int)grant, w->adopted_cmax, start_cmax,
                      best_known, I->cpm, w->best_order, &w->S, w->moves_buf, w->cmax_buf,
                      w->trace_buf, out7);
        w->used = out7[0];
        w->improved = (int)out7[2];
        w->local_best = (int)out7[3];
        w->iterations += out7[0];
        w->evaluations += out7[1];
        w->forced += out7[6];
        if (w->P->collect_trace) trace_append(w, w->trace_buf, out7[0]);
    }
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + ts.tv_nsec * 1e-9;
}

/* compute_levels (instance.py:396-415) via the longest unit-weight depth */
static void levels_of(const oinst_t *I, int32_t *lvl_ptr, int32_t *lvl_dat, int *n_levels) {
    int n = I->n;
    int32_t *depth = calloc((size_t)n, sizeof(int32_t));
    int32_t *indeg = malloc(sizeof(int32_t) * n), *queue = malloc(sizeof(int32_t) * n);
    int qh = 0, qt = 0;
    for (int i = 0; i < n; ++i) {
        indeg[i] = I->pred_ptr[i + 1] - I->pred_ptr[i];
        if (!indeg[i]) queue[qt++] = i;
    }
    while (qh < qt) {
        int i = queue[qh++];
        for (int e = I->succ_ptr[i]; e < I->succ_ptr[i + 1]; ++e) {
            int j = I->succ_dat[e];
            if (depth[i] + 1 > depth[j]) depth[j] = depth[i] + 1;
            if (--indeg[j] == 0) queue[qt++] = j;
        }
    }
    int maxd = 0;
    for (int i = 0; i < n; ++i) if (depth[i] > maxd) maxd = depth[i];
    *n_levels = maxd + 1;
    int p = 0;
    for (int d = 0; d <= maxd; ++d) {
        lvl_ptr[d] = p;
        for (int i = 0; i < n; ++i) if (depth[i] == d) lvl_dat[p++] = i; /* sorted ids */
    }
    lvl_ptr[maxd + 1] = p;
    free(depth); free(indeg); free(queue);
}

/* critical_path_length (instance.py:374-388) */
static int cpm_of(const oinst_t *I) {
    int n = I->n;
    int32_t *dist = calloc((size_t)n, sizeof(int32_t));
    int32_t *indeg = malloc(sizeof(int32_t) * n), *queue = malloc(sizeof(int32_t) * n);
    int qh = 0, qt = 0;
    for (int i = 0; i < n; ++i) {
        indeg[i] = I->pred_ptr[i + 1] - I->pred_ptr[i];
        if (!indeg[i]) queue[qt++] = i;
    }
    while (qh < qt) {
        int i = queue[qh++];
        for (int e = I->succ_ptr[i]; e < I->succ_ptr[i + 1]; ++e) {
            int j = I->succ_dat[e];
            if (dist[i] + I->dur[i] > dist[j]) dist[j] = dist[i] + I->dur[i];
            if (--indeg[j] == 0) queue[qt++] = j;
        }
    }
    int r = dist[n - 1];
    free(dist); free(indeg); free(queue);
    return r;
}

int oracle_critical_path(int n, const int32_t *dur, const int32_t *pred_ptr,
                         const int32_t *pred_dat, const int32_t *succ_ptr,
                         const int32_t *succ_dat) {
    oinst_t I;
    int32_t cap1 = 1;
    inst_fill(&I, n, 0, 0, dur, NULL, &cap1, pred_ptr, pred_dat, succ_ptr, succ_dat);
    return cpm_of(&I);
}

/* Full orchestrate (cooperation.py:237-302) without the dynamic-mode
 * controller.  params7 = {total_iters, workers, delta, tabu_size, phi_steps,
 * phi_max, pool_size}; seeds = 6 uint64 per PCG64 state: [0] is the pool
 * rng default_rng(seed), [1 + w] is worker w's default_rng(seed ^ w).
 * out (int64[16]): best_cmax, iterations(consumed), evaluations, exchanges,
 *   diversifications, forced, stop_reason (1 = critical_path), cpm,
 *   best_mode, pool_evaluations, trace_total, n_chunks_total.
 * wall_time written to *wall.  best_order (n) filled.  If trace != NULL it
 * receives the concatenated traces (capacity trace_cap) and chunk_lens the
 * chunk lengths (capacity chunk_cap), worker-major like RunStats.traces. */
int oracle_orchestrate(int n, int m, int horizon, const int32_t *dur, const int32_t *dem,
                       const int32_t *cap, const int32_t *pred_ptr, const int32_t *pred_dat,
                       const int32_t *succ_ptr, const int32_t *succ_dat, const long *params7,
                       int mode, const uint64_t *seeds, int32_t *best_order, long *out,
                       double *wall, int32_t *trace, long trace_cap, long *chunk_lens,
                       long chunk_cap) {
    oinst_t I;
    inst_fill(&I, n, m, horizon, dur, dem, cap, pred_ptr, pred_dat, succ_ptr, succ_dat);
    uint8_t *adj = build_adj(n, succ_ptr, succ_dat);
    I.adj = adj;
    int32_t *lvl_ptr = malloc(sizeof(int32_t) * (n + 1)), *lvl_dat = malloc(sizeof(int32_t) * n);
    levels_of(&I, lvl_ptr, lvl_dat, &I.n_levels);
    I.cpm = cpm_of(&I);

    oparams_t P;
    P.n = n;
    P.total_iters = params7[0];
    int B = (int)params7[1];
    P.delta = (int)params7[2];
    P.T = (int)params7[3];
    P.phi_steps = (int)params7[4];
    P.phi_max = (int)params7[5];
    int F = (int)params7[6];
    P.mode = mode;
    P.collect_trace = trace != NULL;
    P.block_iters = (P.total_iters + B - 1) / B;
    if (P.block_iters < 1) P.block_iters = 1;

    int n_all;
    int32_t *moves_all = gen_neighborhood(n, P.delta, &n_all);

    double tick = now_s();
    /* initialize_working_set (cooperation.py:138-160) */
    pcg64_t pool_rng;
    pcg_load(&pool_rng, seeds);
    oscratch_t S0;
    scratch_alloc(&S0, &I);
    ows_t ws;
    memset(&ws, 0, sizeof(ws));
    ws.F = F;
    ws.entries = calloc((size_t)F, sizeof(oentry_t));
    int32_t *tmp_order = malloc(sizeof(int32_t) * n);
    for (int idx = 0; idx < F; ++idx) {
        oentry_t *e = &ws.entries[idx];
        e->order = malloc(sizeof(int32_t) * n);
        e->tabu = calloc((size_t)2 * P.T, sizeof(int32_t));
        /* moves.py:42-57 initial_order(shuffle=True) */
        for (int l = 0; l < I.n_levels; ++l) {
            int a = lvl_ptr[l], b = lvl_ptr[l + 1];
            memcpy(tmp_order + a, lvl_dat + a, sizeof(int32_t) * (b - a));
            if (b - a > 1) pcg_permute(&pool_rng, tmp_order + a, b - a);
        }
        if (idx % 2 == 0) {
            fbi_raw(&I, tmp_order, mode, &S0, e->order, NULL);
        } else {
            memcpy(e->order, tmp_order, sizeof(int32_t) * n);
        }
        e->cmax = evaluate_order_raw(e->order, &I, I.pred_ptr, I.pred_dat, mode, &S0, horizon);
        S0.evaluations++;
        e->mode = mode;
    }
    long pool_evals = S0.evaluations;
    scratch_free(&S0);
    free(tmp_order);
    pthread_mutex_init(&ws.lock, NULL);
    ws.total = P.total_iters;
    ws.floor_cmax = I.cpm;
    int best = 0;
    for (int i = 1; i < F; ++i) if (ws.entries[i].cmax < ws.entries[best].cmax) best = i;
    ws.best_cmax = ws.entries[best].cmax;
    ws.best_order = malloc(sizeof(int32_t) * n);
    memcpy(ws.best_order, ws.entries[best].order, sizeof(int32_t) * n);
    ws.best_mode = mode;
    if (ws.best_cmax <= ws.floor_cmax) ws.stop = 1;

    oworker_t *W = calloc((size_t)B, sizeof(oworker_t));
    long budget_cap = P.total_iters + 1;
    for (int b = 0; b < B; ++b) {
        oworker_t *w = &W[b];
        w->I = &I; w->P = &P; w->ws = &ws; w->index = b;
        pcg_load(&w->rng, seeds + 6 * (1 + b));
        w->tabu_list = calloc((size_t)2 * P.T, sizeof(int32_t));
        w->tabu_count = calloc((size_t)n * n, sizeof(int32_t));
        scratch_alloc(&w->S, &I);
        w->moves_all = moves_all; w->n_all = n_all;
        w->moves_buf = malloc(sizeof(int32_t) * 2 * (size_t)(n_all > 0 ? n_all : 1));
        w->cmax_buf = malloc(sizeof(int32_t) * (size_t)(n_all > 0 ? n_all : 1));
        w->best_order = malloc(sizeof(int32_t) * n);
        w->order = malloc(sizeof(int32_t) * n);
        w->trace_buf = malloc(sizeof(int32_t) * (size_t)budget_cap);
        w->entry_index = -1;
    }
    if (!ws.stop) {
        if (B == 1) {
            run_worker(&W[0]);
        } else {
            pthread_t *th = malloc(sizeof(pthread_t) * B);
            for (int b = 0; b < B; ++b) pthread_create(&th[b], NULL, run_worker, &W[b]);
            for (int b = 0; b < B; ++b) pthread_join(th[b], NULL);
            free(th);
        }
    }
    *wall = now_s() - tick;

    long evals = pool_evals, exch = 0, div = 0, forced = 0, tlen = 0, nch = 0;
    for (int b = 0; b < B; ++b) {
        evals += W[b].evaluations;
        exch += W[b].exchanges;
        div += W[b].diversifications;
        forced += W[b].forced;
        if (trace) {
            for (long c = 0; c < W[b].n_chunks && nch < chunk_cap; ++c) chunk_lens[nch++] = W[b].chunk_len[c];
            long take = W[b].trace_len;
            if (tlen + take > trace_cap) take = trace_cap - tlen;
            if (take > 0) memcpy(trace + tlen, W[b].trace_all, sizeof(int32_t) * take);
            tlen += take;
        }
    }
    memcpy(best_order, ws.best_order, sizeof(int32_t) * n);
    out[0] = ws.best_cmax; out[1] = ws.consumed; out[2] = evals; out[3] = exch; out[4] = div;
    out[5] = forced; out[6] = ws.best_cmax <= I.cpm ? 1 : 0; out[7] = I.cpm;
    out[8] = ws.best_mode; out[9] = pool_evals; out[10] = tlen; out[11] = nch;

    for (int b = 0; b < B; ++b) {
        oworker_t *w = &W[b];
        free(w->tabu_list); free(w->tabu_count); scratch_free(&w->S); free(w->moves_buf);
        free(w->cmax_buf); free(w->best_order); free(w->order); free(w->trace_buf);
        free(w->trace_all); free(w->chunk_len);
    }
    free(W);
    for (int i = 0; i < F; ++i) { free(ws.entries[i].order); free(ws.entries[i].tabu); }
    free(ws.entries); free(ws.best_order);
    pthread_mutex_destroy(&ws.lock);
    free(moves_all); free(adj); free(lvl_ptr); free(lvl_dat);
    return 0;
}

/* Diversify stand-alone (search.py:77-94) for parity tests. */
int oracle_diversify(int n, const int32_t *succ_ptr, const int32_t *succ_dat, int32_t *work,
                     int phi_steps, uint64_t *rng_state) {
    oinst_t I;
    memset(&I, 0, sizeof(I));
    I.n = n;
    uint8_t *adj = build_adj(n, succ_ptr, succ_dat);
    I.adj = adj;
    oparams_t P;
    memset(&P, 0, sizeof(P));
    P.phi_steps = phi_steps;
    oworker_t w;
    memset(&w, 0, sizeof(w));
    w.I = &I; w.P = &P;
    pcg_load(&w.rng, rng_state);
    diversify(&w, work);
    pcg_store(&w.rng, rng_state);
    free(adj);
    return 0;
}
