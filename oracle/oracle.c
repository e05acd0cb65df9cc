/*
 * oracle.c -- CPU restatement of the pushrank IFP1/IFP2 hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the *checker*: it is loaded by
 * tests/, by __graft_entry__.smoke() and by bench.py's cpu_baseline /
 * --impl reference legs, never by the product package
 * (paper_2302_03245_b200/), which has no CPU fallback.
 *
 * Every function restates one reference function; the citation is the
 * file:line under /root/reference/pkg/src/pushrank/ it follows.  The
 * restatement is pinned against the real reference (tests/golden/, made by
 * tests/golden/make_golden.py which imports the reference package).
 *
 * Integer work (graph build, classification, IFP2 split) is bit-exact.
 * The synchronous rounds reproduce the reference's np.bincount order
 * (sequential, ascending source, then row order) and its
 * "(c*amount)/degree" rounding, so reserved/pending vectors are bit-exact
 * with sync_simulate; trace float sums (numpy pairwise) are not.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <stdatomic.h>
#include <time.h>
#include <unistd.h>

/* ------------------------------------------------------------------ */
/* from_edges (graph.py:133-177)                                      */
/* ------------------------------------------------------------------ */

/* LSD radix sort of uint64 keys, 11-bit digits, only as many passes as
 * the key range needs.  Equivalent to the np.unique sort at graph.py:152. */
static void radix_sort_u64(uint64_t *keys, uint64_t *tmp, int64_t count, int bits)
{
    const int D = 11, R = 1 << D;
    int64_t *hist = (int64_t *)malloc(sizeof(int64_t) * R);
    uint64_t *a = keys, *b = tmp;
    for (int shift = 0; shift < bits; shift += D) {
        memset(hist, 0, sizeof(int64_t) * R);
        for (int64_t i = 0; i < count; ++i) hist[(a[i] >> shift) & (R - 1)]++;
        int64_t run = 0;
        for (int d = 0; d < R; ++d) { int64_t c = hist[d]; hist[d] = run; run += c; }
        for (int64_t i = 0; i < count; ++i) b[hist[(a[i] >> shift) & (R - 1)]++] = a[i];
        uint64_t *t = a; a = b; b = t;
    }
    if (a != keys) memcpy(keys, a, sizeof(uint64_t) * count);
    free(hist);
}

static int bit_width_u64(uint64_t x) { int b = 0; while (x) { ++b; x >>= 1; } return b; }

/* Returns m (unique edges).  out_targets/in_sources must hold m_raw items.
 * Caller has already range-checked ids (graph.py:148-150 raise in Python). */
int64_t orc_from_edges(int64_t n, const int64_t *src, const int64_t *dst, int64_t m_raw,
                       int64_t *out_offsets, int64_t *out_targets,
                       int64_t *in_offsets, int64_t *in_sources)
{
    uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (m_raw ? m_raw : 1));
    uint64_t *tmp = (uint64_t *)malloc(sizeof(uint64_t) * (m_raw ? m_raw : 1));
    for (int64_t i = 0; i < m_raw; ++i) keys[i] = (uint64_t)src[i] * (uint64_t)n + (uint64_t)dst[i];
    radix_sort_u64(keys, tmp, m_raw, bit_width_u64((uint64_t)n * (uint64_t)n - 1));
    int64_t m = 0;
    for (int64_t i = 0; i < m_raw; ++i)
        if (i == 0 || keys[i] != keys[i - 1]) keys[m++] = keys[i];

    memset(out_offsets, 0, sizeof(int64_t) * (n + 1));
    memset(in_offsets, 0, sizeof(int64_t) * (n + 1));
    for (int64_t e = 0; e < m; ++e) {
        int64_t s = (int64_t)(keys[e] / (uint64_t)n), t = (int64_t)(keys[e] % (uint64_t)n);
        out_targets[e] = t;
        out_offsets[s + 1]++;
        in_offsets[t + 1]++;
    }
    for (int64_t v = 0; v < n; ++v) {
        out_offsets[v + 1] += out_offsets[v];
        in_offsets[v + 1] += in_offsets[v];
    }
    /* stable counting sort by target: ascending source within a target
     * (graph.py:164 argsort(kind="stable")) */
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (n ? n : 1));
    memcpy(cursor, in_offsets, sizeof(int64_t) * n);
    for (int64_t e = 0; e < m; ++e) {
        int64_t s = (int64_t)(keys[e] / (uint64_t)n), t = out_targets[e];
        in_sources[cursor[t]++] = s;
    }
    free(cursor);
    free(keys);
    free(tmp);
    return m;
}

/* ------------------------------------------------------------------ */
/* classify (graph.py:274-318): base sets + joint weak peel            */
/* flags: bit0 dangling, bit1 unreferenced, bit2 weak dangling,        */
/*        bit3 weak unreferenced                                       */
/* ------------------------------------------------------------------ */
int64_t orc_classify(int64_t n, const int64_t *out_offsets, const int64_t *out_targets,
                     const int64_t *in_offsets, const int64_t *in_sources,
                     uint8_t *flags, int64_t *peel_rounds)
{
    int64_t *cur_out = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t *cur_in = (int64_t *)malloc(sizeof(int64_t) * n);
    uint8_t *alive = (uint8_t *)malloc(n);
    uint8_t *doomed = (uint8_t *)malloc(n);
    int64_t m_d = 0, rounds = 0;
    for (int64_t v = 0; v < n; ++v) {
        cur_out[v] = out_offsets[v + 1] - out_offsets[v];
        cur_in[v] = in_offsets[v + 1] - in_offsets[v];
        flags[v] = (uint8_t)((cur_out[v] == 0 ? 1 : 0) | (cur_in[v] == 0 ? 2 : 0));
        if (cur_out[v] == 0) m_d += cur_in[v];           /* graph.py:285 */
        alive[v] = 1;
        doomed[v] = (uint8_t)(cur_out[v] == 0 || cur_in[v] == 0);   /* graph.py:293 */
    }
    for (;;) {
        int any = 0;
        for (int64_t v = 0; v < n; ++v) if (doomed[v]) { any = 1; alive[v] = 0; }
        if (!any) break;
        ++rounds;
        for (int64_t v = 0; v < n; ++v) {
            if (!doomed[v]) continue;
            for (int64_t e = out_offsets[v]; e < out_offsets[v + 1]; ++e)
                if (alive[out_targets[e]]) cur_in[out_targets[e]]--;      /* graph.py:298-300 */
            for (int64_t e = in_offsets[v]; e < in_offsets[v + 1]; ++e)
                if (alive[in_sources[e]]) cur_out[in_sources[e]]--;       /* graph.py:302-304 */
        }
        for (int64_t v = 0; v < n; ++v) {
            int nd = alive[v] && cur_out[v] == 0;
            int nu = alive[v] && cur_in[v] == 0;
            if (nd && !(flags[v] & 1)) flags[v] |= 4;                     /* graph.py:308 */
            if (nu && !(flags[v] & 2)) flags[v] |= 8;                     /* graph.py:309 */
            doomed[v] = (uint8_t)(nd || nu);                              /* graph.py:310 */
        }
    }
    free(cur_out); free(cur_in); free(alive); free(doomed);
    if (peel_rounds) *peel_rounds = rounds;
    return m_d;
}

/* dangling_target_counts (graph.py:334-340) */
void orc_dangling_target_counts(int64_t n, const int64_t *out_offsets, const int64_t *out_targets,
                                const uint8_t *dangling, int64_t *out)
{
    for (int64_t v = 0; v < n; ++v) {
        int64_t c = 0;
        for (int64_t e = out_offsets[v]; e < out_offsets[v + 1]; ++e) c += dangling[out_targets[e]];
        out[v] = c;
    }
}

/* preprocess_ifp2 (graph.py:343-378).  Returns live edge count. */
int64_t orc_preprocess_ifp2(int64_t n, const int64_t *out_offsets, const int64_t *out_targets,
                            const int64_t *in_offsets, const int64_t *in_sources,
                            const uint8_t *dangling,
                            int64_t *live_offsets, int64_t *live_targets, int64_t *live_degree,
                            int64_t *dangling_ids, int64_t *source_offsets, int64_t *source_ids)
{
    int64_t w = 0, nd = 0, s = 0;
    live_offsets[0] = 0;
    for (int64_t v = 0; v < n; ++v) {
        int64_t before = w;
        for (int64_t e = out_offsets[v]; e < out_offsets[v + 1]; ++e)
            if (!dangling[out_targets[e]]) live_targets[w++] = out_targets[e];
        live_degree[v] = w - before;
        live_offsets[v + 1] = w;
    }
    source_offsets[0] = 0;
    for (int64_t v = 0; v < n; ++v) {
        if (!dangling[v]) continue;
        dangling_ids[nd++] = v;
        for (int64_t e = in_offsets[v]; e < in_offsets[v + 1]; ++e) source_ids[s++] = in_sources[e];
        source_offsets[nd] = s;
    }
    return w;
}

/* ------------------------------------------------------------------ */
/* sync_simulate rounds (engines.py:349-456)                           */
/* ------------------------------------------------------------------ */
typedef struct {
    double h_l1, alpha, active_mass, carry_mass;
    int64_t converged, work, push_ops, push_ops_dangling;
    uint64_t digest;
} orc_row;

/* order-independent position-weighted digest of (reserved, pending) bits;
 * the device computes the same value with wrapping atomics */
static uint64_t state_digest(int64_t n, const double *reserved, const double *h)
{
    uint64_t acc = 0;
    for (int64_t v = 0; v < n; ++v) {
        uint64_t a, b;
        memcpy(&a, &reserved[v], 8);
        memcpy(&b, &h[v], 8);
        uint64_t w = ((uint64_t)v * 0x9E3779B97F4A7C15ull) | 1ull;
        acc += (a ^ (b * 0xBF58476D1CE4E5B9ull)) * w;
    }
    return acc;
}

/*
 * variant 0 = ifp1, 1 = ifp2 (offsets/targets are the live CSR),
 * 2 = fp-full.  scan mask = non-dangling (ifp1/ifp2) or all (fp-full).
 * Writes one row per state including the terminal one (engines.py:427-437).
 * Returns the number of iterations, -1 if max_iterations exhausted
 * (engines.py:455-456), -2 if trace_cap too small.
 */
int64_t orc_sync_rounds(int variant, int64_t n, const int64_t *offsets, const int64_t *targets,
                        const int64_t *degree, const int64_t *dt_count,
                        double c, double xi, int64_t max_iterations,
                        double *reserved, double *h, orc_row *rows, int64_t trace_cap,
                        int64_t *n_rows)
{
    const double reserve_frac = variant == 2 ? 1.0 - c : 1.0;     /* engines.py:389-394 */
    double *inflow = (double *)malloc(sizeof(double) * n);
    uint8_t *active = (uint8_t *)malloc(n);
    double *amount = (double *)malloc(sizeof(double) * n);
    int64_t push_ops = 0, push_dang = 0, iterations = 0, r = 0;
    int settled = 0;
    for (int64_t v = 0; v < n; ++v) { reserved[v] = 0.0; h[v] = 1.0; }
    for (int64_t t = 0; t <= max_iterations; ++t) {
        double above_mass = 0.0, nd_above = 0.0, l1 = 0.0;
        int64_t conv = 0, work = 0, nact = 0;
        for (int64_t v = 0; v < n; ++v) {
            int dang = degree[v] == 0;
            int above = h[v] > xi;                                  /* strict, engines.py:421 */
            int scan = variant == 2 ? 1 : !dang;
            l1 += h[v];
            if (above) { above_mass += h[v]; if (!dang) nd_above += h[v]; } else ++conv;
            active[v] = (uint8_t)(above && scan);
            if (active[v]) { work += degree[v] + 1; ++nact; }
        }
        if (r >= trace_cap) { r = -1; break; }
        rows[r].h_l1 = l1;
        rows[r].converged = conv;
        rows[r].alpha = above_mass > 0.0 ? nd_above / above_mass : 1.0;
        rows[r].work = work;
        rows[r].push_ops = push_ops;
        rows[r].push_ops_dangling = push_dang;
        rows[r].active_mass = above_mass;
        rows[r].carry_mass = l1 - above_mass;
        rows[r].digest = state_digest(n, reserved, h);
        ++r;
        if (nact == 0) { settled = 1; break; }
        for (int64_t v = 0; v < n; ++v) inflow[v] = 0.0;
        for (int64_t v = 0; v < n; ++v) {
            if (!active[v]) continue;
            amount[v] = h[v];
            reserved[v] += reserve_frac * h[v];                      /* engines.py:439 */
            int64_t lo = offsets[v], hi = offsets[v + 1];
            if (hi > lo) {
                double share = c * h[v] / (double)degree[v];           /* engines.py:444 */
                for (int64_t e = lo; e < hi; ++e) inflow[targets[e]] += share;   /* bincount order */
            }
            push_ops += hi - lo;
            push_dang += dt_count ? dt_count[v] : 0;
        }
        for (int64_t v = 0; v < n; ++v) h[v] = (active[v] ? 0.0 : h[v]) + inflow[v];  /* engines.py:448 */
        iterations = t + 1;
    }
    free(inflow); free(active); free(amount);
    *n_rows = r < 0 ? trace_cap : r;
    if (r < 0) return -2;
    return settled ? iterations : -1;
}

/*
 * The same rounds as orc_sync_rounds, restated as a pull over the CSC and
 * spread over `threads` POSIX threads, for the full-size configs (C5: 1.06 B
 * edges, where the sequential scatter takes tens of minutes).  Bit-identity
 * with the scatter form: np.bincount (engines.py:444-448) adds target v's
 * contributions in CSR edge order, i.e. ascending source -- exactly the
 * order of v's CSC column (graph.py:161-164, stable argsort) -- and an
 * inactive source contributes +0.0, which leaves a non-negative sum
 * unchanged.  So inflow[v] = sum over v's column of share[u] (share 0 when
 * u is inactive) is the same double, bit for bit.  Receivers: every vertex
 * (ifp1, fp-full) or the non-dangling ones (ifp2: the live CSR drops edges
 * into dangling targets, graph.py:355-360).  `row_len` is the pushed row
 * length (live out-degree for ifp2, out-degree otherwise).  Per-round
 * digests are order-free and equal the sequential form's; trace float sums
 * are combined per thread (not numpy's pairwise order).
 */
typedef struct {
    int variant, tid, nthreads;
    int64_t n;
    const int64_t *in_offsets, *in_sources, *degree, *dt_count, *row_len;
    double c, xi, reserve_frac;
    double *reserved, *h, *share;
    uint8_t *active;
    pthread_barrier_t *bar;
    volatile int *stop;
    /* per-round partials (phase A) */
    double l1, above, nd_above;
    int64_t conv, work, nact, pops, pdang;
    uint64_t digest;
} pull_worker;

static void *pull_worker_main(void *arg)
{
    pull_worker *W = (pull_worker *)arg;
    const int64_t n = W->n;
    const int64_t lo = n * W->tid / W->nthreads, hi = n * (W->tid + 1) / W->nthreads;
    for (;;) {
        /* phase A: statistics of the state, activity, shares, reservation */
        double l1 = 0.0, above_m = 0.0, nd_above = 0.0;
        int64_t conv = 0, work = 0, nact = 0, pops = 0, pdang = 0;
        uint64_t dig = 0;
        for (int64_t v = lo; v < hi; ++v) {
            const double hv = W->h[v];
            const int dang = W->degree[v] == 0;
            const int above = hv > W->xi;
            const int scan = W->variant == 2 ? 1 : !dang;
            uint64_t a, b;
            memcpy(&a, &W->reserved[v], 8);
            memcpy(&b, &W->h[v], 8);
            dig += (a ^ (b * 0xBF58476D1CE4E5B9ull)) * (((uint64_t)v * 0x9E3779B97F4A7C15ull) | 1ull);
            l1 += hv;
            if (above) { above_m += hv; if (!dang) nd_above += hv; } else ++conv;
            W->active[v] = (uint8_t)(above && scan);
            W->share[v] = 0.0;
            if (W->active[v]) {
                work += W->degree[v] + 1;
                ++nact;
            }
        }
        W->l1 = l1; W->above = above_m; W->nd_above = nd_above;
        W->conv = conv; W->work = work; W->nact = nact; W->digest = dig;
        pthread_barrier_wait(W->bar);      /* main: row + termination */
        pthread_barrier_wait(W->bar);
        if (*W->stop) break;
        for (int64_t v = lo; v < hi; ++v) {
            if (!W->active[v]) continue;
            const double hv = W->h[v];
            W->reserved[v] += W->reserve_frac * hv;                            /* engines.py:439 */
            if (W->row_len[v] > 0) W->share[v] = W->c * hv / (double)W->degree[v];   /* engines.py:444 */
            pops += W->row_len[v];
            pdang += W->dt_count ? W->dt_count[v] : 0;
        }
        W->pops = pops; W->pdang = pdang;
        pthread_barrier_wait(W->bar);      /* every share written */
        /* phase B: pull (ascending source = bincount order) */
        for (int64_t v = lo; v < hi; ++v) {
            double acc = 0.0;
            if (W->variant != 1 || W->degree[v] > 0)
                for (int64_t e = W->in_offsets[v]; e < W->in_offsets[v + 1]; ++e) acc += W->share[W->in_sources[e]];
            W->h[v] = (W->active[v] ? 0.0 : W->h[v]) + acc;                    /* engines.py:448 */
        }
        pthread_barrier_wait(W->bar);      /* state t+1 complete */
    }
    return NULL;
}

int64_t orc_sync_rounds_pull(int variant, int64_t n, const int64_t *in_offsets, const int64_t *in_sources,
                             const int64_t *degree, const int64_t *row_len, const int64_t *dt_count,
                             double c, double xi, int64_t max_iterations, int threads,
                             double *reserved, double *h, orc_row *rows, int64_t trace_cap, int64_t *n_rows)
{
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pull_worker *W = (pull_worker *)calloc((size_t)threads, sizeof(pull_worker));
    pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    double *share = (double *)malloc(sizeof(double) * (size_t)(n ? n : 1));
    uint8_t *active = (uint8_t *)malloc((size_t)(n ? n : 1));
    pthread_barrier_t bar;
    pthread_barrier_init(&bar, NULL, (unsigned)threads + 1);
    volatile int stop = 0;
    for (int64_t v = 0; v < n; ++v) { reserved[v] = 0.0; h[v] = 1.0; }
    for (int k = 0; k < threads; ++k) {
        W[k] = (pull_worker){variant, k, threads, n, in_offsets, in_sources, degree, dt_count, row_len,
                             c, xi, variant == 2 ? 1.0 - c : 1.0, reserved, h, share, active, &bar, &stop};
        pthread_create(&th[k], NULL, pull_worker_main, &W[k]);
    }
    int64_t push_ops = 0, push_dang = 0, iterations = 0, r = 0;
    int settled = 0;
    for (int64_t t = 0;; ++t) {
        pthread_barrier_wait(&bar);        /* phase A done */
        double l1 = 0.0, above = 0.0, nd_above = 0.0;
        int64_t conv = 0, work = 0, nact = 0;
        uint64_t dig = 0;
        for (int k = 0; k < threads; ++k) {
            l1 += W[k].l1; above += W[k].above; nd_above += W[k].nd_above;
            conv += W[k].conv; work += W[k].work; nact += W[k].nact; dig += W[k].digest;
        }
        int done = 0;
        if (r >= trace_cap) { r = -1; done = 1; }
        else {
            rows[r].h_l1 = l1;
            rows[r].converged = conv;
            rows[r].alpha = above > 0.0 ? nd_above / above : 1.0;
            rows[r].work = work;
            rows[r].push_ops = push_ops;
            rows[r].push_ops_dangling = push_dang;
            rows[r].active_mass = above;
            rows[r].carry_mass = l1 - above;
            rows[r].digest = dig;
            ++r;
            if (nact == 0) { settled = 1; done = 1; }
            else if (t >= max_iterations) done = 1;
        }
        stop = done;
        pthread_barrier_wait(&bar);
        if (done) break;
        pthread_barrier_wait(&bar);        /* reservation + shares */
        for (int k = 0; k < threads; ++k) { push_ops += W[k].pops; push_dang += W[k].pdang; }
        pthread_barrier_wait(&bar);        /* pull done */
        iterations = t + 1;
    }
    for (int k = 0; k < threads; ++k) pthread_join(th[k], NULL);
    pthread_barrier_destroy(&bar);
    free(W); free(th); free(share); free(active);
    *n_rows = r < 0 ? trace_cap : r;
    if (r < 0) return -2;
    return settled ? iterations : -1;
}

/* _settle_dangling (engines.py:269-289), sequential ascending-source sum */
int64_t orc_settle(int64_t n_d, const int64_t *dangling_ids, const int64_t *source_offsets,
                   const int64_t *source_ids, const int64_t *out_degree, double c,
                   double *reserved, double *h)
{
    for (int64_t i = 0; i < n_d; ++i) {
        double acc = 0.0;
        for (int64_t e = source_offsets[i]; e < source_offsets[i + 1]; ++e) {
            int64_t u = source_ids[e];
            acc += c * reserved[u] / (double)out_degree[u];
        }
        int64_t d = dangling_ids[i];
        reserved[d] = h[d] + acc;
        h[d] = 0.0;
    }
    return n_d ? source_offsets[n_d] : 0;
}

/* ------------------------------------------------------------------ */
/* R-MAT samples of the BASELINE configs (paper_2302_03245_b200/       */
/* synthetic.py rmat_edges + _drop_self_loops), threaded, for C5 on    */
/* the host.  Not a reference function: the reference has no R-MAT    */
/* generator; this restates the repo's seeded definition so the C5     */
/* edge list reaches the oracle independently of the device generator. */
/* ------------------------------------------------------------------ */
static inline uint64_t orc_mix64(uint64_t x)
{
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

typedef struct {
    int scale, pass;
    uint64_t key0, ta, tb, tc;
    int64_t lo, hi, kept, out;
    int64_t *src, *dst;
} rmat_job;

static void *rmat_main(void *arg)
{
    rmat_job *J = (rmat_job *)arg;
    const uint64_t G = 0x9E3779B97F4A7C15ull;
    int64_t k = 0;
    for (int64_t i = J->lo; i < J->hi; ++i) {
        uint64_t base = J->key0 + (uint64_t)i * 64ull * G, s = 0, d = 0;
        for (int l = 0; l < J->scale; ++l) {
            uint64_t u = orc_mix64(base + (uint64_t)l * G) >> 32;
            s = (s << 1) | (uint64_t)(u >= J->tb);
            d = (d << 1) | (uint64_t)((u >= J->ta && u < J->tb) || u >= J->tc);
        }
        if (s == d) continue;                      /* self-loop dropped, order kept */
        if (J->pass) { J->src[J->out + k] = (int64_t)s; J->dst[J->out + k] = (int64_t)d; }
        ++k;
    }
    J->kept = k;
    return NULL;
}

/* ta/tb/tc are the cumulative thresholds (synthetic.rmat_thresholds).
 * src/dst NULL: count only.  Returns the number of non-loop samples. */
int64_t orc_rmat(int scale, int64_t edge_factor, uint64_t ta, uint64_t tb, uint64_t tc, uint64_t seed,
                 int threads, int64_t *src, int64_t *dst)
{
    if (threads < 1) threads = 1;
    const int64_t total = edge_factor << scale;
    rmat_job *J = (rmat_job *)calloc((size_t)threads, sizeof(rmat_job));
    pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    const uint64_t key0 = orc_mix64(seed);
    for (int pass = 0; pass < (src ? 2 : 1); ++pass) {
        int64_t out = 0;
        for (int k = 0; k < threads; ++k) {
            J[k].scale = scale; J[k].pass = pass; J[k].key0 = key0;
            J[k].ta = ta; J[k].tb = tb; J[k].tc = tc;
            J[k].lo = total * k / threads; J[k].hi = total * (k + 1) / threads;
            J[k].src = src; J[k].dst = dst;
            if (pass) { J[k].out = out; out += J[k].kept; }
            pthread_create(&th[k], NULL, rmat_main, &J[k]);
        }
        for (int k = 0; k < threads; ++k) pthread_join(th[k], NULL);
    }
    int64_t kept = 0;
    for (int k = 0; k < threads; ++k) kept += J[k].kept;
    free(J); free(th);
    return kept;
}

/* ------------------------------------------------------------------ */
/* power_method (solvers.py:186-243) with _WalkMultiplier (124-183)    */
/* ------------------------------------------------------------------ */
typedef struct {
    int64_t lo, hi;
    const int64_t *in_offsets, *in_sources;
    const double *z, *p;
    double restart, *nxt;
} power_job;

static void *power_main(void *arg)
{
    power_job *J = (power_job *)arg;
    for (int64_t v = J->lo; v < J->hi; ++v) {
        double y = 0.0;
        for (int64_t e = J->in_offsets[v]; e < J->in_offsets[v + 1]; ++e) y += J->z[J->in_sources[e]];
        J->nxt[v] = y + J->restart * J->p[v];
    }
    return NULL;
}

/* threads > 1: the multiply split by destination range, as
 * _WalkMultiplier(workers) does (solvers.py:124-183) -- identical result */
int64_t orc_power(int64_t n, const int64_t *in_offsets, const int64_t *in_sources,
                  const int64_t *out_degree, double c, const double *p,
                  int64_t iterations, double tolerance, double *pi, double *deltas, int threads)
{
    if (threads < 1) threads = 1;
    double *inv = (double *)malloc(sizeof(double) * n);
    double *z = (double *)malloc(sizeof(double) * n);
    double *nxt = (double *)malloc(sizeof(double) * n);
    power_job *J = (power_job *)calloc((size_t)threads, sizeof(power_job));
    pthread_t *th = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    for (int64_t v = 0; v < n; ++v) {
        inv[v] = out_degree[v] > 0 ? 1.0 / (double)out_degree[v] : 0.0;
        pi[v] = p[v];
    }
    int64_t k;
    for (k = 0; k < iterations; ++k) {
        double dang = 0.0;
        for (int64_t v = 0; v < n; ++v) {
            z[v] = c * pi[v] * inv[v];                                  /* solvers.py:173 */
            if (out_degree[v] == 0) dang += pi[v];
        }
        double restart = c * dang + (1.0 - c);                           /* solvers.py:219 */
        for (int t = 0; t < threads; ++t) {
            J[t] = (power_job){n * t / threads, n * (t + 1) / threads, in_offsets, in_sources, z, p, restart, nxt};
            if (threads > 1) pthread_create(&th[t], NULL, power_main, &J[t]);
            else power_main(&J[t]);
        }
        if (threads > 1)
            for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
        double total = 0.0;
        for (int64_t v = 0; v < n; ++v) total += nxt[v];
        double delta = 0.0;
        for (int64_t v = 0; v < n; ++v) {
            double x = nxt[v] / total;
            delta += x > pi[v] ? x - pi[v] : pi[v] - x;
            pi[v] = x;
        }
        deltas[k] = delta;
        if (tolerance > 0.0 && delta < tolerance) { ++k; break; }
    }
    free(inv); free(z); free(nxt); free(J); free(th);
    return k;
}

/* ------------------------------------------------------------------ */
/* Asynchronous engine: K free-running workers + a quiescence monitor  */
/* restating _kernels.pyx:66-137 and engines.py:120-216.  Used only as  */
/* the "port" CPU baseline when oracle/_ref (the reference's own       */
/* compiled worker loop) is unavailable.                               */
/* ------------------------------------------------------------------ */
typedef struct {
    _Atomic uint64_t *h;           /* doubles as raw bits */
    double *reserved;
    const int64_t *offsets, *targets, *degree, *vertices, *dt_count;
    int64_t nv;
    double xi, c;
    _Atomic int64_t *stop;
    _Atomic int64_t *counters;     /* started, finished, edges, dangling, vertices; 8-stride */
} orc_worker;

static inline double bits2d(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }
static inline uint64_t d2bits(double d) { uint64_t b; memcpy(&b, &d, 8); return b; }

static void *orc_worker_main(void *arg)
{
    orc_worker *w = (orc_worker *)arg;
    while (atomic_load(w->stop) == 0) {
        int64_t done = 0;
        for (int64_t i = 0; i < w->nv; ++i) {
            if (atomic_load(w->stop)) break;
            int64_t v = w->vertices[i];
            if (bits2d(atomic_load(&w->h[v])) <= w->xi) continue;
            atomic_fetch_add(&w->counters[0], 1);
            double mass = bits2d(atomic_exchange(&w->h[v], d2bits(0.0)));
            w->reserved[v] += mass;
            int64_t lo = w->offsets[v], hi = w->offsets[v + 1];
            if (hi > lo) {
                double share = w->c * mass / (double)w->degree[v];
                for (int64_t e = lo; e < hi; ++e) {
                    _Atomic uint64_t *cell = &w->h[w->targets[e]];
                    uint64_t old = atomic_load_explicit(cell, memory_order_relaxed);
                    while (!atomic_compare_exchange_weak(cell, &old, d2bits(bits2d(old) + share))) {}
                }
            }
            atomic_fetch_add(&w->counters[2], hi - lo);
            atomic_fetch_add(&w->counters[3], w->dt_count ? w->dt_count[v] : 0);
            atomic_fetch_add(&w->counters[4], 1);
            atomic_fetch_add(&w->counters[1], 1);
            ++done;
        }
        if (done == 0) usleep(20);
    }
    return NULL;
}

/* vertex sets arrive concatenated: set j is vertices[set_offsets[j] .. set_offsets[j+1]) */
int orc_async_phase(int64_t n, double *h, double *reserved,
                    const int64_t *offsets, const int64_t *targets, const int64_t *degree,
                    const int64_t *vertices, const int64_t *set_offsets, int workers,
                    const int64_t *scan_ids, int64_t n_scan, const int64_t *dt_count,
                    double xi, double c, int64_t *push_ops, int64_t *push_ops_dangling)
{
    (void)n;
    _Atomic int64_t stop = 0;
    _Atomic int64_t *ctr = (_Atomic int64_t *)calloc((size_t)workers * 8, sizeof(int64_t));
    orc_worker *ws = (orc_worker *)calloc((size_t)workers, sizeof(orc_worker));
    pthread_t *th = (pthread_t *)calloc((size_t)workers, sizeof(pthread_t));
    _Atomic uint64_t *hb = (_Atomic uint64_t *)h;
    for (int j = 0; j < workers; ++j) {
        ws[j] = (orc_worker){hb, reserved, offsets, targets, degree,
                             vertices + set_offsets[j], dt_count,
                             set_offsets[j + 1] - set_offsets[j], xi, c, &stop, ctr + 8 * j};
        pthread_create(&th[j], NULL, orc_worker_main, &ws[j]);
    }
    for (;;) {                           /* probe: _kernels.pyx:111-137 */
        int64_t s1 = 0, f1 = 0, s2 = 0, f2 = 0;
        for (int j = 0; j < workers; ++j) s1 += atomic_load(&ctr[8 * j]);
        for (int j = 0; j < workers; ++j) f1 += atomic_load(&ctr[8 * j + 1]);
        int below = s1 == f1;
        for (int64_t i = 0; below && i < n_scan; ++i)
            if (bits2d(atomic_load(&hb[scan_ids[i]])) > xi) below = 0;
        if (below) {
            for (int j = 0; j < workers; ++j) s2 += atomic_load(&ctr[8 * j]);
            for (int j = 0; j < workers; ++j) f2 += atomic_load(&ctr[8 * j + 1]);
            if (s2 != s1 || f2 != f1) below = 0;
        }
        if (below) break;
        if (n_scan > 100000) usleep(500);  /* engines.py:194 */
    }
    atomic_store(&stop, 1);
    for (int j = 0; j < workers; ++j) pthread_join(th[j], NULL);
    int64_t po = 0, pd = 0;
    for (int j = 0; j < workers; ++j) { po += ctr[8 * j + 2]; pd += ctr[8 * j + 3]; }
    *push_ops = po;
    *push_ops_dangling = pd;
    free(ctr); free(ws); free(th);
    return 0;
}
