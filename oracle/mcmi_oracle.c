/* oracle/mcmi_oracle.c — TEST INFRASTRUCTURE ONLY (see mcmi_oracle.h).
 *
 * Serial plain-C restatement of the reference build pipeline.  Each function
 * cites the reference lines it restates (paths relative to
 * /root/reference/proj).  Built with -ffp-contract=off so that no a*b+c is
 * fused, matching the reference's x86-64 build without -march.
 */
#include "mcmi_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- Philox */

/* rng.hpp:44-67 — Philox4x32-10, Random123 constants. */
void orc_philox(const uint32_t ctr[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* rng.hpp:32-41 — two u32 (lo first) -> 53-bit double in [0,1). */
static double u32pair_to_double(uint32_t lo, uint32_t hi) {
    const uint64_t u = ((uint64_t)hi << 32) | lo;
    return (double)(u >> 11) * 0x1.0p-53;
}

/* Reference-mode stream: RngStream(master_seed, row) (mc_engine.cpp:168). */
typedef struct {
    uint32_t key[2];
    uint64_t stream_id;
    uint64_t counter;
    uint32_t block[4];
    int pos;
} stream_t;

static void stream_init(stream_t* s, uint64_t seed, uint64_t id) {
    s->key[0] = (uint32_t)seed;
    s->key[1] = (uint32_t)(seed >> 32);
    s->stream_id = id;
    s->counter = 0;
    s->pos = 4;
}

static uint32_t stream_u32(stream_t* s) { /* rng.hpp:24-30 */
    if (s->pos == 4) {
        const uint32_t ctr[4] = {(uint32_t)s->counter, (uint32_t)(s->counter >> 32),
                                 (uint32_t)s->stream_id, (uint32_t)(s->stream_id >> 32)};
        orc_philox(ctr, s->key, s->block);
        s->counter++;
        s->pos = 0;
    }
    return s->block[s->pos++];
}

static double stream_double(stream_t* s) {
    const uint32_t lo = stream_u32(s);
    const uint32_t hi = stream_u32(s);
    return u32pair_to_double(lo, hi);
}

/* Keyed mode: u(row, chain, step) = double #(step & 1) of
 * philox({step >> 1, chain, row lo, row hi}, seed). */
static double keyed_double(uint64_t seed, uint64_t row, uint64_t chain, uint64_t step) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    const uint32_t ctr[4] = {(uint32_t)(step >> 1), (uint32_t)chain, (uint32_t)row,
                             (uint32_t)(row >> 32)};
    uint32_t b[4];
    orc_philox(ctr, key, b);
    return (step & 1) ? u32pair_to_double(b[2], b[3]) : u32pair_to_double(b[0], b[1]);
}

/* ------------------------------------------------------------------ CSR */

typedef struct {
    int64_t n;
    int64_t* rp;
    int64_t* ci;
    double* v;
} csr_t;

static void csr_free(csr_t* m) {
    free(m->rp);
    free(m->ci);
    free(m->v);
    m->rp = NULL;
    m->ci = NULL;
    m->v = NULL;
}

static int csr_alloc(csr_t* m, int64_t n, int64_t nnz) {
    m->n = n;
    m->rp = calloc((size_t)n + 1, sizeof(int64_t));
    m->ci = malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
    m->v = malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
    return m->rp && m->ci && m->v;
}

static void set_err(char* err, size_t errlen, const char* msg) {
    if (err && errlen) {
        strncpy(err, msg, errlen - 1);
        err[errlen - 1] = 0;
    }
}

/* ----------------------------------------------------------------- drop */

static const double* g_abs_for_sort;
static int cmp_abs_stable(const void* pa, const void* pb) {
    const int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
    const double fa = fabs(g_abs_for_sort[a]), fb = fabs(g_abs_for_sort[b]);
    if (fa < fb) return -1;
    if (fb < fa) return 1;
    return (a > b) - (a < b); /* stable: ties by position (csr.cpp:147-150) */
}

/* csr.cpp:127-157 (+ off_diagonal_range :88-105, filter_entries :109-123).
 * Returns 0 and fills *out (a copy when nothing is dropped). */
static int drop_small_entries(const csr_t* m, double p, int mode, csr_t* out, char* err,
                              size_t errlen) {
    if (!(p >= 0.0 && p <= 1.0)) {
        set_err(err, errlen, "drop fraction must lie in [0,1]");
        return 1;
    }
    const int64_t nnz = m->rp[m->n];
    char* keep = malloc((size_t)(nnz > 0 ? nnz : 1));
    if (!keep) return 5;
    memset(keep, 1, (size_t)(nnz > 0 ? nnz : 1));
    if (p != 0.0) {
        if (mode == 0) {
            double mn = 0.0, mx = 0.0;
            int seen = 0;
            for (int64_t i = 0; i < m->n; ++i)
                for (int64_t k = m->rp[i]; k < m->rp[i + 1]; ++k) {
                    if (m->ci[k] == i) continue;
                    const double a = fabs(m->v[k]);
                    if (!seen) {
                        mn = mx = a;
                        seen = 1;
                    } else {
                        if (a < mn) mn = a;
                        if (a > mx) mx = a;
                    }
                }
            if (mx != 0.0) {
                const double threshold = mn + p * (mx - mn);
                for (int64_t i = 0; i < m->n; ++i)
                    for (int64_t k = m->rp[i]; k < m->rp[i + 1]; ++k)
                        if (m->ci[k] != i && fabs(m->v[k]) < threshold) keep[k] = 0;
            }
        } else {
            int64_t cnt = 0;
            int64_t* off = malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
            if (!off) {
                free(keep);
                return 5;
            }
            for (int64_t i = 0; i < m->n; ++i)
                for (int64_t k = m->rp[i]; k < m->rp[i + 1]; ++k)
                    if (m->ci[k] != i) off[cnt++] = k;
            const size_t n_drop = (size_t)(p * (double)cnt);
            g_abs_for_sort = m->v;
            qsort(off, (size_t)cnt, sizeof(int64_t), cmp_abs_stable);
            for (size_t t = 0; t < n_drop && t < (size_t)cnt; ++t) keep[off[t]] = 0;
            free(off);
        }
    }
    int64_t kept = 0;
    for (int64_t k = 0; k < nnz; ++k) kept += keep[k];
    if (!csr_alloc(out, m->n, kept)) {
        free(keep);
        return 5;
    }
    int64_t o = 0;
    for (int64_t i = 0; i < m->n; ++i) {
        for (int64_t k = m->rp[i]; k < m->rp[i + 1]; ++k)
            if (keep[k]) {
                out->ci[o] = m->ci[k];
                out->v[o] = m->v[k];
                ++o;
            }
        out->rp[i + 1] = o;
    }
    free(keep);
    return 0;
}

/* ---------------------------------------------------------------- split */

typedef struct {
    int64_t n;
    double* b1_diag;
    csr_t a; /* A = I - B1^{-1} B_hat, zero diagonal, v == 0 skipped */
    double* p; /* MAO probabilities on A's pattern */
    double a_norm;
} split_t;

static void split_free(split_t* s) {
    free(s->b1_diag);
    free(s->p);
    csr_free(&s->a);
}

/* split.cpp:46-100 (+ with_explicit_diagonal :10-42, inf_norm csr.cpp:77-86,
 * transition_probabilities split.cpp:102-119). */
static int augment_and_split(const csr_t* b, double alpha, int mode, split_t* s, char* err,
                             size_t errlen) {
    memset(s, 0, sizeof(*s));
    if (!(alpha > 0.0)) {
        set_err(err, errlen, "alpha must be positive");
        return 1;
    }
    const int64_t n = b->n;
    double b_norm = 0.0; /* inf_norm: sequential row sums, then max */
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t k = b->rp[i]; k < b->rp[i + 1]; ++k) acc += fabs(b->v[k]);
        if (acc > b_norm) b_norm = acc;
    }
    s->n = n;
    s->b1_diag = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (!s->b1_diag) return 5;
    for (int64_t i = 0; i < n; ++i) {
        double d = 0.0; /* a structurally missing diagonal is materialized as 0 */
        for (int64_t k = b->rp[i]; k < b->rp[i + 1]; ++k)
            if (b->ci[k] == i) {
                d = b->v[k];
                break;
            }
        double shift = alpha * b_norm;
        if (mode == 1 && d < 0.0) shift = -shift;
        s->b1_diag[i] = d + shift;
        if (s->b1_diag[i] == 0.0) {
            char msg[128];
            snprintf(msg, sizeof msg, "degenerate diagonal after augmentation at row %lld",
                     (long long)i);
            set_err(err, errlen, msg);
            split_free(s);
            return 2;
        }
    }
    const int64_t nnz = b->rp[n];
    if (!csr_alloc(&s->a, n, nnz)) return 5;
    int64_t o = 0;
    double a_norm = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double row_sum = 0.0;
        for (int64_t k = b->rp[i]; k < b->rp[i + 1]; ++k) {
            const int64_t j = b->ci[k];
            if (j == i) continue;
            const double v = -b->v[k] / s->b1_diag[i];
            if (v == 0.0) continue;
            s->a.ci[o] = j;
            s->a.v[o] = v;
            ++o;
            row_sum += fabs(v);
        }
        s->a.rp[i + 1] = o;
        if (row_sum > a_norm) a_norm = row_sum;
    }
    s->a_norm = a_norm;
    if (!(a_norm < 1.0)) {
        char msg[128];
        snprintf(msg, sizeof msg, "diagonal dominance failure: ||A||inf = %f", a_norm);
        set_err(err, errlen, msg);
        split_free(s);
        return 2;
    }
    s->p = malloc(sizeof(double) * (size_t)(o > 0 ? o : 1));
    if (!s->p) return 5;
    for (int64_t i = 0; i < n; ++i) {
        double row_sum = 0.0;
        for (int64_t k = s->a.rp[i]; k < s->a.rp[i + 1]; ++k) row_sum += fabs(s->a.v[k]);
        for (int64_t k = s->a.rp[i]; k < s->a.rp[i + 1]; ++k)
            s->p[k] = fabs(s->a.v[k]) / row_sum;
    }
    return 0;
}

/* ---------------------------------------------------------------- budget */

/* mc_engine.cpp:12-33 */
static int derive_chain_budget(const orc_config* cfg, double a_norm, int64_t* n_chains,
                               int64_t* max_len, char* err, size_t errlen) {
    if (!(a_norm >= 0.0 && a_norm < 1.0)) {
        set_err(err, errlen, "||A|| must lie in [0,1)");
        return 1;
    }
    int64_t nc, ml;
    if (cfg->has_chains_override) {
        nc = cfg->chains_override;
    } else {
        const double root = 0.6745 / (cfg->epsilon * (1.0 - a_norm));
        nc = (int64_t)ceil(root * root);
    }
    if (cfg->has_max_len_override) {
        ml = cfg->max_len_override;
    } else if (a_norm <= 0.0) {
        ml = 1;
    } else {
        const double len = log(cfg->delta) / log(a_norm);
        ml = (int64_t)ceil(len);
        if (ml < 1) ml = 1;
    }
    if (nc < 1) nc = 1;
    *n_chains = nc;
    *max_len = ml;
    return 0;
}

/* ------------------------------------------------------------- row estimate */

typedef struct {
    double* acc;
    char* touched;
    int64_t* cols;
    int64_t ncols;
} workspace_t;

static void ws_deposit(workspace_t* ws, int64_t col, double w) { /* mc_engine.cpp:45-51 */
    if (!ws->touched[col]) {
        ws->touched[col] = 1;
        ws->cols[ws->ncols++] = col;
    }
    ws->acc[col] += w;
}

static void ws_reset(workspace_t* ws) {
    for (int64_t i = 0; i < ws->ncols; ++i) {
        ws->acc[ws->cols[i]] = 0.0;
        ws->touched[ws->cols[i]] = 0;
    }
    ws->ncols = 0;
}

static int cmp_i64(const void* pa, const void* pb) {
    const int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
    return (a > b) - (a < b);
}

typedef struct {
    int64_t col;
    double val;
} entry_t;

/* mc_engine.cpp:80-113 (+ sample_transition :64-78).  Emits the
 * column-sorted row acc[c] * (1 / chains_run). */
static int64_t estimate_row(const split_t* s, int64_t r, int64_t n_chains, int64_t max_len,
                            double delta, const orc_config* cfg, workspace_t* ws,
                            entry_t* row, int64_t* chains_run_out, int64_t* steps,
                            int64_t* deg_sum) {
    ws_reset(ws);
    stream_t rng;
    stream_init(&rng, cfg->master_seed, (uint64_t)r);
    int64_t chains_run = n_chains;
    for (int64_t chain = 0; chain < n_chains; ++chain) {
        int64_t state = r;
        double w = 1.0;
        int drew = 0;
        ws_deposit(ws, r, w);
        for (int64_t step = 0; step < max_len; ++step) {
            const int64_t begin = s->a.rp[state], end = s->a.rp[state + 1];
            int64_t k;
            if (begin == end) break; /* absorbing */
            *steps += 1;
            *deg_sum += end - begin;
            if (end - begin == 1) {
                k = begin; /* forced move, no randomness */
            } else {
                drew = 1;
                const double u = cfg->rng_mode == 0
                                     ? stream_double(&rng)
                                     : keyed_double(cfg->master_seed, (uint64_t)r,
                                                    (uint64_t)chain, (uint64_t)step);
                double cum = 0.0;
                k = end - 1; /* rounding slop lands on the last entry */
                for (int64_t q = begin; q < end; ++q) {
                    cum += s->p[q];
                    if (u < cum) {
                        k = q;
                        break;
                    }
                }
            }
            w *= s->a.v[k] / s->p[k];
            state = s->a.ci[k];
            ws_deposit(ws, state, w);
            if (fabs(w) < delta) break;
        }
        if (chain == 0 && !drew) {
            chains_run = 1;
            break;
        }
    }
    qsort(ws->cols, (size_t)ws->ncols, sizeof(int64_t), cmp_i64);
    const double inv_n = 1.0 / (double)chains_run;
    for (int64_t i = 0; i < ws->ncols; ++i) {
        row[i].col = ws->cols[i];
        row[i].val = ws->acc[ws->cols[i]] * inv_n;
    }
    *chains_run_out = chains_run;
    return ws->ncols;
}

/* mc_engine.cpp:124-145 — order by (diag first, |v| desc, col asc). */
static int64_t g_diag_col;
static int cmp_topk(const void* pa, const void* pb) {
    const entry_t* a = pa;
    const entry_t* b = pb;
    const int da = a->col == g_diag_col, db = b->col == g_diag_col;
    if (da != db) return da ? -1 : 1;
    const double ma = fabs(a->val), mb = fabs(b->val);
    if (ma != mb) return ma > mb ? -1 : 1;
    return (a->col > b->col) - (a->col < b->col);
}
static int cmp_entry_col(const void* pa, const void* pb) {
    const entry_t* a = pa;
    const entry_t* b = pb;
    return (a->col > b->col) - (a->col < b->col);
}

static int64_t retain_top_k(entry_t* row, int64_t len, int64_t k, int64_t diag_col) {
    if (k <= 0 || len <= k) return len;
    g_diag_col = diag_col;
    qsort(row, (size_t)len, sizeof(entry_t), cmp_topk);
    qsort(row, (size_t)k, sizeof(entry_t), cmp_entry_col); /* restore column order */
    return k;
}

/* --------------------------------------------------------------- pipeline */

struct orc_result {
    int64_t n_rows;
    int64_t* rp;
    int64_t* ci;
    double* v;
    int64_t nnz;
    int64_t* chains_used;
    int64_t* entries_before;
    int64_t n_chains, max_len;
    int64_t walk_steps, walk_deg_sum;
    double a_norm;
};

void orc_result_free(orc_result* r) {
    if (!r) return;
    free(r->rp);
    free(r->ci);
    free(r->v);
    free(r->chains_used);
    free(r->entries_before);
    free(r);
}

/* mc_engine.cpp:153-226 (serial branch), restricted to rows [row_begin, row_end). */
int orc_build(int64_t n, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
              const orc_config* cfg, int64_t row_begin, int64_t row_end, orc_result** out,
              char* err, size_t errlen) {
    *out = NULL;
    if (row_begin < 0) row_begin = 0;
    if (row_end < 0 || row_end > n) row_end = n;
    if (row_end < row_begin) row_end = row_begin;
    csr_t b = {n, (int64_t*)row_ptr, (int64_t*)col_idx, (double*)values};
    csr_t red;
    int st = drop_small_entries(&b, cfg->drop_fraction, cfg->drop_mode, &red, err, errlen);
    if (st) return st;
    split_t s;
    st = augment_and_split(&red, cfg->alpha, cfg->mode, &s, err, errlen);
    csr_free(&red);
    if (st) return st;
    int64_t nc, ml;
    st = derive_chain_budget(cfg, s.a_norm, &nc, &ml, err, errlen);
    if (st) {
        split_free(&s);
        return st;
    }
    orc_result* res = calloc(1, sizeof(orc_result));
    const int64_t rows = row_end - row_begin;
    res->n_rows = rows;
    res->n_chains = nc;
    res->max_len = ml;
    res->a_norm = s.a_norm;
    res->rp = calloc((size_t)rows + 1, sizeof(int64_t));
    res->chains_used = calloc((size_t)(rows > 0 ? rows : 1), sizeof(int64_t));
    res->entries_before = calloc((size_t)(rows > 0 ? rows : 1), sizeof(int64_t));
    workspace_t ws;
    ws.acc = calloc((size_t)(n > 0 ? n : 1), sizeof(double));
    ws.touched = calloc((size_t)(n > 0 ? n : 1), 1);
    ws.cols = malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    ws.ncols = 0;
    entry_t* row = malloc(sizeof(entry_t) * (size_t)(n > 0 ? n : 1));
    int64_t cap = 1024, nnz = 0;
    res->ci = malloc(sizeof(int64_t) * (size_t)cap);
    res->v = malloc(sizeof(double) * (size_t)cap);
    for (int64_t r = row_begin; r < row_end; ++r) {
        int64_t chains_run = 0;
        int64_t len = estimate_row(&s, r, nc, ml, cfg->delta, cfg, &ws, row, &chains_run,
                                   &res->walk_steps, &res->walk_deg_sum);
        res->chains_used[r - row_begin] = chains_run;
        res->entries_before[r - row_begin] = len;
        len = retain_top_k(row, len, cfg->retain_k, r);
        for (int64_t i = 0; i < len; ++i) { /* scale_columns, mc_engine.cpp:147-149 */
            const double v = row[i].val / s.b1_diag[row[i].col];
            if (v == 0.0 && row[i].col != r) continue; /* prune, mc_engine.cpp:174-176 */
            if (nnz == cap) {
                cap *= 2;
                res->ci = realloc(res->ci, sizeof(int64_t) * (size_t)cap);
                res->v = realloc(res->v, sizeof(double) * (size_t)cap);
            }
            res->ci[nnz] = row[i].col;
            res->v[nnz] = v;
            ++nnz;
        }
        res->rp[r - row_begin + 1] = nnz;
    }
    res->nnz = nnz;
    free(ws.acc);
    free(ws.touched);
    free(ws.cols);
    free(row);
    split_free(&s);
    *out = res;
    return 0;
}

void orc_result_sizes(const orc_result* r, int64_t* n_rows, int64_t* nnz) {
    *n_rows = r->n_rows;
    *nnz = r->nnz;
}

void orc_result_copy(const orc_result* r, int64_t* row_ptr, int64_t* col_idx, double* values,
                     int64_t* chains_used, int64_t* entries_before, int64_t* n_chains,
                     int64_t* max_len, int64_t* walk_steps, int64_t* walk_deg_sum,
                     double* a_norm) {
    if (row_ptr) memcpy(row_ptr, r->rp, sizeof(int64_t) * (size_t)(r->n_rows + 1));
    if (col_idx) memcpy(col_idx, r->ci, sizeof(int64_t) * (size_t)r->nnz);
    if (values) memcpy(values, r->v, sizeof(double) * (size_t)r->nnz);
    if (chains_used) memcpy(chains_used, r->chains_used, sizeof(int64_t) * (size_t)r->n_rows);
    if (entries_before)
        memcpy(entries_before, r->entries_before, sizeof(int64_t) * (size_t)r->n_rows);
    if (n_chains) *n_chains = r->n_chains;
    if (max_len) *max_len = r->max_len;
    if (walk_steps) *walk_steps = r->walk_steps;
    if (walk_deg_sum) *walk_deg_sum = r->walk_deg_sum;
    if (a_norm) *a_norm = r->a_norm;
}
