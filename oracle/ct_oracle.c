/*
 * ct_oracle.c -- plain, slow, obviously-correct CPU oracle for Compact-Table
 * propagation (arXiv 2507.18413).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this file's library.  The product path
 * (paper_2507_18413_b200/, include/) never includes, links or calls it, and it
 * shares no code, header, table or helper with the CUDA path.
 *
 * What it computes (section 2):
 *   - L52-55  : c is GAC iff every value a of every x_i has a tuple of rel(c)
 *               with a in position i ("a is supported"); unsupported values are
 *               removed; if no solution exists, unsatisfiability is reported.
 *   - L189-193: tuple tau_j is *valid* iff tau_j[i] in dom(x_i) for every i;
 *               currTable bit j = 1 iff tau_j is valid.
 *   - L144-146: Alg. 1 fails iff currTable = 0 (no valid tuple).
 *   - L226-238: Alg. 3 keeps a in dom(x_i) iff currTable & supports[x_i,a] != 0,
 *               i.e. iff some valid tuple has value a in position i.
 * So, given the domains D_in (the domains after the caller's removals), the
 * result is:  V = { j : all i, tau_j[i] in D_in(x_i) };  FAIL iff V is empty;
 * else D_out(x_i) = { tau_j[i] : j in V }.  This is the definition written out
 * as one tuple scan (no supports matrix, no bitsets, no residues, no index).
 *
 * Readings:
 *   - a tuple value outside [lo_i, lo_i + d_i) is never in any domain, so such
 *     a tuple is never valid;
 *   - D_out is not written on FAIL.
 *
 * Encoding (the oracle's own): domains are one byte per (variable, value);
 * variable i's d_i bytes start at rowbase_i = d_0 + ... + d_{i-1}; byte
 * rowbase_i + (v - lo_i) is 1 iff v is in the domain.  tuples is int32
 * [t][n] row-major.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Returns 1 (OK, GAC domains written to dom_out), 0 (FAIL), -1 (bad args).
 * valid_out (may be NULL): t bytes, valid_out[j] = 1 iff tau_j is valid. */
int oracle_gac(int32_t n, const int32_t *lo, const int32_t *d, int64_t t,
               const int32_t *tuples, const uint8_t *dom_in, uint8_t *dom_out,
               uint8_t *valid_out)
{
    if (n < 1) return -1;
    int64_t *rowbase = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    if (!rowbase) return -1;
    int64_t R = 0;
    for (int32_t i = 0; i < n; ++i) { rowbase[i] = R; R += d[i]; }

    uint8_t *acc = (uint8_t *)calloc((size_t)(R > 0 ? R : 1), 1);
    if (!acc) { free(rowbase); return -1; }
    int any_valid = 0;

    for (int64_t j = 0; j < t; ++j) {
        const int32_t *tau = tuples + j * (int64_t)n;
        int valid = 1;
        for (int32_t i = 0; i < n; ++i) {
            int64_t v = (int64_t)tau[i] - lo[i];
            if (v < 0 || v >= d[i] || !dom_in[rowbase[i] + v]) { valid = 0; break; }
        }
        if (valid_out) valid_out[j] = (uint8_t)valid;
        if (valid) {
            any_valid = 1;
            for (int32_t i = 0; i < n; ++i)
                acc[rowbase[i] + ((int64_t)tau[i] - lo[i])] = 1;
        }
    }
    if (any_valid) memcpy(dom_out, acc, (size_t)R);
    free(acc);
    free(rowbase);
    return any_valid;
}

/*
 * The same definition with the tuple scan split into `nthreads` contiguous
 * ranges (timing on all host cores, and parity at the configs' full sizes):
 * V is the union of the ranges' valid sets and D_out the union of their
 * projections, so every range is one oracle_gac call on its slice of the
 * tuples and the results are OR-ed.  nthreads <= 1 is oracle_gac itself.
 * Pinned to oracle_gac on random instances (tests/test_oracle.py).
 */
typedef struct {
    int32_t n; const int32_t *lo, *d; int64_t t; const int32_t *tuples;
    const uint8_t *dom_in; uint8_t *dom_out; uint8_t *valid_out; int result;
} gac_slice;

static void *gac_slice_run(void *arg)
{
    gac_slice *a = (gac_slice *)arg;
    a->result = oracle_gac(a->n, a->lo, a->d, a->t, a->tuples, a->dom_in, a->dom_out, a->valid_out);
    return NULL;
}

int oracle_gac_split(int32_t n, const int32_t *lo, const int32_t *d, int64_t t,
                     const int32_t *tuples, const uint8_t *dom_in, uint8_t *dom_out,
                     uint8_t *valid_out, int32_t nthreads)
{
    if (n < 1) return -1;
    if (nthreads <= 1 || t < 2 * (int64_t)nthreads)
        return oracle_gac(n, lo, d, t, tuples, dom_in, dom_out, valid_out);
    int64_t R = 0;
    for (int32_t i = 0; i < n; ++i) R += d[i];
    gac_slice *sl = (gac_slice *)calloc((size_t)nthreads, sizeof(gac_slice));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    uint8_t *outs = (uint8_t *)calloc((size_t)nthreads * (size_t)(R > 0 ? R : 1), 1);
    if (!sl || !th || !outs) { free(sl); free(th); free(outs); return -1; }
    for (int32_t k = 0; k < nthreads; ++k) {
        int64_t j0 = t * k / nthreads, j1 = t * (k + 1) / nthreads;
        sl[k].n = n; sl[k].lo = lo; sl[k].d = d; sl[k].t = j1 - j0;
        sl[k].tuples = tuples + j0 * (int64_t)n; sl[k].dom_in = dom_in;
        sl[k].dom_out = outs + (size_t)k * (size_t)(R > 0 ? R : 1);
        sl[k].valid_out = valid_out ? valid_out + j0 : NULL;
        if (pthread_create(&th[k], NULL, gac_slice_run, &sl[k]) != 0) gac_slice_run(&sl[k]), th[k] = 0;
    }
    int any = 0, bad = 0;
    for (int32_t k = 0; k < nthreads; ++k) {
        if (th[k]) pthread_join(th[k], NULL);
        if (sl[k].result < 0) bad = 1;
        if (sl[k].result == 1) any = 1;
    }
    if (any && !bad) {
        memset(dom_out, 0, (size_t)R);
        for (int32_t k = 0; k < nthreads; ++k)
            if (sl[k].result == 1)
                for (int64_t r = 0; r < R; ++r) dom_out[r] |= sl[k].dom_out[r];
    }
    free(sl); free(th); free(outs);
    return bad ? -1 : any;
}

/* One row of the static supports matrix, by its definition:
 * out[j] = 1 iff tau_j[i] = value.  (Used to pin the CUDA supports builder.) */
void oracle_supports_row(int32_t n, int64_t t, const int32_t *tuples,
                         int32_t i, int32_t value, uint8_t *out)
{
    for (int64_t j = 0; j < t; ++j)
        out[j] = (uint8_t)(tuples[j * (int64_t)n + i] == value);
}

/*
 * Fixpoint of several table constraints sharing variables (SURVEY §8(f) f1,
 * the engine alternates propagation until nothing changes).
 * Tables are revisited in a fixed round-robin order until a full round changes
 * no domain (the greatest fixpoint is unique) or one fails.
 *
 * Model: nv variables with global domains dom[] (byte per value, variable v at
 * vbase_v = dv_0+...+dv_{v-1}, values lo_v..lo_v+dv_v-1).  Table k has arity
 * ar[k], scope scope[k][0..ar-1] (global var ids), t[k] tuples at tuples[k].
 * Returns 1 OK (dom updated in place), 0 FAIL, -1 bad args.
 */
int oracle_fixpoint_split(int32_t nv, const int32_t *vlo, const int32_t *vd, int32_t ntab,
                          const int32_t *ar, const int32_t *const *scope, const int64_t *t,
                          const int32_t *const *tuples, uint8_t *dom, int32_t nthreads)
{
    int64_t *vbase = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nv + 1));
    if (!vbase) return -1;
    vbase[0] = 0;
    for (int32_t v = 0; v < nv; ++v) vbase[v + 1] = vbase[v] + vd[v];
    int result = 1;
    int changed = 1;
    while (changed && result == 1) {
        changed = 0;
        for (int32_t k = 0; k < ntab && result == 1; ++k) {
            int32_t n = ar[k];
            int32_t *lo = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
            int32_t *d = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
            int64_t R = 0;
            for (int32_t i = 0; i < n; ++i) { lo[i] = vlo[scope[k][i]]; d[i] = vd[scope[k][i]]; R += d[i]; }
            uint8_t *din = (uint8_t *)malloc((size_t)R);
            uint8_t *dout = (uint8_t *)malloc((size_t)R);
            int64_t off = 0;
            for (int32_t i = 0; i < n; ++i) {
                memcpy(din + off, dom + vbase[scope[k][i]], (size_t)d[i]);
                off += d[i];
            }
            int r = oracle_gac_split(n, lo, d, t[k], tuples[k], din, dout, NULL, nthreads);
            if (r != 1) {
                result = r;
            } else {
                off = 0;
                for (int32_t i = 0; i < n; ++i) {
                    uint8_t *g = dom + vbase[scope[k][i]];
                    for (int32_t a = 0; a < d[i]; ++a) {
                        if (g[a] != dout[off + a]) { g[a] = dout[off + a]; changed = 1; }
                    }
                    off += d[i];
                }
            }
            free(lo); free(d); free(din); free(dout);
        }
    }
    free(vbase);
    return result;
}

/* The fixpoint with one thread per table call (the plain definition). */
int oracle_fixpoint(int32_t nv, const int32_t *vlo, const int32_t *vd, int32_t ntab,
                    const int32_t *ar, const int32_t *const *scope, const int64_t *t,
                    const int32_t *const *tuples, uint8_t *dom)
{
    return oracle_fixpoint_split(nv, vlo, vd, ntab, ar, scope, t, tuples, dom, 1);
}

/*
 * ---------------------------------------------------------------- f4: short and
 * negative tables (PAPER.md L66-68 and its footnote: "A table
 * c is positive if its tuples list the allowed values for var(c).  A table
 * explicitly listing the disallowed tuples is said negative.  A table is short
 * if more than one domain value can be specified in each cell.").  The paper
 * defines the tables and leaves their propagation to the cited CT extensions;
 * GAC itself is still L52-55 on the relation the table denotes.
 */

/* Short tables: a cell holding ORACLE_STAR (INT32_MIN) stands for every value
 * of its variable's initial domain (reading R-f4a: the star cell, the
 * short-table form the cited extension propagates); any other cell is one value.
 * A short tuple denotes the Cartesian product of its cells, so rel(c) is the
 * union of those products and, by L52-55:
 *   V = { j : every cell of tau_j meets D_in(x_i) }   (the products meeting D);
 *   FAIL iff V is empty;
 *   D_out(x_i) = union over j in V of (cell_j[i] intersect D_in(x_i)).
 * valid_out (may be NULL): t bytes, 1 iff tau_j in V.  Returns 1/0/-1 as
 * oracle_gac. */
#define ORACLE_STAR (-2147483647 - 1)

int oracle_gac_short(int32_t n, const int32_t *lo, const int32_t *d, int64_t t,
                     const int32_t *tuples, const uint8_t *dom_in, uint8_t *dom_out,
                     uint8_t *valid_out)
{
    if (n < 1) return -1;
    int64_t *rowbase = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    uint8_t *nonempty = (uint8_t *)malloc((size_t)n);
    if (!rowbase || !nonempty) { free(rowbase); free(nonempty); return -1; }
    int64_t R = 0;
    for (int32_t i = 0; i < n; ++i) {
        rowbase[i] = R;
        nonempty[i] = 0;
        for (int32_t a = 0; a < d[i]; ++a) if (dom_in[R + a]) nonempty[i] = 1;
        R += d[i];
    }
    uint8_t *acc = (uint8_t *)calloc((size_t)(R > 0 ? R : 1), 1);
    if (!acc) { free(rowbase); free(nonempty); return -1; }
    int any_valid = 0;
    for (int64_t j = 0; j < t; ++j) {
        const int32_t *tau = tuples + j * (int64_t)n;
        int valid = 1;
        for (int32_t i = 0; i < n; ++i) {
            if (tau[i] == ORACLE_STAR) {                      /* meets D iff D nonempty */
                if (!nonempty[i]) { valid = 0; break; }
            } else {
                int64_t v = (int64_t)tau[i] - lo[i];
                if (v < 0 || v >= d[i] || !dom_in[rowbase[i] + v]) { valid = 0; break; }
            }
        }
        if (valid_out) valid_out[j] = (uint8_t)valid;
        if (valid) {
            any_valid = 1;
            for (int32_t i = 0; i < n; ++i) {
                if (tau[i] == ORACLE_STAR) {
                    for (int32_t a = 0; a < d[i]; ++a)
                        if (dom_in[rowbase[i] + a]) acc[rowbase[i] + a] = 1;
                } else {
                    acc[rowbase[i] + ((int64_t)tau[i] - lo[i])] = 1;
                }
            }
        }
    }
    if (any_valid) memcpy(dom_out, acc, (size_t)R);
    free(acc); free(rowbase); free(nonempty);
    return any_valid;
}

/* Negative tables: the tuples list the FORBIDDEN assignments, so rel(c) is the
 * product of the initial domains minus that list (duplicates list one tuple
 * once; a tuple with a value outside [lo_i, lo_i + d_i) forbids nothing).  By
 * L52-55, value a of x_i is supported iff some assignment of D_in with x_i = a
 * is not forbidden, i.e. iff
 *   c[i][a] = |{ distinct forbidden tau in D_in(x_1) x ... x D_in(x_n) : tau[i] = a }|
 * is smaller than P_i = prod over k != i of |D_in(x_k)|, the number of such
 * assignments.  FAIL iff some D_out(x_i) is empty.  The count is the definition
 * written out; duplicates are removed by sorting the tuple list (qsort).
 * nvalid_out (may be NULL): |distinct forbidden tuples inside D_in|. */
static int32_t g_cmp_n;
static int cmp_tuple(const void *a, const void *b)
{
    const int32_t *x = (const int32_t *)a, *y = (const int32_t *)b;
    for (int32_t i = 0; i < g_cmp_n; ++i) {
        if (x[i] < y[i]) return -1;
        if (x[i] > y[i]) return 1;
    }
    return 0;
}

int oracle_gac_negative(int32_t n, const int32_t *lo, const int32_t *d, int64_t t,
                        const int32_t *tuples, const uint8_t *dom_in, uint8_t *dom_out,
                        int64_t *nvalid_out)
{
    if (n < 1) return -1;
    int64_t *rowbase = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    double *size = (double *)malloc(sizeof(double) * (size_t)n);
    if (!rowbase || !size) { free(rowbase); free(size); return -1; }
    int64_t R = 0;
    for (int32_t i = 0; i < n; ++i) {
        rowbase[i] = R;
        size[i] = 0;
        for (int32_t a = 0; a < d[i]; ++a) size[i] += dom_in[R + a] ? 1 : 0;
        R += d[i];
    }
    int32_t *sorted = (int32_t *)malloc(sizeof(int32_t) * (size_t)(t > 0 ? t * n : 1));
    int64_t *cnt = (int64_t *)calloc((size_t)(R > 0 ? R : 1), sizeof(int64_t));
    if (!sorted || !cnt) { free(rowbase); free(size); free(sorted); free(cnt); return -1; }
    if (t > 0) memcpy(sorted, tuples, sizeof(int32_t) * (size_t)(t * n));
    g_cmp_n = n;   /* single-threaded by construction: the caller serialises */
    if (t > 1) qsort(sorted, (size_t)t, sizeof(int32_t) * (size_t)n, cmp_tuple);
    int64_t nvalid = 0;
    for (int64_t j = 0; j < t; ++j) {
        const int32_t *tau = sorted + j * (int64_t)n;
        if (j > 0 && cmp_tuple(tau - n, tau) == 0) continue;     /* duplicate */
        int inside = 1;
        for (int32_t i = 0; i < n; ++i) {
            int64_t v = (int64_t)tau[i] - lo[i];
            if (v < 0 || v >= d[i] || !dom_in[rowbase[i] + v]) { inside = 0; break; }
        }
        if (!inside) continue;
        ++nvalid;
        for (int32_t i = 0; i < n; ++i) cnt[rowbase[i] + ((int64_t)tau[i] - lo[i])] += 1;
    }
    /* P_i in double: exact while < 2^53, and every count is <= t < 2^53, so the
     * comparison c < P_i is exact whenever it can be false */
    int ok = 1;
    for (int32_t i = 0; i < n && ok; ++i) {
        double P = 1.0;
        for (int32_t k = 0; k < n; ++k) if (k != i) P *= size[k];
        int any = 0;
        for (int32_t a = 0; a < d[i]; ++a) {
            uint8_t keep = (uint8_t)(dom_in[rowbase[i] + a] && (double)cnt[rowbase[i] + a] < P);
            dom_out[rowbase[i] + a] = keep;
            any |= keep;
        }
        if (!any) ok = 0;
    }
    if (nvalid_out) *nvalid_out = nvalid;
    free(rowbase); free(size); free(sorted); free(cnt);
    return ok;
}
