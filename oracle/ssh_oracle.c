/*
 * ssh_oracle.c — CPU restatement of the reference SSH hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for the B200 build.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path (paper_1610_07328_b200) never links or calls it.
 *
 * Every function restates one function of the reference package `sshts`
 * (/root/reference/pkg/src/sshts, cited as file:line) in plain C99 double
 * arithmetic.  Compile with -ffp-contract=off: the reference's numpy matmul
 * inner loop and numba DTW are FMA-free, so every
 * multiply and add here is a separate IEEE operation in reference order.
 *
 * The CWS variates are NOT recomputed here: log() bits come from numpy
 * (wmh.py:70-72) and are passed in as tables r / ln_c / beta / ln_w that
 * oracle.py generates with np.log exactly as the reference does.  oracle.py
 * also carries a direct numpy restatement of _cws_keys that pins the tables.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define SALT_KEY 0xEB44ACCAB455D165ULL

/* wmh.py:34-44 — splitmix64 finalizer, wrapping arithmetic. */
static inline uint64_t mix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t orc_mix64(uint64_t x) { return mix64(x); }

static inline double load_x(const void *X, int is_f32, int64_t idx) {
    return is_f32 ? (double)((const float *)X)[idx] : ((const double *)X)[idx];
}

/* sketch.py:46-48 */
int orc_num_sketch_bits(int m, int W, int delta) { return (m - W) / delta + 1; }

/* sketch.py:51-61 (sketch_values) and sketch.py:69-89 (sketch_matrix):
 * dots = windows @ weights via numpy's non-BLAS matmul loop, i.e. acc starts
 * at 0 and adds x*w in k order; bit = +1 if dot >= 0 else -1.  Optionally
 * reports the raw dots (for near-zero accounting). */
void orc_sketch(const void *X, int is_f32, int64_t N, int m, int64_t ld,
                const double *w, int W, int delta, int8_t *bits, double *dots,
                int threads) {
    int nb = orc_num_sketch_bits(m, W, delta);
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
    for (int64_t s = 0; s < N; s++) {
        for (int i = 0; i < nb; i++) {
            double acc = 0.0;
            for (int k = 0; k < W; k++) {
                double prod = load_x(X, is_f32, s * ld + (int64_t)i * delta + k) * w[k];
                acc = acc + prod;
            }
            bits[s * nb + i] = acc >= 0.0 ? 1 : -1;
            if (dots) dots[s * nb + i] = acc;
        }
    }
}

static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

/* shingle.py:56-68 (tokenize_bits: first bit most significant, +1 -> 1) and
 * np.unique(..., return_counts=True) at index.py:118 / shingle.py:71-75.
 * `scratch` holds nb-n+1 uint64.  Returns the distinct-token count D. */
int orc_shingle(const int8_t *bits, int nb, int n, uint64_t *tokens, int64_t *counts,
                uint64_t *scratch) {
    int nt = nb - n + 1;
    for (int i = 0; i < nt; i++) {
        uint64_t tok = 0;
        for (int j = 0; j < n; j++) tok = (tok << 1) | (uint64_t)(bits[i + j] > 0);
        scratch[i] = tok;
    }
    qsort(scratch, (size_t)nt, sizeof(uint64_t), cmp_u64);
    int D = 0;
    for (int i = 0; i < nt; i++) {
        if (D > 0 && tokens[D - 1] == scratch[i]) {
            counts[D - 1]++;
        } else {
            tokens[D] = scratch[i];
            counts[D] = 1;
            D++;
        }
    }
    return D;
}

/* wmh.py:52-81 (_cws_keys) evaluated from host tables.  Table layout
 * [token][slot] with `S` slots; ln_w[c] = np.log(float(c)).
 *   t    = floor(ln_w / r + beta)          wmh.py:74
 *   ln_y = r * (t - beta)                  wmh.py:75
 *   ln_a = ln_c - ln_y - r                 wmh.py:76
 *   j    = argmin(ln_a) (first occurrence) wmh.py:78
 *   key  = mix64(tok_j ^ mix64(uint64(int64(t_j)) ^ SALT_KEY))   wmh.py:79-81 */
void orc_cws_keys(const uint64_t *tokens, const int64_t *counts, int D, int S,
                  const double *tab_r, const double *tab_lnc, const double *tab_beta,
                  const double *ln_w, uint64_t *keys) {
    for (int s = 0; s < S; s++) {
        double best = 0.0, best_t = 0.0;
        int bj = -1;
        for (int d = 0; d < D; d++) {
            size_t e = (size_t)tokens[d] * (size_t)S + (size_t)s;
            double r = tab_r[e], lnc = tab_lnc[e], beta = tab_beta[e];
            double lw = ln_w[counts[d]];
            double q = lw / r;
            double t = floor(q + beta);
            double tb = t - beta;
            double lny = r * tb;
            double a = lnc - lny;
            a = a - r;
            if (bj < 0 || a < best) {
                best = a;
                best_t = t;
                bj = d;
            }
        }
        uint64_t tt = (uint64_t)(int64_t)best_t;
        keys[s] = mix64(tokens[bj] ^ mix64(tt ^ SALT_KEY));
    }
}

/* wmh.py:107-125 (signature, concat=K): keys.reshape(L, K); acc = k[:,0];
 * acc = mix64(acc ^ k[:, i]) for i = 1..K-1. */
void orc_fold(const uint64_t *keys, int L, int K, uint64_t *sig) {
    for (int j = 0; j < L; j++) {
        uint64_t acc = keys[j * K];
        for (int i = 1; i < K; i++) acc = mix64(acc ^ keys[j * K + i]);
        sig[j] = acc;
    }
}

/* index.py:113-138 (_signature_rows / compute_signatures) with the K-aware
 * fold of wmh.py:107-125.  One row per series, OpenMP over series (rows
 * depend only on their series, index.py:124-125). */
void orc_signatures(const void *X, int is_f32, int64_t N, int m, int64_t ld,
                    const double *w, int W, int delta, int n, int L, int K,
                    const double *tab_r, const double *tab_lnc, const double *tab_beta,
                    const double *ln_w, uint64_t *sig, int threads) {
    int nb = orc_num_sketch_bits(m, W, delta);
    int nt = nb - n + 1;
    int S = L * K;
#pragma omp parallel num_threads(threads > 0 ? threads : 1)
    {
        int8_t *bits = (int8_t *)malloc((size_t)nb);
        uint64_t *tok = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)nt);
        uint64_t *scr = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)nt);
        int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (size_t)nt);
        uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)S);
#pragma omp for schedule(dynamic, 64)
        for (int64_t s = 0; s < N; s++) {
            for (int i = 0; i < nb; i++) {
                double acc = 0.0;
                for (int k = 0; k < W; k++) {
                    double prod = load_x(X, is_f32, s * ld + (int64_t)i * delta + k) * w[k];
                    acc = acc + prod;
                }
                bits[i] = acc >= 0.0 ? 1 : -1;
            }
            int D = orc_shingle(bits, nb, n, tok, cnt, scr);
            orc_cws_keys(tok, cnt, D, S, tab_r, tab_lnc, tab_beta, ln_w, keys);
            orc_fold(keys, L, K, sig + s * L);
        }
        free(bits); free(tok); free(scr); free(cnt); free(keys);
    }
}

/* dtw.py:83-121 (_dtw_band_sq): squared banded DTW, two rolling rows,
 * abandon when every cell of a row exceeds abandon_sq (>= 0 to enable).
 * x = rows (the candidate), y = columns (the query). */
double orc_dtw_band_sq(const double *x, const double *y, int m, int r, double abandon_sq,
                       double *prev, double *curr) {
    for (int j = 0; j < m; j++) { prev[j] = INFINITY; curr[j] = INFINITY; }
    for (int i = 0; i < m; i++) {
        int lo = i - r; if (lo < 0) lo = 0;
        int hi = i + r; if (hi > m - 1) hi = m - 1;
        if (lo > 0) curr[lo - 1] = INFINITY;
        double row_min = INFINITY;
        for (int j = lo; j <= hi; j++) {
            double d = x[i] - y[j];
            d = d * d;
            double c;
            if (i == 0 && j == 0) {
                c = d;
            } else {
                double best = prev[j];
                if (j > 0) {
                    if (curr[j - 1] < best) best = curr[j - 1];
                    if (prev[j - 1] < best) best = prev[j - 1];
                }
                c = d + best;
            }
            curr[j] = c;
            if (c < row_min) row_min = c;
        }
        if (abandon_sq >= 0.0 && row_min > abandon_sq) return INFINITY;
        double *tmp = prev; prev = curr; curr = tmp;
    }
    return prev[m - 1];
}

double orc_dtw(const double *x, const double *y, int m, int r, double abandon_sq) {
    double *buf = (double *)malloc(sizeof(double) * 2 * (size_t)m);
    double v = orc_dtw_band_sq(x, y, m, r, abandon_sq, buf, buf + m);
    free(buf);
    return v;
}

/* dtw.py:124-151 (_envelope_into): running max/min over [i-r, i+r] with
 * monotonic deques (`qmax`, `qmin` scratch of m ints each). */
void orc_envelope(const double *x, int m, int r, double *upper, double *lower, int64_t *qbuf) {
    int64_t *qmax = qbuf, *qmin = qbuf + m;
    int hmax = 0, tmax = 0, hmin = 0, tmin = 0;
    for (int j = 0; j < m + r; j++) {
        if (j < m) {
            while (tmax > hmax && x[qmax[tmax - 1]] <= x[j]) tmax--;
            qmax[tmax++] = j;
            while (tmin > hmin && x[qmin[tmin - 1]] >= x[j]) tmin--;
            qmin[tmin++] = j;
        }
        int i = j - r;
        if (i >= 0) {
            while (qmax[hmax] < i - r) hmax++;
            while (qmin[hmin] < i - r) hmin++;
            upper[i] = x[qmax[hmax]];
            lower[i] = x[qmin[hmin]];
        }
    }
}

/* dtw.py:154-168 (_lb_keogh_sq). */
double orc_lb_keogh_sq(const double *c, const double *upper, const double *lower, int m,
                       double abandon_sq) {
    double total = 0.0;
    for (int i = 0; i < m; i++) {
        double v = c[i];
        if (v > upper[i]) {
            double d = v - upper[i];
            total += d * d;
        } else if (v < lower[i]) {
            double d = lower[i] - v;
            total += d * d;
        }
        if (abandon_sq >= 0.0 && total > abandon_sq) return total;
    }
    return total;
}

static inline void load_row(const void *X, int is_f32, int64_t ld, int64_t id, int m, double *out) {
    for (int i = 0; i < m; i++) out[i] = load_x(X, is_f32, id * ld + i);
}

/* dtw.py:171-236 (_cascade_search): LB_Kim -> LB_Keogh -> LB_Keogh2 -> DTW
 * over cand_ids in the given order; strict prune with id tie-break; sorted
 * top-k by (d2, id).  counters = [kim, keogh, keogh2, dtw_computed,
 * dtw_abandoned].  Returns the number of results (`filled`). */
int orc_cascade_search(const void *X, int is_f32, int64_t ld, int m, const int64_t *cand,
                       int64_t n_cand, const double *q, const double *q_upper,
                       const double *q_lower, int r, int k, int64_t *top_ids, double *top_d2,
                       int64_t *counters) {
    int size = (int64_t)k < n_cand ? k : (int)n_cand;
    for (int i = 0; i < size; i++) { top_ids[i] = -1; top_d2[i] = INFINITY; }
    int filled = 0;
    double *c = (double *)malloc(sizeof(double) * 5 * (size_t)m);
    double *cu = c + m, *cl = c + 2 * m, *prev = c + 3 * m, *curr = c + 4 * m;
    int64_t *qbuf = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)m);
    for (int j = 0; j < 5; j++) counters[j] = 0;

    for (int64_t ci = 0; ci < n_cand; ci++) {
        int64_t idx = cand[ci];
        load_row(X, is_f32, ld, idx, m, c);
        int full = filled == size;
        double bsf = full ? top_d2[size - 1] : INFINITY;
        int64_t bsf_id = full ? top_ids[size - 1] : -1;
        double abandon = full ? bsf : -1.0;

        double d0 = c[0] - q[0];
        double dm = c[m - 1] - q[m - 1];
        double kim = d0 * d0 + dm * dm;
        if (full && (kim > bsf || (kim == bsf && idx > bsf_id))) { counters[0]++; continue; }

        double lb1 = orc_lb_keogh_sq(c, q_upper, q_lower, m, abandon);
        if (full && (lb1 > bsf || (lb1 == bsf && idx > bsf_id))) { counters[1]++; continue; }

        orc_envelope(c, m, r, cu, cl, qbuf);
        double lb2 = orc_lb_keogh_sq(q, cu, cl, m, abandon);
        if (full && (lb2 > bsf || (lb2 == bsf && idx > bsf_id))) { counters[2]++; continue; }

        counters[3]++;
        double d2 = orc_dtw_band_sq(c, q, m, r, abandon, prev, curr);
        if (isinf(d2)) { counters[4]++; continue; }
        if (full && (d2 > bsf || (d2 == bsf && idx > bsf_id))) continue;

        int pos = filled < size ? filled : size - 1;
        while (pos > 0 && (top_d2[pos - 1] > d2 || (top_d2[pos - 1] == d2 && top_ids[pos - 1] > idx))) {
            top_d2[pos] = top_d2[pos - 1];
            top_ids[pos] = top_ids[pos - 1];
            pos--;
        }
        top_d2[pos] = d2;
        top_ids[pos] = idx;
        if (filled < size) filled++;
    }
    free(c);
    free(qbuf);
    return filled;
}

/* ---------------- query_index (index.py:175-273), K-aware -------------- */

typedef struct { double lb; int64_t id; } lb_pair;

static int cmp_lb_pair(const void *a, const void *b) {
    const lb_pair *x = (const lb_pair *)a, *y = (const lb_pair *)b;
    if (x->lb < y->lb) return -1;
    if (x->lb > y->lb) return 1;
    return (x->id > y->id) - (x->id < y->id);
}

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* Binary search of `key` in the sorted unique keys of one table. */
static int64_t find_bucket(const uint64_t *ukeys, int64_t nb, uint64_t key) {
    int64_t lo = 0, hi = nb;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (ukeys[mid] < key) lo = mid + 1; else hi = mid;
    }
    return (lo < nb && ukeys[lo] == key) ? lo : -1;
}

/* One query through the reference query_index (index.py:204-273):
 *   query_signature (index.py:175-181, K-aware fold)      -> qsig[L]
 *   probe_candidates (index.py:184-190)                    -> R ascending
 *   build_envelope + _keogh_lb_batch + lexsort((cand, lb)) (index.py:245-250)
 *   _cascade_search (dtw.py:171-236)
 * Tables are CSR per table: ukeys/offsets/ids concatenated with per-table
 * base pointers tab_kbase (bucket base) and tab_ibase (id base = j*N).
 * Outputs: top ids / d2 (<= k), counters[5], n_cand, qsig.  Returns the
 * number of results; 0 with n_cand == 0 means status "no-candidates". */
int orc_query_one(const void *X, int is_f32, int64_t N, int m, int64_t ld,
                  const double *q, const double *w, int W, int delta, int n, int L, int K,
                  const double *tab_r, const double *tab_lnc, const double *tab_beta,
                  const double *ln_w, const uint64_t *ukeys, const int64_t *offsets,
                  const int64_t *ids, const int64_t *tab_nb, const int64_t *tab_kbase,
                  int r, int k, int64_t *top_ids, double *top_d2, int64_t *counters,
                  int64_t *n_cand_out, uint64_t *qsig) {
    int nb = orc_num_sketch_bits(m, W, delta);
    int nt = nb - n + 1;
    int S = L * K;
    int8_t *bits = (int8_t *)malloc((size_t)nb);
    uint64_t *tok = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)nt * 2);
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (size_t)nt);
    uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)S);
    orc_sketch(q, 0, 1, m, m, w, W, delta, bits, NULL, 1);
    int D = orc_shingle(bits, nb, n, tok, cnt, tok + nt);
    orc_cws_keys(tok, cnt, D, S, tab_r, tab_lnc, tab_beta, ln_w, keys);
    orc_fold(keys, L, K, qsig);
    free(bits); free(tok); free(cnt); free(keys);

    /* probe_candidates: union of the L probed buckets, np.unique -> ascending */
    int64_t total = 0;
    int64_t *bs = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)L);
    for (int j = 0; j < L; j++) {
        int64_t b = find_bucket(ukeys + tab_kbase[j], tab_nb[j], qsig[j]);
        if (b >= 0) {
            int64_t o0 = offsets[tab_kbase[j] + j + b], o1 = offsets[tab_kbase[j] + j + b + 1];
            bs[2 * j] = (int64_t)j * N + o0;
            bs[2 * j + 1] = o1 - o0;
            total += o1 - o0;
        } else {
            bs[2 * j] = 0;
            bs[2 * j + 1] = 0;
        }
    }
    int64_t *cand = (int64_t *)malloc(sizeof(int64_t) * (size_t)(total > 0 ? total : 1));
    int64_t p = 0;
    for (int j = 0; j < L; j++)
        for (int64_t e = 0; e < bs[2 * j + 1]; e++) cand[p++] = ids[bs[2 * j] + e];
    free(bs);
    qsort(cand, (size_t)total, sizeof(int64_t), cmp_i64);
    int64_t nc = 0;
    for (int64_t e = 0; e < total; e++)
        if (nc == 0 || cand[nc - 1] != cand[e]) cand[nc++] = cand[e];
    *n_cand_out = nc;
    for (int j = 0; j < 5; j++) counters[j] = 0;
    if (nc == 0) { free(cand); return 0; }

    /* build_envelope, _keogh_lb_batch, lexsort((cand, lbs)) */
    double *U = (double *)malloc(sizeof(double) * 3 * (size_t)m);
    double *Lw = U + m, *row = U + 2 * m;
    int64_t *qbuf = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)m);
    orc_envelope(q, m, r, U, Lw, qbuf);
    lb_pair *pairs = (lb_pair *)malloc(sizeof(lb_pair) * (size_t)nc);
    for (int64_t e = 0; e < nc; e++) {
        load_row(X, is_f32, ld, cand[e], m, row);
        double sa = 0.0, sb = 0.0;
        for (int i = 0; i < m; i++) {
            double a = row[i] - U[i]; if (a < 0.0) a = 0.0;
            double b = Lw[i] - row[i]; if (b < 0.0) b = 0.0;
            sa += a * a;
            sb += b * b;
        }
        pairs[e].lb = sa + sb;
        pairs[e].id = cand[e];
    }
    qsort(pairs, (size_t)nc, sizeof(lb_pair), cmp_lb_pair);
    for (int64_t e = 0; e < nc; e++) cand[e] = pairs[e].id;
    free(pairs);
    int kk = (int64_t)k < nc ? k : (int)nc;
    int filled = orc_cascade_search(X, is_f32, ld, m, cand, nc, q, U, Lw, r, kk, top_ids,
                                    top_d2, counters);
    free(U); free(qbuf); free(cand);
    return filled;
}

/* A batch of queries, OpenMP over queries (bench.py:129-133 runs query_index
 * under a thread pool; numba is nogil).  Q is (nq, m) float64. */
void orc_query_batch(const void *X, int is_f32, int64_t N, int m, int64_t ld,
                     const double *Q, int nq, const double *w, int W, int delta, int n,
                     int L, int K, const double *tab_r, const double *tab_lnc,
                     const double *tab_beta, const double *ln_w, const uint64_t *ukeys,
                     const int64_t *offsets, const int64_t *ids, const int64_t *tab_nb,
                     const int64_t *tab_kbase, int r, int k, int64_t *top_ids, double *top_d2,
                     int32_t *n_out, int64_t *counters, int64_t *n_cand, uint64_t *qsig,
                     int threads) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : 1)
    for (int qi = 0; qi < nq; qi++) {
        n_out[qi] = orc_query_one(X, is_f32, N, m, ld, Q + (int64_t)qi * m, w, W, delta, n, L, K,
                                  tab_r, tab_lnc, tab_beta, ln_w, ukeys, offsets, ids, tab_nb,
                                  tab_kbase, r, k, top_ids + (int64_t)qi * k,
                                  top_d2 + (int64_t)qi * k, counters + (int64_t)qi * 5,
                                  n_cand + qi, qsig + (int64_t)qi * L);
    }
}

/* bench.py:37-42 (_dtw_all) + bench.py:45-60 (brute_force_topk) over an
 * explicit id list: full DTW (no abandon) of every id, OpenMP over ids. */
void orc_dtw_many(const void *X, int is_f32, int64_t ld, int m, const int64_t *ids_in,
                  int64_t n_ids, const double *q, int r, double *d2_out, int threads) {
#pragma omp parallel num_threads(threads > 0 ? threads : 1)
    {
        double *buf = (double *)malloc(sizeof(double) * 3 * (size_t)m);
#pragma omp for schedule(dynamic, 16)
        for (int64_t e = 0; e < n_ids; e++) {
            load_row(X, is_f32, ld, ids_in[e], m, buf);
            d2_out[e] = orc_dtw_band_sq(buf, q, m, r, -1.0, buf + m, buf + 2 * m);
        }
        free(buf);
    }
}
