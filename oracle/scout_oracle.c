/*
 * scout_oracle.c — CPU restatement of the reference's hot-path arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this; the product path
 * (paper_2603_27138_b200/) never does, and fails loudly without its CUDA
 * library.
 *
 * Parity pinned two ways: against golden vectors produced by
 * the reference headers themselves (oracle/_ref/libscout_ref.so, built by
 * oracle/Makefile from /root/reference; script tests/golden/make_golden.py)
 * and against the reference tests' hand-worked known answers
 * (proj/tests/test_digest.cpp:35-105, test_attention.cpp:130-154).
 *
 * Everything is double precision and sequential, exactly as the reference
 * (SPEC.md:70); built like it (no -march, so no FMA) plus -ffp-contract=off.
 * Citations are to /root/reference/proj/include/scout/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define HEAD_DIM 128
#define BLOCK 64

/* build_digest, minmax branch (digest.hpp:41-50): row 0 seeds lo/hi, then
 * channel-wise std::min / std::max over the remaining rows. */
void oracle_build_digest_minmax(const double* keys, int rows, int d, double* lo, double* hi) {
    for (int c = 0; c < d; ++c) lo[c] = hi[c] = keys[c];
    for (int r = 1; r < rows; ++r)
        for (int c = 0; c < d; ++c) {
            const double v = keys[(size_t)r * d + c];
            lo[c] = (v < lo[c]) ? v : lo[c]; /* std::min(lo, v) */
            hi[c] = (hi[c] < v) ? v : hi[c]; /* std::max(hi, v) */
        }
}

/* build_digest, mean branch (digest.hpp:51-57): column sums from 0.0 in row
 * order, then divide by rows. */
void oracle_build_digest_mean(const double* keys, int rows, int d, double* mean) {
    for (int c = 0; c < d; ++c) mean[c] = 0.0;
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < d; ++c) mean[c] += keys[(size_t)r * d + c];
    for (int c = 0; c < d; ++c) mean[c] /= (double)rows;
}

static double ref_max(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* digest_score (digest.hpp:62-72) on an n-long (stacked) vector. */
double oracle_digest_score_minmax(const double* q, const double* lo, const double* hi, int n) {
    double s = 0.0;
    for (int c = 0; c < n; ++c) {
        s += ref_max(q[c] * lo[c], q[c] * hi[c]);
    }
    return s;
}
double oracle_digest_score_mean(const double* q, const double* mean, int n) {
    double s = 0.0; /* dot (numerics.hpp:62-69) */
    for (int c = 0; c < n; ++c) s += q[c] * mean[c];
    return s;
}

/* GQA stacking rule: the G query heads of a KV head form one
 * G*d vector q_s[c*G+g] = q_g[c]; the digest is tiled G times per channel.
 * Scoring the stacked pair with digest_score is the unit's block score. */
double oracle_stacked_score(const double* q /*[G][d]*/, int G, int d, int method, const double* dig, int nb_stride,
                            int b) {
    double s = 0.0;
    for (int c = 0; c < d; ++c)
        for (int g = 0; g < G; ++g) {
            const double qv = q[(size_t)g * d + c];
            if (method == 0)
                s += ref_max(qv * dig[(size_t)c * nb_stride + b], qv * dig[(size_t)(d + c) * nb_stride + b]);
            else
                s += qv * dig[(size_t)c * nb_stride + b];
        }
    return s;
}

typedef struct {
    double s;
    int64_t id;
} scored_t;

/* select_topk comparator (digest.hpp:108-111): score desc, then id asc. */
static int cmp_scored(const void* pa, const void* pb) {
    const scored_t* a = (const scored_t*)pa;
    const scored_t* b = (const scored_t*)pb;
    if (a->s != b->s) return (a->s > b->s) ? -1 : 1;
    return (a->id < b->id) ? -1 : (a->id > b->id);
}
static int cmp_i64(const void* pa, const void* pb) {
    const int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
    return (a < b) ? -1 : (a > b);
}

/* select_topk (digest.hpp:101-118) given precomputed scores. Returns the
 * number of ids written (ascending), or -1 when k == 0 (the reference throws
 * std::invalid_argument, :103). */
int oracle_select_topk(const double* scores, const int64_t* ids, int n, int k, int64_t* out) {
    if (k == 0) return -1;
    scored_t* v = (scored_t*)malloc(sizeof(scored_t) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) {
        v[i].s = scores[i];
        v[i].id = ids ? ids[i] : i;
    }
    qsort(v, (size_t)n, sizeof(scored_t), cmp_scored);
    const int m = k < n ? k : n;
    for (int i = 0; i < m; ++i) out[i] = v[i].id;
    qsort(out, (size_t)m, sizeof(int64_t), cmp_i64);
    free(v);
    return m;
}

/* Unit-batched score + top-k + split, the CPU statement of K1.
 * q [u][G][d] double; digests [u][2][d][nb_stride] (minmax) or [u][d][nb_stride]
 * (mean) double; table [u][nb_stride] (slot or -1) may be NULL.
 * Split = set_intersection / set_difference with the resident set
 * (engine.hpp:239-241). Returns 0, or -1 when k == 0. */
int oracle_score_topk_split(int n_units, int G, int method, int k, int k_stride, int nb_stride, const double* q,
                            const double* digests, const int32_t* n_tokens, const int32_t* table, int32_t* sel_ids,
                            int32_t* n_sel, int32_t* res_ids, int32_t* res_slots, int32_t* n_res, int32_t* cpu_ids,
                            int32_t* n_cpu, double* scores_out) {
    if (k == 0) return -1;
    const int d = HEAD_DIM;
    double* sc = (double*)malloc(sizeof(double) * (size_t)nb_stride);
    int64_t* out = (int64_t*)malloc(sizeof(int64_t) * (size_t)(k > 0 ? k : 1));
    for (int u = 0; u < n_units; ++u) {
        const int nb = (n_tokens[u] + BLOCK - 1) / BLOCK;
        const double* dig = digests + (size_t)u * (method == 0 ? 2 : 1) * d * nb_stride;
        for (int b = 0; b < nb; ++b) {
            sc[b] = oracle_stacked_score(q + (size_t)u * G * d, G, d, method, dig, nb_stride, b);
            if (scores_out) scores_out[(size_t)u * nb_stride + b] = sc[b];
        }
        const int m = oracle_select_topk(sc, NULL, nb, k, out);
        int nr = 0, nc = 0;
        for (int i = 0; i < m; ++i) {
            sel_ids[(size_t)u * k_stride + i] = (int32_t)out[i];
            if (table) {
                const int32_t slot = table[(size_t)u * nb_stride + out[i]];
                if (slot >= 0) {
                    res_ids[(size_t)u * k_stride + nr] = (int32_t)out[i];
                    res_slots[(size_t)u * k_stride + nr] = slot;
                    ++nr;
                } else {
                    cpu_ids[(size_t)u * k_stride + nc] = (int32_t)out[i];
                    ++nc;
                }
            }
        }
        n_sel[u] = m;
        if (table) {
            n_res[u] = nr;
            n_cpu[u] = nc;
        }
    }
    free(sc);
    free(out);
    return 0;
}

/* PartialAttention {o_acc, max_logit, denom, token_count} (attention.hpp:22-35)
 * built token by token with accumulate_token (:38-50); rows are visited in
 * the given order (blocks ascending, rows ascending, :78-88). */
void oracle_partial_attention(const double* q, int d, const double* keys, const double* values, int rows,
                              double scale, double* o_acc, double* max_logit, double* denom, int64_t* count) {
    double m = -INFINITY, l = 0.0;
    int64_t n = 0;
    for (int c = 0; c < d; ++c) o_acc[c] = 0.0;
    for (int r = 0; r < rows; ++r) {
        double s = 0.0;
        for (int c = 0; c < d; ++c) s += q[c] * keys[(size_t)r * d + c];
        const double logit = scale * s;
        if (logit > m) {
            const double sc = (n == 0) ? 0.0 : exp(m - logit);
            for (int c = 0; c < d; ++c) o_acc[c] *= sc;
            l *= sc;
            m = logit;
        }
        const double w = exp(logit - m);
        for (int c = 0; c < d; ++c) o_acc[c] += w * values[(size_t)r * d + c];
        l += w;
        n += 1;
    }
    *max_logit = m;
    *denom = l;
    *count = n;
}

/* merge (attention.hpp:100-114): empty operands are exact identities. */
void oracle_merge(int d, const double* oa, double ma, double la, int64_t na, const double* ob, double mb, double lb,
                  int64_t nb, double* o, double* m, double* l, int64_t* n) {
    if (na == 0) {
        memmove(o, ob, sizeof(double) * (size_t)d);
        *m = mb; *l = lb; *n = nb;
        return;
    }
    if (nb == 0) {
        memmove(o, oa, sizeof(double) * (size_t)d);
        *m = ma; *l = la; *n = na;
        return;
    }
    const double mm = (ma < mb) ? mb : ma;
    const double wa = exp(ma - mm), wb = exp(mb - mm);
    for (int c = 0; c < d; ++c) o[c] = wa * oa[c] + wb * ob[c];
    *l = wa * la + wb * lb;
    *m = mm;
    *n = na + nb;
}

/* finalize (attention.hpp:117-122); returns -1 for an empty partial (the
 * reference throws std::invalid_argument). */
int oracle_finalize(int d, const double* o_acc, double denom, int64_t count, double* out) {
    if (count == 0) return -1;
    for (int c = 0; c < d; ++c) out[c] = o_acc[c] / denom;
    return 0;
}
