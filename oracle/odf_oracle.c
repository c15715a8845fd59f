/*
 * odf_oracle.c -- CPU ORACLE for oblivious-decision-forest inference.
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, the smoke()
 * check in __graft_entry__.py and bench.py's cpu_baseline / `--impl reference`
 * leg may load, call or execute anything under oracle/.  It shares no code,
 * header, table or constant with the CUDA path in paper_2205_07307_b200/, and
 * neither side includes or imports the other.
 *
 * It is the plain, slow, obviously-correct definition of what the hot path
 * computes, written from the paper (arxiv 2205.07307, /root/reference/PAPER.md,
 * cited as P:<line>) and SURVEY.md section 8(c) (O1..O7):
 *
 *   O1  condition   c(i,t,l) = FACTOR[i][INDEX] < THRESHOLD
 *   O2  leaf index  idx(i,t) = sum_l c(i,t,l) * 2^l                  (P:80 descent,
 *                   P:114-116 "true,false,true -> 5" (polarity true=1),
 *                   P:307 "bit at offset i <-> condition at base + i" (LSB first))
 *   O3  score       s(i) = sum_t leaf[t][idx(i,t)], fp64, tree order (P:80 last sentence)
 *   O4  bins        borders_f = sorted unique-by-== thresholds on f;
 *                   bin(i,f) = #{ j : !(x < borders_f[j]) } by LINEAR scan
 *                   (BASELINE.json north_star; made NaN-safe, SURVEY 8(c) reading 4)
 *   O7  fingerprint FNV-1a-64 over idx(i,0..T-1) as u16 little-endian
 *   NEXT-1          u32 leaves summed in u64, final (R - 2^31) * S + B
 *   NEXT-2          paper-native mixed-height forests: trees in descending height,
 *                   condition indices into a binary-feature list,
 *                   running sums of heights / 2^heights
 *
 * Floating point: fp32 compares are IEEE strict '<' (no -ffast-math, no FTZ/DAZ);
 * sums are in double.  Pinning: see tests/test_oracle_pins.py and DESIGN.md.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <sched.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* O1: one node condition.  P:80: "В узлах деревьев записаны условия вида
 * FACTOR_{INDEX_i} < THRESHOLD_i".  Strict fp32 less-than; NaN -> false.     */
static int oracle_condition(const float *row, int32_t feature, float threshold)
{
    return row[feature] < threshold ? 1 : 0;
}

/* O2: the leaf reached by descending tree t from its root.  P:80: at each step,
 * starting from the root, descend into one of two subtrees depending on the
 * binary feature of that level, until a leaf is reached.  P:114-116: the leaf is
 * found by writing the tree's binary features as a binary number (true -> 1).
 * bit at offset l of that number is the condition listed at base + l,
 * i.e. level l (the root is l = 0) is the least-significant bit.             */
int32_t oracle_leaf_index(const float *row, const int32_t *feature_index,
                          const float *thresholds, int32_t depth, int64_t t)
{
    int32_t idx = 0;
    for (int32_t l = 0; l < depth; ++l) {
        int c = oracle_condition(row, feature_index[t * depth + l],
                                 thresholds[t * depth + l]);
        idx += c << l;
    }
    return idx;
}

/* ---- threading helper (plain static split of documents over threads) ---- */
typedef struct {
    void (*fn)(void *ctx, int64_t d0, int64_t d1);
    void *ctx;
    int64_t d0, d1;
} oracle_job;

static void *oracle_job_run(void *p)
{
    oracle_job *j = (oracle_job *)p;
    j->fn(j->ctx, j->d0, j->d1);
    return NULL;
}

int oracle_default_threads(void)
{
    cpu_set_t set;
    if (sched_getaffinity(0, sizeof(set), &set) == 0) {
        int n = CPU_COUNT(&set);
        if (n > 0) return n;
    }
    return 1;
}

static void oracle_parallel(void (*fn)(void *, int64_t, int64_t), void *ctx,
                            int64_t n, int n_threads)
{
    if (n_threads <= 0) n_threads = oracle_default_threads();
    if (n_threads > 256) n_threads = 256;
    if (n_threads <= 1 || n < 2 * n_threads) {
        fn(ctx, 0, n);
        return;
    }
    pthread_t th[256];
    oracle_job jobs[256];
    for (int k = 0; k < n_threads; ++k) {
        jobs[k].fn = fn;
        jobs[k].ctx = ctx;
        jobs[k].d0 = n * k / n_threads;
        jobs[k].d1 = n * (k + 1) / n_threads;
        pthread_create(&th[k], NULL, oracle_job_run, &jobs[k]);
    }
    for (int k = 0; k < n_threads; ++k) pthread_join(th[k], NULL);
}

/* ---- O3: scores --------------------------------------------------------- */
typedef struct {
    const float *x;
    int64_t ld;
    const int32_t *fi;
    const float *thr;
    const float *leaves;
    int32_t depth;
    int64_t n_trees;
    double *out64;
    float *out32;
} score_ctx;

static void score_range(void *p, int64_t d0, int64_t d1)
{
    score_ctx *c = (score_ctx *)p;
    const int64_t n_leaves = (int64_t)1 << c->depth;
    for (int64_t i = d0; i < d1; ++i) {
        const float *row = c->x + i * c->ld;
        double s = 0.0;
        /* "Итоговой ответ считается как сумма ответов по всем деревьям";
         * summed in tree order t = 0..T-1, in double. */
        for (int64_t t = 0; t < c->n_trees; ++t) {
            int32_t idx = oracle_leaf_index(row, c->fi, c->thr, c->depth, t);
            s += (double)c->leaves[t * n_leaves + idx];
        }
        if (c->out64) c->out64[i] = s;
        if (c->out32) c->out32[i] = (float)s;
    }
}

void oracle_score(const float *x, int64_t n_docs, int64_t ld,
                  const int32_t *feature_index, const float *thresholds,
                  const float *leaf_values, int32_t depth, int64_t n_trees,
                  double *out64, float *out32, int n_threads)
{
    score_ctx c = {x, ld, feature_index, thresholds, leaf_values, depth, n_trees, out64, out32};
    oracle_parallel(score_range, &c, n_docs, n_threads);
}

/* Scores of an explicit list of documents (sampled parity at full size). */
void oracle_score_rows(const float *x, int64_t ld, const int64_t *rows, int64_t n_rows,
                       const int32_t *feature_index, const float *thresholds,
                       const float *leaf_values, int32_t depth, int64_t n_trees,
                       double *out64)
{
    const int64_t n_leaves = (int64_t)1 << depth;
    for (int64_t r = 0; r < n_rows; ++r) {
        const float *row = x + rows[r] * ld;
        double s = 0.0;
        for (int64_t t = 0; t < n_trees; ++t)
            s += (double)leaf_values[t * n_leaves +
                                     oracle_leaf_index(row, feature_index, thresholds, depth, t)];
        out64[r] = s;
    }
}

/* ---- leaf-index window and O7 fingerprint ------------------------------- */
void oracle_leaf_indices(const float *x, int64_t ld, const int32_t *feature_index,
                         const float *thresholds, int32_t depth, int64_t doc0,
                         int64_t ndoc, int64_t tree0, int64_t ntree, uint16_t *out)
{
    for (int64_t d = 0; d < ndoc; ++d)
        for (int64_t t = 0; t < ntree; ++t)
            out[d * ntree + t] = (uint16_t)oracle_leaf_index(
                x + (doc0 + d) * ld, feature_index, thresholds, depth, tree0 + t);
}

typedef struct {
    const float *x;
    int64_t ld;
    const int32_t *fi;
    const float *thr;
    int32_t depth;
    int64_t n_trees;
    uint64_t *out;
} fp_ctx;

static void fp_range(void *p, int64_t d0, int64_t d1)
{
    fp_ctx *c = (fp_ctx *)p;
    for (int64_t i = d0; i < d1; ++i) {
        uint64_t h = 0xcbf29ce484222325ULL; /* FNV-1a 64 offset basis */
        for (int64_t t = 0; t < c->n_trees; ++t) {
            uint16_t idx = (uint16_t)oracle_leaf_index(c->x + i * c->ld, c->fi, c->thr, c->depth, t);
            h ^= (uint64_t)(idx & 0xff);
            h *= 0x100000001b3ULL; /* FNV-1a 64 prime */
            h ^= (uint64_t)(idx >> 8);
            h *= 0x100000001b3ULL;
        }
        c->out[i] = h;
    }
}

void oracle_fingerprint(const float *x, int64_t n_docs, int64_t ld,
                        const int32_t *feature_index, const float *thresholds,
                        int32_t depth, int64_t n_trees, uint64_t *out, int n_threads)
{
    fp_ctx c = {x, ld, feature_index, thresholds, depth, n_trees, out};
    oracle_parallel(fp_range, &c, n_docs, n_threads);
}

/* FNV-1a-64 of a plain byte string (lets tests pin the hash to its published
 * test vectors independently of the forest code). */
uint64_t oracle_fnv1a64(const uint8_t *bytes, int64_t n)
{
    uint64_t h = 0xcbf29ce484222325ULL;
    for (int64_t k = 0; k < n; ++k) {
        h ^= (uint64_t)bytes[k];
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* ---- O4: borders and bins ----------------------------------------------- */
static int cmp_float(const void *a, const void *b)
{
    float fa = *(const float *)a, fb = *(const float *)b;
    return (fa < fb) ? -1 : (fb < fa) ? 1 : 0;
}

/* borders_f = sort(unique-by-==({thr_tl : f_tl = f})) for every feature f.
 * Output: counts[f] and offsets[f] into borders_out (capacity >= n_nodes).
 * Returns the total number of borders.  (P:180 groups thresholds per factor;
 * sorting and deduplication are the north_star's bin format.)               */
int64_t oracle_borders(const int32_t *feature_index, const float *thresholds, int64_t n_nodes,
                       int32_t n_features, float *borders_out, int32_t *counts, int64_t *offsets)
{
    int64_t total = 0;
    float *tmp = (float *)malloc(sizeof(float) * (size_t)(n_nodes > 0 ? n_nodes : 1));
    for (int32_t f = 0; f < n_features; ++f) {
        int64_t n = 0;
        for (int64_t k = 0; k < n_nodes; ++k)
            if (feature_index[k] == f) tmp[n++] = thresholds[k];
        qsort(tmp, (size_t)n, sizeof(float), cmp_float);
        int32_t m = 0;
        offsets[f] = total;
        for (int64_t k = 0; k < n; ++k) {
            if (m > 0 && tmp[k] == borders_out[total + m - 1]) continue; /* dedup by == */
            borders_out[total + m] = tmp[k];
            ++m;
        }
        counts[f] = m;
        total += m;
    }
    free(tmp);
    return total;
}

/* bin(i,f) = #{ j < m_f : !(x[i][f] < borders_f[j]) }, by a linear scan.
 * uint16 output: the count itself, whatever m_f (the north_star's uint8 bins are
 * the m_f <= 254 case; NEXT-4 widens them). */
void oracle_bins(const float *x, int64_t n_docs, int64_t ld, int32_t n_features,
                 const float *borders, const int32_t *counts, const int64_t *offsets,
                 uint16_t *bins_out /* [n_docs][n_features] */)
{
    for (int64_t i = 0; i < n_docs; ++i)
        for (int32_t f = 0; f < n_features; ++f) {
            const float v = x[i * ld + f];
            int32_t b = 0;
            for (int32_t j = 0; j < counts[f]; ++j)
                if (!(v < borders[offsets[f] + j])) ++b;
            bins_out[i * (int64_t)n_features + f] = (uint16_t)b;
        }
}

/* k_tl = position of thr_tl in borders_{f_tl}, by exact == (linear scan).
 * Returns -1 if absent (cannot happen for thresholds that built the borders). */
void oracle_border_index(const int32_t *feature_index, const float *thresholds, int64_t n_nodes,
                         const float *borders, const int32_t *counts, const int64_t *offsets,
                         int32_t *k_out)
{
    for (int64_t n = 0; n < n_nodes; ++n) {
        int32_t f = feature_index[n];
        k_out[n] = -1;
        for (int32_t j = 0; j < counts[f]; ++j)
            if (borders[offsets[f] + j] == thresholds[n]) {
                k_out[n] = j;
                break;
            }
    }
}

/* ---- NEXT-1: MatrixNet integer leaves ------------------------ */
typedef struct {
    const float *x;
    int64_t ld;
    const int32_t *fi;
    const float *thr;
    const uint32_t *leaves;
    int32_t depth;
    int64_t n_trees;
    uint64_t *out;
} score_u64_ctx;

static void score_u64_range(void *p, int64_t d0, int64_t d1)
{
    score_u64_ctx *c = (score_u64_ctx *)p;
    const int64_t n_leaves = (int64_t)1 << c->depth;
    for (int64_t i = d0; i < d1; ++i) {
        /* "Для каждого документа считаем сумму ответов деревьев в
         * беззнаковом 64-битном числе". */
        uint64_t r = 0;
        for (int64_t t = 0; t < c->n_trees; ++t)
            r += (uint64_t)c->leaves[t * n_leaves +
                                     oracle_leaf_index(c->x + i * c->ld, c->fi, c->thr, c->depth, t)];
        c->out[i] = r;
    }
}

void oracle_score_u64(const float *x, int64_t n_docs, int64_t ld,
                      const int32_t *feature_index, const float *thresholds,
                      const uint32_t *leaf_values, int32_t depth, int64_t n_trees,
                      uint64_t *out, int n_threads)
{
    score_u64_ctx c = {x, ld, feature_index, thresholds, leaf_values, depth, n_trees, out};
    oracle_parallel(score_u64_range, &c, n_docs, n_threads);
}

/* final answer (R - 2^31) * S + B, R the u64 sum, S and B real model
 * parameters (SURVEY 8(c) reading 9: applied once per document).            */
void oracle_finalize(const uint64_t *r, int64_t n, double scale, double bias, double *out)
{
    for (int64_t i = 0; i < n; ++i)
        out[i] = ((double)r[i] - 2147483648.0) * scale + bias;
}

/* ---- NEXT-2: paper-native mixed-height model ----------
 * Binary features: descriptor groups (factor index, count) with thresholds in
 * group order.  Trees: STC[h] trees of height h, stored in descending
 * height; condition indices index the binary features; running sums of heights
 * and of 2^heights give each tree's condition and leaf bases.        */
void oracle_binary_features(const float *row, const int32_t *group_factor,
                            const int32_t *group_count, int32_t n_groups,
                            const float *thresholds, uint8_t *bits_out)
{
    int64_t k = 0; /* keep the current binary-feature index and group */
    for (int32_t g = 0; g < n_groups; ++g)
        for (int32_t j = 0; j < group_count[g]; ++j, ++k)
            bits_out[k] = (uint8_t)oracle_condition(row, group_factor[g], thresholds[k]);
}

void oracle_apply_paper(const float *x, int64_t n_docs, int64_t ld,
                        const int32_t *group_factor, const int32_t *group_count, int32_t n_groups,
                        const float *thresholds, int64_t n_binary,
                        const int32_t *stc /* [9], heights 0..8 */,
                        const uint32_t *cond_indices, const uint32_t *leaves, uint64_t *out)
{
    uint8_t *bits = (uint8_t *)malloc((size_t)(n_binary > 0 ? n_binary : 1));
    for (int64_t i = 0; i < n_docs; ++i) {
        oracle_binary_features(x + i * ld, group_factor, group_count, n_groups, thresholds, bits);
        uint64_t r = 0;
        int64_t cond_base = 0, leaf_base = 0;
        for (int32_t h = 8; h >= 0; --h) /* "Рассматриваем деревья по убыванию высоты" */
            for (int32_t t = 0; t < stc[h]; ++t) {
                int32_t idx = 0;
                for (int32_t l = 0; l < h; ++l)
                    idx += (int32_t)bits[cond_indices[cond_base + l]] << l;
                r += (uint64_t)leaves[leaf_base + idx];
                cond_base += h;
                leaf_base += (int64_t)1 << h;
            }
        out[i] = r;
    }
    free(bits);
}

/* ---- NEXT-3: ordered bit format (§5.4) ------------------------
 * One binary feature per (used factor f ascending, border j ascending); word g of
 * binary feature kb holds, at bit i, the condition x[32g + i][f] < borders_f[j]
 * ("на смещении i стоит бит, соответствующий документу номер i + 1").
 * Output: words[g * n_binary + kb], g < ceil(n_docs / 32).                   */
void oracle_condition_words(const float *x, int64_t n_docs, int64_t ld, int32_t n_features,
                            const float *borders, const int32_t *counts, const int64_t *offsets,
                            uint32_t *words, int64_t n_binary)
{
    int64_t n_groups = (n_docs + 31) / 32;
    memset(words, 0, sizeof(uint32_t) * (size_t)(n_groups * n_binary));
    int64_t kb = 0;
    for (int32_t f = 0; f < n_features; ++f)
        for (int32_t j = 0; j < counts[f]; ++j, ++kb)
            for (int64_t i = 0; i < n_docs; ++i)
                if (oracle_condition(x + i * ld, f, borders[offsets[f] + j]))
                    words[(i / 32) * n_binary + kb] |= 1u << (i % 32);
}
