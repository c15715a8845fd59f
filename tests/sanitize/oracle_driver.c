/* Sanitizer driver for the CPU oracle (test infrastructure; tests/test_sanitizers.py).
 * Built with -fsanitize=address,undefined (and separately -fsanitize=thread) together
 * with oracle/odf_oracle.c; calls every entry point on seeded tiny forests, including
 * the threaded ones, and checks a few cross-consistencies so the run is not a no-op:
 * oracle_score == oracle_score_rows, the fingerprint == FNV-1a of the index window,
 * every node condition == (bin <= k) (the O5 invariant).  Exit status 0 = clean. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

int32_t oracle_leaf_index(const float *, const int32_t *, const float *, int32_t, int64_t);
void oracle_score(const float *, int64_t, int64_t, const int32_t *, const float *, const float *,
                  int32_t, int64_t, double *, float *, int);
void oracle_score_rows(const float *, int64_t, const int64_t *, int64_t, const int32_t *,
                       const float *, const float *, int32_t, int64_t, double *);
void oracle_leaf_indices(const float *, int64_t, const int32_t *, const float *, int32_t, int64_t,
                         int64_t, int64_t, int64_t, uint16_t *);
void oracle_fingerprint(const float *, int64_t, int64_t, const int32_t *, const float *, int32_t,
                        int64_t, uint64_t *, int);
uint64_t oracle_fnv1a64(const uint8_t *, int64_t);
int64_t oracle_borders(const int32_t *, const float *, int64_t, int32_t, float *, int32_t *, int64_t *);
void oracle_bins(const float *, int64_t, int64_t, int32_t, const float *, const int32_t *,
                 const int64_t *, uint16_t *);
void oracle_border_index(const int32_t *, const float *, int64_t, const float *, const int32_t *,
                         const int64_t *, int32_t *);
void oracle_score_u64(const float *, int64_t, int64_t, const int32_t *, const float *,
                      const uint32_t *, int32_t, int64_t, uint64_t *, int);
void oracle_finalize(const uint64_t *, int64_t, double, double, double *);
void oracle_apply_paper(const float *, int64_t, int64_t, const int32_t *, const int32_t *, int32_t,
                        const float *, int64_t, const int32_t *, const uint32_t *, const uint32_t *,
                        uint64_t *);
void oracle_condition_words(const float *, int64_t, int64_t, int32_t, const float *, const int32_t *,
                            const int64_t *, uint32_t *, int64_t);

static uint64_t g_state = 0x9E3779B97F4A7C15ull;
static uint32_t rnd(void)
{
    g_state = g_state * 6364136223846793005ull + 1442695040888963407ull;
    return (uint32_t)(g_state >> 33);
}
static float rndf(void) { return (float)(rnd() % 20001) / 10000.0f - 1.0f; }

static int fail(const char *what, int c)
{
    fprintf(stderr, "case %d: %s\n", c, what);
    return 1;
}

static int one_case(int c, int32_t D, int32_t F, int32_t T, int32_t depth, int ld_pad)
{
    const int64_t ld = F + ld_pad, nodes = (int64_t)T * depth, nl = (int64_t)T << depth;
    float *x = malloc(sizeof(float) * (size_t)(D * ld + 1));
    int32_t *fi = malloc(sizeof(int32_t) * (size_t)(nodes + 1));
    float *thr = malloc(sizeof(float) * (size_t)(nodes + 1));
    float *lv = malloc(sizeof(float) * (size_t)(nl + 1));
    uint32_t *lu = malloc(sizeof(uint32_t) * (size_t)(nl + 1));
    for (int64_t k = 0; k < (int64_t)D * ld; ++k) x[k] = rndf();
    for (int64_t k = 0; k < nodes; ++k) {
        fi[k] = (int32_t)(rnd() % (uint32_t)F);
        thr[k] = (float)(rnd() % 11) / 5.0f - 1.0f; /* few distinct values: ties */
    }
    if (D > 3) { x[0] = NAN; x[ld + 1 % F] = -0.0f; x[2 * ld] = 1e-40f; } /* NaN, -0, denormal */
    for (int64_t k = 0; k < nl; ++k) { lv[k] = rndf(); lu[k] = rnd(); }
    double *s64 = malloc(sizeof(double) * (size_t)(D + 1)), *r64 = malloc(sizeof(double) * (size_t)(D + 1));
    float *s32 = malloc(sizeof(float) * (size_t)(D + 1));
    oracle_score(x, D, ld, fi, thr, lv, depth, T, s64, s32, 4);
    int64_t *rows = malloc(sizeof(int64_t) * (size_t)(D + 1));
    for (int64_t i = 0; i < D; ++i) rows[i] = D - 1 - i;
    oracle_score_rows(x, ld, rows, D, fi, thr, lv, depth, T, r64);
    for (int64_t i = 0; i < D; ++i)
        if (r64[i] != s64[D - 1 - i]) return fail("score_rows != score", c);
    uint16_t *idx = malloc(sizeof(uint16_t) * (size_t)(D * (int64_t)T + 1));
    oracle_leaf_indices(x, ld, fi, thr, depth, 0, D, 0, T, idx);
    uint64_t *fp = malloc(sizeof(uint64_t) * (size_t)(D + 1));
    oracle_fingerprint(x, D, ld, fi, thr, depth, T, fp, 4);
    for (int64_t i = 0; i < D; ++i)
        if (fp[i] != oracle_fnv1a64((const uint8_t *)(idx + i * T), 2 * (int64_t)T))
            return fail("fingerprint != FNV-1a(index window)", c);
    float *bord = malloc(sizeof(float) * (size_t)(nodes + 1));
    int32_t *cnt = malloc(sizeof(int32_t) * (size_t)F);
    int64_t *off = malloc(sizeof(int64_t) * (size_t)F);
    const int64_t nb = oracle_borders(fi, thr, nodes, F, bord, cnt, off);
    uint16_t *bins = malloc(sizeof(uint16_t) * (size_t)(D * (int64_t)F + 1));
    oracle_bins(x, D, ld, F, bord, cnt, off, bins);
    int32_t *kk = malloc(sizeof(int32_t) * (size_t)(nodes + 1));
    oracle_border_index(fi, thr, nodes, bord, cnt, off, kk);
    for (int64_t i = 0; i < D; ++i) /* O5: x < thr  <=>  bin <= k */
        for (int64_t n = 0; n < nodes; ++n)
            if ((x[i * ld + fi[n]] < thr[n]) != (bins[i * F + fi[n]] <= kk[n]))
                return fail("O5 invariant", c);
    uint64_t *u = malloc(sizeof(uint64_t) * (size_t)(D + 1));
    double *fin = malloc(sizeof(double) * (size_t)(D + 1));
    oracle_score_u64(x, D, ld, fi, thr, lu, depth, T, u, 4);
    oracle_finalize(u, D, 0.5, 1.25, fin);
    uint32_t *words = malloc(sizeof(uint32_t) * (size_t)(((D + 31) / 32) * (nb > 0 ? nb : 1)));
    oracle_condition_words(x, D, ld, F, bord, cnt, off, words, nb);
    /* paper layout: one group per factor, 3 binary features each, trees of heights 0..8 */
    int32_t gf[64], gc[64], stc[9];
    int64_t K = 0;
    for (int32_t g = 0; g < F && g < 64; ++g) { gf[g] = g; gc[g] = 3; K += 3; }
    float *pth = malloc(sizeof(float) * (size_t)K);
    for (int64_t k = 0; k < K; ++k) pth[k] = rndf();
    int64_t nc = 0, npl = 0;
    for (int h = 0; h <= 8; ++h) { stc[h] = (int32_t)(rnd() % 3); nc += (int64_t)h * stc[h]; npl += ((int64_t)1 << h) * stc[h]; }
    uint32_t *ci = malloc(sizeof(uint32_t) * (size_t)(nc + 1)), *pl = malloc(sizeof(uint32_t) * (size_t)(npl + 1));
    for (int64_t k = 0; k < nc; ++k) ci[k] = rnd() % (uint32_t)K;
    for (int64_t k = 0; k < npl; ++k) pl[k] = rnd();
    uint64_t *pr = malloc(sizeof(uint64_t) * (size_t)(D + 1));
    oracle_apply_paper(x, D, ld, gf, gc, F < 64 ? F : 64, pth, K, stc, ci, pl, pr);
    free(x); free(fi); free(thr); free(lv); free(lu); free(s64); free(r64); free(s32); free(rows);
    free(idx); free(fp); free(bord); free(cnt); free(off); free(bins); free(kk); free(u); free(fin);
    free(words); free(pth); free(ci); free(pl); free(pr);
    return 0;
}

int main(void)
{
    int bad = 0, c = 0;
    const int32_t depths[] = {0, 1, 3, 6, 8, 10};
    for (int di = 0; di < 6; ++di)
        for (int k = 0; k < 3; ++k, ++c)
            bad |= one_case(c, 1 + (int32_t)(rnd() % 70), 1 + (int32_t)(rnd() % 9),
                            (int32_t)(rnd() % 20), depths[di], (int)(rnd() % 4));
    bad |= one_case(c++, 0, 3, 5, 6, 0); /* empty batch */
    printf(bad ? "oracle driver: FAILED\n" : "oracle driver: ok (%d cases)\n", c);
    return bad;
}
