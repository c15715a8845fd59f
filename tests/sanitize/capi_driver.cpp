// Sanitizer driver for the host side of the C ABI (tests/test_sanitizers.py): the
// model compiler (borders, code columns, factor metadata, bank-swizzled tables,
// chunking, NEXT-2 import, validation) on seeded random models of every depth,
// narrow and wide, fp32 and u32 leaves, plus invalid inputs.  Built with
// -fsanitize=address,undefined against tests/sanitize/kernel_stubs.cpp.  Without
// a GPU a valid model returns ODF_E_CUDA (after the host compile), an invalid one
// ODF_E_INVALID_ARG / ODF_E_UNSUPPORTED; exit status 0 = every status as expected.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/odf.h"

static uint64_t g_s = 12345;
static uint32_t rnd()
{
    g_s = g_s * 6364136223846793005ull + 1442695040888963407ull;
    return static_cast<uint32_t>(g_s >> 33);
}

static bool valid_status(odf_status st) { return st == ODF_OK || st == ODF_E_CUDA; }

int main()
{
    int bad = 0, n = 0;
    for (int depth = 0; depth <= ODF_MAX_DEPTH; ++depth)
        for (int variant = 0; variant < 4; ++variant, ++n) {
            const int32_t F = 1 + rnd() % 70;
            const int64_t T = rnd() % 90;
            const bool wide = variant == 2, u32 = variant == 3;
            std::vector<int32_t> fi(T * depth);
            std::vector<float> thr(T * depth);
            for (size_t k = 0; k < fi.size(); ++k) {
                fi[k] = wide && (k % 2) ? 0 : static_cast<int32_t>(rnd() % F);
                thr[k] = wide ? static_cast<float>(k) * 0.5f : static_cast<float>(rnd() % 300) / 7.0f;
            }
            std::vector<float> lf(T << depth);
            std::vector<uint32_t> lu(T << depth);
            for (size_t k = 0; k < lf.size(); ++k) { lf[k] = static_cast<float>(rnd() % 1000) * 1e-3f; lu[k] = rnd(); }
            odf_model_desc d;
            std::memset(&d, 0, sizeof d);
            d.feature_index = fi.data();
            d.thresholds = thr.data();
            d.leaf_values = u32 ? static_cast<const void *>(lu.data()) : static_cast<const void *>(lf.data());
            d.leaf_type = u32 ? ODF_LEAF_U32 : ODF_LEAF_F32;
            d.depth = depth;
            d.n_trees = T;
            d.n_features = F;
            d.scale = 1.0;
            odf_model *m = nullptr;
            odf_status st = odf_load_model_ex(&d, &m);
            if (!valid_status(st)) { std::fprintf(stderr, "depth %d variant %d: %d %s\n", depth, variant, st, odf_last_error()); bad = 1; }
            if (m) odf_free_model(m);
            // invalid: NaN threshold, feature out of range
            if (T > 0 && depth > 0) {
                thr[0] = NAN;
                if (odf_load_model_ex(&d, &m) != ODF_E_INVALID_ARG) { std::fprintf(stderr, "NaN accepted\n"); bad = 1; }
                thr[0] = 0.0f;
                fi[0] = F;
                if (odf_load_model_ex(&d, &m) != ODF_E_INVALID_ARG) { std::fprintf(stderr, "feature accepted\n"); bad = 1; }
            }
        }
    // many code columns (> 512) with skewed usage, depths 4..8
    for (int depth = 4; depth <= 8; ++depth) {
        const int32_t F = 900;
        const int64_t T = 700;
        std::vector<int32_t> fi(T * depth);
        std::vector<float> thr(T * depth);
        for (size_t k = 0; k < fi.size(); ++k) {
            const uint32_t r = rnd() % 1000;  // skewed: low features popular
            fi[k] = static_cast<int32_t>(r < 500 ? r % 40 : rnd() % F);
            thr[k] = static_cast<float>(rnd() % 200) / 9.0f;
        }
        std::vector<float> lf(T << depth);
        for (size_t k = 0; k < lf.size(); ++k) lf[k] = static_cast<float>(rnd() % 1000) * 1e-3f;
        odf_model *m = nullptr;
        odf_status st = odf_load_model(fi.data(), thr.data(), lf.data(), depth, T, F, 0, &m);
        if (!valid_status(st)) { std::fprintf(stderr, "wide forest depth %d: %d %s\n", depth, st, odf_last_error()); bad = 1; }
        if (m) odf_free_model(m);
    }
    // > 2032 borders on one factor: unsupported
    {
        const int depth = 6;
        const int64_t T = 400;
        std::vector<int32_t> fi(T * depth, 0);
        std::vector<float> thr(T * depth);
        for (size_t k = 0; k < thr.size(); ++k) thr[k] = static_cast<float>(k);
        std::vector<float> lf(T << depth, 0.0f);
        odf_model *m = nullptr;
        if (odf_load_model(fi.data(), thr.data(), lf.data(), depth, T, 2, 0, &m) != ODF_E_UNSUPPORTED) {
            std::fprintf(stderr, "2400 borders accepted\n");
            bad = 1;
        }
    }
    // paper-native import (NEXT-2): heights 0..8, three binary features per factor
    {
        const int32_t F = 7;
        std::vector<int32_t> gf(F), gc(F, 3);
        for (int32_t g = 0; g < F; ++g) gf[g] = g;
        std::vector<float> th(3 * F);
        for (size_t k = 0; k < th.size(); ++k) th[k] = static_cast<float>(rnd() % 100) / 50.0f;
        int32_t stc[ODF_MAX_DEPTH + 1] = {2, 1, 0, 3, 1, 0, 4, 1, 2, 0, 0};
        int64_t nc = 0, nl = 0;
        for (int h = 0; h <= ODF_MAX_DEPTH; ++h) { nc += h * stc[h]; nl += (int64_t(1) << h) * stc[h]; }
        std::vector<uint32_t> ci(nc), lv(nl);
        for (auto &v : ci) v = rnd() % (3 * F);
        for (auto &v : lv) v = rnd();
        odf_paper_model_desc p;
        std::memset(&p, 0, sizeof p);
        p.n_features = F;
        p.group_factor = gf.data();
        p.group_count = gc.data();
        p.n_groups = F;
        p.thresholds = th.data();
        p.stc = stc;
        p.cond_indices = ci.data();
        p.leaves = lv.data();
        p.scale = 0.5;
        odf_model *m = nullptr;
        odf_status st = odf_load_model_paper(&p, &m);
        if (!valid_status(st)) { std::fprintf(stderr, "paper import: %d %s\n", st, odf_last_error()); bad = 1; }
        if (m) odf_free_model(m);
        ci[0] = 3 * F;  // out of range
        if (odf_load_model_paper(&p, &m) != ODF_E_INVALID_ARG) { std::fprintf(stderr, "bad cond index accepted\n"); bad = 1; }
    }
    std::printf(bad ? "capi driver: FAILED\n" : "capi driver: ok (%d models)\n", n);
    return bad;
}
