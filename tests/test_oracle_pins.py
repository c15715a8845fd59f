"""Pins of the CPU oracle to things other than itself (SURVEY.md 8(c) "What pins each part").

* paper worked examples and rules (tests/golden/paper_examples.json, each cited);
* hand depth-1 / depth-2 cases fixing polarity, strictness and LSB-first order;
* brute force: each oblivious tree re-expanded into an explicit full binary tree
  (heap-ordered node records with child pointers) and descended pointer by pointer;
* the bin <-> raw-comparison invariant over every (doc, tree, level) with numpy's
  own float32 comparison; special cases (ties, NaN, +-0, denormals, +-inf);
* closed forms for the sum (constant-per-tree leaves, exact-arithmetic leaves
  summed with Python fractions, zero trees, single tree);
* FNV-1a-64 published vectors for the fingerprint.

A plausible mistake in the oracle (dropped term, wrong sign or bit order,
transposed operand, non-strict compare) fails at least one of these.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def _forest_from_conditions(conds):
    """A depth-len(conds) one-tree forest over len(conds) features whose condition
    values for the doc x = 0.5 are exactly `conds` (threshold 1 -> true, 0 -> false)."""
    d = len(conds)
    fi = np.arange(d, dtype=np.int32)
    thr = np.array([1.0 if c else 0.0 for c in conds], np.float32)
    x = np.full((1, d), 0.5, np.float32)
    leaves = np.arange(1 << d, dtype=np.float32)  # leaf j holds value j
    return x, fi, thr, leaves


def test_p116_example_true_false_true_is_5():
    g = GOLD["p116_true_false_true_is_5"]
    x, fi, thr, lv = _forest_from_conditions(g["conditions"])
    assert oracle.leaf_index(x[0], fi, thr, g["depth"], 0) == g["leaf_index"]
    s64, s32 = oracle.score(x, fi, thr, lv, g["depth"])
    assert s64[0] == g["leaf_index"] and s32[0] == g["leaf_index"]


def test_p307_lsb_first_order():
    g = GOLD["p307_lsb_first"]
    for case in g["cases"]:
        x, fi, thr, lv = _forest_from_conditions(case["conditions"])
        assert oracle.leaf_index(x[0], fi, thr, g["depth"], 0) == case["leaf_index"], case


def test_hand_depth1_strict_less():
    # level 0: f0 < 0.5, leaves [a, b]; SURVEY 8(c) pins: 0.3 -> b, 0.5 -> a (tie), 0.7 -> a
    fi = np.array([0], np.int32)
    thr = np.array([0.5], np.float32)
    lv = np.array([10.0, 20.0], np.float32)
    x = np.array([[0.3], [0.5], [0.7]], np.float32)
    s64, _ = oracle.score(x, fi, thr, lv, 1)
    assert list(s64) == [20.0, 10.0, 10.0]


def test_hand_depth2_lsb_convention():
    # level 0: f0 < 0.5, level 1: f1 < 0.25, leaves [l0, l1, l2, l3]
    fi = np.array([0, 1], np.int32)
    thr = np.array([0.5, 0.25], np.float32)
    lv = np.array([100.0, 101.0, 102.0, 103.0], np.float32)
    x = np.array([[0.3, 0.7], [0.6, 0.1], [0.3, 0.1], [0.6, 0.7]], np.float32)
    s64, _ = oracle.score(x, fi, thr, lv, 2)
    assert list(s64) == [101.0, 102.0, 103.0, 100.0]


# ---------------------------------------------------------------------------
# brute force: explicit full binary tree, pointer descent
# ---------------------------------------------------------------------------
class _Node:
    __slots__ = ("feature", "threshold", "left", "right", "value")

    def __init__(self):
        self.feature = self.threshold = self.left = self.right = self.value = None


def _expand_tree(fi, thr, leaves, depth, t):
    """Re-expand oblivious tree t into 2^d-1 internal nodes (each level repeats that
    level's condition) and 2^d leaves; the leaf reached through path bits
    (c_0..c_{d-1}) holds leaves[t*2^d + sum c_l 2^l]."""
    def build(level, path_bits):
        node = _Node()
        if level == depth:
            idx = sum(b << l for l, b in enumerate(path_bits))
            node.value = float(leaves[t * (1 << depth) + idx])
            return node
        node.feature = int(fi[t * depth + level])
        node.threshold = thr[t * depth + level]
        node.left = build(level + 1, path_bits + [0])   # condition false
        node.right = build(level + 1, path_bits + [1])  # condition true
        return node
    return build(0, [])


def _descend(root, row):
    node = root
    while node.value is None:
        go_true = bool(np.float32(row[node.feature]) < np.float32(node.threshold))
        node = node.right if go_true else node.left
    return node.value


@pytest.mark.parametrize("seed,depth,n_trees,n_docs", [(11, 1, 5, 64), (12, 3, 9, 100),
                                                       (13, 6, 7, 129), (14, 4, 16, 37),
                                                       (15, 0, 3, 10)])
def test_brute_force_explicit_trees(seed, depth, n_trees, n_docs):
    c = synth.tiny_case(seed=seed, n_docs=n_docs, n_features=5, n_trees=n_trees, depth=depth,
                        pool=4)
    roots = [_expand_tree(c.feature_index, c.thresholds, c.leaf_values, depth, t)
             for t in range(n_trees)]
    s64, s32 = oracle.score(c.x, c.feature_index, c.thresholds, c.leaf_values, depth)
    for i in range(n_docs):
        vals = [_descend(r, c.x[i]) for r in roots]
        for t, v in enumerate(vals):  # leaf-by-leaf
            idx = oracle.leaf_index(c.x[i], c.feature_index, c.thresholds, depth, t)
            assert c.leaf_values[t * (1 << depth) + idx] == np.float32(v)
        exact = sum(Fraction(v) for v in vals)  # score-by-score, exactly
        assert abs(Fraction(s64[i]) - exact) <= Fraction(1, 2 ** 40) * (1 + abs(exact))


@pytest.mark.parametrize("depth", [1, 2, 5, 6])
def test_every_path_reaches_its_leaf(depth):
    # distinct feature per level; doc for path p sets x_l below (bit 1) or above (bit 0) 0.5
    fi = np.arange(depth, dtype=np.int32)
    thr = np.full(depth, 0.5, np.float32)
    lv = np.arange(1 << depth, dtype=np.float32)
    for p in range(1 << depth):
        row = np.array([0.25 if (p >> l) & 1 else 0.75 for l in range(depth)], np.float32)
        assert oracle.leaf_index(row, fi, thr, depth, 0) == p
        root = _expand_tree(fi, thr, lv, depth, 0)
        assert _descend(root, row) == p


# ---------------------------------------------------------------------------
# bins (O4/O5)
# ---------------------------------------------------------------------------
def test_bins_spec_s146_example():
    g = GOLD["p80_strict_less"]
    thr = np.array(g["thresholds"], np.float32)
    fi = np.zeros(thr.size, np.int32)
    per, flat, counts, offs = oracle.borders(fi, thr, 1)
    x = np.array([[g["factor"]]], np.float32)
    b = oracle.bins(x, 1, flat, counts, offs)[0, 0]
    assert b == 2
    k = oracle.border_index(fi, thr, flat, counts, offs)
    assert [int(b <= kk) for kk in k] == g["bits"]


def test_bins_special_values():
    borders = np.array([-1.0, 0.0, 2.5, 7.0], np.float32)
    fi = np.zeros(4, np.int32)
    _, flat, counts, offs = oracle.borders(fi, borders, 1)
    m = 4
    den = np.float32(1e-45)  # smallest denormal
    xs = [-5.0, -1.0, -0.5, -0.0, 0.0, den, 2.5, 3.0, 7.0, 8.0, np.inf, -np.inf, np.nan]
    want = [0, 1, 1, 2, 2, 2, 3, 3, 4, 4, m, 0, m]
    x = np.array(xs, np.float32).reshape(-1, 1)
    got = oracle.bins(x, 1, flat, counts, offs)[:, 0]
    assert list(got) == want


def test_borders_dedup_signed_zero_and_sort():
    thr = np.array([0.0, -0.0, 3.0, 1.0, 3.0, -2.0], np.float32)
    fi = np.zeros(thr.size, np.int32)
    per, flat, counts, offs = oracle.borders(fi, thr, 1)
    assert counts[0] == 4
    assert list(per[0]) == [-2.0, 0.0, 1.0, 3.0]
    # -0.0 vs a 0.0 border: not less -> counted
    x = np.array([[-0.0]], np.float32)
    assert oracle.bins(x, 1, flat, counts, offs)[0, 0] == 2


@pytest.mark.parametrize("name,n_docs", [("c1", 1024), ("c2", 300), ("c4", 200)])
def test_bins_reproduce_every_raw_comparison(name, n_docs):
    c = synth.make_case(name, n_docs=n_docs, n_trees=64 if name != "c1" else None)
    per, flat, counts, offs = oracle.borders(c.feature_index, c.thresholds, c.n_features)
    # borders: strictly increasing and each equal to np.unique of that feature's thresholds
    for f in range(c.n_features):
        u = np.unique(c.thresholds[c.feature_index == f])
        assert np.array_equal(per[f], u)
        assert np.all(np.diff(per[f]) > 0)
    b = oracle.bins(c.x, c.n_features, flat, counts, offs)
    k = oracle.border_index(c.feature_index, c.thresholds, flat, counts, offs)
    assert np.all(k >= 0)
    raw = c.x[:, c.feature_index] < c.thresholds[None, :]        # numpy fp32 compare
    via_bins = b[:, c.feature_index].astype(np.int32) <= k[None, :]
    assert np.array_equal(raw, via_bins)


@pytest.mark.parametrize("m", [255, 700, 2032])
def test_wide_bins_reproduce_every_raw_comparison(m):
    # NEXT-4: more than 254 borders on one factor -> bins above 255 (uint16); the
    # invariant x < b_k  <=>  bin <= k must hold on every border, ties included
    rng = np.random.default_rng(m)
    thr = np.sort(rng.standard_normal(m).astype(np.float32))
    thr = np.unique(thr)
    fi = np.zeros(thr.size, np.int32)
    per, flat, counts, offs = oracle.borders(fi, thr, 1)
    x = np.concatenate([rng.standard_normal(400).astype(np.float32), thr[::7],
                        np.array([np.inf, -np.inf, np.nan], np.float32)]).reshape(-1, 1)
    b = oracle.bins(x, 1, flat, counts, offs)[:, 0]
    assert b.dtype == np.uint16 and b.max() == thr.size  # +inf / NaN count every border
    k = oracle.border_index(fi, thr, flat, counts, offs)
    assert np.array_equal(k, np.arange(thr.size))
    with np.errstate(invalid="ignore"):
        raw = x[:, 0][:, None] < thr[None, :]
    assert np.array_equal(raw, b.astype(np.int64)[:, None] <= k[None, :])


def test_bins_with_injected_ties_nan_zero_denormal():
    c = synth.tiny_case(seed=21, n_docs=256, n_features=8, n_trees=32, depth=4, pool=6)
    x = c.x.copy()
    rng = np.random.default_rng(5)
    # exact ties: copy thresholds into factors; specials in some cells
    for _ in range(200):
        n = rng.integers(c.feature_index.size)
        x[rng.integers(256), c.feature_index[n]] = c.thresholds[n]
    specials = np.array([np.nan, -0.0, 0.0, 1e-45, -1e-45, np.inf, -np.inf], np.float32)
    for _ in range(100):
        x[rng.integers(256), rng.integers(8)] = specials[rng.integers(specials.size)]
    per, flat, counts, offs = oracle.borders(c.feature_index, c.thresholds, 8)
    b = oracle.bins(x, 8, flat, counts, offs)
    k = oracle.border_index(c.feature_index, c.thresholds, flat, counts, offs)
    with np.errstate(invalid="ignore"):
        raw = x[:, c.feature_index] < c.thresholds[None, :]
    assert np.array_equal(raw, b[:, c.feature_index].astype(np.int32) <= k[None, :])
    # leaf indices from raw comparisons == oracle O2
    s64, _ = oracle.score(x, c.feature_index, c.thresholds, c.leaf_values, 4)
    idx = (raw.reshape(256, 32, 4) * (1 << np.arange(4))).sum(-1)
    want = c.leaf_values.reshape(32, 16)[np.arange(32)[None, :], idx].astype(np.float64)
    assert np.allclose(s64, np.array([sum(map(Fraction, r)) for r in want], float),
                       rtol=0, atol=1e-12)


# ---------------------------------------------------------------------------
# sums (O3) closed forms
# ---------------------------------------------------------------------------
def test_constant_per_tree_leaves_sum_closed_form():
    c = synth.tiny_case(seed=31, n_docs=200, n_features=6, n_trees=50, depth=5)
    const = np.random.default_rng(1).normal(0, 1, 50).astype(np.float32)
    lv = np.repeat(const, 32)
    s64, _ = oracle.score(c.x, c.feature_index, c.thresholds, lv, 5)
    want = float(sum(Fraction(float(v)) for v in const))
    assert np.all(s64 == want)


def test_exact_arithmetic_leaves_are_exact():
    c = synth.tiny_case(seed=32, n_docs=100, n_features=10, n_trees=300, depth=6,
                        exact_leaves=True)
    s64, s32 = oracle.score(c.x, c.feature_index, c.thresholds, c.leaf_values, 6)
    idx = oracle.leaf_indices(c.x, c.feature_index, c.thresholds, 6, 0, 100, 0, 300)
    lv = c.leaf_values.reshape(300, 64)
    for i in range(100):
        exact = sum(Fraction(float(lv[t, idx[i, t]])) for t in range(300))
        assert Fraction(s64[i]) == exact and Fraction(float(s32[i])) == exact


def test_zero_trees_and_single_tree():
    c = synth.tiny_case(seed=33, n_docs=50, n_features=4, n_trees=1, depth=3)
    s64, _ = oracle.score(c.x, c.feature_index[:0], c.thresholds[:0], c.leaf_values[:0], 3,
                          n_trees=0)
    assert np.all(s64 == 0.0)
    s64, s32 = oracle.score(c.x, c.feature_index, c.thresholds, c.leaf_values, 3)
    for i in range(50):
        t = oracle.leaf_index(c.x[i], c.feature_index, c.thresholds, 3, 0)
        assert s32[i] == c.leaf_values[t] and s64[i] == float(c.leaf_values[t])


def test_oracle_threads_do_not_change_results():
    c = synth.tiny_case(seed=34, n_docs=999, n_features=12, n_trees=40, depth=6)
    a, _ = oracle.score(c.x, c.feature_index, c.thresholds, c.leaf_values, 6, n_threads=1)
    b, _ = oracle.score(c.x, c.feature_index, c.thresholds, c.leaf_values, 6, n_threads=7)
    assert np.array_equal(a, b)
    rows = np.array([0, 5, 998, 400], np.int64)
    r = oracle.score_rows(c.x, rows, c.feature_index, c.thresholds, c.leaf_values, 6)
    assert np.array_equal(r, a[rows])


# ---------------------------------------------------------------------------
# fingerprint (O7)
# ---------------------------------------------------------------------------
def test_fnv1a64_published_vectors():
    for case in GOLD["fnv1a64_vectors"]["cases"]:
        assert oracle.fnv1a64(bytes.fromhex(case["bytes_hex"])) == int(case["hash"], 16)


def test_fingerprint_is_fnv_of_u16_le_indices():
    c = synth.tiny_case(seed=35, n_docs=40, n_features=16, n_trees=30, depth=10, pool=16)
    fp = oracle.fingerprint(c.x, c.feature_index, c.thresholds, 10, 30)
    idx = oracle.leaf_indices(c.x, c.feature_index, c.thresholds, 10, 0, 40, 0, 30)
    for i in range(40):
        assert int(fp[i]) == oracle.fnv1a64(idx[i].astype("<u2").tobytes())


# ---------------------------------------------------------------------------
# NEXT-1 integer mode / NEXT-2 paper-native layout
# ---------------------------------------------------------------------------
def test_finalize_p309_examples():
    for case in GOLD["p309_finalize"]["cases"]:
        out = oracle.finalize(np.array([case["R"]], np.uint64), case["S"], case["B"])
        assert out[0] == case["score"]


def test_u64_sums_closed_form_and_no_u32_overflow():
    c = synth.tiny_case(seed=36, n_docs=64, n_features=4, n_trees=8, depth=3)
    lv = np.full(8 * 8, 0xFFFFFFFF, np.uint32)
    r = oracle.score_u64(c.x, c.feature_index, c.thresholds, lv, 3)
    assert np.all(r == np.uint64(8 * 0xFFFFFFFF))
    lv = np.random.default_rng(2).integers(0, 2 ** 32, 64, dtype=np.uint64).astype(np.uint32)
    r = oracle.score_u64(c.x, c.feature_index, c.thresholds, lv, 3)
    idx = oracle.leaf_indices(c.x, c.feature_index, c.thresholds, 3, 0, 64, 0, 8)
    want = [sum(int(lv[t * 8 + idx[i, t]]) for t in range(8)) for i in range(64)]
    assert [int(v) for v in r] == want


def test_paper_layout_lengths_and_bases():
    g = GOLD["p304_p305_lengths"]
    stc = g["stc"]
    assert sum(h * stc[h] for h in range(9)) == g["n_conditions"]
    assert sum((1 << h) * stc[h] for h in range(9)) == g["n_leaves"]
    g = GOLD["p307_tree_layout"]
    cb, lb, c0, l0 = [], [], 0, 0
    for h in g["heights"]:
        cb.append(c0)
        lb.append(l0)
        c0 += h
        l0 += 1 << h
    assert cb == g["cond_base"] and lb == g["leaf_base"]


def test_paper_native_apply_matches_brute_force():
    rng = np.random.default_rng(7)
    F, D = 5, 40
    x = rng.random((D, F), dtype=np.float32)
    group_factor = np.array([0, 2, 3, 4], np.int32)
    group_count = np.array([3, 1, 4, 2], np.int32)
    K = int(group_count.sum())
    thr = rng.random(K, dtype=np.float32)
    stc = np.zeros(9, np.int32)
    stc[[0, 2, 3, 6]] = [2, 3, 1, 2]
    heights = [h for h in range(8, -1, -1) for _ in range(stc[h])]  # descending height
    cond = rng.integers(0, K, sum(heights)).astype(np.uint32)
    leaves = rng.integers(0, 2 ** 32, sum(1 << h for h in heights), dtype=np.uint64).astype(np.uint32)
    got = oracle.apply_paper(x, group_factor, group_count, thr, stc, cond, leaves)
    # brute force: binary features by group walk, explicit trees with pointer descent
    feat_of_bf = np.repeat(group_factor, group_count)
    for i in range(D):
        bits = oracle.binary_features(x[i], group_factor, group_count, thr)
        assert list(bits) == [int(x[i, feat_of_bf[k]] < thr[k]) for k in range(K)]
        total, cb, lb = 0, 0, 0
        for h in heights:
            fi = feat_of_bf[cond[cb:cb + h]].astype(np.int32)
            th = thr[cond[cb:cb + h]]
            root = _expand_tree(fi, th, leaves[lb:lb + (1 << h)].astype(np.float64), h, 0)
            total += int(_descend(root, x[i]))
            cb += h
            lb += 1 << h
        assert int(got[i]) == total


def test_condition_words_ordered_bits():
    # bit i of a word <-> document i; each bit is the raw condition x < border
    c = synth.tiny_case(seed=81, n_docs=70, n_features=5, n_trees=20, depth=3, pool=6)
    per, flat, counts, offs = oracle.borders(c.feature_index, c.thresholds, 5)
    w = oracle.condition_words(c.x, 5, flat, counts, offs)
    kb = 0
    for f in range(5):
        for j in range(counts[f]):
            for i in range(70):
                bit = (int(w[i // 32, kb]) >> (i % 32)) & 1
                assert bit == int(np.float32(c.x[i, f]) < per[f][j])
            kb += 1
    assert w.shape == (3, int(counts.sum()))


def test_o5_invariant_every_condition_of_c2():
    """SURVEY 8(c) O5 in full on config c2 (BASELINE size): for every document (100,000),
    every tree (2,000) and level (6), the raw fp32 condition x < thr (numpy's own
    compare) equals bin <= k from the oracle's bins and border indices -- 1.2e9 checks,
    one node at a time over all documents."""
    from concurrent.futures import ThreadPoolExecutor
    c = synth.make_case("c2")
    per, flat, counts, offs = oracle.borders(c.feature_index, c.thresholds, c.n_features)
    n = c.n_docs
    b = np.empty((n, c.n_features), np.uint16)
    step = 8192

    def job(r0):  # the oracle's linear-scan bins, in row blocks (ctypes releases the GIL)
        b[r0:r0 + step] = oracle.bins(c.x[r0:r0 + step], c.n_features, flat, counts, offs)

    with ThreadPoolExecutor(8) as ex:
        list(ex.map(job, range(0, n, step)))
    k = oracle.border_index(c.feature_index, c.thresholds, flat, counts, offs)
    assert np.all(k >= 0)
    xt = np.ascontiguousarray(c.x[:, :c.n_features].T)   # [feature][doc]
    bt = np.ascontiguousarray(b.T)
    bad = 0
    for node in range(c.feature_index.size):
        f = c.feature_index[node]
        bad += int(np.count_nonzero((xt[f] < c.thresholds[node]) != (bt[f] <= k[node])))
    assert bad == 0
