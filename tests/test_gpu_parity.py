"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by
element on the same seeded inputs.

Bar (BASELINE.json north_star):
  * bins and leaf indices bit-exact (window export + per-document FNV fingerprint);
  * scores |s_gpu - s_oracle64| <= 1e-5 * sum_t max_j |L_t[j]|;
  * exact-arithmetic leaves (integer * 2^-20) -> scores bit-exact;
  * fused odf_score == odf_binarize + odf_apply bit-for-bit (same summation order);
  * a document's score does not depend on the batch it is scored in (bit-exact).
"""
import numpy as np
import pytest

import oracle
import synth
from helpers import cuda_model, oracle_bins_used, run_cuda, to_dev, tolerance

pytestmark = pytest.mark.gpu

SPEC_DOC_COUNTS = [1, 7, 16, 100, 127, 128, 129, 257, 1000, 1024]


def _ld(f):
    return (f + 3) // 4 * 4


def full_check(case, check_fp=True, exact=False, idx_window=None):
    import torch
    n = case.n_docs
    m = cuda_model(case)
    x = to_dev(case.x)
    bins, s_fused, s_two = run_cuda(m, x, n)
    # bins bit-exact
    want_bins, used, _ = oracle_bins_used(case)
    assert np.array_equal(m.used_feature_ids, used)
    got_bins = m.canonical_bins(bins, n).cpu().numpy()
    assert np.array_equal(got_bins, want_bins), "bins differ"
    # scores
    s64, s32 = oracle.score(case.x, case.feature_index, case.thresholds, case.leaf_values,
                            case.depth, n_trees=case.n_trees)
    f = s_fused.cpu().numpy()
    t = s_two.cpu().numpy()
    assert np.array_equal(f.view(np.uint32), t.view(np.uint32)), "fused != two-stage"
    if exact:
        assert np.array_equal(f, s32), "exact-arithmetic leaves must give bit-exact scores"
    else:
        err = np.abs(f.astype(np.float64) - s64)
        tol = tolerance(case.leaf_values, case.depth)
        assert err.max(initial=0.0) <= tol, (err.max(), tol)
    # leaf indices: fingerprint of every document, and a window
    if check_fp and case.n_trees > 0:
        fp = m.index_fingerprint(bins, n).cpu().numpy().view(np.uint64)
        want_fp = oracle.fingerprint(case.x, case.feature_index, case.thresholds, case.depth,
                                     case.n_trees)
        assert np.array_equal(fp, want_fp), "leaf-index fingerprints differ"
    if idx_window and case.n_trees > 0:
        d0, nd, t0, nt = idx_window
        got = m.leaf_indices(bins, n, d0, nd, t0, nt).cpu().numpy().view(np.uint16)
        want = oracle.leaf_indices(case.x, case.feature_index, case.thresholds, case.depth,
                                   d0, nd, t0, nt)
        assert np.array_equal(got, want)
    torch.cuda.synchronize()
    m.close()
    return f


@pytest.mark.parametrize("seed", range(1, 21))
def test_c1_twenty_seeds(seed):
    case = synth.make_case("c1", seed=seed)
    full_check(case, idx_window=(0, case.n_docs, 0, case.n_trees))


@pytest.mark.parametrize("n_docs", SPEC_DOC_COUNTS)
def test_spec_doc_counts(n_docs):
    case = synth.tiny_case(seed=100 + n_docs, n_docs=n_docs, n_features=37, ld=40, n_trees=83,
                           depth=6, pool=16)
    full_check(case, idx_window=(0, n_docs, 0, 83))


@pytest.mark.parametrize("depth", list(range(0, 11)))
def test_every_depth(depth):
    case = synth.tiny_case(seed=200 + depth, n_docs=300, n_features=19, ld=20, n_trees=45,
                           depth=depth, pool=12)
    full_check(case, idx_window=(0, 300, 0, 45))


@pytest.mark.parametrize("depth", [3, 6, 10])
def test_exact_arithmetic_leaves_bit_exact(depth):
    case = synth.tiny_case(seed=300 + depth, n_docs=777, n_features=24, n_trees=210,
                           depth=depth, pool=20, exact_leaves=True)
    full_check(case, exact=True)


def test_special_values_ties_nan_zero_denormal_inf():
    case = synth.tiny_case(seed=41, n_docs=1000, n_features=16, n_trees=128, depth=6, pool=10)
    x = case.x
    rng = np.random.default_rng(3)
    for _ in range(3000):  # exact ties: a factor equal to a threshold on it
        k = rng.integers(case.feature_index.size)
        x[rng.integers(case.n_docs), case.feature_index[k]] = case.thresholds[k]
    specials = np.array([np.nan, -0.0, 0.0, 1e-45, -1e-45, 1e-40, np.inf, -np.inf,
                         np.finfo(np.float32).max, -np.finfo(np.float32).max], np.float32)
    for _ in range(3000):
        x[rng.integers(case.n_docs), rng.integers(16)] = specials[rng.integers(specials.size)]
    # thresholds that are themselves +-0.0 and denormal
    case.thresholds[:20:4] = np.float32(-0.0)
    case.thresholds[1:20:4] = np.float32(0.0)
    case.thresholds[2:20:4] = np.float32(1e-45)
    full_check(case, idx_window=(0, 1000, 0, 128))


@pytest.mark.parametrize("n_borders", [127, 128, 200, 254, 255, 381, 700, 2032])
def test_many_borders_split_columns(n_borders):
    # one factor carries n_borders distinct thresholds: > 127 uses C = ceil(m/127) code
    # columns; > 254 makes the model wide (uint16 bins, NEXT-4)
    rng = np.random.default_rng(n_borders)
    F, d, D = 8, 6, 700
    T = max(96, (3 * n_borders) // (2 * d))
    pool = np.sort(rng.standard_normal(n_borders).astype(np.float32))
    fi = rng.integers(0, F, T * d).astype(np.int32)
    fi[fi == 3] = 4  # factor 3 gets exactly the pool's n_borders thresholds
    thr = rng.standard_normal(T * d).astype(np.float32)
    first = np.arange(n_borders)
    fi[first] = 3
    thr[first] = pool
    hot = rng.random(T * d) < 0.3
    hot[:n_borders] = False  # keep every pool value: exactly n_borders distinct borders
    fi[hot] = 3
    thr[hot] = pool[rng.integers(0, n_borders, hot.sum())]
    x = rng.standard_normal((D, F)).astype(np.float32)
    x[::3, 3] = pool[rng.integers(0, n_borders, x[::3, 3].size)]  # ties on the hot factor
    lv = rng.normal(0, 0.01, T << d).astype(np.float32)
    case = synth.ForestCase("split", x, F, fi, thr, lv, d, T)
    f = full_check(case, idx_window=(0, D, 0, T))
    m = cuda_model(case)
    assert m.info["bins_elem_bytes"] == (2 if n_borders > 254 else 1)
    xd = to_dev(case.x)
    # the other consumers of bins / codes on the same model
    bins = m.binarize(xd)
    nbytes, k = m.bits_layout(D)
    words = m.bits_from_bins(bins, D)[: nbytes // 4].cpu().numpy().view(np.uint32).reshape(-1, k)
    per, flat, counts, offs = oracle.borders(case.feature_index, case.thresholds, case.n_features)
    assert np.array_equal(words, oracle.condition_words(case.x, F, flat, counts, offs))
    assert np.array_equal(m.apply_bits(m.bits_from_bins(bins, D), D).cpu().numpy().view(np.uint32),
                          f.view(np.uint32))
    ws = m.latency_workspace(D)
    lat = m.score_latency(xd, ws).cpu().numpy()
    assert np.abs(lat.astype(np.float64) - f).max() <= tolerance(case.leaf_values, d)
    m.close()


def test_too_many_borders_unsupported():
    from paper_2205_07307_b200 import MAX_BORDERS_WIDE, OdfError
    n = MAX_BORDERS_WIDE + 1
    rng = np.random.default_rng(5)
    d = 6
    T = (n + d - 1) // d
    fi = np.zeros(T * d, np.int32)
    thr = np.zeros(T * d, np.float32)
    thr[:n] = np.sort(rng.standard_normal(n).astype(np.float32))
    thr[n:] = thr[0]
    assert np.unique(thr).size == n
    case = synth.ForestCase("toomany", np.zeros((4, 2), np.float32), 2, fi, thr,
                            np.zeros(T << d, np.float32), d, T)
    with pytest.raises(OdfError) as e:
        cuda_model(case)
    assert e.value.status == 2  # ODF_E_UNSUPPORTED


def test_zero_docs_zero_trees_depth0():
    import torch
    case = synth.tiny_case(seed=51, n_docs=10, n_features=8, n_trees=0, depth=6)
    m = cuda_model(case)
    x = to_dev(case.x)
    assert np.all(m.score(x).cpu().numpy() == 0.0)
    assert m.n_used == 0
    empty = torch.empty((0, 8), dtype=torch.float32, device="cuda")
    assert m.score(empty).numel() == 0
    m.close()
    case = synth.tiny_case(seed=52, n_docs=130, n_features=8, n_trees=5, depth=0)
    full_check(case)


def test_ld_padding_and_ragged_features():
    case = synth.tiny_case(seed=61, n_docs=513, n_features=45, ld=64, n_trees=70, depth=5,
                           pool=9)
    case.x[:, 45:] = np.nan  # padding columns must never be read as factors
    full_check(case, idx_window=(100, 300, 3, 60))


def test_invalid_factor_layouts_rejected():
    import torch
    from paper_2205_07307_b200 import OdfError
    case = synth.tiny_case(seed=62, n_docs=64, n_features=6, ld=6, n_trees=4, depth=3)
    m = cuda_model(case)
    x = torch.from_numpy(case.x).cuda()
    with pytest.raises(OdfError) as e:
        m.score(x)  # ld = 6 is not a multiple of 4 (TMA row alignment)
    assert e.value.status == 1
    m.close()


def test_score_independent_of_batch_and_offset():
    import torch
    case = synth.make_case("c2", n_docs=5000, n_trees=300)
    m = cuda_model(case)
    x = to_dev(case.x)
    full = m.score(x).cpu().numpy()
    for a, b in [(0, 1), (1, 130), (127, 4000), (4999, 5000), (333, 4444)]:
        part = m.score(x[a:b].contiguous()).cpu().numpy()
        assert np.array_equal(part.view(np.uint32), full[a:b].view(np.uint32)), (a, b)
    torch.cuda.synchronize()
    m.close()


def test_score_host_e2e_matches_device():
    import torch
    case = synth.make_case("c2", n_docs=20000, n_trees=200)
    m = cuda_model(case)
    dev = m.score(to_dev(case.x)).cpu().numpy()
    xh = torch.from_numpy(case.x).pin_memory()
    host = m.score_host(xh, chunk_docs=3000)
    assert np.array_equal(host.numpy().view(np.uint32), dev.view(np.uint32))
    host2 = m.score_host(case.x, chunk_docs=1 << 20)
    assert np.array_equal(host2.view(np.uint32), dev.view(np.uint32))
    # caller-supplied outputs are checked before any copy is queued
    from paper_2205_07307_b200 import OdfError
    for bad in (np.empty(100, np.float32), np.empty(20000, np.float64)):
        with pytest.raises(OdfError):
            m.score_host(case.x, out=bad)
    with pytest.raises(OdfError):
        m.score_host(xh, out=torch.empty(10, dtype=torch.float32))
    m.close()


def test_concurrent_streams_one_model():
    import torch
    case = synth.make_case("c2", n_docs=3000, n_trees=500)
    m = cuda_model(case)
    x = to_dev(case.x)
    ref = m.score(x).cpu().numpy()
    streams = [torch.cuda.Stream() for _ in range(4)]
    outs = []
    for s in streams:
        with torch.cuda.stream(s):
            outs.append(m.score(x, stream=s))
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(o.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    m.close()


# ---------------------------------------------------------------------------
# BASELINE.json sizes, in the launch configuration bench.py times
# ---------------------------------------------------------------------------
def _oracle_bins_rows(case, rows_x, used, threads=8):
    """Oracle bins (used features) of the rows in rows_x, in parallel row chunks (the
    ctypes call releases the GIL; the oracle's arithmetic is unchanged)."""
    from concurrent.futures import ThreadPoolExecutor
    per, flat, counts, offs = oracle.borders(case.feature_index, case.thresholds, case.n_features)
    n = rows_x.shape[0]
    out = np.empty((n, used.size), np.uint16)
    step = max(1, -(-n // (threads * 4)))

    def job(r0):
        r1 = min(n, r0 + step)
        out[r0:r1] = oracle.bins(rows_x[r0:r1], case.n_features, flat, counts, offs)[:, used]

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(job, range(0, n, step)))
    return out


def _full_size(name, every=1, block=4096):
    """BASELINE size in bench.py's launch configuration (automatic tile width).  Checked
    against the oracle on EVERY document (every=1) or on every `every`-th block of
    `block` documents plus the last block: scores within the tolerance, bins and
    leaf-index fingerprints bit-exact; fused == two-stage bit for bit on all documents."""
    import torch
    case = synth.make_case(name)
    n = case.n_docs
    m = cuda_model(case)
    x = to_dev(case.x)
    bins, s_fused, s_two = run_cuda(m, x, n)
    f = s_fused.cpu().numpy()
    assert np.array_equal(f.view(np.uint32), s_two.cpu().numpy().view(np.uint32))
    starts = list(range(0, n, block))
    sel = starts[::every] + ([starts[-1]] if (len(starts) - 1) % every else [])
    rows = np.concatenate([np.arange(s0, min(s0 + block, n)) for s0 in sel])
    xs = case.x if every == 1 else case.x[rows]
    s64, _ = oracle.score(xs, case.feature_index, case.thresholds, case.leaf_values, case.depth)
    err = np.abs(f[rows].astype(np.float64) - s64)
    assert err.max() <= tolerance(case.leaf_values, case.depth), err.max()
    fp = m.index_fingerprint(bins, n).cpu().numpy().view(np.uint64)
    want_fp = oracle.fingerprint(xs, case.feature_index, case.thresholds, case.depth, case.n_trees)
    assert np.array_equal(fp[rows], want_fp)
    used = m.used_feature_ids
    canon = m.canonical_bins(bins, n)
    want = _oracle_bins_rows(case, xs, used)
    rows_t = torch.from_numpy(rows).cuda()
    for r0 in range(0, rows.size, 262144):
        got = canon[rows_t[r0:r0 + 262144]].cpu().numpy()
        assert np.array_equal(got, want[r0:r0 + 262144]), f"bins differ in rows {r0}.."
    got_idx = m.leaf_indices(bins, n, 1000, 64, case.n_trees - 100, 100).cpu().numpy().view(np.uint16)
    want_idx = oracle.leaf_indices(case.x, case.feature_index, case.thresholds, case.depth,
                                   1000, 64, case.n_trees - 100, 100)
    assert np.array_equal(got_idx, want_idx)
    m.close()
    del x, bins, canon
    torch.cuda.empty_cache()


def test_c2_full_size():
    _full_size("c2")


def test_c3_full_size():
    _full_size("c3")


def test_c4_full_size():
    _full_size("c4", every=4)  # 25 % of the 4 M documents (1.6e10 doc-trees in full)


# ---------------------------------------------------------------------------
# Tile width (odf_score_tiles / odf_apply_tiles): 128- and 256-document tiles
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,depth_note", [("c4", "depth 10"), ("c1", "depth 6")])
@pytest.mark.parametrize("n_docs", [1, 100, 128, 129, 255, 256, 257, 1000, 5000])
def test_tile_widths_bit_identical(name, depth_note, n_docs):
    """256-document tiles (two halves sharing every staged tree chunk) give the same
    scores, bit for bit, as 128-document tiles, fused and two-stage; ragged tiles
    include a fully empty second half (n_docs <= 128 mod 256)."""
    import torch
    case = synth.make_case(name, n_docs=max(n_docs, 65536) if name != "c1" else n_docs,
                           n_trees=48 if name == "c4" else None)
    case.x = np.ascontiguousarray(case.x[:n_docs])
    m = cuda_model(case)
    assert m.info["max_tile_docs"] == 256, m.info
    x = to_dev(case.x)
    bins = m.binarize(x)
    outs = [m.score(x, tile_docs=t) for t in (128, 256, 0)] + \
           [m.apply(bins, n_docs, tile_docs=t) for t in (128, 256, 0)]
    torch.cuda.synchronize()
    ref = outs[0].cpu().numpy()
    for o in outs[1:]:
        assert np.array_equal(o.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    s64, _ = oracle.score(case.x, case.feature_index, case.thresholds, case.leaf_values, case.depth)
    assert np.abs(ref.astype(np.float64) - s64).max() <= tolerance(case.leaf_values, case.depth)
    m.close()


def test_tile_256_exact_leaves_and_many_tiles():
    """Exact-arithmetic leaves: 256-document tiles are bit-exact against the oracle's
    fp32 rounding over many tiles (every SM runs several tiles, the ring wraps)."""
    import torch
    case = synth.make_case("c4", n_docs=200_000, n_trees=160, exact_leaves=True)
    m = cuda_model(case)
    x = to_dev(case.x)
    s256 = m.score(x, tile_docs=256)
    s128 = m.score(x, tile_docs=128)
    torch.cuda.synchronize()
    _, s32 = oracle.score(case.x, case.feature_index, case.thresholds, case.leaf_values, case.depth)
    assert np.array_equal(s256.cpu().numpy(), s32)
    assert np.array_equal(s128.cpu().numpy(), s32)
    m.close()


@pytest.mark.parametrize("depth", list(range(0, 11)))
def test_tile_256_every_depth_exact(depth):
    """256-document tiles at every depth (each depth has its own tree-item size, ring
    sub-slot count and factor-job span): exact-arithmetic leaves, fused and two-stage
    bit-exact against the oracle's fp32 rounding and equal to 128-document tiles, over
    many tiles per SM (the sub-slot ring wraps many times; ragged last tile)."""
    import torch
    n_docs = 148 * 256 * 3 + 77
    case = synth.tiny_case(seed=700 + depth, n_docs=n_docs, n_features=40, n_trees=48 + 16 * depth,
                           depth=depth, pool=24, exact_leaves=True)
    m = cuda_model(case)
    assert m.info["max_tile_docs"] == 256, m.info
    x = to_dev(case.x)
    bins = m.binarize(x)
    outs = [m.score(x, tile_docs=256), m.apply(bins, n_docs, tile_docs=256),
            m.score(x, tile_docs=128)]
    torch.cuda.synchronize()
    _, s32 = oracle.score(case.x, case.feature_index, case.thresholds, case.leaf_values, case.depth)
    for o in outs:
        assert np.array_equal(o.cpu().numpy(), s32)
    m.close()


def test_tile_width_errors():
    from paper_2205_07307_b200 import OdfError
    case = synth.tiny_case(3, n_docs=300)
    m = cuda_model(case)
    x = to_dev(case.x)
    for bad in (64, 512, -1):
        with pytest.raises(OdfError) as e:
            m.score(x, tile_docs=bad)
        assert e.value.status == 1
    m.close()
    # a wide model (a factor with > 254 borders, uint16 bins) has no 256-document tiles
    rng = np.random.default_rng(6)
    d, nb = 6, 300
    T = (nb + d - 1) // d
    fi = np.zeros(T * d, np.int32)
    thr = np.sort(rng.standard_normal(T * d).astype(np.float32))
    lv = rng.normal(0, 0.01, T << d).astype(np.float32)
    case = synth.ForestCase("wide", rng.standard_normal((300, 4)).astype(np.float32), 4, fi, thr,
                            lv, d, T)
    m = cuda_model(case)
    assert m.info["bins_elem_bytes"] == 2
    assert m.info["max_tile_docs"] == 128
    with pytest.raises(OdfError) as e:
        m.score(to_dev(case.x), tile_docs=256)
    assert e.value.status == 2
    s = m.score(to_dev(case.x), tile_docs=128)
    assert s.shape[0] == 300
    m.close()


# ---------------------------------------------------------------------------
# K4 latency path (config c5 shape): tolerance parity, determinism
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("batch,splits", [(1, 0), (100, 0), (100, 37), (1000, 0), (5000, 0),
                                          (777, 1)])
def test_latency_path(batch, splits):
    import torch
    case = synth.make_case("c5", n_docs=12000)
    m = cuda_model(case)
    x = to_dev(case.x)
    offs = synth.latency_queries(5, case.n_docs, batch, 3)
    ws = m.latency_workspace(batch, splits)
    tol = tolerance(case.leaf_values, case.depth)
    for o in offs:
        q = x[o:o + batch]
        a = m.score_latency(q, ws, splits=splits).cpu().numpy()
        b = m.score_latency(q, ws, splits=splits).cpu().numpy()
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), "not deterministic"
        rows = np.arange(o, o + batch)
        if batch > 300:
            rows = rows[np.random.default_rng(int(o)).choice(batch, 300, replace=False)]
        s64 = oracle.score_rows(case.x, rows, case.feature_index, case.thresholds,
                                case.leaf_values, case.depth)
        err = np.abs(a[rows - o].astype(np.float64) - s64)
        assert err.max() <= tol, (err.max(), tol)
        fused = m.score(q).cpu().numpy()
        assert np.abs(fused.astype(np.float64) - a).max() <= 2 * tol
    torch.cuda.synchronize()
    m.close()


def test_latency_path_depth10_and_small_workspace_error():
    import torch
    from paper_2205_07307_b200 import OdfError
    case = synth.tiny_case(seed=71, n_docs=300, n_features=20, n_trees=40, depth=10, pool=30)
    m = cuda_model(case)
    x = to_dev(case.x)
    ws = m.latency_workspace(300)
    got = m.score_latency(x, ws).cpu().numpy()
    s64, _ = oracle.score(case.x, case.feature_index, case.thresholds, case.leaf_values, 10)
    assert np.abs(got - s64).max() <= tolerance(case.leaf_values, 10)
    with pytest.raises(OdfError):
        m.score_latency(x, ws[:16])
    torch.cuda.synchronize()
    m.close()


# ---------------------------------------------------------------------------
# NEXT-1: MatrixNet integer leaves (u32 answers, u64 sums, (R - 2^31) S + B), zero tolerance
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("batch", [100, 1000, 5000])
def test_latency_graph(batch):
    """The K4 latency path captured in a CUDA graph (binarize kernel + apply kernel
    with a programmatic dependent launch) replays bit-identically to direct calls on
    the same input buffer, whatever that buffer holds, within the tolerance of the
    oracle; replays reuse the captured workspace and tensor map."""
    import torch
    case = synth.make_case("c5", n_docs=65536, n_trees=1000)
    m = cuda_model(case)
    x = to_dev(case.x)
    buf = x[:batch].clone()
    ws = m.latency_workspace(batch)
    out = torch.empty(batch, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # warm-up outside the capture
        m.score_latency(buf, ws, out=out)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        m.score_latency(buf, ws, out=out)
    tol = tolerance(case.leaf_values, case.depth)
    for q, off in enumerate([0, 7000, 65536 - batch]):
        buf.copy_(x[off:off + batch])
        g.replay()
        torch.cuda.synchronize()
        got = out.clone()
        ws2 = m.latency_workspace(batch)
        direct = m.score_latency(buf, ws2)
        torch.cuda.synchronize()
        assert torch.equal(got.view(torch.int32), direct.view(torch.int32)), q
        rows = np.arange(off, off + batch)[:: max(1, batch // 200)]
        s64 = oracle.score_rows(case.x, rows, case.feature_index, case.thresholds,
                                case.leaf_values, case.depth)
        assert np.abs(got.cpu().numpy()[rows - off].astype(np.float64) - s64).max() <= tol
    m.close()


def test_latency_path_rejects_too_many_tiles():
    from paper_2205_07307_b200 import OdfError
    case = synth.tiny_case(2, n_docs=128)
    m = cuda_model(case)
    big = 65535 * 128 + 1
    x = torch_empty_cuda((big, case.n_features))
    with pytest.raises(OdfError) as e:
        m.score_latency(x, m.latency_workspace(128))
    assert e.value.status == 1
    m.close()


def torch_empty_cuda(shape):
    import torch
    return torch.empty(shape, dtype=torch.float32, device="cuda")


@pytest.mark.parametrize("depth,n_docs,n_trees", [(6, 1000, 300), (3, 129, 1000), (10, 257, 40),
                                                  (0, 50, 7)])
def test_integer_leaves_exact(depth, n_docs, n_trees):
    import torch
    from paper_2205_07307_b200 import Model
    case = synth.tiny_case(seed=400 + depth, n_docs=n_docs, n_features=28, n_trees=n_trees,
                           depth=depth, pool=20)
    rng = np.random.default_rng(depth)
    lv = rng.integers(0, 2 ** 32, n_trees << depth, dtype=np.uint64).astype(np.uint32)
    S, B = 0.5 ** 20, -3.25
    m = Model(case.feature_index, case.thresholds, lv, depth, case.n_features, leaf_type="u32",
              scale=S, bias=B)
    x = to_dev(case.x)
    sums, sc = m.score_u64(x)
    bins = m.binarize(x)
    sums2, sc2 = m.apply_u64(bins, n_docs)
    want = oracle.score_u64(case.x, case.feature_index, case.thresholds, lv, depth)
    got = sums.cpu().numpy().view(np.uint64)
    assert np.array_equal(got, want)
    assert np.array_equal(sums2.cpu().numpy().view(np.uint64), want)
    fin = oracle.finalize(want, S, B)
    assert np.array_equal(sc.cpu().numpy(), fin) and np.array_equal(sc2.cpu().numpy(), fin)
    # the latency path (K4): u64 partials per split, exact -> bit-identical for any split
    for splits in (0, 1, 3):
        ws = m.latency_workspace(n_docs, splits)
        s3, sc3 = m.score_latency_u64(x, ws, splits=splits)
        assert np.array_equal(s3.cpu().numpy().view(np.uint64), want)
        assert np.array_equal(sc3.cpu().numpy(), fin)
    from paper_2205_07307_b200 import OdfError
    with pytest.raises(OdfError):
        m.score(x)
    with pytest.raises(OdfError):
        m.score_latency(x, m.latency_workspace(n_docs))
    torch.cuda.synchronize()
    m.close()


# ---------------------------------------------------------------------------
# Models wider than one 128-document code block (1,950 factors): 64-document
# tiles in every kernel
# ---------------------------------------------------------------------------
def _wide_columns_case(n_docs, depth=6, n_trees=1200, seed=1950):
    """Every one of F = 1950 factors used (1950+ code columns, ~250 KB for 128
    documents), factor 7 with 200 distinct thresholds (two code columns), ties."""
    rng = np.random.default_rng(seed)
    F = 1950
    nodes = n_trees * depth
    fi = np.concatenate([np.arange(F), rng.integers(0, F, nodes - F)]).astype(np.int32)
    rng.shuffle(fi)
    thr = (rng.integers(0, 40, nodes) / 10.0 - 2.0).astype(np.float32)
    pool = np.sort(rng.standard_normal(200).astype(np.float32))
    hot = np.flatnonzero(fi == 7)
    extra = rng.choice(np.flatnonzero(fi != 7), 200, replace=False)
    fi[extra] = 7
    thr[extra] = pool
    thr[hot] = pool[rng.integers(0, 200, hot.size)]
    ld = (F + 3) // 4 * 4
    x = np.zeros((n_docs, ld), np.float32)
    x[:, :F] = rng.standard_normal((n_docs, F)).astype(np.float32)
    x[::5, 7] = pool[rng.integers(0, 200, x[::5, 7].size)]  # ties on the split factor
    x[1::7, :F] = np.round(x[1::7, :F] * 10) / 10  # ties with the 0.1-grid thresholds
    lv = rng.normal(0, 0.01, n_trees << depth).astype(np.float32)
    return synth.ForestCase("wide_cols", x, F, fi, thr, lv, depth, n_trees)


@pytest.mark.parametrize("n_docs,depth", [(1, 6), (63, 6), (64, 6), (65, 6), (1000, 6), (4097, 6),
                                          (777, 8), (300, 3)])
def test_wide_column_model_64_document_tiles(n_docs, depth):
    case = _wide_columns_case(n_docs, depth=depth, n_trees=1200 if depth < 8 else 400)
    m = cuda_model(case)
    assert m.info["bins_tile_docs"] == 64 and m.info["n_columns"] > 1800, m.info
    assert m.info["max_tile_docs"] == 64
    m.close()
    full_check(case, idx_window=(0, min(n_docs, 70), case.n_trees - 40, 40))


def test_wide_column_model_integer_and_latency_path():
    import torch
    from paper_2205_07307_b200 import Model, OdfError
    case = _wide_columns_case(500, n_trees=600)
    rng = np.random.default_rng(9)
    lv = rng.integers(0, 2 ** 32, case.n_trees << 6, dtype=np.uint64).astype(np.uint32)
    m = Model(case.feature_index, case.thresholds, lv, 6, case.n_features, leaf_type="u32")
    assert m.info["bins_tile_docs"] == 64
    x = to_dev(case.x)
    sums, _ = m.score_u64(x)
    sums2, _ = m.apply_u64(m.binarize(x), 500)
    want = oracle.score_u64(case.x, case.feature_index, case.thresholds, lv, 6)
    assert np.array_equal(sums.cpu().numpy().view(np.uint64), want)
    assert np.array_equal(sums2.cpu().numpy().view(np.uint64), want)
    sums3, _ = m.score_latency_u64(x, m.latency_workspace(500))  # K4, 64-document tiles
    assert np.array_equal(sums3.cpu().numpy().view(np.uint64), want)
    m.close()
    # depth 10 at this width: 16-tree chunks of 4 KB tables (66 KB) x 2 ring slots do not
    # fit next to even a 64-document code block -> ODF_E_UNSUPPORTED, naming the bound
    deep = _wide_columns_case(10, depth=10, n_trees=200)
    with pytest.raises(OdfError) as e:
        cuda_model(deep)
    assert e.value.status == 2 and "64 documents" in str(e.value)
    m = cuda_model(case)
    s = m.score(x, tile_docs=0)
    s64 = m.score(x, tile_docs=64)
    assert torch.equal(s.view(torch.int32), s64.view(torch.int32))
    for td, st in ((128, 2), (256, 2), (32, 1)):
        with pytest.raises(OdfError) as e:
            m.score(x, tile_docs=td)
        assert e.value.status == st
    torch.cuda.synchronize()
    m.close()


@pytest.mark.parametrize("n_docs", [1, 63, 64, 65, 129, 500])
@pytest.mark.parametrize("splits", [0, 1, 3])
def test_wide_column_latency_path(n_docs, splits):
    """K4 on a 64-document-tile model (1,950 factors, P:168's width): within the
    tolerance of the oracle and of odf_score, deterministic, graph-capturable."""
    import torch
    case = _wide_columns_case(n_docs, n_trees=400)
    m = cuda_model(case)
    assert m.info["bins_tile_docs"] == 64
    x = to_dev(case.x)
    ws = m.latency_workspace(n_docs, splits)
    a = m.score_latency(x, ws, splits=splits).cpu().numpy()
    b = m.score_latency(x, ws, splits=splits).cpu().numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    tol = tolerance(case.leaf_values, case.depth)
    s64, _ = oracle.score(case.x, case.feature_index, case.thresholds, case.leaf_values, case.depth)
    assert np.abs(a.astype(np.float64) - s64).max() <= tol
    assert np.abs(a - m.score(x).cpu().numpy()).max() <= tol
    out = torch.empty(n_docs, device="cuda")
    g = torch.cuda.CUDAGraph()
    m.score_latency(x, ws, out=out, splits=splits)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        m.score_latency(x, ws, out=out, splits=splits)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), a.view(np.uint32))
    m.close()


# ---------------------------------------------------------------------------
# NEXT-2: paper-native mixed-height model import, exact u64 parity
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("pad_heights", [False, True], ids=["per_height", "padded"])
@pytest.mark.parametrize("stc,n_binary,n_features", [
    ([100] * 9, 100, 100),             # Table 6.1 synthetic: 100 trees of each height 0..8
    ([3, 0, 5, 0, 0, 0, 40, 0, 0], 150, 20),
    ([0, 0, 0, 0, 0, 0, 64, 0, 0], 64, 64),
    ([7, 0, 0, 0, 0, 0, 0, 0, 0], 10, 4),   # only constant (height-0) trees
    ([1, 1, 1, 1, 1, 1, 1990, 2, 3], 2000, 500),  # P:168's mix: ~99.9 % depth 6
])
def test_paper_native_import(stc, n_binary, n_features, pad_heights):
    import torch
    from paper_2205_07307_b200 import Model
    pm = synth.paper_model(11, n_features, n_binary, stc)
    pm.scale, pm.bias = 2.0 ** -31, 1.5
    rng = np.random.default_rng(3)
    D = 1024
    x = np.zeros((D, (n_features + 3) // 4 * 4), np.float32)
    x[:, :n_features] = rng.random((D, n_features), dtype=np.float32)
    for _ in range(500):  # ties with thresholds
        k = rng.integers(pm.thresholds.size)
        f = np.repeat(pm.group_factor, pm.group_count)[k]
        x[rng.integers(D), f] = pm.thresholds[k]
    m = Model.from_paper(pm.n_features, pm.group_factor, pm.group_count, pm.thresholds, pm.stc,
                         pm.cond_indices, pm.leaves, pm.scale, pm.bias, pad_heights=pad_heights)
    xd = torch.from_numpy(x).cuda()
    sums, sc = m.score_u64(xd)
    want = oracle.apply_paper(x, pm.group_factor, pm.group_count, pm.thresholds, pm.stc,
                              pm.cond_indices, pm.leaves)
    assert np.array_equal(sums.cpu().numpy().view(np.uint64), want)
    assert np.array_equal(sc.cpu().numpy(), oracle.finalize(want, pm.scale, pm.bias))
    # two-stage (binarize + apply_u64) gives the same exact sums
    s2, _ = m.apply_u64(m.binarize(xd), D)
    assert np.array_equal(s2.cpu().numpy().view(np.uint64), want)
    # the latency path (K4, per-height segments of a mixed model included), exact
    for splits in (0, 5):
        s3, sc3 = m.score_latency_u64(xd, m.latency_workspace(D, splits), splits=splits)
        assert np.array_equal(s3.cpu().numpy().view(np.uint64), want)
        assert np.array_equal(sc3.cpu().numpy(), oracle.finalize(want, pm.scale, pm.bias))
    heights = [h for h in range(len(stc)) if stc[h] > 0]
    if not pad_heights and len(heights) > 1:  # mixed model: no per-tree index export
        from paper_2205_07307_b200 import OdfError
        with pytest.raises(OdfError) as e:
            m.index_fingerprint(m.binarize(xd), D)
        assert e.value.status == 2
    m.close()


# ---------------------------------------------------------------------------
# NEXT-4: feature-major (pre-transposed, §5.5) input, bit-identical to doc-major
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n_docs,name", [(1, "c1"), (129, "c1"), (1024, "c1"), (3000, "c2"),
                                         (777, "c4")])
def test_feature_major_input(n_docs, name):
    import torch
    case = synth.make_case(name, n_docs=n_docs, n_trees=None if name == "c1" else 300)
    m = cuda_model(case)
    x = to_dev(case.x)
    ldt = (n_docs + 3) // 4 * 4 + 4
    xt_h = np.full((case.n_features, ldt), np.nan, np.float32)
    xt_h[:, :n_docs] = case.x[:, :case.n_features].T
    xt = to_dev(xt_h)
    b_dm = m.binarize(x)
    b_fm = m.binarize_fm(xt, n_docs)
    assert np.array_equal(m.canonical_bins(b_fm, n_docs).cpu().numpy(),
                          m.canonical_bins(b_dm, n_docs).cpu().numpy())
    s_dm = m.score(x).cpu().numpy()
    s_fm = m.score_fm(xt, n_docs).cpu().numpy()
    assert np.array_equal(s_dm.view(np.uint32), s_fm.view(np.uint32))
    want_bins, _, _ = oracle_bins_used(case)
    assert np.array_equal(m.canonical_bins(b_fm, n_docs).cpu().numpy(), want_bins)
    torch.cuda.synchronize()
    m.close()


# ---------------------------------------------------------------------------
# tree sharding on one GPU: per-shard partials summed == whole forest (tolerance / exact)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("world,exact", [(2, False), (3, True), (8, False)])
def test_tree_shards_sum_to_forest(world, exact):
    import torch
    from paper_2205_07307_b200 import Model
    from paper_2205_07307_b200.parallel import tree_shard
    case = synth.make_case("c4", n_docs=2000, n_trees=203, exact_leaves=exact)
    x = to_dev(case.x)
    total = torch.zeros(case.n_docs, dtype=torch.float32, device="cuda")
    for r in range(world):
        fi, th, lv, _ = tree_shard(case.feature_index, case.thresholds, case.leaf_values,
                                   case.depth, world, r)
        m = Model(fi, th, lv, case.depth, case.n_features)
        total += m.score(x)
        m.close()
    got = total.cpu().numpy()
    s64, s32 = oracle.score(case.x, case.feature_index, case.thresholds, case.leaf_values,
                            case.depth)
    if exact:
        assert np.array_equal(got, s32)
    else:
        assert np.abs(got - s64).max() <= tolerance(case.leaf_values, case.depth)


# ---------------------------------------------------------------------------
# determinism across many tiles and CTAs (WAR hazards on the TMA ring would show here)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,n_docs,n_trees", [("c4", 300_000, 1000), ("c2", 300_000, 2000)])
def test_deterministic_over_many_tiles(name, n_docs, n_trees):
    import torch
    case = synth.make_case(name, n_docs=n_docs, n_trees=n_trees)
    m = cuda_model(case)
    x = to_dev(case.x)
    ref = m.score(x)
    bins = m.binarize(x)
    for _ in range(3):
        assert torch.equal(m.score(x).view(torch.int32), ref.view(torch.int32))
        assert torch.equal(m.apply(bins, n_docs).view(torch.int32), ref.view(torch.int32))
    torch.cuda.synchronize()
    m.close()


# ---------------------------------------------------------------------------
# NEXT-3: bit-packed ordered condition words (ballot) and the apply over them
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,n_docs,n_trees", [("c1", 1024, None), ("c1", 33, None),
                                                 ("c2", 5000, 300), ("c4", 1000, 64)])
def test_condition_words_and_bits_apply(name, n_docs, n_trees):
    import torch
    case = synth.make_case(name, n_docs=n_docs, n_trees=n_trees)
    m = cuda_model(case)
    x = to_dev(case.x)
    bins = m.binarize(x)
    words = m.bits_from_bins(bins, n_docs)
    nbytes, k = m.bits_layout(n_docs)
    per, flat, counts, offs = oracle.borders(case.feature_index, case.thresholds, case.n_features)
    want = oracle.condition_words(case.x, case.n_features, flat, counts, offs)
    got = words[: nbytes // 4].cpu().numpy().view(np.uint32).reshape(-1, k)
    assert np.array_equal(got, want)
    s_bits = m.apply_bits(words, n_docs).cpu().numpy()
    s_main = m.score(x).cpu().numpy()
    assert np.array_equal(s_bits.view(np.uint32), s_main.view(np.uint32))
    torch.cuda.synchronize()
    m.close()


# ---------------------------------------------------------------------------
# Many code columns (more than tensor memory would hold: the round-2 TMEM code-cache
# experiment, profiles/r2_tmem_experiment.json) with skewed column usage
# ---------------------------------------------------------------------------
def _many_column_case(depth, n_docs=3000, n_trees=700, n_features=900, seed=41, exact=True):
    rng = np.random.default_rng(seed + depth)
    x = rng.standard_normal((n_docs, n_features)).astype(np.float32)
    pools = np.sort(rng.standard_normal((n_features, 24)).astype(np.float32), axis=1)
    popular = rng.random(n_trees * depth) < 0.6  # skewed usage: hot and cold columns
    fi = np.where(popular, rng.integers(0, 100, n_trees * depth),
                  rng.integers(0, n_features, n_trees * depth)).astype(np.int32)
    thr = pools[fi, rng.integers(0, 24, fi.size)].astype(np.float32)
    lv = synth.leaves(seed, n_trees, depth, 0.01, exact=exact)
    return synth.ForestCase("many-columns", x, n_features, fi, thr, lv, depth, n_trees)


@pytest.mark.parametrize("depth", [4, 5, 6, 7, 8])
def test_many_columns_exact(depth):
    """> 512 code columns, skewed usage: with exact-arithmetic leaves the fused and
    two-stage scores are bit-exact against the oracle, bins / fingerprints / the full
    leaf-index export are exact, and the bit-word apply and the latency path agree bit
    for bit."""
    import torch
    case = _many_column_case(depth)
    f = full_check(case, exact=True, idx_window=(0, case.n_docs, 0, case.n_trees))
    m = cuda_model(case)
    assert m.info["n_columns"] > 512, m.info
    x = to_dev(case.x)
    bins = m.binarize(x)
    s_bits = m.apply_bits(m.bits_from_bins(bins, case.n_docs), case.n_docs).cpu().numpy()
    assert np.array_equal(s_bits.view(np.uint32), f.view(np.uint32))
    lat = m.score_latency(x, m.latency_workspace(case.n_docs)).cpu().numpy()
    assert np.array_equal(lat, f)
    torch.cuda.synchronize()
    m.close()


@pytest.mark.parametrize("n_docs", [1, 129, 5000])
def test_many_columns_fp32_tolerance(n_docs):
    """fp32 leaves on a many-column model: scores within the tolerance, fused ==
    two-stage bit for bit."""
    case = _many_column_case(6, n_docs=n_docs, exact=False)
    full_check(case)


@pytest.mark.parametrize("extra_tiles,tail", [(1, 0), (20, 37), (74, 0), (75, 5)])
def test_partial_last_wave_as_64_document_tiles(extra_tiles, tail):
    """odf_score's partly filled last wave (<= half of the SMs) runs as 64-document tiles
    in a programmatic dependent launch: bit-identical to 128-document tiles throughout
    (tile_docs=128 never splits) and to the two-stage path, and bit-exact against the
    oracle with exact-arithmetic leaves; 75 extra tiles (> half) keep one launch."""
    import torch
    probe = cuda_model(synth.tiny_case(seed=91, n_docs=128, n_features=40, n_trees=64, depth=6, pool=24))
    sms = probe.info["num_sms"]
    probe.close()
    n_docs = (sms + extra_tiles) * 128 + tail
    case = synth.tiny_case(seed=90 + extra_tiles, n_docs=n_docs, n_features=40, n_trees=96, depth=6, pool=24,
                           exact_leaves=True)
    m = cuda_model(case)
    x = to_dev(case.x)
    auto = m.score(x)
    t128 = m.score(x, tile_docs=128)
    two = m.apply(m.binarize(x), n_docs)
    torch.cuda.synchronize()
    _, s32 = oracle.score(case.x, case.feature_index, case.thresholds, case.leaf_values, case.depth)
    a = auto.cpu().numpy()
    assert np.array_equal(a.view(np.uint32), t128.cpu().numpy().view(np.uint32))
    assert np.array_equal(a.view(np.uint32), two.cpu().numpy().view(np.uint32))
    assert np.array_equal(a, s32)
    m.close()
