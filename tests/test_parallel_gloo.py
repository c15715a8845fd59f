"""Multi-process (world size 2, gloo, CPU) checks of the multi-GPU host logic in
paper_2205_07307_b200/parallel.py.  The per-rank compute is the oracle (these
tests exercise sharding, gathering and reductions, not the kernels)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2205_07307_b200.parallel import shard_bounds, tree_shard


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_bounds_partition():
    for n in [0, 1, 7, 100, 1_000_000]:
        for w in [1, 2, 3, 8]:
            b = [shard_bounds(n, w, r) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_tree_shard_covers_forest():
    rng = np.random.default_rng(0)
    T, d = 37, 3
    fi = rng.integers(0, 5, T * d).astype(np.int32)
    th = rng.random(T * d).astype(np.float32)
    lv = rng.random(T << d).astype(np.float32)
    parts = [tree_shard(fi, th, lv, d, 4, r) for r in range(4)]
    assert np.array_equal(np.concatenate([p[0] for p in parts]), fi)
    assert np.array_equal(np.concatenate([p[1] for p in parts]), th)
    assert np.array_equal(np.concatenate([p[2] for p in parts]), lv)


def _worker(rank, world, port, exact, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import oracle
    import synth
    from paper_2205_07307_b200.parallel import DocSharded, TreeSharded, tree_shard
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = synth.tiny_case(seed=77, n_docs=301, n_features=12, n_trees=50, depth=6,
                               exact_leaves=exact)
        x = torch.from_numpy(case.x)

        def full_scorer(xx):
            return torch.from_numpy(oracle.score(xx.numpy(), case.feature_index, case.thresholds,
                                                 case.leaf_values, 6)[1])
        ds = DocSharded(full_scorer)
        got_doc = ds.score(x, gather=True).numpy()
        fi, th, lv, _ = tree_shard(case.feature_index, case.thresholds, case.leaf_values, 6,
                                   world, rank)

        def shard_scorer(xx):
            return torch.from_numpy(oracle.score(xx.numpy(), fi, th, lv, 6, n_trees=lv.size >> 6)[1])
        ts = TreeSharded(shard_scorer)
        got_tree = ts.score(x, op="all_reduce").numpy()
        got_red = ts.score(x, op="reduce", root=0).numpy()
        got_rs = ts.score(x, op="reduce_scatter").numpy()
        q.put((rank, got_doc, got_tree, got_red, got_rs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exact", [False, True])
def test_two_rank_doc_and_tree_sharding(exact):
    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, exact, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, a, b, c, d = q.get(timeout=120)
        res[r] = (a, b, c, d)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    case = synth.tiny_case(seed=77, n_docs=301, n_features=12, n_trees=50, depth=6,
                           exact_leaves=exact)
    s64, s32 = oracle.score(case.x, case.feature_index, case.thresholds, case.leaf_values, 6)
    tol = 1e-5 * np.abs(case.leaf_values.astype(np.float64)).reshape(-1, 64).max(1).sum()
    for r in range(2):
        doc, tree, red, rs = res[r]
        lo, hi = shard_bounds(301, 2, r)
        assert np.array_equal(rs, tree[lo:hi])  # reduce-scatter = doc-sharded totals
        assert np.array_equal(doc.view(np.uint32), s32.view(np.uint32))  # doc shard: identical
        assert np.abs(tree - s64).max() <= tol
        if exact:
            assert np.array_equal(tree, s32)  # exact partial sums: bit-exact
    assert np.abs(res[0][2] - s64).max() <= tol  # reduce to root


def _worker_bench_shard(rank, world, port, n_docs, q):
    """bench.py --gpus N (doc sharding) host logic: rank r generates only its rows of
    the batch (synth rows=), scores them, and the padded all-gather into a
    preallocated buffer rebuilds the whole score vector on every rank."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import oracle
    import synth
    from paper_2205_07307_b200.parallel import DocSharded
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_bounds(n_docs, world, rank)
        case = synth.make_case("c2", n_docs=n_docs, n_trees=40, rows=(lo, hi))
        assert case.x.shape[0] == hi - lo
        _, s32 = oracle.score(case.x, case.feature_index, case.thresholds, case.leaf_values,
                              case.depth)
        ds = DocSharded(lambda t: t)
        m = DocSharded.padded_size(n_docs, world)
        loc = torch.zeros(m, dtype=torch.float32)
        loc[:hi - lo] = torch.from_numpy(s32)
        out = torch.empty(m * world, dtype=torch.float32)
        ds.gather_into(loc, out)
        q.put((rank, ds.unpad(out, n_docs).numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_docs", [(2, 3001), (3, 1000)])
def test_bench_doc_shard_gather(world, n_docs):
    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker_bench_shard, args=(r, world, port, n_docs, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    case = synth.make_case("c2", n_docs=n_docs, n_trees=40)
    _, s32 = oracle.score(case.x, case.feature_index, case.thresholds, case.leaf_values, case.depth)
    for r in range(world):
        assert np.array_equal(res[r].view(np.uint32), s32.view(np.uint32))
