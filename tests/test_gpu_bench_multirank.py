"""bench.py's multi-rank code path, run functionally on a one-GPU box: torchrun with 2
ranks over gloo, both on cuda:0 (--dist-backend gloo exists for this test only).  It
checks what the driver's 8-GPU run relies on -- row-range generation per rank, the
padded all-gather / the reduce of tree-shard partials inside the step, max-over-ranks
timing, one JSON line from rank 0 -- and the bench's own correctness checks (doc shard
bit-identical to one GPU, tree shard within the tolerance).  Timings of such a run mean
nothing and are not asserted."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("shard", ["docs", "trees", "weak"])
def test_bench_two_ranks_gloo_one_gpu(shard):
    extra = ["--shard", "docs", "--weak"] if shard == "weak" else ["--shard", shard]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--dist-backend", "gloo", "--config", "c2", *extra, "--steps", "3",
           "--warmup", "3", "--secondary", "none", "--no-cpu-baseline", "--e2e-steps", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["n_docs"] == 100_000 and d["per_rank_docs"] in (50_000, 100_000)
    if shard == "weak":  # every rank its own full batch, no collective, no cross-rank check
        assert d["scaling"] == "weak" and d["check"] is None and d["per_rank_docs"] == 100_000
        assert d["config"]["parallelism"] == "doc batches x2, no collective (weak)"
        assert d["e2e"]["h2d_bytes_per_step"] >= 2 * 100_000 * d["config"]["n_features"] * 4
        return
    assert d["scaling"] == "strong"
    if shard == "docs":
        assert d["check"]["bit_identical"] is True, d["check"]
        assert d["config"]["parallelism"] == "doc-shard x2 + NCCL all-gather"
    else:
        assert d["check"]["ok"] is True, d["check"]
