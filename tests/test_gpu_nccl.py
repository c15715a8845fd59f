"""NCCL on the real backend, one GPU (world size 1): the collectives bench.py times in
its multi-GPU steps (the padded all-gather of doc-sharded scores, the reduce of
tree-shard partials) run through torch.distributed's NCCL communicator on the CUDA
path's outputs.  (More ranks need more GPUs: the host logic at world size 2/3 is
covered by tests/test_parallel_gloo.py.)"""
import os
import socket

import numpy as np
import pytest

import synth
from helpers import cuda_model, to_dev

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_world1_gather_and_reduce():
    import torch
    import torch.distributed as dist
    from paper_2205_07307_b200.parallel import DocSharded, TreeSharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        assert dist.get_backend() == "nccl"
        case = synth.tiny_case(21, n_docs=1000)
        m = cuda_model(case)
        x = to_dev(case.x)
        ref = m.score(x)
        ds = DocSharded(lambda t: m.score(t))
        mp = DocSharded.padded_size(1000, 1)
        loc = torch.zeros(mp, device="cuda")
        out = torch.empty(mp, device="cuda")
        m.score(x, out=loc[:1000])
        ds.gather_into(loc, out)
        dist.all_gather_into_tensor(out, loc)  # the NCCL collective itself
        assert torch.equal(ds.unpad(out, 1000).view(torch.int32), ref.view(torch.int32))
        ts = TreeSharded(lambda t: m.score(t))
        red = ts.score(x, op="reduce", root=0)
        part = m.score(x)
        dist.reduce(part, dst=0, op=dist.ReduceOp.SUM)
        torch.cuda.synchronize()
        assert torch.equal(red.view(torch.int32), ref.view(torch.int32))
        assert torch.equal(part.view(torch.int32), ref.view(torch.int32))
        m.close()
    finally:
        dist.destroy_process_group()
