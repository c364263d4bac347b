"""GPU test of the sharded plan path on one device: G logical shards, each a
libf3m plan over its row slice, with the three all-reduces done in-process (sum of the
shards' tensors) -- the result must match the unsharded f3m_matvec.  Plus the real
torch.distributed flow with a single-rank NCCL group."""
import os
import socket

import numpy as np
import pytest
import torch

import datagen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def f3m():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2202_01085_b200 as m
    return m


@pytest.mark.parametrize("G,n,ev", [(2, 200000, 1.0), (4, 300001, 10.0), (3, 100000, 0.1)])
def test_logical_shards_match_unsharded(f3m, G, n, ev):
    from paper_2202_01085_b200.sharded import DevicePlan
    X = datagen.points("uniform", n, 3, seed=0).cuda()
    b = datagen.weights(n, seed=1).cuda()
    g = datagen.gamma_for_ev("uniform", 3, ev)
    vref = f3m.matvec(X, b, g)
    cuts = [r * n // G for r in range(G + 1)]
    plans = [DevicePlan(X[cuts[r]:cuts[r + 1]].contiguous(), b[cuts[r]:cuts[r + 1]].contiguous(), g) for r in range(G)]
    try:
        mms = torch.stack([p.bbox() for p in plans])
        D = 3
        gmm = torch.cat([mms[:, :D].min(0).values, mms[:, D:].max(0).values])
        cs = [p.counts(gmm) for p in plans]
        tot = torch.stack(cs).sum(0)
        for c in cs:
            c.copy_(tot)
        ws = [p.s2m() for p in plans]
        totw = torch.stack(ws).sum(0)
        for w in ws:
            w.copy_(totw)
        outs = [p.evaluate(torch.empty(cuts[r + 1] - cuts[r], device="cuda")) for r, p in enumerate(plans)]
    finally:
        for p in plans:
            p.close()
    v = torch.cat(outs).double()
    err = (torch.linalg.norm(v - vref.double()) / torch.linalg.norm(vref.double())).item()
    assert err <= 1e-5, err


def test_single_rank_nccl_flow(f3m):
    import torch.distributed as dist
    from paper_2202_01085_b200.sharded import sharded_matvec
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        X = datagen.points("uniform", 150000, 3, seed=3).cuda()
        b = datagen.weights(150000, seed=4).cuda()
        g = datagen.gamma_for_ev("uniform", 3, 1.0)
        v, st = sharded_matvec(X, b, g)
        assert torch.equal(v, f3m.matvec(X, b, g))
        assert st.kernel_launches > 0
    finally:
        dist.destroy_process_group()
