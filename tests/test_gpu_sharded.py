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


def logical_shards(f3m, X, b, g, G, **cfg):
    """G library plans over contiguous row slices of X (device), the collectives done in-process:
    MIN / MAX of the boxes, the concatenated sparse leaf lists, the SUM of the charges."""
    from paper_2202_01085_b200.sharded import DevicePlan
    n, D = X.shape
    cuts = [r * n // G for r in range(G + 1)]
    plans = [DevicePlan(X[cuts[r]:cuts[r + 1]].contiguous(), b[cuts[r]:cuts[r + 1]].contiguous(), g,
                        Yfull=X, bfull=b, **cfg) for r in range(G)]
    try:
        mms = torch.stack([p.bbox() for p in plans])
        gmm = torch.cat([mms[:, :D].min(0).values, mms[:, D:].max(0).values])
        lv = [p.leaves(gmm) for p in plans]
        keys = torch.cat([k for k, _ in lv])
        cnts = torch.cat([c for _, c in lv])
        for p in plans:
            p.set_leaves(keys, cnts)
        ws = [p.s2m() for p in plans]
        totw = torch.stack(ws).sum(0)
        for w in ws:
            w.copy_(totw)
        outs = [p.evaluate(torch.empty(cuts[r + 1] - cuts[r], device="cuda")) for r, p in enumerate(plans)]
        stats = plans[0].stats
    finally:
        for p in plans:
            p.close()
    return torch.cat(outs), stats


def rel(a, b):
    a, b = a.double(), b.double()
    return (torch.linalg.norm(a - b) / torch.linalg.norm(b)).item()


@pytest.mark.parametrize("G,n,ev", [(2, 200000, 1.0), (4, 300001, 10.0), (3, 100000, 0.1)])
def test_logical_shards_match_unsharded(f3m, G, n, ev):
    X = datagen.points("uniform", n, 3, seed=0).cuda()
    b = datagen.weights(n, seed=1).cuda()
    g = datagen.gamma_for_ev("uniform", 3, ev)
    vref = f3m.matvec(X, b, g)
    v, _ = logical_shards(f3m, X, b, g, G)
    assert rel(v, vref) <= 1e-5


# complete levels at D = 5 / 7 (uniform): the counted smooth level and the mode-product M2L
# (reading R29) on the all-reduced tree, with the register-blocked S2M / L2T on each shard
@pytest.mark.parametrize("n,D,P,G,extra", [(120000, 5, 4, 2, {}), (300000, 7, 2, 3, {}),
                                           (300000, 7, 3, 2, {"node_cap": 4096})])
def test_logical_shards_complete_levels(f3m, n, D, P, G, extra):
    X = datagen.points("uniform", n, D, seed=0).cuda()
    b = datagen.weights(n, seed=1).cuda()
    g = datagen.gamma_for_ev("uniform", D, 1.0)
    vref, st = f3m.matvec(X, b, g, P=P, return_stats=True, **extra)
    assert st.m2l_grid_groups >= 1
    v, sst = logical_shards(f3m, X, b, g, G, P=P, **extra)
    assert sst.m2l_grid_groups >= 1
    assert rel(v, vref) <= 1e-5


# near / small field present (normal data: small pairs in the tails, a deep multi-pass tree),
# and D * T_sort = 28 > 24 bits (normal D = 7): the sparse leaf lists and the replicated sources
@pytest.mark.parametrize("kind,n,D,P,G,extra", [
    ("normal", 120000, 3, 4, 2, {}),
    ("normal", 90001, 3, 4, 3, {"zeta": 16, "rho": 40}),
    ("normal", 20000, 7, 2, 2, {}),
])
def test_logical_shards_near_field(f3m, kind, n, D, P, G, extra):
    import oracle
    X = datagen.points(kind, n, D, seed=0)
    b = datagen.weights(n, seed=1)
    g = datagen.gamma_for_ev(kind, D, 1.0)
    vref, st = f3m.matvec(X.cuda(), b.cuda(), g, P=P, return_stats=True, **extra)
    assert st.near_pairs > 0
    v, sst = logical_shards(f3m, X.cuda(), b.cuda(), g, G, P=P, **extra)
    assert sst.near_pairs > 0
    assert rel(v, vref) <= 1e-5
    if D != 3:
        return
    # and against the oracle on the first rows (subset-target mode)
    m = 300
    r = oracle.f3m(X, b, g, P=P, n_eval=m, details=False, **extra)
    ve = torch.from_numpy(r.v[:m])
    assert rel(v[:m].cpu(), ve) <= 1e-5


def test_sharded_without_replicated_sources_is_rejected(f3m):
    from paper_2202_01085_b200 import F3MError
    from paper_2202_01085_b200.sharded import DevicePlan
    X = datagen.points("normal", 50000, 3, seed=0).cuda()
    b = datagen.weights(50000, seed=1).cuda()
    g = datagen.gamma_for_ev("normal", 3, 1.0)
    p = DevicePlan(X, b, g)
    try:
        mm = p.bbox()
        p.set_leaves(*p.leaves(mm))
        with pytest.raises(F3MError, match="replicated sources"):
            p.s2m()
    finally:
        p.close()


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


def _two_rank_worker(rank, world, port, n, out_path, kind="uniform"):
    import torch.distributed as dist
    from paper_2202_01085_b200.sharded import sharded_matvec
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    # two ranks on one GPU: gloo carries the three all-reduces (NCCL needs one GPU per rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X = datagen.points(kind, n, 3, seed=21).cuda()
        b = datagen.weights(n, seed=22).cuda()
        g = datagen.gamma_for_ev(kind, 3, 1.0)
        lo, hi = rank * n // world, (rank + 1) * n // world
        v, _ = sharded_matvec(X[lo:hi].contiguous(), b[lo:hi].contiguous(), g, Yfull=X, bfull=b)
        torch.save(v.cpu(), f"{out_path}.{rank}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["uniform", "normal"])
def test_two_rank_flow_on_one_gpu(f3m, tmp_path, kind):
    """The real multi-process flow of bench.py --gpus 2 (torch.distributed, row shards, the
    collectives) with two ranks sharing the one GPU, against the unsharded call; normal data
    has a near / small field (sources from the replicated full set)."""
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    n = 400_003
    out = str(tmp_path / "v")
    mp.start_processes(_two_rank_worker, args=(2, port, n, out, kind), nprocs=2, join=True, start_method="spawn")
    v = torch.cat([torch.load(f"{out}.{r}") for r in range(2)]).double()
    X = datagen.points(kind, n, 3, seed=21).cuda()
    b = datagen.weights(n, seed=22).cuda()
    vref = f3m.matvec(X, b, datagen.gamma_for_ev(kind, 3, 1.0)).cpu().double()
    assert (torch.linalg.norm(v - vref) / torch.linalg.norm(vref)).item() <= 1e-5
