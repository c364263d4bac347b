"""World-size-2 gloo test (CPU) of the sharded driver's host logic
(paper_2202_01085_b200.sharded.run_sharded).

The device plan is replaced by a CPU test double with the same interface whose bbox /
leaves / charges / evaluate are simple functions of the local shard; the sharded result
must equal the unsharded result of the same double, which holds only if the driver
all-reduces MIN of the minima and MAX of the maxima, hands every rank the concatenation of
all ranks' sparse leaf lists (the double sums equal keys), SUMs the charges and keeps every
rank's rows in order.  The double also keys its leaves on a 2^40-wide grid (no dense
histogram could hold it) and reports a near-field term that needs every rank's sources."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class FakePlan:
    """CPU double of sharded.DevicePlan: 4 bins per dimension over the global cube."""

    def __init__(self, X: np.ndarray, b: np.ndarray):
        self.X, self.b = X, b
        self.D = X.shape[1]

    def bbox(self):
        return torch.from_numpy(np.concatenate([self.X.min(0), self.X.max(0)]).astype(np.float64))

    def leaves(self, gmm):
        gmm = gmm.numpy()
        lo, hi = gmm[: self.D], gmm[self.D:]
        self.lo, self.E = lo, (hi - lo).max()
        c = np.minimum(np.floor((self.X - lo) / self.E * 4), 3).astype(np.int64)
        self.bin = (c * (4 ** np.arange(self.D))).sum(1)
        keys = self.bin << 34  # sparse keys far beyond any dense histogram
        uk, cnt = np.unique(keys, return_counts=True)
        return torch.from_numpy(uk.astype(np.int64)), torch.from_numpy(cnt.astype(np.int64))

    def set_leaves(self, keys, counts):
        k, c = keys.numpy(), counts.numpy()
        self.h = np.zeros(4 ** self.D, dtype=np.int64)
        np.add.at(self.h, k >> 34, c)  # the concatenation of every rank's list, equal keys summed

    def s2m(self):
        w = np.bincount(self.bin, weights=self.b, minlength=4 ** self.D)
        self.local_charges = torch.from_numpy(w.astype(np.float64))
        return self.local_charges

    def evaluate(self, out):
        W = self.local_charges.numpy()  # all-reduced in place by the driver
        v = W[self.bin] * (1.0 + self.X.sum(1)) + 0.001 * W.sum() + 1e-4 * self.h[self.bin]
        out.copy_(torch.from_numpy(v.astype(np.float32)))
        return out

    def close(self):
        pass


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, X, b, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_01085_b200.sharded import run_sharded
        n = X.shape[0]
        lo, hi = rank * n // world, (rank + 1) * n // world
        plan = FakePlan(X[lo:hi], b[lo:hi])
        out = torch.empty(hi - lo)
        run_sharded(plan, out)
        q.put((rank, out.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_driver_matches_unsharded(world):
    try:
        import paper_2202_01085_b200  # noqa: F401  (needs libf3m.so to import)
    except ImportError as e:
        pytest.skip(str(e))
    rng = np.random.default_rng(0)
    X = rng.normal(size=(1001, 3))
    b = rng.normal(size=1001)
    ref = FakePlan(X, b)
    ref.set_leaves(*ref.leaves(ref.bbox()))
    ref.s2m()
    vref = ref.evaluate(torch.empty(1001)).numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, b, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    v = np.concatenate([res[r] for r in range(world)])
    np.testing.assert_allclose(v, vref, rtol=1e-6)
