#!/usr/bin/env python
"""Benchmark of the F^3M KMVM hot path on B200 (BASELINE.json metric, config C4).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl f3m|reference]
    torchrun --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 --master-port P bench.py --gpus N ...

One step = one full F^3M KMVM (Alg. 1: bbox, keys, counting sort, tree, S2M, M2L, L2T,
near field, sigma) over n = 1e9 uniform points in [0,1)^3 (k(X,X), Gaussian, EV = 1,
P = 4, eta = 0.5), inputs resident in HBM.  N > 1 shards the targets (and S2M sources)
over N ranks with three NCCL all-reduces (strong scaling: n fixed).  Timing: W warm-up
steps, K timed steps between barrier + synchronize, CUDA events on the launch stream,
max over ranks; inputs (12 GB) are far larger than L2 (126 MB).  Rank 0 prints ONE JSON
line.  ``--impl reference`` times the CPU oracle (the reference arm of this tier) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("F3M_TIMING", "1")  # per-phase CUDA events inside the library (launch stream)

METRIC = "F3M KMVM points/sec (n=1e9,D=3) at 1/2/4/8 B200; rel. error vs exact"
UNIT = "points/s"

# Algorithmic work per unit of each timed phase (SURVEY.md 8(d) "Which roofline binds"; DESIGN.md
# sec. 5).  unit = what the phase processes (points, interacting box pairs, point pairs);
# bytes = HBM bytes the method must move per unit; flops = FP32 operations per unit.
def sparse_size(D: int, q: int) -> int:
    """|H| of the level-q Smolyak grid (reading R27): the union of the combination technique's
    tensor grids over nested Chebyshev levels (level 0: 1 point, level j: 2^j + 1)."""
    import itertools
    n1 = 2 ** q + 1
    H = set()
    for js in itertools.product(range(q + 1), repeat=D):
        if sum(js) > q:
            continue
        axes = [[2 ** (q - 1)] if j == 0 else [k * 2 ** (q - j) for k in range(2 ** j + 1)] for j in js]
        H.update(itertools.product(*axes))
    return len(H)


def phase_work(D: int, P: int, local: bool, passes: int = 1, sparse_level: int = 0) -> dict:
    """{phase: (unit, HBM bytes per unit, FP32 flops per unit)}."""
    m = P ** D
    s2m_flops = 2 * m + 4 * D * P + sum(P ** j for j in range(D))         # 197 at D = 3, P = 4
    l2t_flops = 2 * sum(P ** j for j in range(1, D + 1)) + 4 * D * P      # 216 at D = 3, P = 4
    m2l_flops = 2 * D * P ** (D + 1)
    if sparse_level:
        # sparse grid (kernels_sparse.cu): per point |H| basis products of <= q + 1 factors
        # (q + 1 flops each, the last an FMA) plus the D Chebyshev recurrences; per pair |H|^2
        # node-pair kernels of D table factors (D - 1 multiplies and one FMA: D + 1 flops)
        q, n1 = sparse_level, 2 ** sparse_level + 1
        mh = sparse_size(D, q)
        s2m_flops = l2t_flops = (q + 1) * mh + 3 * D * n1
        m2l_flops = (D + 1) * mh * mh
    return {
        "bbox": ("point", 4 * D, 0),
        # LSD pass 0: rank (read X, write the tile order) and scatter (read X, b, order; write
        # sorted coords, weights, pi, keys); later passes re-read / re-write the sorted copies
        "count": ("point", 4 * D + 2, 0),
        "scatter": ("point", (4 * D + 4 + 2) + (4 * D + 4 + 4 + 8), 0),
        "sort_misc": ("point", max(0, passes - 1) * ((8 + 2) + (8 + 4 + 4 * D + 4 + 2) + (4 * D + 4 + 4 + 8)), 0),
        # tile-local S2M ranks the tile (reads X, b; writes the 2-byte tile order); L2T reads X and
        # the order, writes v in input order and pi at the counting-sort destinations
        "s2m": ("point", (4 * D + 4 + 2) if local else (4 * D + 4), s2m_flops),
        "l2t": ("point", (4 * D + 2 + 4 + 4) if local else (4 * D + 8), l2t_flops),
        # separable M2L (SURVEY 8(a) note 2): 2 D P^{D+1} flops per far / smooth pair (D P^2 exps)
        "m2l": ("pair", 0, m2l_flops),
        # exact near / small field: one ex2 + (3D + 2) flops per point pair
        "near": ("point pair", 0, 3 * D + 3),
        "unpermute": ("point", 12, 0),
    }


def phase_units(phase: str, st, n_pts: float) -> float:
    if phase == "s2m":
        return st.s2m_points
    if phase == "l2t":
        return st.l2t_points
    if phase == "m2l":  # pairs of the pairwise (separable) M2L; complete-level groups: grid_flops()
        return float(sum(st.m_far) - sum(st.m_far_dropped) + sum(st.m_smooth) - st.m2l_grid_pairs)
    if phase == "near":
        return float(st.near_pairs)
    return n_pts


def grid_flops(phase: str, st) -> float:
    """FP32-equivalent flops of the complete-level M2L (kernels_grid.cu, reading R29):
    its fp64 FMAs at 2 flops each, counted twice against the FP32 peak (sm_100 DFMA runs at half
    the FFMA rate: 64 vs 128 lanes per SM per clock)."""
    return 4.0 * st.m2l_grid_fma if phase == "m2l" else 0.0


def fp32_peak(sm_max_mhz: float):
    """FP32 FFMA peak: the committed microbenchmark (tools/fp32_peak.cu, profiles/fp32_peak.json:
    best of its variants on this pool's B200), else the unit-count derivation."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp32_peak.json")) as f:
            j = json.load(f)
        return float(j["tflops"]), f"measured FFMA microbenchmark ({j['variant']}, profiles/fp32_peak.json)"
    except Exception:
        return 148 * 128 * 2 * sm_max_mhz * 1e6 / 1e12, "derived: 148 SM x 128 FP32 lanes x 2 flop x sm_max_mhz"


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz, self.ok = [], set(), None, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return j.get("hbm_gbs", 6650.0), "measured", j.get("sm_max_mhz", 1965.0)
    except Exception:
        return 6650.0, "fallback", 1965.0


def lengthscale(args, X) -> float:
    """--gamma, else from the effective variance: the population variance for
    uniform / normal data, the sample variance for the App. A datasets."""
    import datagen
    if args.gamma:
        return args.gamma
    if args.kind in ("uniform", "normal"):
        return datagen.gamma_for_ev(args.kind, args.D, args.ev)
    return datagen.gamma_for_ev_sample(X, args.ev)


def method_kw(args) -> dict:
    """Method parameters beyond P and eta: node cap, ablation flags."""
    kw = {}
    if args.node_cap != 2048:
        kw["node_cap"] = args.node_cap
    if args.flags:
        kw["flags"] = args.flags
    if args.sparse_level:
        kw["sparse_level"] = args.sparse_level
    return kw


def config_name(args) -> str:
    """Which BASELINE.json config this run is."""
    if args.D in (5, 7):
        return "C5"
    if args.D == 3 and args.kind == "normal" and args.n == 1_000_000:
        return "C2"
    if args.D == 3 and args.kind == "uniform":
        return {10_000: "C1", 100_000_000: "C3", 1_000_000_000: "C4"}.get(args.n, "custom")
    return "custom"


def dist_label(kind: str, D: int) -> str:
    return {"uniform": f"U[0,1)^{D}", "normal": f"N(0,I_{D})"}.get(kind, f"{kind} (datagen.py)")


def workload_config(args, gamma, world, sample_n=None):
    name = config_name(args)
    scale = f"ls={gamma:.4g}" if args.gamma else f"EV={args.ev} (gamma={gamma:.4f})"
    wl = (f"{name}: n={args.n:.0e} D={args.D} X=Y~{dist_label(args.kind, args.D)}, Gaussian k, {scale}, "
          f"P={args.P} (r={args.P ** args.D}), eta={args.eta}")
    if args.flags:
        wl += f", flags={args.flags}"
    if args.sparse_level:
        wl += f", sparse grid level {args.sparse_level}"
    if args.b == "planted":
        wl += ", planted b (KRR targets)"
    cfg = {
        "workload": wl, "baseline_config": name,
        "n": args.n, "D": args.D, "kind": args.kind, "ev": args.ev, "gamma": gamma, "P": args.P, "eta": args.eta,
        "rho": 2 * args.P ** args.D, "zeta": args.P ** args.D, "case": "k(X,X)",
        "node_cap": args.node_cap, "flags": args.flags, "b": args.b, "sparse_level": args.sparse_level,
        "l2": "inputs larger than L2 (X alone is 12 B/pt x n)" if args.n * 4 * args.D > 126e6
              else "inputs smaller than L2 (126 MB): warm-L2 timing, context only",
        "parallelism": f"targets sharded over {world} rank(s)" if world > 1 else "single GPU",
    }
    if sample_n is not None:
        cfg["timed_sample_n"] = sample_n
        cfg["workload"] += f" -- timed on the first {sample_n:.0e} points of it (bounded CPU sample)"
    return cfg


def host_cpu() -> dict:
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def run_reference(args):
    """The reference arm of this tier: the CPU oracle, as it stands, on a bounded sample."""
    import datagen
    import oracle
    rank, world, _ = env_rank()
    if rank != 0:
        return
    n_s = args.ref_sample
    Xt = datagen.points(args.kind, n_s, args.D, seed=0)
    gamma = lengthscale(args, Xt)
    X = Xt.double().numpy()
    b = datagen.weights(n_s, seed=1).double().numpy()
    oracle.build()
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.f3m(X, b, gamma, P=args.P, eta=args.eta, **method_kw(args), details=False)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    sec = statistics.mean(times)
    val = n_s / sec
    ladder = None
    if args.oracle_ladder:  # SURVEY 8(d) "Oracle timing": full single-threaded runs, pts/s per n
        ladder = []
        for nl in (10_000, 100_000, 1_000_000, 10_000_000):
            Xl = datagen.points(args.kind, nl, args.D, seed=0)
            gl = lengthscale(args, Xl)
            bl = datagen.weights(nl, seed=1).double().numpy()
            t0 = time.perf_counter()
            oracle.f3m(Xl.double().numpy(), bl, gl, P=args.P, eta=args.eta, **method_kw(args), details=False)
            dt = time.perf_counter() - t0
            ladder.append({"n": nl, "seconds": dt, "points_per_s": nl / dt})
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, gamma, args.gpus, sample_n=n_s),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", **host_cpu(),
                         "sample": f"first {n_s} points of the seeded workload per step (single-threaded fp64 oracle)"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if ladder is not None:
        line["oracle_ladder"] = {"runs": ladder, "cores": 1, **host_cpu(),
                                 "what": "full oracle F3M (stage 2 for every target) per n, single-threaded fp64"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="f3m", choices=["f3m", "reference"])
    ap.add_argument("--n", type=float, default=1e9)
    ap.add_argument("--D", type=int, default=3)
    ap.add_argument("--kind", default="uniform")
    ap.add_argument("--ev", type=float, default=1.0)
    ap.add_argument("--P", type=int, default=4)
    ap.add_argument("--eta", type=float, default=0.5)
    ap.add_argument("--gamma", type=float, default=0.0, help="lengthscale (overrides --ev; C1 / C3 quote ls)")
    ap.add_argument("--b", default="normal", choices=["normal", "planted"], help="b ~ N(0,1) or the KRR targets (PAPER.md:346)")
    ap.add_argument("--node-cap", type=int, default=2048, help="P^D cap (PAPER.md:286: 2048; 3^7 = 2187 needs more)")
    ap.add_argument("--flags", type=int, default=0, help="F3M_* ablation / admissibility flags (include/f3m.h)")
    ap.add_argument("--sparse-level", type=int, default=0,
                    help="Smolyak sparse grid of this level instead of the P^D tensor grid (PAPER.md:214, reading R27)")
    ap.add_argument("--subset", type=int, default=5000,
                    help="targets of the exact fp64 error subset (PAPER.md:286: 5000 rows)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-sample", type=int, default=5_000_000)
    ap.add_argument("--ref-sample", type=int, default=1_000_000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-op", action="store_true", help="skip the plan-reuse (operator API) measurement")
    ap.add_argument("--oracle-ladder", action="store_true",
                    help="--impl reference: also time the full oracle at n = 1e4 .. 1e7 (SURVEY 8(d) oracle timing)")
    args = ap.parse_args()
    args.n = int(args.n)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import datagen
    import paper_2202_01085_b200 as f3m
    from paper_2202_01085_b200 import sharded

    rank, world, local = env_rank()
    if world != args.gpus:
        args.gpus = world
    if local >= torch.cuda.device_count():  # the gloo single-GPU test of the N > 1 flow
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("F3M_DIST_BACKEND", "nccl")  # gloo: test the N > 1 flow on one GPU
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    n = args.n
    # the same seeded global X on every rank; rank g keeps rows [g n/N, (g+1) n/N)
    lo, hi = rank * n // world, (rank + 1) * n // world
    Xg = datagen.points(args.kind, n, args.D, seed=0, device=dev)
    gamma = lengthscale(args, Xg)
    bg = datagen.weights(n, seed=1, device=dev)
    if args.b == "planted":
        # the KRR targets of Sec. 5: b = k(X, D) alpha + eps, D = 1000 points of X,
        # alpha ~ N(0, I), eps ~ N(0, 0.1); the kernel sum is the library's exact direct sum
        alpha = datagen.weights(1000, seed=2, device=dev)
        bg = f3m.direct(Xg, alpha, gamma, Y=Xg[:1000].contiguous()) + math.sqrt(0.1) * bg
    X = Xg[lo:hi].contiguous() if world > 1 else Xg
    b = bg[lo:hi].contiguous() if world > 1 else bg
    # N > 1: Xg / bg stay resident as the replicated sources of the near / small field (the
    # library sorts them only when the tree has such pairs; none at C4)
    v = torch.empty(hi - lo, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        if world == 1:
            _, st = f3m.matvec(X, b, gamma, P=args.P, eta=args.eta, **method_kw(args), out=v, return_stats=True)
        else:
            plan = sharded.DevicePlan(X, b, gamma, Yfull=Xg, bfull=bg, P=args.P, eta=args.eta, **method_kw(args))
            try:
                sharded.run_sharded(plan, v)
                st = plan.stats
            finally:
                plan.close()
        return st

    def barrier():
        if world > 1:
            if dist.get_backend() == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    barrier()
    phases = f3m._ffi.phase_names()
    ph_ms = {p: 0.0 for p in phases}
    launches = 0
    last = None
    sampler = ClockSampler(local)
    with sampler:
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            st = step()
            last = st
            launches += st.kernel_launches
            for i, p in enumerate(phases):
                ph_ms[p] += st.ms_phase[i]
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    value = n / (ms * 1e-3)

    # ---- exact error on the first `subset` targets (fp64 on the device, validated vs the oracle)
    err = None
    if rank == 0 and args.subset > 0:
        Xall = Xg
        ball = bg
        m = min(args.subset, hi - lo)
        ve = f3m.direct(X[:m].contiguous(), ball, gamma, Y=Xall, fp64=True)
        vh = v[:m].double()
        num = torch.sum((vh - ve) ** 2).item()
        den = torch.sum(ve ** 2).item()
        err = {"err2": num / den, "err": math.sqrt(num / den), "subset": f"first {m} rows vs all {n} sources, fp64"}
    if world > 1:
        barrier()

    # ---- roofline of the dominant kernel phase (CUDA events on the launch stream, timed region)
    hbm_peak, peak_kind, sm_max = peaks()
    alu_peak, alu_src = fp32_peak(sm_max)
    local = last.far_groups_local > 0 and last.far_groups_sorted == 0
    work = phase_work(args.D, args.P, local, last.num_sort_passes, args.sparse_level)
    kern = {p: t / args.steps for p, t in ph_ms.items() if p != "total" and t > 0}
    phase_roof = {}
    for p_, t_ms in kern.items():
        e = {"ms": round(t_ms, 4)}
        if p_ in work:
            unit, per_b, per_f = work[p_]
            units = phase_units(p_, last, n / world)
            t_s = t_ms * 1e-3
            e.update({"unit": unit, "units": units, "bytes_per_unit": per_b, "flops_per_unit": per_f})
            fl = per_f * units + grid_flops(p_, last)
            if grid_flops(p_, last):
                e["grid_m2l"] = {"groups": last.m2l_grid_groups, "pairs": last.m2l_grid_pairs,
                                 "fp64_fma": last.m2l_grid_fma, "fp32_equiv_flops": grid_flops(p_, last)}
            if per_b:
                e["hbm_frac"] = round(per_b * units / t_s / 1e9 / hbm_peak, 4)
            if fl:
                e["alu_frac"] = round(fl / t_s / 1e12 / alu_peak, 4)
            e["ideal_ms"] = round(max(per_b * units / (hbm_peak * 1e9), fl / (alu_peak * 1e12)) * 1e3, 4)
        else:
            e["bound"] = "latency (host tree logic / O(boxes + pairs) kernels; no roofline model)"
        phase_roof[p_] = e
    modelled = {p_: t for p_, t in kern.items() if "ideal_ms" in phase_roof[p_]}
    top = max(modelled, key=modelled.get) if modelled else None
    roof = None
    if top:
        unit, per_b, per_f = work[top]
        units = phase_units(top, last, n / world)
        t_s = kern[top] * 1e-3
        hbm = per_b * units / t_s / 1e9
        alu = (per_f * units + grid_flops(top, last)) / t_s / 1e12
        if per_f == 0 or hbm / hbm_peak >= alu / alu_peak:
            roof = {"bound": "hbm", "kernel": top, "achieved": hbm, "peak": hbm_peak, "unit": "GB/s",
                    "frac": hbm / hbm_peak, "traffic": None, "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                    "bytes_per_unit": per_b, "work_unit": unit, "units_per_launch": units}
        else:
            roof = {"bound": "alu", "kernel": top, "achieved": alu, "peak": alu_peak, "unit": "TFLOP/s",
                    "frac": alu / alu_peak, "traffic": None, "peak_source": alu_src,
                    "flops_per_unit": per_f, "work_unit": unit, "units_per_launch": units,
                    "hbm_frac": hbm / hbm_peak}
            if grid_flops(top, last):  # achieved = (flops_per_unit x units + these) / time
                roof["grid_m2l_fp32_equiv_flops"] = grid_flops(top, last)
        tr_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tr_path):
            try:
                tr = json.load(open(tr_path))
                if top in tr and tr[top].get("n") == n // world:
                    roof["traffic"] = tr[top]["dram_bytes"]
            except Exception:
                pass
    phase_ms = {p: round(t / args.steps, 4) for p, t in ph_ms.items()}
    ideal_ms = sum(e.get("ideal_ms", 0.0) for e in phase_roof.values())
    phase_roof["overall"] = {"ideal_ms": round(ideal_ms, 3), "frac": round(ideal_ms / ms, 4),
                             "what": "sum over modelled phases of max(bytes / HBM peak, flops / FP32 peak) / ms_per_step"}

    # ---- config C2 context: the exact KeOps-style tiled sum (f3m_direct, fp32) on the same input
    exact = None
    if world == 1 and n <= 2_000_000:
        f3m.direct(X, b, gamma)
        torch.cuda.synchronize(dev)
        d0 = torch.cuda.Event(enable_timing=True)
        d1 = torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        f3m.direct(X, b, gamma)
        d1.record(stream)
        torch.cuda.synchronize(dev)
        dms = d0.elapsed_time(d1)
        exact = {"ms": dms, "value": n / (dms * 1e-3), "unit": UNIT, "f3m_speedup": dms / ms,
                 "kernel_pairs_per_s": n * n / (dms * 1e-3),
                 "what": "exact KMVM, KeOps-style tiled map-reduce (f3m_direct, fp32 eval, fp64 cross-tile sums)"}

    # ---- plan reuse (operator API): the same X, new b per apply
    reuse = None
    if world == 1 and not args.no_op:
        op = f3m.Operator(X, gamma, P=args.P, eta=args.eta, **method_kw(args))
        for _ in range(args.warmup):
            op.apply(b, out=v)
        torch.cuda.synchronize(dev)
        r0 = torch.cuda.Event(enable_timing=True)
        r1 = torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for _ in range(args.steps):
            _, ost = op.apply(b, out=v, return_stats=True)
        r1.record(stream)
        torch.cuda.synchronize(dev)
        rms = r0.elapsed_time(r1) / args.steps
        reuse = {"value": n / (rms * 1e-3), "unit": UNIT, "ms_per_apply": rms, "reuses_plan": op.reuses_plan,
                 "phase_ms": {p: round(ost.ms_phase[i], 4) for i, p in enumerate(phases) if ost.ms_phase[i] > 0},
                 "what": "f3m_op_apply: the b-dependent stages only (tile-local: S2M from the stored tile orders, M2L, "
                         "L2T; multi-pass trees: b gathered into the sorted order, S2M, M2L, near field, L2T, "
                         "LSD un-scatter); sort, tree and lists built once by f3m_op_create"}
        op.close()

    # ---- e2e: public API with pinned host buffers, H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        Xh = X.cpu().pin_memory()
        bh = b.cpu().pin_memory()
        vh = torch.empty(hi - lo, dtype=torch.float32).pin_memory()

        def e2e_step():
            if world == 1:
                f3m.matvec(Xh, bh, gamma, P=args.P, eta=args.eta, **method_kw(args), out=vh)
            else:
                Xd = Xh.to(dev, non_blocking=True)
                bd = bh.to(dev, non_blocking=True)
                vd, _ = sharded.sharded_matvec(Xd, bd, gamma, Yfull=Xg, bfull=bg, P=args.P, eta=args.eta, **method_kw(args))
                vh.copy_(vd, non_blocking=True)
            torch.cuda.synchronize(dev)

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        barrier()
        el = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            t = torch.tensor([el], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = t.item()
        e2e = {"value": n / el, "unit": UNIT, "h2d_bytes_per_step": int(n * (4 * args.D + 4)),
               "d2h_bytes_per_step": int(n * 4), "ms_per_step": el * 1e3}
        del Xh, bh, vh

    # ---- CPU baseline: the oracle as it stands on a bounded sample (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle
        n_s = min(args.cpu_sample, n)
        Xs = X[:n_s].cpu().double().numpy()
        bs = b[:n_s].cpu().double().numpy()
        oracle.build()
        t0 = time.perf_counter()
        oracle.f3m(Xs, bs, gamma, P=args.P, eta=args.eta, **method_kw(args), details=False)
        dt = time.perf_counter() - t0
        cpu = {"value": n_s / dt, "unit": UNIT, "cores": 1, "kind": "oracle", **host_cpu(),
               "sample": f"first {n_s} of the {n} seeded points, same gamma/P/eta, {dt:.1f} s single-threaded fp64"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, gamma, world),
            "roofline": roof, "phase_ms": phase_ms, "phase_roofline": phase_roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": sampler.summary(), "error_vs_exact": err, "plan_reuse": reuse,
            "exact_direct": exact,
            "tree": {"t_star": last.t_star, "t_sort": last.t_sort, "depth": last.depth_reached,
                     "sort_passes": last.num_sort_passes, "far_pairs": int(sum(last.m_far)),
                     "smooth_pairs": int(sum(last.m_smooth)), "near_pairs_points": int(last.near_pairs)},
            "paper_context": "F3M on 1x V100: 125.9 s at n=1e9, D=3, r=64, eta=0.5 (7.9e6 points/s; Table 2, "
                             "PAPER.md:302) -- other hardware and dataset, not the target",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
