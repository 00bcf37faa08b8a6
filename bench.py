"""Benchmark: recursive-DAG site evaluations per second on B200.

Default workload (BASELINE.json configs[1], the single-GPU DAG-kernel
baseline): cfg2 -- O3, D=12, nu<=4 (50,909 DAG nodes), seeded complex-normal
A per site ([S, 819] complex128, resident in HBM), one real N(0,1)
coefficient per target (48,665), output Re(phi) per site.  One step = one pass
of the recursive kernel K2 over 100,000 sites per GPU (weak scaling: every
rank evaluates its own shard; sites are independent, so there is no
data-path collective).  `--config cfg1|cfg3|cfg4|cfg5` runs the other
BASELINE configurations (cfg3/cfg5 from Cartesian neighbour shells with the
total-energy all-reduce; cfg3/cfg5 shard a fixed global site count).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfgX]
    torchrun --nproc-per-node N bench.py --gpus N ...

Rank 0 prints ONE JSON line.  `--impl reference` times the reference's CPU
algorithm (the oracle port, oracle/acedag_oracle.py -- the reference is pure
Python and is not installed on the GPU box) on all host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "site evals/sec (recursive DAG contraction)"
UNIT = "sites/s"
R_IN, R_CUT = 0.8, 5.0

CONFIGS = {
    "cfg1": {"D": 8, "nu": 3, "sites": 1_000, "input": "A", "n_out": 1, "scaling": "weak", "cpu_sites": 64,
             "sha256": "ff6f09143cbc28f844d568e9ad810f830a215cab27570f8db4d757801e099b09",
             "desc": "cfg1 (BASELINE configs[0]): O3 D=8 nu<=3, 1e3 sites/GPU, A-given"},
    "cfg2": {"D": 12, "nu": 4, "sites": 100_000, "input": "A", "n_out": 1, "scaling": "weak", "cpu_sites": 32,
             "sha256": "cf46bc8f5590ee62f6f33a4ef6e8e1d14d972d2e4db4744d64edfff5215bd6bd",
             "desc": "cfg2 (BASELINE configs[1]): O3 D=12 nu<=4, 1e5 sites/GPU, A-given"},
    "cfg3": {"D": 12, "nu": 4, "sites": 1_000_000, "input": "positions", "J": 30, "n_out": 1,
             "scaling": "strong", "cpu_sites": 2,
             "sha256": "cf46bc8f5590ee62f6f33a4ef6e8e1d14d972d2e4db4744d64edfff5215bd6bd",
             "desc": "cfg3 (BASELINE configs[2]): O3 D=12 nu<=4 from J=30 neighbours, 1e6 sites total, energy all-reduce"},
    "cfg4": {"D": 16, "nu": 6, "sites": 200_000, "input": "A", "n_out": 1, "scaling": "weak", "cpu_sites": 1,
             "sha256": "bcc01406b9d7172f0b9601986ad7ae553aa2b1a44d0c9f1fddc2eab3ff1ec3a1",
             "desc": "cfg4 (BASELINE configs[3]): O3 D=16 nu<=6 (3,711,466 nodes), 2e5 sites/GPU, A-given"},
    "cfg5": {"D": 14, "nu": 5, "sites": 500_000, "input": "positions", "J": 40, "n_out": 64,
             "scaling": "strong", "cpu_sites": 1,
             "sha256": "4b1e54f455dac3196538dc8194cfbdaa83eab30f3a66604bdcba5dccba504cd9",
             "desc": "cfg5 (BASELINE configs[4]): O3 D=14 nu<=5 from J=40 neighbours, 64 outputs, 5e5 sites total"},
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--prec", default="f64", choices=["f64", "f32"])
    ap.add_argument("--alg", default="orig", choices=["orig", "gen"],
                    help="DAG construction: Algorithm 1 (orig) or Algorithm 2 (gen, insert_generalized)")
    ap.add_argument("--n", type=int, default=2, help="block size n of Algorithm 2 (--alg gen)")
    ap.add_argument("--sites", type=int, default=None, help="override the config's site count")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-naive", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------- workload
def with_alg(cfg, alg, n):
    """The config with its DAG built by Algorithm 2 (graphbuild.py:169-202)
    instead of Algorithm 1: same targets and coefficients, another node set."""
    if alg == "orig":
        return dict(cfg, alg="orig", n=1)
    return dict(cfg, alg="gen", n=n, sha256=None, desc=cfg["desc"] + f" [Alg. 2 DAG: insert_generalized n={n}]")


def workload(cfg, seed=1):
    """The graph (native builder, SHA-pinned) and coefficients [T] / [T, n_out]."""
    import paper_2202_04140_b200 as P
    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, cfg["D"]), cfg["nu"], cfg.get("alg", "orig"), cfg.get("n", 1))
    rng = np.random.default_rng(seed)
    n_out = cfg["n_out"]
    c = rng.normal(size=len(g.target_ids)) if n_out == 1 else rng.normal(size=(len(g.target_ids), n_out))
    return g, c


def dag_census(pa, pb, n_seeds, n_targets, cfg, used_seeds):
    """P, L_f, P_int, T and the algorithmic flops/bytes per site,
    from the DAG's parent arrays (either arm: native graph or oracle graph)."""
    N, L = len(pa), n_seeds
    child = np.zeros(N, np.int64)
    np.add.at(child, np.asarray(pa[L:], np.int64), 1)
    np.add.at(child, np.asarray(pb[L:], np.int64), 1)
    P_ = N - L
    L_f = int(np.sum(child[L:] == 0))
    P_int = P_ - L_f
    T = int(n_targets)
    n_out = cfg["n_out"]
    F = 6 * P_int + 3 * L_f + 2 * T * n_out
    if cfg["input"] == "positions":
        F += 4 * cfg["J"] * used_seeds
        B = 24 * cfg["J"] + 8 * n_out
    else:
        B = 16 * L + 8 * n_out
    return {"P": P_, "L_f": L_f, "P_int": P_int, "T": T, "F_site": F, "B_site": B}


def config_block(cfg, S, global_sites, world, n_nodes, census, in_bytes):
    """The `config` object, identical for both arms at the same N (workload
    keys only; plan details go to the separate "plan" key)."""
    pos = cfg["input"] == "positions"
    return {"workload": cfg["desc"], "sites_per_gpu": S, "global_sites": global_sites,
            "dag_nodes": n_nodes, "dag_products": census["P"], "targets": census["T"], "n_out": cfg["n_out"],
            "l2": ("inputs %.2f GB per GPU > 126 MB L2 (no flush)" % (in_bytes / 1e9)) if in_bytes > 126e6
            else "inputs fit L2; timed steps reuse them",
            "parallelism": f"dp{world} (sites sharded" + (", energy all-reduce)" if pos else ", no collective)")}


def shard_sizes(cfg, total_sites, rank, world):
    """(sites on this rank, global sites): weak configs give every rank the
    full count, strong configs split a fixed total evenly (distributed.shard_range)."""
    if cfg["scaling"] == "strong":
        base, rem = divmod(total_sites, world)
        return base + (1 if rank < rem else 0), total_sites
    return total_sites, world * total_sites


def input_bytes(cfg, S, n_seeds, prec):
    if cfg["input"] == "positions":
        return S * cfg["J"] * 3 * 8
    return S * n_seeds * (16 if prec == "f64" else 8)


def positions(S, J, gen, device):
    import torch
    d = torch.randn(S, J, 3, dtype=torch.float64, device=device, generator=gen)
    d = d / d.norm(dim=-1, keepdim=True)
    u = torch.rand(S, J, 1, dtype=torch.float64, device=device, generator=gen)
    r = (R_IN ** 3 + u * (R_CUT ** 3 - R_IN ** 3)) ** (1.0 / 3.0)
    return (d * r).contiguous()


# --------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no nvidia-smi samples"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[2:]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------- CPU baseline
_CPU_CTX = {}


def _cpu_worker(args):
    """Oracle port of the path (pool for position inputs, evaluate_graph +
    sequential c-dot) over a block of sites; the DAG arrays come from the
    parent through fork (no CUDA in the workers)."""
    S, seed = args
    from oracle import acedag_oracle as O
    pa, pb, tg, c, L, cfg = _CPU_CTX["graph"]
    rng = np.random.default_rng(seed)
    if cfg["input"] == "positions":
        J = cfg["J"]
        d = rng.normal(size=(S, J, 3))
        d /= np.linalg.norm(d, axis=-1, keepdims=True)
        r = (R_IN ** 3 + rng.uniform(size=(S, J)) * (R_CUT ** 3 - R_IN ** 3)) ** (1.0 / 3.0)
        xyz = d * r[..., None]
    else:
        A = rng.normal(0, math.sqrt(0.5), (S, L)) + 1j * rng.normal(0, math.sqrt(0.5), (S, L))
    t0 = time.perf_counter()
    if cfg["input"] == "positions":
        A = np.array([O.pool_positions(cfg["D"], xyz[s]) for s in range(S)])
    re, im = O.evaluate_nodes(pa, pb, A)
    if c.ndim == 1:
        O.model_sum(re, im, tg, c)
    else:
        for o in range(c.shape[1]):
            O.model_sum(re, im, tg, c[:, o])
    return S, time.perf_counter() - t0


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_pool(g, c, cfg, procs):
    _CPU_CTX["graph"] = (g.parents[:, 0].copy(), g.parents[:, 1].copy(), g.target_ids.copy(), c,
                         g.num_seeds, cfg)
    return mp.get_context("fork").Pool(procs)


def cpu_rate(g, c, cfg, procs, reps=1):
    per = cfg["cpu_sites"]
    with cpu_pool(g, c, cfg, procs) as pool:
        pool.map(_cpu_worker, [(1, i) for i in range(procs)])  # warm imports
        tot, wall = 0, 0.0
        for r in range(reps):
            t0 = time.perf_counter()
            res = pool.map(_cpu_worker, [(per, 100 + r * procs + i) for i in range(procs)])
            wall += time.perf_counter() - t0
            tot += sum(s for s, _ in res)
    return tot / wall, tot


def cpu_sample_text(cfg, procs, n):
    what = "pool_positions + " if cfg["input"] == "positions" else ""
    return (f"{n} sites: {procs} processes x {cfg['cpu_sites']} sites per step (oracle/acedag_oracle.py "
            f"{what}evaluate_nodes + model_sum, NumPy, fork pool)")


# --------------------------------------------------------- reference arm
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_workload(cfg, seed=1):
    """The reference arm's graph: the oracle's restatement of build_graph
    (graphbuild.py:243-268), SHA-256-checked against the reference's pinned
    hash -- no repo library is loaded on this arm."""
    from oracle import acedag_oracle as O
    og = O.build_graph("O3", O.Spec(1, cfg["D"]), cfg["nu"], cfg.get("alg", "orig"), cfg.get("n", 1))
    sha = O.graph_sha256(og)
    if cfg["sha256"] and sha != cfg["sha256"]:
        raise SystemExit(f"oracle graph SHA-256 {sha} != pinned {cfg['sha256']}")
    pa, pb, _aux, tg = O.graph_arrays(og)
    rng = np.random.default_rng(seed)
    n_out = cfg["n_out"]
    c = rng.normal(size=len(tg)) if n_out == 1 else rng.normal(size=(len(tg), n_out))
    L = len(O.one_particle_indices("O3", cfg["D"]))
    return pa, pb, tg, c, L


def used_seed_count(pa, pb, tg, L):
    used = np.zeros(L, bool)
    for arr in (pa[L:], pb[L:]):
        used[np.asarray(arr)[np.asarray(arr) < L]] = True
    used[np.asarray(tg)[np.asarray(tg) < L]] = True
    return int(used.sum())


def run_reference(a):
    """The reference's CPU algorithm on the box's host cores: the oracle port
    of evaluate_graph + the sequential c-dot (evaluator.py:93-142; pool for
    position inputs), NumPy, one forked process per core.  Rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    assert "paper_2202_04140_b200" not in sys.modules
    cfg = with_alg(CONFIGS[a.config], a.alg, a.n)
    cores = host_cores()
    pa, pb, tg, c, L = oracle_workload(cfg)
    census = dag_census(pa, pb, L, len(tg), cfg, used_seed_count(pa, pb, tg, L))
    S, global_sites = shard_sizes(cfg, a.sites or cfg["sites"], 0, a.gpus)
    _CPU_CTX["graph"] = (pa, pb, tg, c, L, cfg)
    # one core: the same per-process sample, alone
    with mp.get_context("fork").Pool(1) as pool1:
        pool1.map(_cpu_worker, [(1, 0)])
        t0 = time.perf_counter()
        n1 = sum(s for s, _ in pool1.map(_cpu_worker, [(cfg["cpu_sites"], 7)]))
        rate1 = n1 / (time.perf_counter() - t0)
    with mp.get_context("fork").Pool(cores) as pool:
        for w in range(a.warmup):
            pool.map(_cpu_worker, [(1, w * cores + i) for i in range(cores)])
        sites = 0
        t0 = time.perf_counter()
        for k in range(a.steps):
            res = pool.map(_cpu_worker, [(cfg["cpu_sites"], 1000 + k * cores + i) for i in range(cores)])
            sites += sum(s for s, _ in res)
        wall = time.perf_counter() - t0
    value = sites / wall
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * wall / a.steps,
            "higher_is_better": True, "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "f64",
            "data": ("synthetic: seeded uniform neighbour shells 0.8-5.0" if cfg["input"] == "positions" else
                     "synthetic: seeded complex-normal A") + ", N(0,1) coefficients per target",
            "config": config_block(cfg, S, global_sites, a.gpus, len(pa), census,
                                   input_bytes(cfg, S, L, "f64")),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "value_1core": rate1, "cpu_model": cpu_model(),
                             "graph": "oracle build_graph restatement" + (
                                 ", SHA-256 == reference " + cfg["sha256"][:16] if cfg["sha256"] else ""),
                             "sample": cpu_sample_text(cfg, cores, sites // max(1, a.steps)) + f" x {a.steps} steps"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- our arm
def fp64_peak_tflops(dev):
    """cuBLAS DGEMM 8192^3 (the FP64 analogue of MEASURED_PEAKS' bf16 probe)."""
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    del a, b
    return best


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def run_ours(a):
    import torch
    import torch.distributed as dist

    import paper_2202_04140_b200 as P
    from paper_2202_04140_b200.distributed import shard_range, total_energy

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # under torchrun the NCCL group is set up even for one rank, so the
    # barrier / max-over-ranks / energy all-reduce path always runs there
    distributed = world > 1 or "RANK" in os.environ
    if distributed:
        dist.init_process_group("nccl", init_method="env://", device_id=dev)

    def barrier():
        if distributed:
            dist.barrier()

    def max_over_ranks(x):
        if distributed:
            t = torch.tensor([x], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return x

    cfg = with_alg(CONFIGS[a.config], a.alg, a.n)
    S, global_sites = shard_sizes(cfg, a.sites or cfg["sites"], rank, world)
    if cfg["scaling"] == "strong":
        lo, hi = shard_range(global_sites, rank, world)
        assert hi - lo == S
    n_out = cfg["n_out"]
    g, c = workload(cfg)
    import hashlib
    graph_sha = hashlib.sha256(P.serialize_graph(g)).hexdigest()
    t_plan = time.perf_counter()
    plan = P.SitePlan(g, local).set_coefficients(node_ids=g.target_ids, values=c)
    t_plan = time.perf_counter() - t_plan
    info = plan.info()
    census = dag_census(g.parents[:, 0], g.parents[:, 1], g.num_seeds, len(g.target_ids), cfg, info["used_seeds"])
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    L = g.num_seeds
    pos = cfg["input"] == "positions"
    if pos:
        X = positions(S, cfg["J"], gen, dev)
    else:
        X = torch.complex(torch.randn(S, L, device=dev, dtype=torch.float64, generator=gen),
                          torch.randn(S, L, device=dev, dtype=torch.float64, generator=gen)) * math.sqrt(0.5)
        if a.prec == "f32":
            X = X.to(torch.complex64)
    out = torch.empty((S,) if n_out == 1 else (S, n_out), dtype=torch.float64, device=dev)
    energy = torch.zeros(n_out, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    launches = {"k": 0}

    def step():
        if pos:
            plan.evaluate_positions(X, result=out)
            energy.zero_()
            plan.reduce_sites(out, energy)
            total_energy(energy)
        else:
            plan.evaluate(X, result=out)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_launch0 = P.launch_count()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(a.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    # our kernels launched inside the timed region (the library's own count)
    gpu_launches = P.launch_count() - n_launch0
    barrier()
    torch.cuda.synchronize()
    ms_step = max_over_ranks(e0.elapsed_time(e1)) / a.steps
    value = global_sites / (ms_step * 1e-3)

    # per-phase device time of the K2 evaluations (CUDA events the library
    # records on the launching stream around the seed copy and the K2 kernel)
    nt = max(3, min(a.steps, 10))
    plan.timing(True)
    for _ in range(nt):
        step()
    ph = plan.read_timing()
    plan.timing(False)
    k2_ms = max_over_ranks(ph["main"] / nt)
    phases = {"prep_ms": ph["prep"] / nt, "k2_ms": ph["main"] / nt, "post_ms": ph["post"] / nt}

    naive = None
    if not pos and not a.no_naive and a.prec == "f64":
        nsteps = max(3, a.steps // 10)
        plan.evaluate(X, method="naive", result=out)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(nsteps):
            plan.evaluate(X, method="naive", result=out)
        e1.record(stream)
        torch.cuda.synchronize()
        naive_ms = max_over_ranks(e0.elapsed_time(e1) / nsteps)
        naive = {"value": global_sites / (naive_ms * 1e-3), "unit": UNIT, "ms_per_step": naive_ms,
                 "naive_products_per_site": info["naive_products"]}

    # end to end through the public API on pinned host buffers
    e2e = None
    if not a.no_e2e:
        Xh = X.cpu().pin_memory()
        res = torch.empty(out.shape, dtype=torch.float64, pin_memory=True)

        def e2e_step():
            if pos:
                plan.evaluate_positions_host(Xh, result=res)
            else:
                plan.evaluate_host(Xh, result=res)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        k = max(3, a.steps // 10)
        e0.record(stream)
        for _ in range(k):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks(e0.elapsed_time(e1) / k)
        e2e = {"value": global_sites / (ems * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(Xh.numel() * Xh.element_size()) if pos else int(plan.last_h2d_bytes),
               "d2h_bytes_per_step": int(res.numel() * 8), "ms_per_step": ems,
               "path": ("SitePlan.evaluate_positions_host: pinned host xyz -> 2-stream chunked H2D / "
                        "pool + K2 / D2H") if pos else
                       ("SitePlan.evaluate_host -> acedag_eval_host: pinned host A read in place over PCIe, "
                        "used seed columns only (k_gather_seeds on 4 SMs) pipelined with K2 on the rest, D2H")}
        del Xh

    F = census["F_site"]
    if cfg["D"] <= 8 and not pos:  # cfg1 is bandwidth-bound (F/B = 1.9)
        peak, src = hbm_peak()
        achieved = census["B_site"] * S / (k2_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_source": src, "bytes_per_site": census["B_site"]}
    else:
        peak = fp64_peak_tflops(dev)
        if a.prec == "f32":
            peak *= 2.0  # FFMA rate is 2x DFMA on B200 (72.6 vs 34.2 TF measured, profiles/r01)
        # position inputs: F includes the pool flops, so it is divided by the
        # whole step (pool + K2), not by the K2 phase alone
        t_roof = ms_step if pos else k2_ms
        achieved = F * S / (t_roof * 1e-3) / 1e12
        roof = {"bound": "fp64" if a.prec == "f64" else "fp32", "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak,
                "peak_source": "measured in this run: cuBLAS DGEMM 8192^3" + (" x2 (fp32)" if a.prec == "f32" else "")
                               + "; MEASURED_PEAKS.json has no FP64 entry",
                "flops_per_site": F,
                "flop_model": "F_site = 6 P_int + 3 L_f + 2 T n_out" + (" + 4 J U_used" if pos else "") + " (SURVEY.md 8d)"}
    roof["kernel"] = plan.kernel_name(prec=a.prec, sites=S)
    if pos:
        roof["kernel"] = "pool_positions + " + roof["kernel"]
        roof["timed_over"] = "whole step (pool + K2 + reduce): F_site includes the pool flops"
    roof["kernel_ms"] = ms_step if pos else k2_ms
    roof["step_share"] = roof["kernel_ms"] / ms_step
    roof["phases_ms"] = phases
    # DRAM bytes of the same kernel on the same workload from the committed
    # ncu --set full capture (only when kernel and site count match this run)
    roof["traffic"] = None
    for rnd in ("r02", "r01"):
        prof = os.path.join(ROOT, "profiles", rnd, "traffic.json")
        if roof["traffic"] is None and os.path.exists(prof) and a.alg == "orig" and a.prec == "f64":
            try:
                ent = json.load(open(prof)).get(a.config)
                if ent and ent.get("kernel") == roof.get("kernel") and ent.get("sites", S) == S:
                    roof["traffic"] = ent["bytes"]
                    roof["traffic_source"] = ent.get("source", prof)
            except Exception:
                pass

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cores = host_cores()
        rate, n = cpu_rate(g, c, cfg, cores, reps=1)
        rate1, _ = cpu_rate(g, c, cfg, 1, reps=1)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "value_1core": rate1,
               "cpu_model": cpu_model(), "sample": cpu_sample_text(cfg, cores, n)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": cfg["scaling"],
            "vs_baseline": None, "dtype": a.prec,
            "data": ("synthetic: seeded uniform neighbour shells 0.8-5.0 [S,J,3] f64" if pos else
                     "synthetic: seeded complex-normal A [S,%d] %s" % (L, "c128" if a.prec == "f64" else "c64"))
                    + " in HBM, N(0,1) coefficients per target",
            "config": config_block(cfg, S, global_sites, world, g.num_nodes, census,
                                   X.numel() * X.element_size()),
            "plan": {"products": info["recursive_products"], "extra_nodes": info["extra_nodes"],
                     "used_seeds": info["used_seeds"], "build_s": round(t_plan, 2),
                     "graph_sha256": graph_sha, "graph_sha_pinned": graph_sha == cfg["sha256"] if cfg["sha256"] else None},
            "dag_products_per_s": value * census["P"],
            "naive": naive,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()
    return 0


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
