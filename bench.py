"""Benchmark: recursive-DAG site evaluations per second on B200.

Workload (BASELINE.json configs[1], the single-GPU DAG-kernel baseline):
cfg2 -- O3, D=12, nu<=4 (50,909 DAG nodes), seeded complex-normal A per site
([S, 819] complex128, resident in HBM), one real N(0,1) coefficient per
target (48,665), output Re(phi) per site.  One step = one pass of the
recursive kernel K2 over 100,000 sites per GPU (weak scaling: every rank
evaluates its own 100,000-site shard; sites are independent, so there is no
data-path collective).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Rank 0 prints ONE JSON line.  `--impl reference` times the reference's CPU
algorithm (the oracle port, oracle/acedag_oracle.py -- the reference is
pure Python and cannot be installed on the GPU box) on all host cores.
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
CFG = {"D": 12, "nu": 4, "sites_per_gpu": 100_000}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sites", type=int, default=CFG["sites_per_gpu"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------- workload
def workload(D, nu, seed=1):
    """The graph (native builder, SHA-pinned) and coefficients."""
    import paper_2202_04140_b200 as P
    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, D), nu)
    c = np.random.default_rng(seed).normal(size=len(g.target_ids))
    return g, c


def dag_census(g):
    """P, L_f, P_int, T and F_site of the reference DAG."""
    N, L = g.num_nodes, g.num_seeds
    par = g.parents[L:]
    child = np.zeros(N, np.int64)
    np.add.at(child, par[:, 0], 1)
    np.add.at(child, par[:, 1], 1)
    P_ = N - L
    L_f = int(np.sum(child[L:] == 0))
    P_int = P_ - L_f
    T = len(g.target_ids)
    F = 6 * P_int + 3 * L_f + 2 * T
    return {"P": P_, "L_f": L_f, "P_int": P_int, "T": T, "F_site": F, "F_naive_min": None}


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
    """Oracle port of evaluate_graph + sequential c-dot over a site block.
    The DAG arrays come from the parent through fork (no CUDA in workers)."""
    S, seed = args
    from oracle import acedag_oracle as O
    pa, pb, tg, c, L = _CPU_CTX["graph"]
    rng = np.random.default_rng(seed)
    A = rng.normal(0, math.sqrt(0.5), (S, L)) + 1j * rng.normal(0, math.sqrt(0.5), (S, L))
    t0 = time.perf_counter()
    re, im = O.evaluate_nodes(pa, pb, A)
    O.model_sum(re, im, tg, c)
    return S, time.perf_counter() - t0


def cpu_rate(g, c, sites_per_proc, procs, reps=1):
    _CPU_CTX["graph"] = (g.parents[:, 0].copy(), g.parents[:, 1].copy(), g.target_ids.copy(), c, g.num_seeds)
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        pool.map(_cpu_worker, [(2, 0)] * procs)  # warm imports
        tot_s, wall = 0, 0.0
        for r in range(reps):
            t0 = time.perf_counter()
            res = pool.map(_cpu_worker, [(sites_per_proc, 100 + r * procs + i) for i in range(procs)])
            wall += time.perf_counter() - t0
            tot_s += sum(s for s, _ in res)
    return tot_s / wall, tot_s


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# --------------------------------------------------------- reference arm
def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    cores = host_cores()
    per = 32
    g, c = workload(CFG["D"], CFG["nu"])
    _CPU_CTX["graph"] = (g.parents[:, 0].copy(), g.parents[:, 1].copy(), g.target_ids.copy(), c, g.num_seeds)
    with mp.get_context("fork").Pool(cores) as pool:
        for w in range(a.warmup):
            pool.map(_cpu_worker, [(4, w * cores + i) for i in range(cores)])
        sites = 0
        t0 = time.perf_counter()
        for k in range(a.steps):
            res = pool.map(_cpu_worker, [(per, 1000 + k * cores + i) for i in range(cores)])
            sites += sum(s for s, _ in res)
        wall = time.perf_counter() - t0
    value = sites / wall
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * wall / a.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded complex-normal A, N(0,1) coefficients",
            "config": {"workload": "cfg2: O3 D=12 nu<=4 recursive DAG + c-dot, Re(phi)",
                       "sites_per_step": per * cores},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{per} sites per process x {cores} processes per step "
                                       "(oracle/acedag_oracle.py evaluate_nodes + model_sum, NumPy)"},
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


def run_ours(a):
    import torch
    import torch.distributed as dist

    import paper_2202_04140_b200 as P

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    D, nu, S = CFG["D"], CFG["nu"], a.sites
    g, c = workload(D, nu)
    census = dag_census(g)
    plan = P.SitePlan(g, local).set_coefficients(node_ids=g.target_ids, values=c)
    info = plan.info()
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    L = g.num_seeds
    A = torch.complex(torch.randn(S, L, device=dev, dtype=torch.float64, generator=gen),
                      torch.randn(S, L, device=dev, dtype=torch.float64, generator=gen)) * math.sqrt(0.5)
    out = torch.empty(S, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        plan.evaluate(A, result=out)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(a.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / a.steps
    value = world * S / (ms_step * 1e-3)

    # naive comparison path (same inputs), a few steps
    nsteps = max(3, a.steps // 10)
    plan.evaluate(A, method="naive", result=out)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(nsteps):
        plan.evaluate(A, method="naive", result=out)
    e1.record(stream)
    torch.cuda.synchronize()
    naive_ms = e0.elapsed_time(e1) / nsteps

    # end to end through the public API on pinned host buffers
    e2e = None
    if not a.no_e2e:
        Ah = A.cpu().pin_memory()
        res = torch.empty(S, dtype=torch.float64, pin_memory=True)
        for _ in range(2):
            plan.evaluate_host(Ah, result=res)
        torch.cuda.synchronize()
        barrier()
        k = max(3, a.steps // 10)
        e0.record(stream)
        for _ in range(k):
            plan.evaluate_host(Ah, result=res)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / k
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": world * S / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(Ah.numel() * 16),
               "d2h_bytes_per_step": int(S * 8), "ms_per_step": ems,
               "path": "SitePlan.evaluate_host: pinned host A -> 2-stream chunked H2D/K2/D2H"}
        del Ah

    peak = fp64_peak_tflops(dev)
    achieved = census["F_site"] * S / (ms_step * 1e-3) / 1e12
    prof = os.path.join(ROOT, "profiles", "ncu_k2_summary.json")
    traffic = None
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cores = host_cores()
        rate, n = cpu_rate(g, c, 32, cores, reps=2)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{n} sites: 2 x {cores} processes x 32 sites (oracle/acedag_oracle.py "
                         "evaluate_nodes + model_sum, NumPy, fork pool)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded complex-normal A [S,819] c128 in HBM, N(0,1) coefficient per target",
            "config": {"workload": "cfg2 (BASELINE configs[1]): O3 D=12 nu<=4, recursive DAG K2, real c, Re(phi)",
                       "sites_per_gpu": S, "global_sites": world * S, "dag_nodes": g.num_nodes,
                       "dag_products": census["P"], "targets": census["T"],
                       "plan_products": info["recursive_products"], "plan_extra_nodes": info["extra_nodes"],
                       "used_seeds": info["used_seeds"],
                       "l2": f"inputs {S * L * 16 / 1e9:.2f} GB per GPU > 126 MB L2 (no flush)",
                       "parallelism": f"dp{world} (sites sharded, no collective)"},
            "dag_products_per_s": value * census["P"],
            "naive": {"value": world * S / (naive_ms * 1e-3), "unit": UNIT, "ms_per_step": naive_ms,
                      "naive_products_per_site": info["naive_products"]},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": "measured in this run: cuBLAS DGEMM 8192^3 (MEASURED_PEAKS.json has no FP64 entry)",
                         "flops_per_site": census["F_site"],
                         "flop_model": "F_site = 6 P_int + 3 L_f + 2 T (SURVEY.md 8d)",
                         "kernel": "k2_fast (one launch per step; duration = step time)"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": a.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
