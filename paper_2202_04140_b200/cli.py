"""Command line for the evaluation path: the callers of the hot path that the
reference's `acedag` CLI exposes (/root/reference/pkg/src/acedag/cli.py),
backed by the native builder and the CUDA kernels.

    python -m paper_2202_04140_b200 build  --group O3 --D 8 --numax 3 --out g.txt
    python -m paper_2202_04140_b200 eval   --graph g.txt --config conf.txt [--coeffs c.txt] [--real-part]
    python -m paper_2202_04140_b200 verify --suite oracle|invariance|all [--group O3 --D 6 --numax 4]
    python -m paper_2202_04140_b200 sites  --graph g.txt --sites 100000    # batched throughput probe

`build` writes the reference's versioned graph format byte for byte
(graphbuild.py:355-384); `eval` prints what `acedag eval` prints
(cli.py:213-236) -- node values are bit-identical; `verify` runs the oracle
(cli.py:261-279) and invariance (cli.py:282-311) suites on the GPU.  Errors
exit 1 with `error: ...` like the reference (cli.py:351-357).
"""

from __future__ import annotations

import argparse
import contextlib
import math
import random
import sys
import time

from .graph import build_graph, read_graph, write_graph
from .indexsets import DegreeSpec, Group, format_elements


def _p(text: str):
    return math.inf if text == "inf" else int(text)


@contextlib.contextmanager
def _out(path):
    if path is None:
        yield sys.stdout
    else:
        with open(path, "w", encoding="utf-8", newline="\n") as fh:
            yield fh


def cmd_build(a) -> int:
    t0 = time.perf_counter()
    g = build_graph(Group(a.group), DegreeSpec(_p(a.p), a.D), a.numax, a.alg, a.n)
    write_graph(g, a.out)
    print(f"built {g.num_nodes} nodes ({g.num_targets} targets, {g.num_aux} auxiliary) "
          f"in {time.perf_counter() - t0:.2f}s -> {a.out}", file=sys.stderr)
    return 0


def cmd_eval(a) -> int:
    from .evaluator import evaluate_graph, evaluate_model, pool, read_coefficients, read_particles
    g = read_graph(a.graph)
    group, particles = read_particles(a.config)
    if group is not g.group:
        raise ValueError(f"configuration group {group.value} does not match graph group {g.group.value}")
    with _out(a.out) as out:
        if a.coeffs is not None:
            value = evaluate_model(g, read_coefficients(a.coeffs, group), particles, real_part=a.real_part)
            out.write(f"{value!r}\n" if a.real_part else f"{value.real!r} {value.imag!r}\n")
        else:
            values = evaluate_graph(g, pool(group, g.spec, particles))
            for i in range(g.num_nodes):
                v = values[i]
                out.write(f"{i} {int(g.aux[i])} {format_elements(g.elements_of(i))} {v.real!r} {v.imag!r}\n")
    return 0


def _suite_oracle(a):
    """Every node of orig and gen(2) graphs vs the direct product, on GPU."""
    import numpy as np
    import torch

    from .evaluator import naive_products, pool_batched, random_particles
    group = Group(a.group or "T")
    spec = DegreeSpec(_p(a.p), a.D)
    rng = random.Random(a.seed)
    worst = 0.0
    nc = group.components
    for alg, n in (("orig", 1), ("gen", 2)):
        g = build_graph(group, spec, a.numax, alg, n)
        confs = [random_particles(group, rng) for _ in range(a.configs)]
        J = max(len(c) for c in confs)
        coords = np.zeros((len(confs), J, nc))
        counts = np.array([len(c) for c in confs], np.int32)
        for s, c in enumerate(confs):
            coords[s, : len(c)] = c
        dev = torch.device("cuda", torch.cuda.current_device())
        A = pool_batched(group, spec.int_cap(), torch.from_numpy(coords).to(dev), torch.from_numpy(counts).to(dev))
        vals = g.plan().evaluate_nodes(A)                     # [S, N]
        idx = np.zeros((g.num_nodes, g.max_order), np.int64)
        lens = np.zeros(g.num_nodes, np.int32)
        index = {e: i for i, e in enumerate(g.labels)}
        for k in range(g.num_nodes):
            ids = [index[e] for e in g.elements_of(k)]
            idx[k, : len(ids)] = ids
            lens[k] = len(ids)
        rows = A[:, torch.from_numpy(idx).to(dev)].reshape(-1, g.max_order).contiguous()
        ref = naive_products(rows, torch.from_numpy(np.tile(lens, A.shape[0])).to(dev)).reshape(vals.shape)
        worst = max(worst, float(((vals - ref).abs() / (1.0 + ref.abs())).max().item()))
    return worst <= 1e-12, f"group={group.value} worst deviation {worst:.3e} (tolerance 1e-12)"


def _suite_invariance(a):
    from .evaluator import invariance_check, naive_eval, pool, random_particles, rotate_particles
    group = Group(a.group or "T")
    spec = DegreeSpec(_p(a.p), a.D)
    g = build_graph(group, spec, a.numax, a.alg, a.n)
    rng = random.Random(a.seed)
    worst = 0.0
    for _ in range(a.configs):
        rep = invariance_check(group, g, random_particles(group, rng), trials=a.trials, seed=rng.randrange(2 ** 32))
        worst = max(worst, rep.rotation_max_dev, rep.inversion_max_dev or 0.0)
    # negative control: a non-invariant pair picks up e^{2 i alpha}
    pair = {Group.T: ((1,), (1,)), Group.SO2: ((0, 1), (0, 1)), Group.O3: ((0, 1, 1), (0, 1, 1)),
            Group.O3F: ((0, 1, 1, 0), (0, 1, 1, 0))}[group]
    base = {Group.T: (0.0,), Group.SO2: (0.9, 0.0), Group.O3: (0.9, 1.0, 0.0),
            Group.O3F: (0.9, 1.0, 0.0, 0.5)}[group]
    parts = [rotate_particles(group, [base], 0.4 * j)[0] for j in range(3)]
    before = naive_eval(pair, pool(group, spec, parts))
    after = naive_eval(pair, pool(group, spec, rotate_particles(group, parts, math.pi / 2)))
    control = abs(after - before) / (1.0 + abs(before))
    ok = worst <= 1e-10 and control > 1e-2
    return ok, (f"group={group.value} worst invariant deviation {worst:.3e} (tolerance 1e-10), "
                f"negative control {control:.3e} (must exceed 1e-2)")


_SUITES = {"oracle": _suite_oracle, "invariance": _suite_invariance}


def cmd_verify(a) -> int:
    names = list(_SUITES) if a.suite == "all" else [a.suite]
    failed = False
    for name in names:
        ok, detail = _SUITES[name](a)
        print(f"{'PASS' if ok else 'FAIL'} {name}: {detail}")
        failed |= not ok
    return 1 if failed else 0


def cmd_sites(a) -> int:
    """Batched throughput probe: recursive and naive kernels on S random sites."""
    import numpy as np
    import torch

    from .evaluator import SitePlan
    g = read_graph(a.graph)
    dev = torch.device("cuda", torch.cuda.current_device())
    gen = torch.Generator(device=dev).manual_seed(a.seed)
    A = torch.complex(torch.randn(a.sites, g.num_seeds, dtype=torch.float64, device=dev, generator=gen),
                      torch.randn(a.sites, g.num_seeds, dtype=torch.float64, device=dev, generator=gen))
    c = np.random.default_rng(a.seed).normal(size=len(g.target_ids))
    plan = SitePlan(g).set_coefficients(node_ids=g.target_ids, values=c)
    for method in ("recursive", "naive"):
        plan.evaluate(A, method=method)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            plan.evaluate(A, method=method)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        print(f"{method:9s} {a.sites / (ms * 1e-3):.4g} sites/s ({ms:.3f} ms per {a.sites} sites)")
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2202_04140_b200")
    sub = ap.add_subparsers(dest="command", required=True)
    groups = [g.value for g in Group]

    p = sub.add_parser("build", help="build an evaluation graph file (native)")
    p.add_argument("--group", choices=groups, required=True)
    p.add_argument("--p", choices=["1", "2", "inf"], default="1")
    p.add_argument("--D", type=float, required=True)
    p.add_argument("--numax", type=int, required=True)
    p.add_argument("--alg", choices=["orig", "gen"], default="orig")
    p.add_argument("--n", type=int, default=1)
    p.add_argument("--out", required=True)

    p = sub.add_parser("eval", help="evaluate a graph on a particle configuration (GPU)")
    p.add_argument("--graph", required=True)
    p.add_argument("--config", required=True)
    p.add_argument("--coeffs", default=None)
    p.add_argument("--real-part", action="store_true")
    p.add_argument("--out", default=None)

    p = sub.add_parser("verify", help="GPU verification suites")
    p.add_argument("--suite", choices=["oracle", "invariance", "all"], required=True)
    p.add_argument("--group", choices=groups, default=None)
    p.add_argument("--p", choices=["1", "2", "inf"], default="1")
    p.add_argument("--D", type=float, default=8)
    p.add_argument("--numax", type=int, default=4)
    p.add_argument("--alg", choices=["orig", "gen"], default="orig")
    p.add_argument("--n", type=int, default=1)
    p.add_argument("--configs", type=int, default=10)
    p.add_argument("--trials", type=int, default=5)
    p.add_argument("--seed", type=int, default=0)

    p = sub.add_parser("sites", help="batched throughput probe on random sites (GPU)")
    p.add_argument("--graph", required=True)
    p.add_argument("--sites", type=int, default=100_000)
    p.add_argument("--reps", type=int, default=10)
    p.add_argument("--seed", type=int, default=0)
    return ap


_COMMANDS = {"build": cmd_build, "eval": cmd_eval, "verify": cmd_verify, "sites": cmd_sites}


def main(argv=None) -> int:
    a = build_parser().parse_args(argv)
    try:
        return _COMMANDS[a.command](a)
    except (OSError, ValueError, KeyError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
