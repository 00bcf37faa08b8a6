"""Generate the golden fixtures in tests/golden from the REFERENCE itself.

Runs only where the read-only reference is mounted (/root/reference); the
outputs are committed so the GPU box (which has no reference) can check
against them.  Every number below comes from the unmodified reference code
(/root/reference/pkg/src/acedag): build_graph/serialize_graph, pool,
one_particle, evaluate_graph, naive_eval and the evaluate_model sum order.

    python tests/golden/make_golden.py

Fixtures:
  graph_hashes.json   SHA-256 + counts of serialize_graph(build_graph(...))
  pool_golden.npz     pool() per group on seeded random_particles configs
  eval_cfg1.npz       cfg1 (O3 D=8 nu=3): A, node values, coefficients, phi
  eval_cfg2.npz       cfg2 (O3 D=12 nu=4): A, coefficients, phi (4 sites)
  positions_cfg3.npz  cfg3 pool from Cartesian shells (cutoff applied around
                      the reference's one_particle), 3 sites x 30 neighbours
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from acedag.evaluator import evaluate_graph, naive_eval, one_particle, pool, random_particles  # noqa: E402
from acedag.graphbuild import build_graph, serialize_graph  # noqa: E402
from acedag.indexsets import DegreeSpec, Group, one_particle_indices  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# BASELINE cfg4 (D=16, nu=6) takes 6-8 minutes in the reference; its hash is
# the one the survey recorded from two independent reference builds
# and is listed separately, not regenerated here.
CFG4 = {"group": "O3", "p": 1, "D": 16, "nu": 6, "alg": "orig", "n": 1, "bytes": 201068448,
        "sha256": "bcc01406b9d7172f0b9601986ad7ae553aa2b1a44d0c9f1fddc2eab3ff1ec3a1",
        "nodes": 3711466, "targets": 3698926, "aux": 10836, "source": "SURVEY.md 8c"}


def _counts(g):
    targets = sum(1 for n in g.nodes if not n.auxiliary and g.is_target(n.elements))
    return len(g.nodes), targets, sum(n.auxiliary for n in g.nodes)


def graph_hashes():
    builds = []
    for grp in ("T", "SO2", "O3", "O3F"):
        for p in (1, 2, math.inf):
            for D, nu in ((4, 3), (5, 3), (6, 4), (3.5, 3)):
                if p != 1 and D > 5:
                    continue
                for alg, n in (("orig", 1), ("gen", 2), ("gen", 3)):
                    builds.append((grp, p, D, nu, alg, n))
    builds += [("T", 1, 10, 5, "orig", 1), ("T", 1, 12, 4, "orig", 1), ("SO2", 1, 8, 4, "gen", 2),
               ("O3", 1, 8, 3, "orig", 1), ("O3", 1, 12, 4, "orig", 1), ("O3", 1, 10, 5, "orig", 1),
               ("O3", 1, 14, 5, "orig", 1), ("O3", 1, 10, 5, "gen", 2), ("O3F", 1, 6, 4, "orig", 1)]
    out = []
    for grp, p, D, nu, alg, n in builds:
        g = build_graph(Group(grp), DegreeSpec(p, D), nu, alg, n)
        s = serialize_graph(g)
        nodes, targets, aux = _counts(g)
        out.append({"group": grp, "p": "inf" if p == math.inf else p, "D": D, "nu": nu, "alg": alg, "n": n,
                    "bytes": len(s), "sha256": hashlib.sha256(s).hexdigest(), "nodes": nodes,
                    "targets": targets, "aux": aux, "source": "reference"})
        print("graph", grp, p, D, nu, alg, n, nodes, flush=True)
    out.append(CFG4)
    with open(os.path.join(HERE, "graph_hashes.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def pool_golden():
    data = {}
    rng = random.Random(2024)
    for grp, cap in (("T", 5), ("SO2", 5), ("O3", 6), ("O3F", 4)):
        group = Group(grp)
        confs = [random_particles(group, rng) for _ in range(6)]
        nc = group.components
        J = max(len(c) for c in confs)
        coords = np.zeros((len(confs), J, nc))
        counts = np.zeros(len(confs), np.int32)
        labels = one_particle_indices(group, cap)
        A = np.zeros((len(confs), len(labels)), np.complex128)
        for s, conf in enumerate(confs):
            counts[s] = len(conf)
            coords[s, : len(conf)] = conf
            pooled = pool(group, DegreeSpec(1, cap), conf)
            A[s] = [pooled[e] for e in labels]
        data[f"{grp}_coords"] = coords
        data[f"{grp}_counts"] = counts
        data[f"{grp}_cap"] = np.array(cap)
        data[f"{grp}_A"] = A
    np.savez_compressed(os.path.join(HERE, "pool_golden.npz"), **data)


def _seeded_A(S, L, seed):
    rng = np.random.default_rng(seed)
    return (rng.normal(0, math.sqrt(0.5), (S, L)) + 1j * rng.normal(0, math.sqrt(0.5), (S, L)))


def _model(g, A, c_by_target, target_ids):
    """evaluate_graph + sequential sum from 0j in coefficient (node-id) order."""
    labels = one_particle_indices(g.group, g.spec.int_cap())
    vals_all, phi = [], []
    for s in range(A.shape[0]):
        pooled = {e: complex(A[s, i]) for i, e in enumerate(labels)}
        vals = evaluate_graph(g, pooled)
        acc = 0j
        for i, c in zip(target_ids, c_by_target):
            acc = acc + c * vals[i]
        vals_all.append(vals)
        phi.append(acc)
    return np.array(vals_all, np.complex128), np.array(phi, np.complex128)


def eval_cfg1():
    g = build_graph(Group.O3, DegreeSpec(1, 8), 3)
    target_ids = [n.id for n in g.nodes if not n.auxiliary and g.is_target(n.elements)]
    A = _seeded_A(8, len(one_particle_indices(Group.O3, 8)), 11)
    c = np.random.default_rng(12).normal(0, 1, len(target_ids))
    vals, phi = _model(g, A, [float(x) for x in c], target_ids)
    # naive products of the targets on site 0 (naive_eval, evaluator.py:113-121)
    labels = one_particle_indices(Group.O3, 8)
    pooled0 = {e: complex(A[0, i]) for i, e in enumerate(labels)}
    naive0 = np.array([naive_eval(g.nodes[i].elements, pooled0) for i in target_ids])
    np.savez_compressed(os.path.join(HERE, "eval_cfg1.npz"), A=A, coef=c, target_ids=np.array(target_ids),
                        node_values=vals, phi=phi, naive_site0=naive0)


def eval_cfg2():
    g = build_graph(Group.O3, DegreeSpec(1, 12), 4)
    target_ids = [n.id for n in g.nodes if not n.auxiliary and g.is_target(n.elements)]
    A = _seeded_A(4, len(one_particle_indices(Group.O3, 12)), 21)
    c = np.random.default_rng(22).normal(0, 1, len(target_ids))
    vals, phi = _model(g, A, [float(x) for x in c], target_ids)
    scale = np.abs(c[None, :] * vals[:, target_ids].real).sum(axis=1)
    np.savez_compressed(os.path.join(HERE, "eval_cfg2.npz"), A=A, coef=c, target_ids=np.array(target_ids),
                        phi=phi, scale=scale)


def positions_cfg3():
    """A_k = sum_j f_c(r_j) one_particle(O3, k, (x_j, theta_j, phi_j))."""
    r_in, r_cut = 0.8, 5.0
    rng = np.random.default_rng(31)
    S, J, cap = 3, 30, 12
    d = rng.normal(size=(S, J, 3))
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    r = (r_in ** 3 + rng.uniform(size=(S, J)) * (r_cut ** 3 - r_in ** 3)) ** (1.0 / 3.0)
    xyz = d * r[..., None]
    labels = one_particle_indices(Group.O3, cap)
    A = np.zeros((S, len(labels)), np.complex128)
    for s in range(S):
        parts = []
        for j in range(J):
            x, y, z = map(float, xyz[s, j])
            rr = math.sqrt(x * x + y * y + z * z)
            xs = min(1.0, max(0.0, (rr - r_in) / (r_cut - r_in)))
            th = math.acos(max(-1.0, min(1.0, z / rr)))
            ph = math.atan2(y, x)
            w = 0.5 * (1.0 + math.cos(math.pi * rr / r_cut)) if rr < r_cut else 0.0
            parts.append((w, (xs, th, ph)))
        for k, e in enumerate(labels):
            acc = 0j
            for w, c in parts:
                acc = acc + w * one_particle(Group.O3, e, c)
            A[s, k] = acc
    np.savez_compressed(os.path.join(HERE, "positions_cfg3.npz"), xyz=xyz, A=A, cap=np.array(cap),
                        r_in=np.array(r_in), r_cut=np.array(r_cut))


if __name__ == "__main__":
    which = sys.argv[1:] or ["graphs", "pool", "cfg1", "cfg2", "cfg3"]
    if "graphs" in which:
        graph_hashes()
    if "pool" in which:
        pool_golden()
    if "cfg1" in which:
        eval_cfg1()
    if "cfg2" in which:
        eval_cfg2()
    if "cfg3" in which:
        positions_cfg3()
    print("done")
