"""Golden fixtures at the BASELINE production shapes, from the REFERENCE itself.

Companion of make_golden.py (same rules: every number comes from the
unmodified reference code under /root/reference/pkg/src/acedag; runs only
where that tree is mounted; the outputs are committed).  Inputs are NOT
stored: each is regenerated bit-for-bit from its NumPy seed by the GPU tests
(tests/_helpers.py seeded_A / seeded_shells), so the fixtures stay small.

    python tests/golden/make_golden_prod.py [cfg1] [cfg2] [cfg3] [cfg4] [cfg5]

For each config the reference builds the graph (build_graph, graphbuild.py:
243-268; SHA-256 of serialize_graph recorded), pools (pool/one_particle,
evaluator.py:61-90, with the cutoff weight and radial map applied around
one_particle for the position configs, as in make_golden.positions_cfg3),
evaluates (evaluate_graph, evaluator.py:93-110) and sums c * value
sequentially in node-id order from 0j (evaluate_model, evaluator.py:141),
on the check sites only, one forked process per core.

Fixtures (prod_<cfg>.npz): S (sites the GPU test evaluates), seeds, the check
site indices, Re phi on them [n_check] or [n_check, n_out], the gate scale
sum_k |c_k Re A_k| of each, and the graph SHA-256.  prod_cfg5 also holds the
pooled A of its check sites (pool_positions4<14> is compared label by label).
"""

from __future__ import annotations

import hashlib
import math
import multiprocessing as mp
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from acedag.evaluator import evaluate_graph, one_particle  # noqa: E402
from acedag.graphbuild import build_graph, serialize_graph  # noqa: E402
from acedag.indexsets import DegreeSpec, Group, one_particle_indices  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
R_IN, R_CUT = 0.8, 5.0

# config: (D, nu, input, S on the GPU, check sites, J, n_out, input seed, coefficient seed)
PROD = {
    "cfg1": dict(D=8, nu=3, input="A", S=1_000, n_check=1000, J=0, n_out=1, seed=101, cseed=102),
    "cfg2": dict(D=12, nu=4, input="A", S=100_000, n_check=2000, J=0, n_out=1, seed=201, cseed=202),
    "cfg3": dict(D=12, nu=4, input="positions", S=20_000, n_check=1000, J=30, n_out=1, seed=301, cseed=302),
    "cfg4": dict(D=16, nu=6, input="A", S=19_000, n_check=24, J=0, n_out=1, seed=401, cseed=402),
    "cfg5": dict(D=14, nu=5, input="positions", S=6_000, n_check=24, J=40, n_out=64, seed=501, cseed=502),
}


def seeded_A(S, L, seed):
    """Same draw as tests/_helpers.seeded_A."""
    rng = np.random.default_rng(seed)
    s = np.sqrt(0.5)
    return rng.normal(0, s, (S, L)) + 1j * rng.normal(0, s, (S, L))


def seeded_shells(S, J, seed):
    """Same draw as tests/_helpers.seeded_shells: uniform in volume in the
    0.8-5.0 shell, Gaussian directions."""
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(S, J, 3))
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    r = (R_IN ** 3 + rng.uniform(size=(S, J)) * (R_CUT ** 3 - R_IN ** 3)) ** (1.0 / 3.0)
    return d * r[..., None]


def check_sites(S, n):
    """Evenly spread, always including the first and the last site."""
    return np.unique(np.linspace(0, S - 1, n).round().astype(np.int64))


def shell_pool(xyz, labels):
    """A_k = sum_j f_c(r_j) one_particle(O3, k, (x_j, theta_j, phi_j)) -- the
    reference's one_particle with the builder's radial map and cutoff."""
    parts = []
    for x, y, z in map(lambda p: map(float, p), xyz):
        rr = math.sqrt(x * x + y * y + z * z)
        xs = min(1.0, max(0.0, (rr - R_IN) / (R_CUT - R_IN)))
        th = math.acos(max(-1.0, min(1.0, z / rr)))
        ph = math.atan2(y, x)
        w = 0.5 * (1.0 + math.cos(math.pi * rr / R_CUT)) if rr < R_CUT else 0.0
        parts.append((w, (xs, th, ph)))
    out = []
    for e in labels:
        acc = 0j
        for w, c in parts:
            acc = acc + w * one_particle(Group.O3, e, c)
        out.append(acc)
    return out


_CTX = {}


def _site(args):
    """One check site: pooled dict -> evaluate_graph -> sequential sums."""
    row, = args
    g, labels, target_ids, C = _CTX["g"], _CTX["labels"], _CTX["target_ids"], _CTX["C"]
    pooled_list = shell_pool(row, labels) if _CTX["positions"] else [complex(v) for v in row]
    pooled = dict(zip(labels, pooled_list))
    vals = evaluate_graph(g, pooled)
    n_out = C.shape[1]
    phi = np.zeros(n_out)
    scale = np.zeros(n_out)
    for o in range(n_out):
        acc = 0j
        sc = 0.0
        for i, c in zip(target_ids, C[:, o].tolist()):
            v = vals[i]
            acc = acc + c * v
            sc += abs(c * v.real)
        phi[o] = acc.real
        scale[o] = sc
    return phi, scale, np.array(pooled_list, np.complex128)


def make(name):
    p = PROD[name]
    t0 = time.time()
    g = build_graph(Group.O3, DegreeSpec(1, p["D"]), p["nu"])
    sha = hashlib.sha256(serialize_graph(g)).hexdigest()
    print(name, "graph", len(g.nodes), sha[:16], f"{time.time() - t0:.0f}s", flush=True)
    labels = one_particle_indices(Group.O3, p["D"])
    target_ids = [n.id for n in g.nodes if not n.auxiliary and g.is_target(n.elements)]
    rng = np.random.default_rng(p["cseed"])
    C = rng.normal(size=(len(target_ids), p["n_out"]))
    idx = check_sites(p["S"], p["n_check"])
    if p["input"] == "A":
        rows = seeded_A(p["S"], len(labels), p["seed"])[idx]
    else:
        rows = seeded_shells(p["S"], p["J"], p["seed"])[idx]
    _CTX.update(g=g, labels=labels, target_ids=target_ids, C=C, positions=p["input"] == "positions")
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        res = pool.map(_site, [(r,) for r in rows], chunksize=1)
    phi = np.array([r[0] for r in res])
    scale = np.array([r[1] for r in res])
    if p["n_out"] == 1:
        phi, scale = phi[:, 0], scale[:, 0]
    extra = {}
    if name == "cfg5":
        extra["A_check"] = np.array([r[2] for r in res])
    np.savez_compressed(os.path.join(HERE, f"prod_{name}.npz"), S=np.array(p["S"]), seed=np.array(p["seed"]),
                        cseed=np.array(p["cseed"]), J=np.array(p["J"]), n_out=np.array(p["n_out"]),
                        D=np.array(p["D"]), nu=np.array(p["nu"]), sites=idx, phi=phi, scale=scale,
                        sha256=np.array(sha), n_targets=np.array(len(target_ids)), **extra)
    print(name, "done", len(idx), "sites", f"{time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:] or list(PROD):
        make(name)
