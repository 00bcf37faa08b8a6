"""Host logic of the plan compiler (csrc/plan.cpp): the DFS program that K2
walks is simulated here in NumPy and must reproduce the oracle's model sum.
CPU only -- exercises re-parenting, seed slots and warp chunking."""

import numpy as np
import pytest

import paper_2202_04140_b200 as P
from oracle import acedag_oracle as O
from paper_2202_04140_b200.program import ROW_BYTES, compile_program
from _helpers import phi_gate, seeded_A


def simulate(prog, A):
    """Walk the program exactly as k2_fast does (per chunk, preorder):
    a root is two records (two seeds; slot U is the constant ONE), every
    other record multiplies its seed into the parent value."""
    ops, slots = prog["ops"], prog["slot_label"]
    U = len(slots)
    seeds = np.concatenate([A[:, slots], np.ones((A.shape[0], 1), A.dtype)], axis=1)  # [S, U+1]
    acc = np.zeros(A.shape[0])
    pos = 0

    def seed(r):
        assert r["off"] % ROW_BYTES == 0 and r["off"] // ROW_BYTES <= U
        return seeds[:, r["off"] // ROW_BYTES]

    def visit(parent, count):
        nonlocal pos, acc
        for _ in range(count):
            r = ops[pos]
            start = pos
            pos += 1
            v = seed(r) * parent
            acc += r["c"] * v.real
            visit(v, r["nch"])
            assert r["skip"] <= r["nch"]  # leading TMEM-resident children

    chunk = prog["chunk"]
    for w in range(len(chunk) - 1):
        pos = chunk[w]
        while pos < chunk[w + 1]:
            r0, r1 = ops[pos], ops[pos + 1]
            assert r1["c"] == 0 and r1["nch"] == 0
            pos += 2
            start = pos
            v = seed(r0) * seed(r1)
            acc += r0["c"] * v.real
            visit(v, r0["nch"])
        assert pos == chunk[w + 1]
    return acc


@pytest.mark.parametrize("D,nu", [(8, 3), (12, 4), (10, 5)])
def test_program_reproduces_oracle(D, nu):
    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, D), nu)
    rng = np.random.default_rng(D * 10 + nu)
    c = rng.normal(size=len(g.target_ids))
    prog = compile_program(g, g.target_ids, c, warps=64)
    assert prog["chunk"][0] == 0 and prog["chunk"][-1] == len(prog["ops"])
    assert np.all(np.diff(prog["chunk"]) >= 0)
    A = seeded_A(6, g.num_seeds, 7)
    got = simulate(prog, A)
    re, im = O.evaluate_nodes(g.parents[:, 0], g.parents[:, 1], A)
    ref, _ = O.model_sum(re, im, g.target_ids, c)
    ok, worst = phi_gate(got, ref, O.energy_scale(re, g.target_ids, c))
    assert ok, worst
    # every reference product node is evaluated once; extras are plan-only nodes
    assert prog["recursive_products"] == (g.num_nodes - g.num_seeds) + prog["extra_nodes"]


def test_program_subset_of_coefficients():
    g = P.build_graph(P.Group.SO2, P.DegreeSpec(1, 7), 4)
    ids = g.target_ids[::3]
    c = np.linspace(-1, 1, len(ids))
    prog = compile_program(g, ids, c, warps=7)
    A = seeded_A(3, g.num_seeds, 3)
    re, im = O.evaluate_nodes(g.parents[:, 0], g.parents[:, 1], A)
    ref, _ = O.model_sum(re, im, ids, c)
    ok, worst = phi_gate(simulate(prog, A), ref, O.energy_scale(re, ids, c))
    assert ok, worst


def test_program_rejects_non_target():
    g = P.build_graph(P.Group.T, P.DegreeSpec(1, 4), 3)
    aux_id = g.id_of(((1,), (1,)))
    with pytest.raises(ValueError, match="non-target"):
        compile_program(g, [aux_id], [1.0])
