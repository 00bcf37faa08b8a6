"""Host logic of the plan compiler (csrc/plan.cpp): the DFS program that K2
walks is simulated here in NumPy and must reproduce the oracle's model sum.
CPU only -- exercises re-parenting, seed slots and warp chunking."""

import numpy as np
import pytest

import paper_2202_04140_b200 as P
from oracle import acedag_oracle as O
from paper_2202_04140_b200.program import SINGLE, compile_program
from _helpers import phi_gate, seeded_A


def simulate(prog, A, n_out=1):
    """Walk the program exactly as k2_fast does (per chunk, preorder)."""
    ops, slots = prog["ops"], prog["slot_label"]
    seeds = A[:, slots]  # [S, U]
    acc = np.zeros(A.shape[0], np.complex128)
    pos = 0

    def visit(parent, count):
        nonlocal pos, acc
        for _ in range(count):
            r = ops[pos]
            pos += 1
            v = seeds[:, r["sa"]] * parent
            acc += r["c"] * v.real
            visit(v, r["nch"])

    chunk = prog["chunk"]
    for w in range(len(chunk) - 1):
        pos = chunk[w]
        while pos < chunk[w + 1]:
            r = ops[pos]
            pos += 1
            v = seeds[:, r["sa"]] if r["sb"] == SINGLE else seeds[:, r["sa"]] * seeds[:, r["sb"]]
            acc += r["c"] * v.real
            visit(v, r["nch"])
        assert pos == chunk[w + 1]
    return acc.real


@pytest.mark.parametrize("D,nu", [(8, 3), (12, 4), (10, 5)])
def test_program_reproduces_oracle(D, nu):
    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, D), nu)
    rng = np.random.default_rng(D * 10 + nu)
    c = rng.normal(size=len(g.target_ids))
    prog = compile_program(g, g.target_ids, c, warps=32)
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
