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
    """Walk the program in the kernels' order (per chunk, preorder):
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


# --------------------------------------------------------------- k2_horner
def simulate_horner(h, A):
    """Walk copy 0 of the k2_horner program exactly as the kernel does (per
    chunk: croots roots; children by seed class hot / shared / global from
    the counts in w; H_u = c_u + sum_children s_q H_q; phi = Re(s_a s_b H))."""
    from paper_2202_04140_b200.program import HORNER_MAX_LEAVES
    ops, slots, hot, us = h["ops"][0], h["slot_label"], h["hot"], h["us"]
    nu = simulate_horner.nu
    seeds = A[:, slots]  # [S, U]

    def seed(z, cls):
        if cls == 0:
            assert z % 16 == 0 and z // 16 < hot
            return seeds[:, z // 16]
        assert z % 2048 == 0
        s = hot + z // 2048 + (us if cls == 2 else 0)
        assert (cls == 1 and s < hot + us) or (cls == 2 and s >= hot + us)
        return seeds[:, s]

    def leaf_cls(j, w):  # last inner order: byte ends hot | shared << 10 | all << 20
        return 0 if 16 * j < (w & 1023) else (1 if 16 * j < ((w >> 10) & 1023) else 2)

    pos = 0

    def leaves(w, H):
        nonlocal pos
        n = (w >> 20) // 16
        assert (w >> 20) % 16 == 0 and n <= HORNER_MAX_LEAVES
        for j in range(n):
            r = ops[pos]
            pos += 1
            assert r["w"] == 0
            H = H + r["c"] * seed(r["z"], leaf_cls(j, w))
        return H

    def children(w, D, Hp, counts=None):
        nonlocal pos
        if counts is None:  # inner record: nch | nhot << 15 | nsm << 22
            nh, ns = (w >> 15) & 127, w >> 22
            counts = (nh, ns, (w & 0x7FFF) - nh - ns)
        for c, n in enumerate(counts):
            for _ in range(n):
                r = ops[pos]
                pos += 1
                H = np.full(A.shape[0], r["c"], complex)
                H = leaves(r["w"], H) if D == nu - 1 else children(r["w"], D + 1, H)
                Hp = Hp + seed(r["z"], c) * H
        return Hp

    def root4_counts(r0, r1):
        """Order-4 roots: the children are sorted by seed class and, inside a
        class, into S1 (one hot leaf), S2 (two hot leaves) and general runs;
        r0.w = general runs (10 bits per class), r1.c bits = S1 | S2 << 16 of
        the hot (low word) / shared (high word) classes, r1.w >> 8 = S1 | S2 << 12
        of the global class.  Returns (per-class totals, S1/S2 runs)."""
        wg, fl = int(r0["w"]), int(r1["w"])
        bits = int(np.array([r1["c"]], "<f8").view("<u8")[0])
        wh, ws = bits & 0xFFFFFFFF, bits >> 32
        runs = [(wh & 0xFFFF, wh >> 16), (ws & 0xFFFF, ws >> 16), ((fl >> 8) & 0xFFF, fl >> 20)]
        gen = [wg & 1023, (wg >> 10) & 1023, wg >> 20]
        return tuple(a + b + g for (a, b), g in zip(runs, gen)), runs

    phi = np.zeros(A.shape[0])
    chunk, croots = h["chunk"], h["croots"]
    for ci in range(len(croots)):
        pos = chunk[ci]
        for _ in range(croots[ci]):
            r0, r1 = ops[pos], ops[pos + 1]
            pos += 2
            fl = int(r1["w"])
            H = np.full(A.shape[0], r0["c"], complex)
            if nu == 3:
                H = leaves(int(r0["w"]), H)
            elif nu == 4 and not fl & 16:
                counts, runs = root4_counts(r0, r1)
                p0 = pos
                H = children(0, 3, H, counts)
                # the S1 / S2 runs really are one- / two-hot-leaf nodes, in that order per class
                q = p0
                for c, n in enumerate(counts):
                    for j in range(n):
                        w = int(ops[q]["w"])
                        if j < runs[c][0]:
                            assert w == (16 | 16 << 10 | 16 << 20)
                        elif j < runs[c][0] + runs[c][1]:
                            assert w == (32 | 32 << 10 | 32 << 20)
                        q += 1 + (w >> 20) // 16
                assert q == pos
            elif nu > 4:
                H = children(int(r0["w"]), 3, H)
            sa = seed(r0["z"], fl & 3)
            phi = phi + (r0["c"] * sa.real if fl & 16 else (sa * seed(r1["z"], (fl >> 2) & 3) * H).real)
        assert pos == chunk[ci + 1]
    return phi


@pytest.mark.parametrize("D,nu,hot,us", [(8, 3, 32, 97), (10, 4, 32, 97), (12, 4, 32, 97), (12, 4, 8, 20),
                                         (12, 3, 4, 6), (6, 2, 32, 0), (9, 5, 16, 40), (14, 4, 32, 97)])
def test_horner_program_reproduces_oracle(D, nu, hot, us):
    """The k2_horner encoding (class-sorted children, class-scaled seed
    offsets, nodes with more than 30 leaves split into copies, per-quadrant
    copies) evaluated bottom-up on the CPU equals the oracle's model sum;
    small hot / shared budgets exercise all three seed classes."""
    from paper_2202_04140_b200.program import compile_horner
    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, D), nu)
    c = np.random.default_rng(D + nu).normal(size=len(g.target_ids))
    h = compile_horner(g, g.target_ids, c, warps=32, hot=hot, us=us)
    ops = h["ops"]
    # copies differ only in the lane-quadrant bits of TMEM (class 0) offsets
    for q in range(1, 4):
        d = ops[q]["z"].astype(np.int64) - ops[0]["z"].astype(np.int64)
        assert set(np.unique(d)) <= {0, q << 21}
        assert np.array_equal(ops[q]["c"], ops[0]["c"]) and np.array_equal(ops[q]["w"], ops[0]["w"])
    A = seeded_A(5, g.num_seeds, 11)
    simulate_horner.nu = max(2, g.max_order)
    phi = simulate_horner(h, A)
    re, im = O.evaluate_nodes(g.parents[:, 0], g.parents[:, 1], A)
    ref, _ = O.model_sum(re, im, g.target_ids, c)
    ok, worst = phi_gate(phi, ref, O.energy_scale(re, g.target_ids, c))
    assert ok, worst
