"""Parity at the BASELINE production shapes, through the C ABI, against
fixtures the REFERENCE produced (tests/golden/make_golden_prod.py).

Each test regenerates the config's inputs from their NumPy seed, evaluates
the full batch on the GPU with the kernel the bench runs at that shape (the
kernel name is asserted), and gates the reference's check sites with the
SURVEY.md 8d criterion |phi_gpu - phi_ref| <= tol * sum_k |c_k Re A_k|
(fp64: 1e-11; fp32 mode: 1e-5).  The native graph's SHA-256 must equal the
reference build's.

    cfg2  D=12 nu=4, 100,000 sites, 2,000 checked   (k2_horner; naive; fp32)
    cfg3  D=12 nu=4 from J=30 shells, 20,000 sites, 1,000 checked
                                                     (pool_positions4<12> + k2_horner)
    cfg4  D=16 nu=6, 19,000 sites, 24 checked        (k2_quad<6>; fp32 k2_horner<6>)
    cfg5  D=14 nu=5 from J=40 shells, 64 outputs, 6,000 sites, 24 checked
                                                     (pool_positions4<14> vs the
                                                      reference pool; k2_mma<5>)
"""

import hashlib

import numpy as np
import pytest
import torch

import paper_2202_04140_b200 as P
from _helpers import phi_gate, seeded_A, seeded_shells

pytestmark = pytest.mark.gpu


def _setup(golden, name):
    d = golden(f"prod_{name}.npz")
    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, int(d["D"])), int(d["nu"]))
    assert hashlib.sha256(P.serialize_graph(g)).hexdigest() == str(d["sha256"])
    assert len(g.target_ids) == int(d["n_targets"])
    n_out = int(d["n_out"])
    C = np.random.default_rng(int(d["cseed"])).normal(size=(len(g.target_ids), n_out))
    plan = P.SitePlan(g).set_coefficients(node_ids=g.target_ids, values=C[:, 0] if n_out == 1 else C)
    return d, g, plan


def _gate(got, d, tol=1e-11):
    ok, worst = phi_gate(got, d["phi"], d["scale"], tol=tol)
    assert ok, worst
    return worst


def test_cfg2_bench_shape(cuda, golden):
    d, g, plan = _setup(golden, "cfg2")
    S, idx = int(d["S"]), d["sites"]
    assert len(idx) >= 2000
    assert plan.kernel_name(sites=S) == "k2_horner"
    A = torch.from_numpy(seeded_A(S, g.num_seeds, int(d["seed"]))).to(cuda)
    _gate(plan.evaluate(A).cpu().numpy()[idx], d)
    _gate(plan.evaluate(A, method="naive").cpu().numpy()[idx], d)
    assert plan.kernel_name(prec="f32", sites=S) == "k2_horner (fp32)"
    _gate(plan.evaluate(A.to(torch.complex64)).cpu().numpy()[idx], d, tol=1e-5)


def test_cfg3_bench_shape_from_positions(cuda, golden):
    d, g, plan = _setup(golden, "cfg3")
    S, idx = int(d["S"]), d["sites"]
    assert len(idx) >= 1000
    xyz = torch.from_numpy(seeded_shells(S, int(d["J"]), int(d["seed"]))).to(cuda)
    _gate(plan.evaluate_positions(xyz).cpu().numpy()[idx], d)


def test_cfg4_bench_shape_k2_quad(cuda, golden):
    d, g, plan = _setup(golden, "cfg4")
    S, idx = int(d["S"]), d["sites"]
    assert len(idx) >= 20 and S >= 148 * 128
    assert plan.kernel_name(sites=S) == "k2_quad"
    A = torch.from_numpy(seeded_A(S, g.num_seeds, int(d["seed"]))).to(cuda)
    full = plan.evaluate(A)
    _gate(full.cpu().numpy()[idx], d)
    # the same sites in a small batch: the order 5-6 kernel does not depend on S
    sub = torch.from_numpy(idx).to(cuda)
    assert torch.equal(plan.evaluate(A[sub].contiguous()), full[sub])
    assert plan.kernel_name(prec="f32", sites=S) == "k2_horner (fp32)"
    _gate(plan.evaluate(A.to(torch.complex64)).cpu().numpy()[idx], d, tol=1e-5)


def test_cfg5_bench_shape_pool_and_k2_mma(cuda, golden):
    d, g, plan = _setup(golden, "cfg5")
    S, idx = int(d["S"]), d["sites"]
    n_out = int(d["n_out"])
    assert len(idx) >= 20 and n_out == 64
    assert plan.kernel_name(sites=S) == "k2_mma"
    xyz_np = seeded_shells(S, int(d["J"]), int(d["seed"]))
    # pool_positions4<14> (J = 40) on the check sites vs the reference's pool
    A = P.pool_positions(14, torch.from_numpy(xyz_np[idx]).to(cuda)).cpu().numpy()
    ref = d["A_check"]
    assert A.shape == ref.shape
    assert np.all(np.abs(A - ref) <= 1e-12 * (1 + np.abs(ref)))
    got = plan.evaluate_positions(torch.from_numpy(xyz_np).to(cuda)).cpu().numpy()
    assert got.shape == (S, n_out)
    _gate(got[idx], d)


def test_cfg1_every_site(cuda, golden):
    """BASELINE configs[0]: all 1,000 sites against the reference, recursive
    and naive (cfg1 all sites)."""
    d, g, plan = _setup(golden, "cfg1")
    S, idx = int(d["S"]), d["sites"]
    assert len(idx) == S == 1000
    A = torch.from_numpy(seeded_A(S, g.num_seeds, int(d["seed"]))).to(cuda)
    _gate(plan.evaluate(A).cpu().numpy()[idx], d)
    _gate(plan.evaluate(A, method="naive").cpu().numpy()[idx], d)
    _gate(plan.evaluate(A.to(torch.complex64)).cpu().numpy()[idx], d, tol=1e-5)
