"""CUDA path vs the oracle / the reference's golden vectors, through the C ABI.

Gates:
  * node values (acedag_eval_nodes): bit-identical to evaluate_graph;
  * fp64 phi: |phi_gpu - phi_ref| <= 1e-11 * sum_k |c_k Re A_k| per site;
  * fp32 mode: same normalisation with 1e-5;
  * naive_eval rows: bit-identical.
"""

import math

import numpy as np
import pytest
import torch

import paper_2202_04140_b200 as P
from _helpers import phi_gate, seeded_A
from oracle import acedag_oracle as O

pytestmark = pytest.mark.gpu


def _oracle_phi(g, A, ids, c):
    re, im = O.evaluate_nodes(g.parents[:, 0], g.parents[:, 1], A)
    pr, pi = O.model_sum(re, im, ids, c)
    return pr, pi, O.energy_scale(re, ids, c)


@pytest.fixture(scope="module")
def cfg1():
    return P.build_graph(P.Group.O3, P.DegreeSpec(1, 8), 3)


@pytest.fixture(scope="module")
def cfg2():
    return P.build_graph(P.Group.O3, P.DegreeSpec(1, 12), 4)


def test_eval_nodes_bit_exact_vs_reference_cfg1(cuda, golden, cfg1):
    d = golden("eval_cfg1.npz")
    A = torch.from_numpy(d["A"]).to(cuda)
    vals = cfg1.plan().evaluate_nodes(A).cpu().numpy()
    assert np.array_equal(vals.view(np.float64), d["node_values"].view(np.float64))


@pytest.mark.parametrize("method", ["recursive", "naive"])
def test_phi_vs_reference_golden_cfg1(cuda, golden, cfg1, method):
    d = golden("eval_cfg1.npz")
    plan = P.SitePlan(cfg1).set_coefficients(node_ids=d["target_ids"], values=d["coef"])
    phi = plan.evaluate(torch.from_numpy(d["A"]).to(cuda), method=method).cpu().numpy()
    re, im = O.evaluate_nodes(cfg1.parents[:, 0], cfg1.parents[:, 1], d["A"])
    ok, worst = phi_gate(phi, d["phi"].real, O.energy_scale(re, d["target_ids"], d["coef"]))
    assert ok, worst


@pytest.mark.parametrize("method", ["recursive", "naive"])
def test_phi_vs_reference_golden_cfg2(cuda, golden, cfg2, method):
    d = golden("eval_cfg2.npz")
    plan = P.SitePlan(cfg2).set_coefficients(node_ids=d["target_ids"], values=d["coef"])
    phi = plan.evaluate(torch.from_numpy(d["A"]).to(cuda), method=method).cpu().numpy()
    ok, worst = phi_gate(phi, d["phi"].real, d["scale"])
    assert ok, worst


def test_phi_cfg2_subsample_vs_oracle(cuda, cfg2):
    S = 96
    A = seeded_A(S, cfg2.num_seeds, 5)
    c = np.random.default_rng(6).normal(size=len(cfg2.target_ids))
    pr, _, scale = _oracle_phi(cfg2, A, cfg2.target_ids, c)
    plan = P.SitePlan(cfg2).set_coefficients(node_ids=cfg2.target_ids, values=c)
    At = torch.from_numpy(A).to(cuda)
    for method in ("recursive", "naive"):
        ok, worst = phi_gate(plan.evaluate(At, method=method).cpu().numpy(), pr, scale)
        assert ok, (method, worst)


def test_fp32_mode_within_1e5(cuda, cfg2):
    S = 64
    A = seeded_A(S, cfg2.num_seeds, 8)
    c = np.random.default_rng(9).normal(size=len(cfg2.target_ids))
    pr, _, scale = _oracle_phi(cfg2, A, cfg2.target_ids, c)
    plan = P.SitePlan(cfg2).set_coefficients(node_ids=cfg2.target_ids, values=c)
    got = plan.evaluate(torch.from_numpy(A.astype(np.complex64)).to(cuda)).cpu().numpy()
    ok, worst = phi_gate(got, pr, scale, tol=1e-5)
    assert ok, worst


def test_complex_coefficients_multi_output(cuda, cfg1):
    S, n_out = 40, 3
    A = seeded_A(S, cfg1.num_seeds, 10)
    rng = np.random.default_rng(11)
    ids = cfg1.target_ids[::2]
    C = rng.normal(size=(len(ids), n_out)) + 1j * rng.normal(size=(len(ids), n_out))
    plan = P.SitePlan(cfg1).set_coefficients(node_ids=ids, values=C)
    got = plan.evaluate(torch.from_numpy(A).to(cuda), out="complex").cpu().numpy()
    gotn = plan.evaluate(torch.from_numpy(A).to(cuda), method="naive", out="complex").cpu().numpy()
    re, im = O.evaluate_nodes(cfg1.parents[:, 0], cfg1.parents[:, 1], A)
    for o in range(n_out):
        pr, pi = O.model_sum(re, im, ids, C[:, o].real, C[:, o].imag)
        scale = np.abs(C[:, o, None] * (re[ids] + 1j * im[ids])).sum(axis=0)
        for res in (got, gotn):
            assert phi_gate(res[:, o].real, pr, scale)[0]
            assert phi_gate(res[:, o].imag, pi, scale)[0]


def test_hybrid_seed_cache_cfg5_graph(cuda):
    """D=14, nu=5 references 575 seeds: 32-site tiles overflow shared memory and
    the cold tail of the seed table lives in the per-CTA global cache."""
    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, 14), 5)
    S = 40
    A = seeded_A(S, g.num_seeds, 12)
    c = np.random.default_rng(13).normal(size=len(g.target_ids))
    plan = P.SitePlan(g).set_coefficients(node_ids=g.target_ids, values=c)
    assert plan.info()["used_seeds"] > 440
    At = torch.from_numpy(A).to(cuda)
    rec = plan.evaluate(At).cpu().numpy()
    nai = plan.evaluate(At, method="naive").cpu().numpy()
    pr, _, scale = _oracle_phi(g, A[:4], g.target_ids, c)
    assert phi_gate(rec[:4], pr, scale)[0]
    assert phi_gate(nai[:4], pr, scale)[0]


def test_full_size_properties_cfg2(cuda, cfg2):
    """Size-independent checks at BASELINE cfg2 size (1e5 sites): recursive ==
    naive, determinism, z-rotation invariance (A_nlm -> e^{i m a} A_nlm leaves
    every target invariant) and homogeneity (A -> 2A scales order o by 2^o)."""
    S = 100_000
    gen = torch.Generator(device=cuda).manual_seed(3)
    A = torch.complex(torch.randn(S, cfg2.num_seeds, device=cuda, dtype=torch.float64, generator=gen),
                      torch.randn(S, cfg2.num_seeds, device=cuda, dtype=torch.float64, generator=gen)) * math.sqrt(0.5)
    c = np.random.default_rng(4).normal(size=len(cfg2.target_ids))
    plan = P.SitePlan(cfg2).set_coefficients(node_ids=cfg2.target_ids, values=c)
    rec = plan.evaluate(A)
    assert torch.equal(rec, plan.evaluate(A))
    nai = plan.evaluate(A, method="naive")
    # sum_k |c_k| prod |A| >= sum_k |c_k Re A_k|: the gate's normalisation, bounded
    pabs = P.SitePlan(cfg2).set_coefficients(node_ids=cfg2.target_ids, values=np.abs(c))
    bound = 1e-11 * pabs.evaluate(A.abs().to(torch.complex128))
    assert torch.all((rec - nai).abs() <= bound)
    ms = torch.tensor([e[2] for e in cfg2.labels], device=cuda, dtype=torch.float64)
    rot = A * torch.exp(1j * 0.7 * ms)
    assert torch.all((plan.evaluate(rot) - rec).abs() <= bound)
    # homogeneity on the order-4 terms only
    ids4 = cfg2.target_ids[cfg2.order[cfg2.target_ids] == 4]
    c4 = np.random.default_rng(5).normal(size=len(ids4))
    p4 = P.SitePlan(cfg2).set_coefficients(node_ids=ids4, values=c4)
    r1 = p4.evaluate(A[:4096])
    r2 = p4.evaluate(2 * A[:4096])
    assert torch.allclose(r2, 16 * r1, rtol=1e-9, atol=1e-9 * float(r1.abs().max()))


def test_eval_nodes_exact_on_generalized_graph(cuda):
    g = P.build_graph(P.Group.SO2, P.DegreeSpec(1, 8), 4, "gen", 2)
    A = seeded_A(5, g.num_seeds, 14)
    re, im = O.evaluate_nodes(g.parents[:, 0], g.parents[:, 1], A)
    vals = g.plan().evaluate_nodes(torch.from_numpy(A).to(cuda)).cpu().numpy()
    assert np.array_equal(vals.real, re.T) and np.array_equal(vals.imag, im.T)


def test_naive_products_bit_exact(cuda, golden, cfg1):
    d = golden("eval_cfg1.npz")
    index = {e: i for i, e in enumerate(cfg1.labels)}
    rows = [[index[e] for e in cfg1.elements_of(t)] for t in d["target_ids"]]
    width = max(len(r) for r in rows)
    vals = np.ones((len(rows), width), np.complex128)
    lens = np.array([len(r) for r in rows], np.int32)
    for i, r in enumerate(rows):
        vals[i, : len(r)] = d["A"][0, r]
    got = P.naive_products(torch.from_numpy(vals).to(cuda), torch.from_numpy(lens).to(cuda)).cpu().numpy()
    assert np.array_equal(got.view(np.float64), d["naive_site0"].view(np.float64))


@pytest.mark.parametrize("grp", ["T", "SO2", "O3", "O3F"])
def test_pool_vs_reference_golden(cuda, golden, grp):
    d = golden("pool_golden.npz")
    group = P.Group(grp)
    A = P.pool_batched(group, int(d[f"{grp}_cap"]), torch.from_numpy(d[f"{grp}_coords"]).to(cuda),
                       torch.from_numpy(d[f"{grp}_counts"]).to(cuda)).cpu().numpy()
    ref = d[f"{grp}_A"]
    assert np.all(np.abs(A - ref) <= 1e-13 * (1 + np.abs(ref)))


def test_positions_pool_vs_reference_golden(cuda, golden):
    d = golden("positions_cfg3.npz")
    A = P.pool_positions(int(d["cap"]), torch.from_numpy(d["xyz"]).to(cuda)).cpu().numpy()
    ref = d["A"]
    assert np.all(np.abs(A - ref) <= 1e-12 * (1 + np.abs(ref)))


def test_fused_positions_eval_vs_oracle(cuda, golden, cfg2):
    d = golden("positions_cfg3.npz")
    c = np.random.default_rng(15).normal(size=len(cfg2.target_ids))
    plan = P.SitePlan(cfg2).set_coefficients(node_ids=cfg2.target_ids, values=c)
    xyz = torch.from_numpy(d["xyz"]).to(cuda)
    got = plan.evaluate_positions(xyz).cpu().numpy()
    pr, _, scale = _oracle_phi(cfg2, d["A"], cfg2.target_ids, c)
    assert phi_gate(got, pr, scale, tol=1e-10)[0]
    # ragged neighbour counts: a site with k neighbours == the first k only
    counts = torch.tensor([30, 7, 0], dtype=torch.int32, device=cuda)
    rag = plan.evaluate_positions(xyz, counts).cpu().numpy()
    assert rag[2] == plan.evaluate(torch.zeros(1, cfg2.num_seeds, dtype=torch.complex128, device=cuda)).item()
    one = plan.evaluate_positions(xyz[1:2, :7].contiguous()).cpu().numpy()
    assert abs(rag[1] - one[0]) <= 1e-12 * (1 + abs(one[0]))


def test_reduce_sites_matches_sum(cuda, cfg1):
    c = np.random.default_rng(16).normal(size=len(cfg1.target_ids))
    plan = P.SitePlan(cfg1).set_coefficients(node_ids=cfg1.target_ids, values=c)
    A = torch.from_numpy(seeded_A(1000, cfg1.num_seeds, 17)).to(cuda)
    phi = plan.evaluate(A)
    tot = plan.reduce_sites(phi)
    assert torch.allclose(tot[0], phi.sum(), rtol=1e-12)


def test_edge_sizes(cuda, cfg1):
    c = np.ones(len(cfg1.target_ids))
    plan = P.SitePlan(cfg1).set_coefficients(node_ids=cfg1.target_ids, values=c)
    empty = torch.zeros((0, cfg1.num_seeds), dtype=torch.complex128, device=cuda)
    assert plan.evaluate(empty).shape == (0,)
    for S in (1, 31, 33, 32 * 148 + 5):
        A = torch.from_numpy(seeded_A(S, cfg1.num_seeds, S)).to(cuda)
        rec = plan.evaluate(A).cpu().numpy()
        nai = plan.evaluate(A, method="naive").cpu().numpy()
        pr, _, scale = _oracle_phi(cfg1, A[:3].cpu().numpy(), cfg1.target_ids, c)
        assert phi_gate(rec[:3], pr, scale)[0] and phi_gate(nai[:3], pr, scale)[0]
    zero = plan.evaluate(torch.zeros((3, cfg1.num_seeds), dtype=torch.complex128, device=cuda))
    assert torch.all(zero == 0)


@pytest.mark.parametrize("n_out", [2, 64])
def test_multi_output_real_coefficients(cuda, cfg2, n_out):
    """Several real outputs: k2_general (n_out < 8) and the DMMA kernel k2_mma
    (n_out >= 8; BASELINE cfg5 uses 64)."""
    S = 48
    A = seeded_A(S, cfg2.num_seeds, 20 + n_out)
    C = np.random.default_rng(21).normal(size=(len(cfg2.target_ids), n_out))
    plan = P.SitePlan(cfg2).set_coefficients(node_ids=cfg2.target_ids, values=C)
    got = plan.evaluate(torch.from_numpy(A).to(cuda)).cpu().numpy()
    assert got.shape == (S, n_out)
    re, im = O.evaluate_nodes(cfg2.parents[:, 0], cfg2.parents[:, 1], A[:6])
    for o in range(0, n_out, max(1, n_out // 8)):
        pr, _ = O.model_sum(re, im, cfg2.target_ids, C[:, o])
        assert phi_gate(got[:6, o], pr, O.energy_scale(re, cfg2.target_ids, C[:, o]))[0], o
    tot = plan.reduce_sites(torch.from_numpy(got).to(cuda)).cpu().numpy()
    assert np.allclose(tot, got.sum(axis=0), rtol=1e-12, atol=1e-9)


def test_host_pipelines_match_device(cuda, cfg2, golden):
    c = np.random.default_rng(30).normal(size=len(cfg2.target_ids))
    plan = P.SitePlan(cfg2).set_coefficients(node_ids=cfg2.target_ids, values=c)
    A = torch.from_numpy(seeded_A(70_000, cfg2.num_seeds, 31))
    dev_phi = plan.evaluate(A.to(cuda)).cpu()
    host_phi = plan.evaluate_host(A.pin_memory())
    assert plan.last_h2d_bytes == 70_000 * plan.info()["used_seeds"] * 16  # used columns only
    assert torch.equal(dev_phi, host_phi)
    assert torch.equal(dev_phi, plan.evaluate_host(A))  # pageable: row-chunk copies
    assert plan.last_h2d_bytes == A.numel() * 16
    xyz = torch.from_numpy(golden("positions_cfg3.npz")["xyz"])
    assert torch.equal(plan.evaluate_positions(xyz.to(cuda)).cpu(),
                       plan.evaluate_positions_host(xyz.pin_memory(), chunk=2).clone())


def test_batch_independent_results(cuda, cfg2):
    """A site's phi does not depend on the batch it is evaluated in: the
    default kernel (k2_horner for order <= 4) sums one partial per program
    chunk in chunk order, so the grid, the last-round split and the site
    count leave every value bit-identical."""
    c = np.random.default_rng(34).normal(size=len(cfg2.target_ids))
    plan = P.SitePlan(cfg2).set_coefficients(node_ids=cfg2.target_ids, values=c)
    A = torch.from_numpy(seeded_A(40_000, cfg2.num_seeds, 35)).to(cuda)
    full = plan.evaluate(A)
    for n in (1, 63, 64, 1000, 9_500, 19_000, 30_001):
        assert torch.equal(plan.evaluate(A[:n]), full[:n]), n
    assert torch.equal(plan.evaluate(A[7_000:27_000]), full[7_000:27_000])


def test_eval_host_variants(cuda, cfg2):
    """acedag_eval_host for the naive method, fp32 mode, several outputs and
    complex output agrees bit for bit with acedag_eval on the device."""
    rng = np.random.default_rng(32)
    A = torch.from_numpy(seeded_A(5_000, cfg2.num_seeds, 33))
    Ad = A.to(cuda)
    plan = P.SitePlan(cfg2).set_coefficients(node_ids=cfg2.target_ids, values=rng.normal(size=len(cfg2.target_ids)))
    assert torch.equal(plan.evaluate(Ad, method="naive").cpu(), plan.evaluate_host(A.pin_memory(), method="naive"))
    A32 = A.to(torch.complex64)
    assert torch.equal(plan.evaluate(A32.to(cuda)).cpu(), plan.evaluate_host(A32.pin_memory()))
    assert plan.last_h2d_bytes == 5_000 * plan.info()["used_seeds"] * 8
    C = rng.normal(size=(len(cfg2.target_ids), 3)) + 1j * rng.normal(size=(len(cfg2.target_ids), 3))
    plan3 = P.SitePlan(cfg2).set_coefficients(node_ids=cfg2.target_ids, values=C)
    Ap = A.pin_memory()
    assert torch.equal(plan3.evaluate(Ad, out="complex").cpu(), plan3.evaluate_host(Ap, out="complex"))
    res = torch.empty(5_000, 3, dtype=torch.float64)
    plan3.evaluate_host(Ap, result=res)
    assert torch.equal(plan3.evaluate(Ad).cpu(), res)
    assert plan3.evaluate_host(Ap[:0]).shape == (0, 3)


@pytest.mark.parametrize("env", [{"ACEDAG_K2": "quad"}, {"ACEDAG_K2": "horner"}, {"ACEDAG_TAIL_PARTS": "1"}])
def test_kernel_variants_in_subprocess(cuda, env):
    """The fp64 single-output kernel forced either way (k2_quad for order <= 4,
    k2_horner above) and the last-round split switched off are selected once
    per process by environment variables; each is checked against the oracle."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, sys
sys.path.insert(0, "tests")
import paper_2202_04140_b200 as P
from oracle import acedag_oracle as O
from _helpers import phi_gate, seeded_A
g = P.build_graph(P.Group.O3, P.DegreeSpec(1, 10), 4)
A = seeded_A(70, g.num_seeds, 3)
re, im = O.evaluate_nodes(g.parents[:, 0], g.parents[:, 1], A[:5])
for n_out in (1, 8):
    C = np.random.default_rng(4).normal(size=(len(g.target_ids), n_out))
    plan = P.SitePlan(g).set_coefficients(node_ids=g.target_ids, values=C if n_out > 1 else C[:, 0])
    got = plan.evaluate(torch.from_numpy(A).cuda()).cpu().numpy().reshape(70, n_out)
    for o in range(n_out):
        pr, _ = O.model_sum(re, im, g.target_ids, C[:, o])
        ok, w = phi_gate(got[:5, o], pr, O.energy_scale(re, g.target_ids, C[:, o]))
        assert ok, (n_out, o, w)
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("group,p,D,nu,alg,n", [
    ("T", 1, 10, 5, "orig", 1), ("SO2", 1, 7, 4, "gen", 2), ("O3", 2, 4, 4, "orig", 1),
    ("O3", math.inf, 3, 3, "gen", 3), ("O3F", 1, 5, 4, "orig", 1), ("O3", 1, 9, 6, "orig", 1)])
def test_all_groups_and_specs_through_k2_k3(cuda, group, p, D, nu, alg, n):
    """K2/K3 are group-agnostic: every group, p-norm and insertion rule."""
    g = P.build_graph(P.Group(group), P.DegreeSpec(p, D), nu, alg, n)
    S = 37
    A = seeded_A(S, g.num_seeds, D * 10 + nu)
    c = np.random.default_rng(nu).normal(size=len(g.target_ids))
    plan = P.SitePlan(g).set_coefficients(node_ids=g.target_ids, values=c)
    At = torch.from_numpy(A).to(cuda)
    pr, _, scale = _oracle_phi(g, A, g.target_ids, c)
    for method in ("recursive", "naive"):
        ok, worst = phi_gate(plan.evaluate(At, method=method).cpu().numpy(), pr, scale)
        assert ok, (method, worst)
    ok, worst = phi_gate(plan.evaluate(At.to(torch.complex64)).cpu().numpy(), pr, scale, tol=1e-5)
    assert ok, ("fp32", worst)


def test_fp32_horner_many_tiles_and_batch_independent(cuda, cfg2):
    """The fp32 k2_horner over more tiles than SMs (tail split): within 1e-5
    of the oracle, and a site's value independent of its batch."""
    S = 20_001
    A = seeded_A(S, cfg2.num_seeds, 41).astype(np.complex64)
    c = np.random.default_rng(42).normal(size=len(cfg2.target_ids))
    plan = P.SitePlan(cfg2).set_coefficients(node_ids=cfg2.target_ids, values=c)
    assert plan.kernel_name(prec="f32", sites=S) == "k2_horner (fp32)"
    At = torch.from_numpy(A).to(cuda)
    full = plan.evaluate(At)
    idx = [0, 12_345, S - 1]
    pr, _, scale = _oracle_phi(cfg2, A[idx].astype(np.complex128), cfg2.target_ids, c)
    ok, worst = phi_gate(full.cpu().numpy()[idx], pr, scale, tol=1e-5)
    assert ok, worst
    assert torch.equal(plan.evaluate(At[12_000:12_700]), full[12_000:12_700])


@pytest.mark.parametrize("cap,J", [(12, 30), (14, 40)])
def test_pool_v4_matches_v2(cuda, cap, J):
    """pool_positions4 (compile-time cap, warp per site) agrees with the
    CTA-per-site pool_positions2 (ACEDAG_POOL=2, in a subprocess) to
    1e-13 (1 + |A|), with ragged neighbour counts."""
    import os
    import subprocess
    import sys
    code = rf'''
import numpy as np, torch, sys
import paper_2202_04140_b200 as P
rng = np.random.default_rng({cap})
S = 300
d = rng.normal(size=(S, {J}, 3)); d /= np.linalg.norm(d, axis=2, keepdims=True)
r = (0.8 ** 3 + rng.uniform(size=(S, {J}, 1)) * (5.0 ** 3 - 0.8 ** 3)) ** (1 / 3)
xyz = torch.from_numpy(d * r).cuda()
counts = torch.from_numpy(rng.integers(0, {J} + 1, S).astype(np.int32)).cuda()
np.save(sys.argv[1], P.pool_positions({cap}, xyz, counts).cpu().numpy())
'''
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    with tempfile.TemporaryDirectory() as tmp:
        for v in ("4", "2"):
            path = os.path.join(tmp, f"pool_v{v}.npy")
            r = subprocess.run([sys.executable, "-c", code, path], cwd=root,
                               env={**os.environ, "ACEDAG_POOL": v}, capture_output=True, text=True, timeout=600)
            assert r.returncode == 0, r.stderr[-2000:]
            out[v] = np.load(path)
    assert np.all(np.abs(out["4"] - out["2"]) <= 1e-13 * (1 + np.abs(out["2"])))
