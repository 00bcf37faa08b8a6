"""Drop-in API on the GPU: the reference's evaluator tests
(/root/reference/pkg/tests/test_evaluator.py) restated against this package.
Each case names the reference test it mirrors."""

import cmath
import math
import random

import numpy as np
import pytest
import torch

import paper_2202_04140_b200 as P
from paper_2202_04140_b200 import DegreeSpec, Group, canonical
from _helpers import seeded_A
from oracle import acedag_oracle as O

pytestmark = pytest.mark.gpu


def T(*ms):
    return tuple((m,) for m in ms)


def dev(a, b):
    return abs(a - b) / (1 + abs(b))


def test_one_particle_kats(cuda):  # test_evaluator.py:35-58
    for th in (0.0, 1.0, 5.5):
        assert P.one_particle(Group.T, (0,), (th,)) == 1
    assert P.one_particle(Group.T, (3,), (0.7,)) == pytest.approx(cmath.exp(2.1j))
    assert P.one_particle(Group.SO2, (0, 2), (1.0, 0.5)) == pytest.approx(cmath.exp(-1j), abs=1e-12)
    assert P.one_particle(Group.O3, (0, 0, 0), (0.3, 1.0, 2.0)) == pytest.approx(1 / (2 * math.sqrt(math.pi)))
    assert abs(P.one_particle(Group.O3, (0, 1, 0), (0.5, math.pi / 2, 1.0))) < 1e-15
    base = P.one_particle(Group.O3, (1, 1, -1), (0.5, 1.0, 2.0))
    with_f = P.one_particle(Group.O3F, (1, 1, -1, 2), (0.5, 1.0, 2.0, 0.25))
    assert with_f == pytest.approx(base * (2 * 0.25 ** 2 - 1))


def test_one_particle_domain_errors(cuda):  # test_evaluator.py:60-68
    with pytest.raises(ValueError):
        P.one_particle(Group.SO2, (0, 1), (1.5, 0.0))
    with pytest.raises(ValueError):
        P.one_particle(Group.O3F, (0, 0, 0, 1), (0.5, 1.0, 2.0, 1.5))
    with pytest.raises(ValueError):
        P.one_particle(Group.O3, (0, 0, 0), (0.5, 1.0))


def test_pool_kats(cuda):  # test_evaluator.py:71-89
    pooled = P.pool(Group.T, DegreeSpec(1, 3), [(0.4,)])
    for m in range(-3, 4):
        assert pooled[(m,)] == pytest.approx(cmath.exp(1j * m * 0.4))
    pooled = P.pool(Group.T, DegreeSpec(1, 2), [(0.9,), (-0.9,)])
    assert pooled[(1,)] == pytest.approx(2 * math.cos(0.9))
    pooled = P.pool(Group.O3, DegreeSpec(1, 2), [])
    assert pooled and all(v == 0 for v in pooled.values())
    spec = DegreeSpec(1, 4)
    assert set(P.pool(Group.SO2, spec, [(0.5, 1.0)])) == {n.elements[0] for n in P.seed_graph(Group.SO2, spec).nodes}


def test_pool_matches_oracle_all_groups(cuda):
    rng = random.Random(99)
    for group in Group:
        parts = P.random_particles(group, rng)
        got = P.pool(group, DegreeSpec(1, 5), parts)
        ref = O.pool(group.value, O.Spec(1, 5), parts)
        for (e, a), b in zip(got.items(), ref):
            assert abs(a - b) <= 1e-13 * (1 + abs(b)), (group, e)


def test_evaluate_graph_kats(cuda):  # test_evaluator.py:93-113
    g = P.build_graph(Group.T, DegreeSpec(1, 3), 2)
    parts = [(0.3,), (1.1,), (4.0,)]
    pooled = P.pool(Group.T, g.spec, parts)
    vals = P.evaluate_graph(g, pooled)
    assert vals[g.id_of(T(-1, 1))] == pytest.approx(abs(pooled[(1,)]) ** 2)
    g = P.build_graph(Group.T, DegreeSpec(1, 4), 3)
    pooled = P.pool(Group.T, g.spec, [(0.2,), (2.5,)])
    vals = P.evaluate_graph(g, pooled)
    assert vals[g.id_of(T(-1, 0, 1))] == pytest.approx(pooled[(0,)] * abs(pooled[(1,)]) ** 2)
    g = P.build_graph(Group.T, DegreeSpec(1, 2), 2)
    pooled = P.pool(Group.T, g.spec, [(0.1,)])
    del pooled[(2,)]
    with pytest.raises(KeyError, match=r"\(2,\)"):
        P.evaluate_graph(g, pooled)


@pytest.mark.parametrize("group", list(Group))
@pytest.mark.parametrize("alg,n", [("orig", 1), ("gen", 2)])
def test_oracle_equivalence(cuda, group, alg, n):  # test_evaluator.py:115-126
    g = P.build_graph(group, DegreeSpec(1, 6), 4, alg, n)
    rng = random.Random(17)
    for _ in range(3):
        parts = P.random_particles(group, rng)
        pooled = P.pool(group, g.spec, parts)
        vals = P.evaluate_graph(g, pooled)
        for node in g.nodes:
            assert dev(vals[node.id], P.naive_eval(node.elements, pooled)) <= 1e-12


def test_naive_eval_kats(cuda):  # test_evaluator.py:140-152
    assert P.naive_eval(T(1), {(1,): 2 + 1j}) == 2 + 1j
    pooled = P.pool(Group.T, DegreeSpec(1, 2), [(0.1,), (2.2,), (3.3,)])
    assert P.naive_eval(T(0, 0, 0), pooled) == pytest.approx(27)
    with pytest.raises(KeyError):
        P.naive_eval(T(5), {})


def test_evaluate_model_cases(cuda):  # test_evaluator.py:155-199
    g = P.build_graph(Group.T, DegreeSpec(1, 4), 3)
    assert P.evaluate_model(g, {T(-1, 1): 0j, T(0, 0): 0j}, [(0.4,), (1.0,)]) == 0
    g2 = P.build_graph(Group.T, DegreeSpec(1, 4), 2)
    parts = [(0.4,), (2.0,)]
    pooled = P.pool(Group.T, g2.spec, parts)
    assert P.evaluate_model(g2, {T(-1, 1): 1.0}, parts) == pytest.approx(abs(pooled[(1,)]) ** 2)
    g3 = P.build_graph(Group.SO2, DegreeSpec(1, 5), 3)
    rng = random.Random(5)
    targets = [n.elements for n in g3.nodes if not n.auxiliary and g3.is_target(n.elements)]
    coeffs = {t: complex(rng.uniform(-1, 1), rng.uniform(-1, 1)) for t in targets[::3]}
    parts = P.random_particles(Group.SO2, rng)
    pooled = P.pool(Group.SO2, g3.spec, parts)
    expected = sum(c * P.naive_eval(t, pooled) for t, c in coeffs.items())
    assert dev(P.evaluate_model(g3, coeffs, parts), expected) < 1e-12
    with pytest.raises(KeyError):
        P.evaluate_model(g2, {T(-9, 9): 1.0}, [(0.1,)])
    with pytest.raises(ValueError):
        P.evaluate_model(g, {T(1, 1): 1.0}, [(0.1,)])
    assert P.evaluate_model(g, {T(-1, 1): 2.0, T(0,): 1.5}, []) == 0
    g4 = P.build_graph(Group.SO2, DegreeSpec(1, 4), 2)
    parts = [(0.8, 0.3), (0.2, 2.0)]
    coeffs = {canonical([(0, 1), (0, -1)]): 1j}
    full = P.evaluate_model(g4, coeffs, parts)
    assert P.evaluate_model(g4, coeffs, parts, real_part=True) == full.real


@pytest.mark.parametrize("group", list(Group))
def test_invariance(cuda, group):  # test_evaluator.py:202-212
    g = P.build_graph(group, DegreeSpec(1, 6), 3)
    parts = P.random_particles(group, random.Random(23))
    rep = P.invariance_check(group, g, parts, trials=6, seed=99)
    assert rep.rotation_max_dev < 1e-10
    if group.has_l:
        assert rep.inversion_max_dev < 1e-10
    else:
        assert rep.inversion_max_dev is None


def test_reference_graph_objects_are_accepted(cuda):
    """A reference-style EvalGraph (duck-typed nodes/parents) goes through the
    same kernels via acedag_graph_from_parents."""
    og = O.build_graph("O3", O.Spec(1, 5), 3)

    class Node:
        def __init__(self, i):
            self.parents = og.parents[i]
            self.auxiliary = og.aux[i]
            self.elements = og.elements[i]

    class RefGraph:
        group = Group.O3
        spec = DegreeSpec(1, 5)
        nu_max = 3
        alg = "orig"
        n = 1
        nodes = [Node(i) for i in range(len(og.elements))]

    parts = P.random_particles(Group.O3, random.Random(1))
    pooled = P.pool(Group.O3, DegreeSpec(1, 5), parts)
    vals = P.evaluate_graph(RefGraph(), pooled)
    pa, pb, _, _ = O.graph_arrays(og)
    import numpy as np
    A = np.array([[pooled[e] for e in O.one_particle_indices("O3", 5)]])
    re, im = O.evaluate_nodes(pa, pb, A)
    assert all(v == complex(r, i) for v, r, i in zip(vals, re[:, 0], im[:, 0]))


def test_rejected_coefficients_keep_the_previous_program(cuda):
    """a rejected set_coefficients (non-target id) raises and leaves
    the plan evaluating its previous coefficients bit for bit."""
    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, 8), 3)
    rng = np.random.default_rng(50)
    c = rng.normal(size=len(g.target_ids))
    plan = P.SitePlan(g).set_coefficients(node_ids=g.target_ids, values=c)
    A = torch.from_numpy(seeded_A(300, g.num_seeds, 51)).to(cuda)
    before = plan.evaluate(A).clone()
    before_n = plan.evaluate(A, method="naive").clone()
    aux = int(np.flatnonzero(g.aux)[0])
    with pytest.raises(ValueError):
        plan.set_coefficients(node_ids=[aux], values=[1.0])
    assert torch.equal(plan.evaluate(A), before)
    assert torch.equal(plan.evaluate(A, method="naive"), before_n)
    # the complex-output kernel (k2_general) sums in another order: same
    # coefficients, equal to rounding
    assert torch.allclose(plan.evaluate(A, out="complex").real, before, rtol=1e-10, atol=1e-9)


def test_device_entry_points_validate_tensors(cuda):
    """wrong dtype / shape / device / contiguity of caller tensors
    is a ValueError before any pointer reaches a kernel."""
    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, 8), 3)
    plan = P.SitePlan(g).set_coefficients(node_ids=g.target_ids, values=np.ones(len(g.target_ids)))
    A = torch.from_numpy(seeded_A(40, g.num_seeds, 52)).to(cuda)
    with pytest.raises(ValueError):
        plan.evaluate(A.cpu())
    with pytest.raises(ValueError):
        plan.evaluate(A.real.contiguous())
    with pytest.raises(ValueError):
        plan.evaluate(A, result=torch.empty(39, dtype=torch.float64, device=cuda))
    with pytest.raises(ValueError):
        plan.evaluate(A, result=torch.empty(40, dtype=torch.float32, device=cuda))
    with pytest.raises(ValueError):
        plan.evaluate(A, result=torch.empty(80, dtype=torch.float64, device=cuda)[::2])
    xyz = torch.rand(5, 7, 3, dtype=torch.float64, device=cuda) + 1.0
    with pytest.raises(ValueError):
        plan.evaluate_positions(xyz.float())
    with pytest.raises(ValueError):
        plan.evaluate_positions(xyz[..., :2].contiguous())
    with pytest.raises(ValueError):
        plan.evaluate_positions(xyz, counts=torch.zeros(4, dtype=torch.int32, device=cuda))
    with pytest.raises(ValueError):
        P.pool_batched(P.Group.O3, 4, xyz.float())
    with pytest.raises(ValueError):
        plan.reduce_sites(torch.zeros(5, 2, dtype=torch.float64, device=cuda))
    # counts above J are clamped to the row (pool_ref), not read past it
    coords = torch.rand(2, 3, 3, dtype=torch.float64, device=cuda)
    big = P.pool_batched(P.Group.O3, 3, coords, torch.tensor([99, 3], dtype=torch.int32, device=cuda))
    full = P.pool_batched(P.Group.O3, 3, coords)
    assert torch.equal(big, full)


def test_pool_keys_cover_seeds(cuda):  # test_evaluator.py:85-89
    spec = DegreeSpec(1, 4)
    g = P.seed_graph(Group.SO2, spec)
    pooled = P.pool(Group.SO2, spec, [(0.5, 1.0)])
    assert set(pooled) == {n.elements[0] for n in g.nodes}


def test_multiplication_count_below_naive():  # test_evaluator.py:128-137 (host only)
    for numax in (3, 4, 5):
        g = P.build_graph(Group.T, DegreeSpec(1, 10), numax)
        graph_muls = sum(1 for node in g.nodes if node.order >= 2)
        naive_muls = sum(node.order - 1 for node in g.nodes if not node.auxiliary and g.is_target(node.elements))
        assert graph_muls < naive_muls


def test_invariance_negative_control(cuda):  # test_evaluator.py:214-222
    spec = DegreeSpec(1, 3)
    parts = [(0.0,), (0.5,), (1.2,)]
    before = P.naive_eval(T(1, 1), P.pool(Group.T, spec, parts))
    after = P.naive_eval(T(1, 1), P.pool(Group.T, spec, P.rotate_particles(Group.T, parts, math.pi / 2)))
    assert dev(after, before) > 1e-2
    assert after == pytest.approx(-before)  # phase e^(i pi)


def test_conjugation_of_negated_tuple(cuda):  # test_evaluator.py:224-233
    g = P.build_graph(Group.T, DegreeSpec(1, 6), 3)
    parts = [(0.4,), (1.9,), (2.7,)]
    vals = P.evaluate_graph(g, P.pool(Group.T, g.spec, parts))
    for node in g.nodes:
        if node.auxiliary or not g.is_target(node.elements):
            continue
        negated = canonical((-m,) for (m,) in node.elements)
        assert vals[g.id_of(negated)] == pytest.approx(vals[node.id].conjugate(), abs=1e-12)
