"""Native DAG builder and graph file format vs the reference's golden
hashes (tests/golden/graph_hashes.json).  CPU only (host code of the .so)."""

import hashlib
import math

import numpy as np
import pytest

import paper_2202_04140_b200 as P
from oracle import acedag_oracle as O


def _spec(r):
    return P.DegreeSpec(math.inf if r["p"] == "inf" else r["p"], r["D"])


def test_native_build_matches_every_reference_hash(golden):
    recs = [r for r in golden("graph_hashes.json") if r["nodes"] < 1_000_000]
    assert any(r["nodes"] == 458484 for r in recs)  # cfg5 (D=14, nu=5)
    for r in recs:
        g = P.build_graph(P.Group(r["group"]), _spec(r), r["nu"], r["alg"], r["n"])
        s = P.serialize_graph(g)
        assert hashlib.sha256(s).hexdigest() == r["sha256"], r
        assert (g.num_nodes, g.num_targets, g.num_aux) == (r["nodes"], r["targets"], r["aux"])


def test_soa_arrays_equal_oracle_cfg2():
    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, 12), 4)
    og = O.build_graph("O3", O.Spec(1, 12), 4)
    pa, pb, aux, tg = O.graph_arrays(og)
    assert np.array_equal(g.parents[:, 0], pa) and np.array_equal(g.parents[:, 1], pb)
    assert np.array_equal(g.aux, aux) and np.array_equal(g.target_ids, tg)
    assert np.array_equal(g.order, [len(t) for t in og.elements])


def test_roundtrip_serialize_deserialize():
    g = P.build_graph(P.Group.SO2, P.DegreeSpec(1, 8), 4, "gen", 2)
    s = P.serialize_graph(g)
    h = P.deserialize_graph(s)
    assert P.serialize_graph(h) == s
    assert h.alg == "gen" and h.n == 2 and h.nu_max == 4


def test_from_parents_rebuilds_tuples():
    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, 6), 4)
    h = P.graph_from_parents(g.group, g.spec, g.parents, g.aux, nu_max=4)
    assert P.serialize_graph(h) == P.serialize_graph(g)
    bad = g.parents.copy()
    bad[g.num_seeds + 3] = [g.num_seeds + 5, 0]
    with pytest.raises(ValueError):
        P.graph_from_parents(g.group, g.spec, bad, nu_max=4)


def test_nodes_and_lookup_api():
    g = P.build_graph(P.Group.T, P.DegreeSpec(1, 4), 3)
    t = ((1,), (1,))
    assert t in g and g.nodes[g.id_of(t)].auxiliary  # test_evaluator.py:185
    assert not g.is_target(t)
    assert g.nodes[g.id_of(((-1,), (0,), (1,)))].order == 3
    with pytest.raises(KeyError):
        g.id_of(((-9,), (9,)))
    assert [n.elements for n in P.seed_graph(P.Group.T, P.DegreeSpec(1, 2)).nodes] == [
        ((-2,),), ((-1,),), ((0,),), ((1,),), ((2,),)]


def test_insertion_traces_of_reference_tests():
    # graphbuild tests: independent tuple splits off the max label (:48-55)
    g = P.build_graph(P.Group.T, P.DegreeSpec(1, 8), 4, "gen", 2)
    assert g.num_nodes > 0
    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, 5), 3)
    assert len(g) == 268 and int(g.aux.sum()) == 10


def test_build_argument_errors():
    with pytest.raises(ValueError):
        P.build_graph(P.Group.T, P.DegreeSpec(1, 4), 0)
    with pytest.raises(ValueError):
        P.build_graph(P.Group.T, P.DegreeSpec(1, 4), 3, "fancy")
    with pytest.raises(ValueError):
        P.DegreeSpec(3, 4)


def test_deserialize_errors():
    with pytest.raises(P.UnsupportedVersionError):
        P.deserialize_graph(b"ACEDAG v2 group=T p=1 D=2 numax=2 alg=orig n=1\n")
    with pytest.raises(P.GraphFormatError) as ei:
        P.deserialize_graph(b"ACEDAG v1 group=T p=1 D=1 numax=2 alg=orig n=1\n0 0 -1 -\nbad\n")
    assert ei.value.offset > 0
