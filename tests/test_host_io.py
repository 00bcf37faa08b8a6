"""Host-side callers of the path: symmetry transforms and the particle /
coefficient text files (evaluator.py:149-186, 231-290).  Where the reference
is mounted (this container) they are compared with it directly; elsewhere
the round-trip and error-text checks still run."""

import math
import os
import random
import sys

import pytest

import paper_2202_04140_b200 as P

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(REF):
        pytest.skip("reference not mounted")
    sys.path.insert(0, REF)
    import acedag.evaluator as R
    from acedag.indexsets import Group
    return R, Group


@pytest.mark.parametrize("grp", ["T", "SO2", "O3", "O3F"])
def test_transforms_and_files_match_reference(ref, grp, tmp_path):
    R, RG = ref
    for seed in range(5):
        a = P.random_particles(P.Group(grp), random.Random(seed))
        b = R.random_particles(RG(grp), random.Random(seed))
        assert a == b
        assert P.rotate_particles(P.Group(grp), a, 1.1) == R.rotate_particles(RG(grp), b, 1.1)
        if grp in ("O3", "O3F"):
            assert P.invert_particles(P.Group(grp), a) == R.invert_particles(RG(grp), b)
        else:
            with pytest.raises(ValueError, match="inversion applies to O3/O3F"):
                P.invert_particles(P.Group(grp), a)
        P.write_particles(tmp_path / "ours", P.Group(grp), a)
        R.write_particles(tmp_path / "ref", RG(grp), b)
        assert (tmp_path / "ours").read_bytes() == (tmp_path / "ref").read_bytes()
        g, parts = P.read_particles(tmp_path / "ref")
        assert g is P.Group(grp) and parts == R.read_particles(tmp_path / "ref")[1]


def test_coefficient_files_match_reference(ref, tmp_path):
    R, RG = ref
    coef = {((0, 1, -1), (0, 1, 1)): 0.25 - 1.5j, ((1, 0, 0),): 2.0, ((0, 0, 0), (0, 2, 0), (1, 1, 0)): -0.125j}
    P.write_coefficients(tmp_path / "ours", coef)
    R.write_coefficients(tmp_path / "ref", coef)
    assert (tmp_path / "ours").read_bytes() == (tmp_path / "ref").read_bytes()
    (tmp_path / "ref").write_text("# comment\n\n" + (tmp_path / "ref").read_text())
    assert P.read_coefficients(tmp_path / "ref", P.Group.O3) == R.read_coefficients(tmp_path / "ref", RG.O3)


@pytest.mark.parametrize("body,msg", [
    ("0.5 1.0 2.0\n", "missing '# group=...' header before data"),
    ("# hello\n", "missing '# group=...' header"),
    ("# group=O3\n0.5 x 2.0\n", ":2: bad coordinate line: '0.5 x 2.0'"),
    ("# group=O3\n1.5 1.0 2.0\n", "radius must lie in [0, 1]"),
    ("# group=O3\n0.5 1.0\n", "O3 particles take 3 coordinates"),
])
def test_particle_file_errors(tmp_path, body, msg):
    path = tmp_path / "p.txt"
    path.write_text(body)
    with pytest.raises(ValueError) as err:
        P.read_particles(path)
    assert msg in str(err.value)


@pytest.mark.parametrize("body,msg", [
    ("0,0,0 1.0\n", ":1: expected '<tuple> <re> <im>', got '0,0,0 1.0'"),
    ("0,0,0 1.0 zz\n", ":1: bad coefficient values: '0,0,0 1.0 zz'"),
    ("0,0 1.0 0.0\n", "expected a multiple of 3 components for O3, got 2"),
])
def test_coefficient_file_errors(tmp_path, body, msg):
    path = tmp_path / "c.txt"
    path.write_text(body)
    with pytest.raises(ValueError) as err:
        P.read_coefficients(path, P.Group.O3)
    assert msg in str(err.value)


def test_rotation_is_azimuthal():
    parts = [(0.5, 1.0, 2.0, 0.25)]
    assert P.rotate_particles(P.Group.O3F, parts, 0.5) == [(0.5, 1.0, 2.5, 0.25)]
    assert P.invert_particles(P.Group.O3F, parts) == [(0.5, math.pi - 1.0, 2.0 + math.pi, 0.25)]


class TestParticleFiles:  # reference tests/test_evaluator.py:240-265, restated
    def test_roundtrip(self, tmp_path):
        parts = [(0.5, 1.0, 2.0, -0.25), (0.1, 0.2, 0.3, 0.4)]
        path = tmp_path / "conf.txt"
        P.write_particles(path, P.Group.O3F, parts)
        group, got = P.read_particles(path)
        assert group is P.Group.O3F and got == parts

    def test_missing_header(self, tmp_path):
        path = tmp_path / "conf.txt"
        path.write_text("0.1 0.2\n")
        with pytest.raises(ValueError):
            P.read_particles(path)

    def test_bad_line(self, tmp_path):
        path = tmp_path / "conf.txt"
        path.write_text("# group=T\nnot-a-number\n")
        with pytest.raises(ValueError):
            P.read_particles(path)

    def test_empty_config(self, tmp_path):
        path = tmp_path / "conf.txt"
        P.write_particles(path, P.Group.T, [])
        group, got = P.read_particles(path)
        assert group is P.Group.T and got == []


class TestCoefficientFiles:  # reference tests/test_evaluator.py:268-279, restated
    def test_roundtrip(self, tmp_path):
        coeffs = {((-1,), (1,)): 1.5 + 0.5j, ((0,),): -2.0 + 0j}
        path = tmp_path / "c.txt"
        P.write_coefficients(path, coeffs)
        assert P.read_coefficients(path, P.Group.T) == coeffs

    def test_bad_line(self, tmp_path):
        path = tmp_path / "c.txt"
        path.write_text("-1,1 1.0\n")
        with pytest.raises(ValueError):
            P.read_coefficients(path, P.Group.T)
