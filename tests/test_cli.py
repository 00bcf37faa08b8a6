"""Command line (callers of the path).  `build` is host-only; `eval`/`verify`
run the CUDA kernels and are marked gpu."""

import hashlib
import math
import subprocess
import sys

import pytest

from paper_2202_04140_b200.cli import main


def test_build_writes_reference_bytes(tmp_path, golden):
    rec = next(r for r in golden("graph_hashes.json") if (r["group"], r["D"], r["nu"]) == ("O3", 8, 3))
    out = tmp_path / "g.txt"
    assert main(["build", "--group", "O3", "--D", "8", "--numax", "3", "--out", str(out)]) == 0
    assert hashlib.sha256(out.read_bytes()).hexdigest() == rec["sha256"]


def test_errors_exit_1(tmp_path, capsys):
    assert main(["build", "--group", "T", "--D", "4", "--numax", "0", "--out", str(tmp_path / "x")]) == 1
    assert "error:" in capsys.readouterr().err


@pytest.mark.gpu
def test_eval_node_lines_and_model(tmp_path, cuda):
    from oracle import acedag_oracle as O
    import paper_2202_04140_b200 as P
    g = tmp_path / "g.txt"
    assert main(["build", "--group", "SO2", "--D", "5", "--numax", "3", "--out", str(g)]) == 0
    conf = tmp_path / "conf.txt"
    parts = [(0.8, 0.3), (0.2, 2.0), (0.5, 4.0)]
    P.write_particles(conf, P.Group.SO2, parts)
    out = tmp_path / "vals.txt"
    assert main(["eval", "--graph", str(g), "--config", str(conf), "--out", str(out)]) == 0
    og = O.build_graph("SO2", O.Spec(1, 5), 3)
    pa, pb, _, _ = O.graph_arrays(og)
    import numpy as np
    A = np.array([O.pool("SO2", O.Spec(1, 5), parts)])
    re, im = O.evaluate_nodes(pa, pb, A)
    lines = out.read_text().splitlines()
    assert len(lines) == len(pa)
    for k, line in enumerate(lines):
        parts_ = line.split()
        assert int(parts_[0]) == k
        assert abs(float(parts_[3]) - re[k, 0]) <= 1e-13 * (1 + abs(re[k, 0]))
    coeffs = tmp_path / "c.txt"
    coeffs.write_text("0,-1,0,1 1.5 0.0\n")
    assert main(["eval", "--graph", str(g), "--config", str(conf), "--coeffs", str(coeffs),
                 "--real-part", "--out", str(out)]) == 0
    k = og.ids[((0, -1), (0, 1))]
    assert math.isclose(float(out.read_text()), 1.5 * re[k, 0], rel_tol=1e-12, abs_tol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("group", ["T", "O3"])
def test_verify_suites_pass(cuda, group, capsys):
    assert main(["verify", "--suite", "all", "--group", group, "--D", "6", "--numax", "4", "--configs", "4"]) == 0
    assert capsys.readouterr().out.count("PASS") == 2
