"""GPU check of the selected K2 kernel (ACEDAG_K2) against the oracle on a
few sites and against the naive kernel K3 on every site.

usage: ACEDAG_K2=horner python tools/check_k2.py"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2202_04140_b200 as P  # noqa: E402
from _helpers import phi_gate, seeded_A  # noqa: E402
from oracle import acedag_oracle as O  # noqa: E402

for D, nu, S in ((8, 3, 1000), (10, 4, 3000), (12, 4, 20000), (6, 2, 500), (12, 4, 100000)):
    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, D), nu)
    A = seeded_A(S, g.num_seeds, 7)
    c = np.random.default_rng(1).normal(size=len(g.target_ids))
    plan = P.SitePlan(g).set_coefficients(node_ids=g.target_ids, values=c)
    Ad = torch.from_numpy(A).cuda()
    name = plan.kernel_name(sites=S)
    got = plan.evaluate(Ad).cpu().numpy()
    nai = plan.evaluate(Ad, method="naive").cpu().numpy()
    k = 6
    re, im = O.evaluate_nodes(g.parents[:, 0], g.parents[:, 1], A[:k])
    ref, _ = O.model_sum(re, im, g.target_ids, c)
    scale = O.energy_scale(re, g.target_ids, c)
    ok, w = phi_gate(got[:k], ref, scale)
    d = np.abs(got - nai)
    rel_naive = float((d / np.maximum(np.abs(nai), 1e-300)).max())
    got2 = plan.evaluate(Ad).cpu().numpy()
    print(f"D={D} nu={nu} S={S} kernel={name}: oracle {'OK' if ok else 'FAIL'} worst={w:.3e}; "
          f"max|rec-naive|={d.max():.3e} (max rel {rel_naive:.2e}); deterministic={np.array_equal(got, got2)}",
          flush=True)
