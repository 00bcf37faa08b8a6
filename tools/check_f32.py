"""GPU check of the fp32 mode (complex64 input) against the oracle at 1e-5
of sum|c Re A| for orders 3-6.  usage: python tools/check_f32.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2202_04140_b200 as P  # noqa: E402
from _helpers import phi_gate, seeded_A  # noqa: E402
from oracle import acedag_oracle as O  # noqa: E402

for D, nu, S in ((8, 3, 1000), (12, 4, 20000), (10, 5, 3000), (9, 6, 3000), (12, 6, 3000)):
    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, D), nu)
    A = seeded_A(S, g.num_seeds, 3).astype(np.complex64)
    c = np.random.default_rng(1).normal(size=len(g.target_ids))
    plan = P.SitePlan(g).set_coefficients(node_ids=g.target_ids, values=c)
    got = plan.evaluate(torch.from_numpy(A).cuda()).cpu().numpy()
    k = 4
    re, im = O.evaluate_nodes(g.parents[:, 0], g.parents[:, 1], A[:k].astype(np.complex128))
    ref, _ = O.model_sum(re, im, g.target_ids, c)
    ok, w = phi_gate(got[:k], ref, O.energy_scale(re, g.target_ids, c), tol=1e-5)
    print(f"D={D} nu={nu} S={S} {plan.kernel_name(prec='f32', sites=S)}: {'OK' if ok else 'FAIL'} worst={w:.3e}",
          flush=True)
