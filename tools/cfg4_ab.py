"""cfg4 A/B: k2_quad (default) vs fp64 k2_horner (ACEDAG_K2=horner) on the
prod_cfg4 fixture sites; run twice with the env var set or not."""
import hashlib, os, sys, time
import numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import paper_2202_04140_b200 as P
from _helpers import phi_gate, seeded_A
d = dict(np.load("tests/golden/prod_cfg4.npz"))
g = P.build_graph(P.Group.O3, P.DegreeSpec(1, 16), 6)
C = np.random.default_rng(int(d["cseed"])).normal(size=(len(g.target_ids), 1))
plan = P.SitePlan(g).set_coefficients(node_ids=g.target_ids, values=C[:, 0])
S = int(d["S"])
A = torch.from_numpy(seeded_A(S, g.num_seeds, int(d["seed"]))).cuda()
got = plan.evaluate(A).cpu().numpy()
ok, worst = phi_gate(got[d["sites"]], d["phi"], d["scale"])
print(os.environ.get("ACEDAG_K2", "auto"), plan.kernel_name(sites=S), "gate", ok, round(worst, 6))
A2 = torch.from_numpy(seeded_A(40000, g.num_seeds, 5)).cuda()
for _ in range(2): plan.evaluate(A2)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3): plan.evaluate(A2)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print("40k sites", round(ms, 2), "ms ->", round(40000 / ms * 1e3), "sites/s")
