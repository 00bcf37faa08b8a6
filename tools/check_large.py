import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2202_04140_b200 as P
from _helpers import seeded_A
g = P.build_graph(P.Group.O3, P.DegreeSpec(1, 12), 4)
c = np.random.default_rng(1).normal(size=len(g.target_ids))
plan = P.SitePlan(g).set_coefficients(node_ids=g.target_ids, values=c)
for S in (1_000_003, 18_945, 148 * 128 * 3 + 1):
    rng = np.random.default_rng(S)
    A = torch.complex(torch.from_numpy(rng.normal(0, 0.5 ** 0.5, (S, g.num_seeds))), torch.from_numpy(rng.normal(0, 0.5 ** 0.5, (S, g.num_seeds)))).cuda()
    a = plan.evaluate(A); b = plan.evaluate(A, method="naive")
    d = (a - b).abs() / b.abs().clamp_min(1e-300)
    sub = plan.evaluate(A[S // 2: S // 2 + 1000])
    print(S, plan.kernel_name(sites=S), "max rel vs naive", float(d.max()), "batch-independent", bool(torch.equal(sub, a[S // 2: S // 2 + 1000])), flush=True)
    del A
