import torch, numpy as np, sys, time
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2202_04140_b200 as P
g=P.build_graph(P.Group.O3,P.DegreeSpec(1,12),4)
plan=P.SitePlan(g).set_coefficients(node_ids=g.target_ids, values=np.random.default_rng(0).normal(size=len(g.target_ids)))
S=100000
A=torch.complex(torch.randn(S,g.num_seeds,dtype=torch.float64),torch.randn(S,g.num_seeds,dtype=torch.float64)).pin_memory()
for _ in range(3): plan.evaluate_host(A)
t=time.perf_counter(); plan.evaluate_host(A); print("wall ms", (time.perf_counter()-t)*1e3, flush=True)
