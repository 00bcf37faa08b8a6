"""The sharded GPU path as a system: two ranks (processes)
on cuda:0 with the gloo backend, each evaluating its shard with SitePlan
(positions -> K1 + K2, cfg3-shaped), reducing its sites on the device and
all-reducing the energy -- exactly what bench.py runs per GPU, with NCCL
replaced by gloo because this box has one GPU.  The ranks' kernels never wait
on one another (the only exchange is the host-side collective).  Checked
against one process evaluating all sites: per-site phi bit-identical (the
kernels do not depend on the batch), total energy to rounding."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from _helpers import seeded_shells

pytestmark = pytest.mark.gpu

S, J = 5_003, 30


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _plan():
    import paper_2202_04140_b200 as P
    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, 12), 4)
    c = np.random.default_rng(70).normal(size=len(g.target_ids))
    return P.SitePlan(g, 0).set_coefficients(node_ids=g.target_ids, values=c)


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2202_04140_b200.distributed import ShardedSites
    plan = _plan()
    sh = ShardedSites(S, plan=plan, positions=True)
    xyz = torch.from_numpy(seeded_shells(S, J, 71)[sh.lo:sh.hi]).cuda()
    phi, total = sh.run(xyz)
    torch.cuda.synchronize()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), lo=sh.lo, hi=sh.hi, phi=phi.cpu().numpy(),
             total=total.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_shard_reduce_allreduce(cuda, tmp_path):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    r = [np.load(tmp_path / f"rank{k}.npz") for k in range(2)]
    assert r[0]["lo"] == 0 and r[0]["hi"] == r[1]["lo"] and r[1]["hi"] == S
    plan = _plan()
    full = plan.evaluate_positions(torch.from_numpy(seeded_shells(S, J, 71)).to(cuda)).cpu().numpy()
    assert np.array_equal(np.concatenate([r[0]["phi"], r[1]["phi"]]), full)
    for k in range(2):  # every rank holds the global total
        assert np.isclose(r[k]["total"][0], full.sum(), rtol=1e-12, atol=1e-8)
    assert r[0]["total"][0] == r[1]["total"][0]
