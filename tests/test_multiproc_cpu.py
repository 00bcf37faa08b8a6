"""Multi-rank host logic on CPU (gloo, world_size 2): site sharding and the
total-energy all-reduce.  The per-rank evaluator here is the oracle (the CPU
checker); on GPUs it is SitePlan -- the sharding code is the same."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2202_04140_b200.distributed import ShardedSites, shard_range


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 7, 100_000, 1_000_003):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import acedag_oracle as O
    import paper_2202_04140_b200 as P

    g = P.build_graph(P.Group.O3, P.DegreeSpec(1, 6), 3)
    c = np.random.default_rng(0).normal(size=len(g.target_ids))
    S = 37
    rng = np.random.default_rng(1)
    A_all = rng.normal(size=(S, g.num_seeds)) + 1j * rng.normal(size=(S, g.num_seeds))

    def oracle_eval(A):
        re, im = O.evaluate_nodes(g.parents[:, 0], g.parents[:, 1], A.numpy())
        pr, _ = O.model_sum(re, im, g.target_ids, c)
        return torch.from_numpy(pr)

    sh = ShardedSites(S, evaluate=oracle_eval)
    phi, total = sh.run(torch.from_numpy(A_all[sh.lo:sh.hi]))
    sizes = [shard_range(S, r, world)[1] - shard_range(S, r, world)[0] for r in range(world)]
    pad = torch.zeros(max(sizes), dtype=torch.float64)
    pad[: phi.shape[0]] = phi
    gathered = [torch.zeros(max(sizes), dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, pad)
    if rank == 0:
        full = oracle_eval(torch.from_numpy(A_all))
        sharded = torch.cat([g[:n] for g, n in zip(gathered, sizes)])
        np.savez(result_path, full=full.numpy(), sharded=sharded.numpy(), total=total.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_evaluation_and_energy_allreduce(tmp_path):
    path = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    r = np.load(path)
    assert np.array_equal(r["sharded"], r["full"])  # sharding is exact: same per-site arithmetic
    assert np.isclose(r["total"][0], r["full"].sum(), rtol=1e-12, atol=1e-9)
