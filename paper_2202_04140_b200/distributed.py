"""Site sharding across GPUs (one process per GPU, torch.distributed).

Sites are independent (phi_s depends only on site s's basis row and the
shared DAG/coefficients), so the data path shards with NO collective: every
rank evaluates a contiguous block of sites against its own copy of the
plan.  The only exchange is the optional total energy, sum_s phi_s, reduced
with one all-reduce of n_out float64 values (BASELINE cfg3/cfg5) -- NCCL over
NVLink on B200s, gloo in the CPU tests.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_sites: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of sites owned by ``rank``: sizes differ by at most 1,
    lower ranks take the remainder."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, rem = divmod(int(n_sites), world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def rank_world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def total_energy(local_total: torch.Tensor) -> torch.Tensor:
    """All-reduce (sum) of per-rank site totals, in place; identity when no
    process group is initialised (a group of one still runs the collective)."""
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(local_total, op=dist.ReduceOp.SUM)
    return local_total


class ShardedSites:
    """Evaluate this rank's shard of a global batch of sites.

    ``evaluate`` maps a tensor of local inputs (A rows or neighbour shells)
    to per-site phi; by default it is ``SitePlan.evaluate`` /
    ``SitePlan.evaluate_positions`` of the given plan.  ``run`` returns the
    local phi block and the globally reduced total.
    """

    def __init__(self, n_sites: int, plan=None, evaluate=None, positions: bool = False):
        self.rank, self.world = rank_world()
        self.lo, self.hi = shard_range(n_sites, self.rank, self.world)
        self.plan = plan
        if evaluate is None:
            evaluate = plan.evaluate_positions if positions else plan.evaluate
        self._evaluate = evaluate

    @property
    def local_sites(self) -> int:
        return self.hi - self.lo

    def run(self, local_inputs: torch.Tensor):
        if local_inputs.shape[0] != self.local_sites:
            raise ValueError(f"rank {self.rank} owns {self.local_sites} sites, got {local_inputs.shape[0]}")
        phi = self._evaluate(local_inputs)
        if self.plan is not None and phi.is_cuda:
            total = self.plan.reduce_sites(phi)
        else:
            total = phi.reshape(phi.shape[0], -1).sum(dim=0).to(torch.float64)
        return phi, total_energy(total)
