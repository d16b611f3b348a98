"""Data parallelism over rollout groups (PAPER.md :258-261 "data parallelism").

Rank r of W owns the contiguous prompt-group range [floor(r P / W), floor((r+1) P / W)).  Rows are independent
once the global kept-token count is known, so the only cross-rank traffic of a learner step is two tiny
all-reduces of counts and statistics (NCCL over NVLink on the GPU box; gloo in the CPU tests).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def shard_groups(n_groups: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous group range [lo, hi) owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return (rank * n_groups) // world, ((rank + 1) * n_groups) // world


def init_from_env(backend: str = "nccl"):
    """Initialise torch.distributed from torchrun's environment (RANK/WORLD_SIZE/MASTER_*); returns (rank, world)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            local = int(os.environ.get("LOCAL_RANK", rank))
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world


def world_info():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def allreduce_sum_(t: torch.Tensor, group=None) -> torch.Tensor:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def allreduce_max_(t: torch.Tensor, group=None) -> torch.Tensor:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


# Layout of the two statistics vectors exchanged per step.
STATS1 = ("n_tokens", "sum_adv", "sum_adv2", "sum_reward", "sum_reward2", "n_zero_std_groups", "n_rollouts_kept",
          "n_groups_kept", "n_groups_dropped")
LOSS_STATS = ("sum_loss", "sum_logp_minus_old", "sum_kl_k3", "n_clipped", "n_nonfinite", "rho_min", "rho_max",
              "sum_logp", "n_tokens", "sum_rho", "sum_weighted_loss")


def reduce_loss_stats_(stats: torch.Tensor, group=None) -> torch.Tensor:
    """All-reduce a loss-stats vector: SUM for the sums/counts, MIN/MAX for the ratio range (in place)."""
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1):
        return stats
    mm = torch.stack([-stats[5], stats[6]])
    sums = stats.clone()
    sums[5] = 0.0
    sums[6] = 0.0
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(mm, op=dist.ReduceOp.MAX, group=group)
    stats.copy_(sums)
    stats[5] = -mm[0]
    stats[6] = mm[1]
    return stats
