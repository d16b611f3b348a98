"""Data parallelism over rollout groups (PAPER.md :258-261 "data parallelism").

Rank r of W owns the contiguous prompt-group range [floor(r P / W), floor((r+1) P / W)).  Rows are independent
once the global kept-token count is known, so the only cross-rank traffic of a learner step is two tiny
all-reduces of counts and statistics (NCCL over NVLink on the GPU box; gloo in the CPU tests).

f3: the stale filter (PAPER.md :224) drops whole groups, so the ranks' kept-token counts
diverge and the step waits for the busiest rank.  ``balanced_bounds`` / ``reshard_plan`` split the global
sequence of kept rollouts (rank-major = group order) into W contiguous ranges of ~N_global / W tokens, and
``exchange`` moves the packed arrays there with one all-to-all per array.  Whole rollouts move (a trainer
reshards before the model's forward pass, which needs whole sequences); the advantage is computed before.
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


# ---------------------------------------------------------------------------------------------------- f3
def balanced_bounds(lengths, world: int) -> list[int]:
    """Rollout boundaries b_0 = 0 <= b_1 <= ... <= b_W = n of a contiguous split of kept rollouts with these
    token lengths into ``world`` ranges of ~equal token count: b_k is the rollout boundary whose token prefix is
    nearest to k N / W (ties to the smaller index), made monotone.  Each range then holds N/W +- max_len tokens."""
    import numpy as np
    if world < 1:
        raise ValueError("world must be >= 1")
    lens = np.maximum(np.asarray(lengths, np.int64), 0)
    pre = np.concatenate([[0], np.cumsum(lens)])
    n, N = len(lens), int(pre[-1])
    b = [0]
    for k in range(1, world):
        target = k * N / world
        i = int(np.searchsorted(pre, target, side="left"))   # first prefix >= target
        if i > 0 and (i > n or target - pre[i - 1] <= pre[i] - target):
            i -= 1
        b.append(min(max(i, b[-1]), n))
    b.append(n)
    return b


def reshard_plan(counts, lengths, world: int, rank: int) -> dict:
    """All-to-all split sizes for ``rank``: ``counts[r]`` is rank r's number of kept rollouts (their lengths are
    ``lengths[sum(counts[:r]) : sum(counts[:r+1])]``, i.e. ``lengths`` is the global rank-major list).
    Returns send/recv rollout and token counts per peer, and the balanced token count of every rank."""
    import numpy as np
    lens = np.maximum(np.asarray(lengths, np.int64), 0)
    pre = np.concatenate([[0], np.cumsum(lens)])
    own = np.concatenate([[0], np.cumsum(np.asarray(counts, np.int64))])
    b = balanced_bounds(lens, world)

    def span(lo, hi, k):  # rollouts of [lo, hi) that land on rank k
        a, c = max(lo, b[k]), min(hi, b[k + 1])
        return (a, c) if c > a else (a, a)

    send_r, send_t, recv_r, recv_t = [], [], [], []
    for k in range(world):
        a, c = span(own[rank], own[rank + 1], k)
        send_r.append(int(c - a))
        send_t.append(int(pre[c] - pre[a]))
        a, c = span(own[k], own[k + 1], rank)
        recv_r.append(int(c - a))
        recv_t.append(int(pre[c] - pre[a]))
    return {"bounds": b, "send_rollouts": send_r, "send_tokens": send_t, "recv_rollouts": recv_r,
            "recv_tokens": recv_t, "tokens_after": [int(pre[b[k + 1]] - pre[b[k]]) for k in range(world)],
            "tokens_before": [int(pre[own[k + 1]] - pre[own[k]]) for k in range(world)]}


def exchange(tensors, send_splits, recv_splits, group=None):
    """All-to-all of each 1-D tensor (same split sizes for all of them); returns the received tensors.  Works on
    device tensors with NCCL and on CPU tensors with gloo."""
    out = []
    for t in tensors:
        r = t.new_empty(sum(recv_splits))
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_to_all_single(r, t[: sum(send_splits)].contiguous(), output_split_sizes=list(recv_splits),
                                   input_split_sizes=list(send_splits), group=group)
        else:
            r.copy_(t[: sum(send_splits)])
        out.append(r)
    return out
