"""Host-side data parallelism (paper_2508_05387_b200.parallel) on CPU: world-size-2 gloo process groups.

The per-rank compute here is the oracle (test infrastructure); what is under test is the product's sharding
(`shard_groups`) and the collectives that combine a step's counts and statistics across ranks
(`allreduce_sum_`, `reduce_loss_stats_`), whose results must equal the single-rank step.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2508_05387_b200.parallel import allreduce_sum_, reduce_loss_stats_, shard_groups


def test_shard_groups_partition():
    for P in (1, 7, 64, 128, 256):
        for W in (1, 2, 3, 4, 8):
            ranges = [shard_groups(P, W, r) for r in range(W)]
            assert ranges[0][0] == 0 and ranges[-1][1] == P
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_groups(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _step_stats(cfg, r0, r1, n_global=None):
    """One rank's step with the oracle: (stats1 without N_global normalisation, loss stats on sampled rows)."""
    b = synth.make_batch(cfg, r0, r1, lengths="ragged")
    pk = oracle.pack_batch(b.version, b.resp_len, b.action, b.old_logp, b.ref_logp, group_size=cfg.G, max_len=cfg.S,
                           vocab=cfg.V, t_train=synth.T_TRAIN, max_lag=cfg.max_lag, rollout_base=r0)
    adv, adv_stats = oracle.group_advantage(b.reward, pk.kept_rollout, group_size=cfg.G, rollout_base=r0)
    n_groups = (r1 - r0) // cfg.G
    stats1 = np.concatenate([[pk.n_tokens], adv_stats, [pk.n_groups_kept, n_groups - pk.n_groups_kept]])
    return pk, adv, stats1


# 16 groups of 4 (f32, V = 1024) with the 7B config's async staleness: 5 of 16 groups dropped, so ranks at W = 4 and 8
# keep uneven token counts (the north_star's 8-GPU split; PAPER.md :224 drops whole groups)
ASYNC16 = synth.Config("async16", 16, 4, 64, 1024, "f32", 2, 0.001, "async", 0, stale_groups=5, lengths="ragged")


def _cfg(name):
    return ASYNC16 if name == "async16" else synth.CONFIGS[name]


def _worker(rank, world, port, cfg_name, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = _cfg(cfg_name)
        g0, g1 = shard_groups(cfg.P, world, rank)
        pk, adv, stats1 = _step_stats(cfg, g0 * cfg.G, g1 * cfg.G)
        s1 = torch.tensor(stats1, dtype=torch.float64)
        allreduce_sum_(s1)
        n_global = float(s1[0])
        keys = (pk.kept_rollout[pk.tok_slot].astype(np.int64) * cfg.S
                + (np.arange(pk.n_tokens, dtype=np.int64) - pk.kept_offset[pk.tok_slot]))
        z = synth.logits_rows(keys, pk.tok_action, cfg.V, cfg.seed, "f32")
        lo = oracle.policy_loss(z, pk.tok_action, pk.tok_old, pk.tok_ref, pk.tok_slot, adv, n_global=n_global,
                                kl_coef=cfg.kl_coef, want_dlogits=False)
        st = torch.tensor(lo.stats, dtype=torch.float64)
        reduce_loss_stats_(st)
        out[rank] = (s1.numpy().copy(), st.numpy().copy(), pk.kept_rollout.copy(), lo.coef.copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name", [(2, "tiny"), (4, "async16"), (8, "async16"), (8, "tiny")])
def test_multi_rank_step_equals_single_rank(world, name):
    """W gloo ranks (W = 8: the north_star's 8-GPU split; with "tiny" at W = 8 half the ranks own no group) give
    the single-rank step's all-reduced counts, loss statistics and per-token coefficients."""
    cfg = _cfg(name)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), name, out), nprocs=world, join=True)
    # single-rank reference
    pk, adv, stats1 = _step_stats(cfg, 0, cfg.R)
    keys = (pk.kept_rollout[pk.tok_slot].astype(np.int64) * cfg.S
            + (np.arange(pk.n_tokens, dtype=np.int64) - pk.kept_offset[pk.tok_slot]))
    z = synth.logits_rows(keys, pk.tok_action, cfg.V, cfg.seed, "f32")
    lo = oracle.policy_loss(z, pk.tok_action, pk.tok_old, pk.tok_ref, pk.tok_slot, adv, n_global=pk.n_tokens,
                            kl_coef=cfg.kl_coef, want_dlogits=False)
    s1_all = [out[r][0] for r in range(world)]
    for s in s1_all:                          # every rank sees the same all-reduced counts
        np.testing.assert_allclose(s, stats1, rtol=1e-12, atol=1e-12)
    st = out[0][1]
    np.testing.assert_allclose(st[[0, 1, 2, 7, 9]], lo.stats[[0, 1, 2, 7, 9]], rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(st[[3, 4, 8]], lo.stats[[3, 4, 8]])
    assert st[5] == lo.stats[5] and st[6] == lo.stats[6]      # min / max exact
    if name == "async16":
        assert stats1[8] == 5 and len({out[r][2].size for r in range(world)}) > 1   # uneven ranks
    # the union of rank outputs is the single-rank output (global ids, W-invariant per-token coefficients)
    np.testing.assert_array_equal(np.concatenate([out[r][2] for r in range(world)]), pk.kept_rollout)
    np.testing.assert_array_equal(np.concatenate([out[r][3] for r in range(world)]), lo.coef)


# ------------------------------------------------------------------------------------------------ f3
from paper_2508_05387_b200.parallel import balanced_bounds, exchange, reshard_plan  # noqa: E402


def test_balanced_bounds_nearest_prefix_and_load_bound():
    rng = np.random.default_rng(3)
    for _ in range(300):
        n = int(rng.integers(0, 40))
        L = rng.integers(0, 50, n)
        W = int(rng.integers(1, 9))
        b = balanced_bounds(L, W)
        pre = np.concatenate([[0], np.cumsum(L)])
        N = pre[-1]
        assert len(b) == W + 1 and b[0] == 0 and b[-1] == n and all(x <= y for x, y in zip(b, b[1:]))
        for k in range(1, W):
            t = k * N / W
            best = np.min(np.abs(pre - t))
            # the boundary's prefix is the nearest one to k N / W unless monotonicity pinned it to b_{k-1}
            assert abs(pre[b[k]] - t) == best or b[k] == b[k - 1]
        loads = [pre[b[k + 1]] - pre[b[k]] for k in range(W)]
        if n:
            assert max(loads) <= N / W + L.max() + 1e-9


def test_reshard_plan_is_a_consistent_all_to_all():
    rng = np.random.default_rng(4)
    for _ in range(100):
        W = int(rng.integers(1, 7))
        counts = rng.integers(0, 9, W)
        L = rng.integers(1, 30, counts.sum())
        plans = [reshard_plan(counts, L, W, r) for r in range(W)]
        for r in range(W):
            for k in range(W):
                assert plans[r]["send_rollouts"][k] == plans[k]["recv_rollouts"][r]
                assert plans[r]["send_tokens"][k] == plans[k]["recv_tokens"][r]
            assert sum(plans[r]["send_rollouts"]) == counts[r]
            assert sum(plans[r]["recv_tokens"]) == plans[0]["tokens_after"][r]
        assert sum(plans[0]["tokens_after"]) == L.sum()


def _rebalance_worker(rank, world, port, cfg_name, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = _cfg(cfg_name)
        g0, g1 = shard_groups(cfg.P, world, rank)
        pk, adv, stats1 = _step_stats(cfg, g0 * cfg.G, g1 * cfg.G)
        s1 = torch.tensor(stats1, dtype=torch.float64)
        allreduce_sum_(s1)
        lens = np.diff(pk.kept_offset[: pk.n_rollouts_kept + 1]).astype(np.int32)
        gathered = [None] * world
        dist.all_gather_object(gathered, lens)
        plan = reshard_plan([len(x) for x in gathered], np.concatenate(gathered), world, rank)
        ro = [torch.from_numpy(pk.kept_rollout[: pk.n_rollouts_kept].copy()), torch.from_numpy(adv.copy()),
              torch.from_numpy(lens)]
        to = [torch.from_numpy(x[: pk.n_tokens].copy()) for x in (pk.tok_action, pk.tok_old, pk.tok_ref)]
        kr, ad, ln = exchange(ro, plan["send_rollouts"], plan["recv_rollouts"])
        ta, told, tref = exchange(to, plan["send_tokens"], plan["recv_tokens"])
        off, slot = oracle.csr_from_lengths(ln.numpy())
        keys = kr.numpy()[slot].astype(np.int64) * cfg.S + (np.arange(len(slot)) - off[slot])
        z = synth.logits_rows(keys, ta.numpy(), cfg.V, cfg.seed, "f32")
        lo = oracle.policy_loss(z, ta.numpy(), told.numpy(), tref.numpy(), slot, ad.numpy(), n_global=float(s1[0]),
                                kl_coef=cfg.kl_coef, want_dlogits=False)
        st = torch.tensor(lo.stats, dtype=torch.float64)
        reduce_loss_stats_(st)
        out[rank] = (plan, kr.numpy().copy(), keys, lo.coef.copy(), st.numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name", [(2, "tiny"), (3, "tiny"), (4, "async16"), (8, "async16")])
def test_rebalanced_step_equals_single_rank(world, name):
    """f3: after the exchange every rank holds a contiguous, token-balanced range of the global kept sequence,
    and the per-token results and step statistics equal the single-rank step's (W up to 8, uneven ranks)."""
    cfg = _cfg(name)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rebalance_worker, args=(world, _free_port(), name, out), nprocs=world, join=True)
    pk, adv, stats1 = _step_stats(cfg, 0, cfg.R)
    keys = (pk.kept_rollout[pk.tok_slot].astype(np.int64) * cfg.S
            + (np.arange(pk.n_tokens, dtype=np.int64) - pk.kept_offset[pk.tok_slot]))
    z = synth.logits_rows(keys, pk.tok_action, cfg.V, cfg.seed, "f32")
    lo = oracle.policy_loss(z, pk.tok_action, pk.tok_old, pk.tok_ref, pk.tok_slot, adv, n_global=pk.n_tokens,
                            kl_coef=cfg.kl_coef, want_dlogits=False)
    plan = out[0][0]
    before, after = plan["tokens_before"], plan["tokens_after"]
    assert max(after) - min(after) <= max(before) - min(before)
    assert max(after) <= pk.n_tokens / world + cfg.S
    np.testing.assert_array_equal(np.concatenate([out[r][1] for r in range(world)]), pk.kept_rollout)
    np.testing.assert_array_equal(np.concatenate([out[r][2] for r in range(world)]), keys)
    np.testing.assert_array_equal(np.concatenate([out[r][3] for r in range(world)]), lo.coef)
    st = out[0][4]
    np.testing.assert_allclose(st[[0, 1, 2, 7, 9]], lo.stats[[0, 1, 2, 7, 9]], rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(st[[3, 4, 8]], lo.stats[[3, 4, 8]])


def test_csr_from_lengths_oracle_matches_pack():
    """The oracle's CSR rebuild reproduces pack's kept_offset / tok_slot from the kept lengths."""
    cfg = synth.CONFIGS["tiny"]
    b = synth.make_batch(cfg, lengths="ragged")
    pk = oracle.pack_batch(b.version, b.resp_len, b.action, b.old_logp, b.ref_logp, group_size=cfg.G, max_len=cfg.S,
                           vocab=cfg.V, t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
    off, slot = oracle.csr_from_lengths(np.diff(pk.kept_offset[: pk.n_rollouts_kept + 1]))
    np.testing.assert_array_equal(off, pk.kept_offset[: pk.n_rollouts_kept + 1])
    np.testing.assert_array_equal(slot, pk.tok_slot[: pk.n_tokens])
    # brute force on small inputs
    rng = np.random.default_rng(9)
    for _ in range(50):
        L = rng.integers(-2, 6, int(rng.integers(0, 12))).astype(np.int32)
        off, slot = oracle.csr_from_lengths(L)
        exp = np.concatenate([[i] * max(int(x), 0) for i, x in enumerate(L)] + [[]]).astype(np.int32)
        np.testing.assert_array_equal(slot, exp)
        assert off[-1] == len(exp) and off[0] == 0
