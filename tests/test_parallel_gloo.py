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


def _worker(rank, world, port, cfg_name, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.CONFIGS[cfg_name]
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


@pytest.mark.parametrize("world", [2])
def test_two_rank_step_equals_single_rank(world):
    cfg = synth.CONFIGS["tiny"]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), "tiny", out), nprocs=world, join=True)
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
    # the union of rank outputs is the single-rank output (global ids, W-invariant per-token coefficients)
    np.testing.assert_array_equal(np.concatenate([out[r][2] for r in range(world)]), pk.kept_rollout)
    np.testing.assert_array_equal(np.concatenate([out[r][3] for r in range(world)]), lo.coef)
