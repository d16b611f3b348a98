"""Pins of the oracle's step (2), GRPO group-relative advantage (SPEC.md :206-214, :238; PAPER.md :374).

SPEC.md's worked examples (tests/golden/advantage_examples.json), the G = 2 closed form, the
sqrt(G-1) bound, shift invariance / positive-scale equivariance (SPEC.md :238) and a brute-force check
against numpy's population mean/std on 10^3 random groups (SPEC.md :677, <= 1e-10).
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def adv64(returns, eps=1e-8):
    r = np.asarray(returns, np.float32)
    G = r.shape[0]
    a32, stats, a64 = oracle.group_advantage(r, np.arange(G, dtype=np.int32), group_size=G, eps=eps, want_f64=True)
    return a32, stats, a64


def test_spec_worked_examples():
    ex = json.load(open(os.path.join(GOLD, "advantage_examples.json")))
    for e in ex["examples"]:
        a32, _, a64 = adv64(e["returns"], ex["eps"])
        if "expect" in e:
            if e["abs_tol"] == 0.0:
                assert np.all(a32 == 0.0) and np.all(a64 == 0.0), e["cite"]
            else:
                np.testing.assert_allclose(a64, e["expect"], atol=e["abs_tol"], rtol=0, err_msg=e["cite"])
        if "expect_sum" in e:
            assert abs(a64.sum() - e["expect_sum"]) <= e["sum_tol"], e["cite"]


def test_zero_variance_is_exact_zero_without_special_case():
    for v in [0.1, 0.3, 0.7, 1.0 / 3.0, -2.5, 10.0]:
        for G in [2, 4, 8, 16]:
            a32, stats, a64 = adv64([v] * G)
            assert np.all(a64 == 0.0) and stats[4] == 1.0


def test_closed_form_g2():
    rng = np.random.default_rng(0)
    for _ in range(200):
        r = rng.normal(size=2).astype(np.float32)
        _, _, a = adv64(r)
        sigma = abs(float(r[1]) - float(r[0])) / 2.0
        expect = sigma / (sigma + float(np.float32(1e-8)))
        s = np.sign(float(r[1]) - float(r[0]))
        np.testing.assert_allclose(a, [-s * expect, s * expect], rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("G", [2, 4, 8, 16])
def test_brute_force_vs_numpy_and_bound(G):
    rng = np.random.default_rng(G)
    for _ in range(1000 // G + 50):
        r = (rng.normal(size=G) * rng.choice([0.1, 1.0, 10.0])).astype(np.float32)
        a32, _, a = adv64(r)
        x = r.astype(np.float64)
        ref = (x - np.mean(x)) / (np.std(x, ddof=0) + float(np.float32(1e-8)))
        assert np.max(np.abs(a - ref)) <= 1e-10
        assert np.all(np.abs(a) <= np.sqrt(G - 1) + 1e-12)
        assert abs(a.sum()) <= 1e-9
        np.testing.assert_array_equal(a32, a.astype(np.float32))


def test_shift_invariance_and_scale_equivariance():
    rng = np.random.default_rng(5)
    eps = float(np.float32(1e-8))
    for _ in range(100):
        r = rng.integers(-8, 9, size=8).astype(np.float32)
        if np.all(r == r[0]):
            continue
        _, _, a = adv64(r)
        _, _, a_shift = adv64(r + np.float32(3.0))
        np.testing.assert_allclose(a_shift, a, rtol=0, atol=1e-14)
        k = 4.0
        _, _, a_scale = adv64(r * np.float32(k))
        sigma = np.std(r.astype(np.float64))
        np.testing.assert_allclose(a_scale, a * k * (sigma + eps) / (k * sigma + eps), rtol=1e-13, atol=1e-15)


def test_stats_and_multi_group_layout():
    rng = np.random.default_rng(9)
    G, n_groups = 8, 10
    reward = (rng.random(G * n_groups) < 0.5).astype(np.float32)
    kept = np.arange(G * n_groups, dtype=np.int32)
    a, stats = oracle.group_advantage(reward, kept, group_size=G)
    per = [adv64(reward[g * G:(g + 1) * G])[0] for g in range(n_groups)]
    np.testing.assert_array_equal(a, np.concatenate(per))
    assert stats[5] == G * n_groups
    assert stats[2] == reward.sum() and stats[3] == (reward.astype(np.float64) ** 2).sum()
    assert stats[4] == sum(1 for g in range(n_groups) if np.all(reward[g * G:(g + 1) * G] == reward[g * G]))
    np.testing.assert_allclose(stats[1], (a.astype(np.float64) ** 2).sum(), rtol=1e-14)
    # kept_rollout with a base offset addresses the local reward table
    a2, _ = oracle.group_advantage(reward[G:], kept[:G] + 104, group_size=G, rollout_base=104)
    np.testing.assert_array_equal(a2, a[G:2 * G])


def test_invalid_group():
    with pytest.raises(ValueError):
        oracle.group_advantage(np.zeros(3, np.float32), np.arange(3, dtype=np.int32), group_size=1)


def test_partial_groups_use_their_survivors():
    """f3 partial groups (pack filter_mode 1): a group is the run of kept rollouts with the same rollout / G and
    its statistics use the n_g survivors; a lone survivor gets A = 0; whole groups are unchanged."""
    rng = np.random.default_rng(12)
    G = 4
    reward = rng.random(6 * G).astype(np.float32)
    kept = np.array([0, 1, 3, 4, 5, 6, 7, 9, 16, 17, 18, 21], np.int32)   # runs: {0,1,3} {4..7} {9} {16,17,18} {21}
    a, stats = oracle.group_advantage(reward, kept, group_size=G)
    runs = [[0, 1, 3], [4, 5, 6, 7], [9], [16, 17, 18], [21]]
    exp = np.concatenate([adv64(reward[r])[0] if len(r) > 1 else np.zeros(1, np.float32) for r in runs])
    np.testing.assert_array_equal(a, exp)
    assert a[kept.tolist().index(9)] == 0.0 and a[kept.tolist().index(21)] == 0.0
    assert stats[4] == 2 and stats[5] == len(kept)                          # two singleton runs have std 0
    full, _ = oracle.group_advantage(reward, np.arange(6 * G, dtype=np.int32), group_size=G)
    np.testing.assert_array_equal(a[3:7], full[4:8])                        # the whole group {4..7}
