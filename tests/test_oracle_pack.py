"""Pins of the oracle's step (1), version-lag filter + pack (PAPER.md :192, :224; SPEC.md :44-49, :341-359).

The pins are (a) the SPEC coordinator / buffer worked examples (tests/golden/lag_filter_examples.json),
(b) a brute-force enumeration written in the replay buffer's own terms -- ``pull(min_version)`` keeps
trajectories with ``param_version >= min_version`` (SPEC.md :344) -- over all 3^4 lag patterns of the
tiny config with ragged lengths, (c) conservation laws, (d) shard invariance.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _batch(lags, lengths, G=4, S=8, V=50, t_train=1000, seed=7):
    R = len(lags) * G
    rng = np.random.default_rng(seed)
    version = np.repeat(t_train - np.asarray(lags, np.int64), G)
    action = rng.integers(0, V, size=(R, S), dtype=np.int32)
    old = -rng.random((R, S), dtype=np.float32)
    ref = -rng.random((R, S), dtype=np.float32)
    return version, np.asarray(lengths, np.int32), action, old, ref


def _brute_force(version, resp_len, action, old, ref, G, S, t_train, max_lag, base=0):
    """Replay-buffer formulation: admit rollouts with version >= min_version = t_train - max_lag, then
    emit (rollout, position) pairs in rollout order."""
    min_version = t_train - max_lag
    kept = [i for i in range(len(version)) if version[i] >= min_version]
    toks = [(k, i, j) for k, i in enumerate(kept) for j in range(resp_len[i])]
    return (np.array([base + i for i in kept], np.int32),
            np.array([k for k, _, _ in toks], np.int32),
            np.array([action[i, j] for _, i, j in toks], np.int32),
            np.array([old[i, j] for _, i, j in toks], np.float32),
            np.array([ref[i, j] for _, i, j in toks], np.float32))


def test_lag_filter_golden_examples():
    ex = json.load(open(os.path.join(GOLD, "lag_filter_examples.json")))["examples"]
    for e in ex:
        version, resp_len, action, old, ref = _batch([e["t_train"] - e["version"]], [3, 3, 3, 3], t_train=e["t_train"])
        out = oracle.pack_batch(version, resp_len, action, old, ref, group_size=4, max_len=8, vocab=50,
                                t_train=e["t_train"], max_lag=e["max_lag"])
        assert out.status == oracle.DATA_OK
        assert (out.n_groups_kept == 1) == e["keep"], e["cite"]


def test_pack_exhaustive_lag_patterns_vs_brute_force():
    rng = np.random.default_rng(3)
    for lags in itertools.product([0, 1, 2], repeat=4):
        lengths = rng.integers(1, 9, size=16)
        version, resp_len, action, old, ref = _batch(lags, lengths)
        out = oracle.pack_batch(version, resp_len, action, old, ref, group_size=4, max_len=8, vocab=50,
                                t_train=1000, max_lag=1)
        kr, ts, ta, to, tr = _brute_force(version, resp_len, action, old, ref, 4, 8, 1000, 1)
        assert out.status == oracle.DATA_OK
        np.testing.assert_array_equal(out.kept_rollout, kr)
        np.testing.assert_array_equal(out.tok_slot, ts)
        np.testing.assert_array_equal(out.tok_action, ta)
        assert out.tok_old.tobytes() == to.tobytes() and out.tok_ref.tobytes() == tr.tobytes()
        # conservation: kept + dropped = R; offsets are the prefix sums of kept lengths
        dropped = sum(4 for l in lags if l > 1)
        assert out.n_rollouts_kept + dropped == 16
        assert out.n_groups_kept == sum(1 for l in lags if l <= 1)
        assert out.kept_offset[0] == 0 and out.kept_offset[-1] == out.n_tokens == len(ts)
        np.testing.assert_array_equal(np.diff(out.kept_offset), resp_len[kr])


def test_boundary_lag_equal_max_kept_and_plus_one_dropped():
    for max_lag in [0, 1, 2, 5]:
        version, resp_len, action, old, ref = _batch([max_lag, max_lag + 1], [2] * 8)
        out = oracle.pack_batch(version, resp_len, action, old, ref, group_size=4, max_len=8, vocab=50,
                                t_train=1000, max_lag=max_lag)
        np.testing.assert_array_equal(out.kept_rollout, [0, 1, 2, 3])


def test_tiny_config_drops_one_group():
    cfg = synth.CONFIGS["tiny"]
    b = synth.make_batch(cfg)
    out = oracle.pack_batch(b.version, b.resp_len, b.action, b.old_logp, b.ref_logp, group_size=cfg.G,
                            max_len=cfg.S, vocab=cfg.V, t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
    assert out.status == 0 and out.n_groups_kept == 3 and out.n_tokens == 768
    np.testing.assert_array_equal(out.kept_rollout, [0, 1, 2, 3, 4, 5, 6, 7, 12, 13, 14, 15])


def test_7b_config_stale_fraction():
    cfg = synth.CONFIGS["qwen2.5-7b"]
    lags = synth.group_lags(cfg)
    assert (lags > cfg.max_lag).sum() == 38 and set(lags[lags > cfg.max_lag]) <= {3, 4}
    assert set(lags[lags <= cfg.max_lag]) <= {0, 1, 2}


@pytest.mark.parametrize("world", [2, 3, 4])
def test_shard_union_equals_whole(world):
    """W-invariance: union of per-shard outputs (global ids via rollout_base) == the W=1 output."""
    rng = np.random.default_rng(11)
    P, G, S = 12, 4, 8
    lags = rng.integers(0, 3, size=P)
    lengths = rng.integers(1, 9, size=P * G)
    version, resp_len, action, old, ref = _batch(lags, lengths, G=G, S=S)
    whole = oracle.pack_batch(version, resp_len, action, old, ref, group_size=G, max_len=S, vocab=50,
                              t_train=1000, max_lag=1)
    parts = []
    for r in range(world):
        g0, g1 = (r * P) // world, ((r + 1) * P) // world
        sl = slice(g0 * G, g1 * G)
        parts.append(oracle.pack_batch(version[sl], resp_len[sl], action[sl], old[sl], ref[sl], group_size=G,
                                       max_len=S, vocab=50, t_train=1000, max_lag=1, rollout_base=g0 * G))
    np.testing.assert_array_equal(np.concatenate([p.kept_rollout for p in parts]), whole.kept_rollout)
    np.testing.assert_array_equal(np.concatenate([p.tok_action for p in parts]), whole.tok_action)
    assert sum(p.n_tokens for p in parts) == whole.n_tokens


def test_errors_and_first_bad_lexicographic():
    version, resp_len, action, old, ref = _batch([0, 0, 0], [4] * 12)
    kw = dict(group_size=4, max_len=8, vocab=50, t_train=1000, max_lag=1)
    v = version.copy(); v[5] = 1001          # future version
    out = oracle.pack_batch(v, resp_len, action, old, ref, **kw)
    assert (out.status, out.first_bad_rollout) == (oracle.DATA_FUTURE_VERSION, 5)
    v = version.copy(); v[6] = 999            # mixed within group 1
    out = oracle.pack_batch(v, resp_len, action, old, ref, **kw)
    assert (out.status, out.first_bad_rollout) == (oracle.DATA_MIXED_GROUP_VERSION, 6)
    L = resp_len.copy(); L[9] = 0             # SPEC.md :39 sequences have length >= 1
    out = oracle.pack_batch(version, L, action, old, ref, **kw)
    assert (out.status, out.first_bad_rollout) == (oracle.DATA_BAD_LENGTH, 9)
    L[9] = 9
    out = oracle.pack_batch(version, L, action, old, ref, **kw)
    assert (out.status, out.first_bad_rollout) == (oracle.DATA_BAD_LENGTH, 9)
    a = action.copy(); a[7, 3] = 50; a[2, 0] = -1
    out = oracle.pack_batch(version, resp_len, a, old, ref, **kw)
    assert (out.status, out.first_bad_rollout) == (oracle.DATA_BAD_ACTION, 2)
    a = action.copy(); a[2, 6] = 99          # beyond L = 4: padding is never read
    out = oracle.pack_batch(version, resp_len, a, old, ref, **kw)
    assert out.status == oracle.DATA_OK
    # lower rollout wins even if its check comes later in the order
    v = version.copy(); v[8] = 1001; a = action.copy(); a[1, 0] = 77
    out = oracle.pack_batch(v, resp_len, a, old, ref, **kw)
    assert (out.status, out.first_bad_rollout) == (oracle.DATA_BAD_ACTION, 1)
    out = oracle.pack_batch(version, resp_len, action, old, ref, token_capacity=47, **kw)
    assert (out.status, out.first_bad_rollout, out.n_tokens) == (oracle.DATA_CAPACITY, -1, 48)
    out = oracle.pack_batch(version, resp_len, action, old, ref, token_capacity=48, **kw)
    assert out.status == oracle.DATA_OK
    with pytest.raises(ValueError):
        oracle.pack_batch(version[:10], resp_len[:10], action[:10], old[:10], ref[:10], **kw)  # R % G != 0
    with pytest.raises(ValueError):
        oracle.pack_batch(version, resp_len, action, old, ref, **{**kw, "group_size": 1})     # SPEC.md :210


def test_empty_batch_and_all_dropped():
    kw = dict(group_size=4, max_len=8, vocab=50, t_train=1000, max_lag=0)
    version, resp_len, action, old, ref = _batch([1, 2], [3] * 8)
    out = oracle.pack_batch(version, resp_len, action, old, ref, **kw)
    assert out.status == 0 and out.n_tokens == 0 and out.n_rollouts_kept == 0
    e = np.zeros((0,), np.int64)
    out = oracle.pack_batch(e, e.astype(np.int32), np.zeros((0, 8), np.int32), np.zeros((0, 8), np.float32),
                            None, **kw)
    assert out.status == 0 and out.n_tokens == 0


def test_staleness_histogram_pins():
    """f3 staleness histogram: brute force per rollout; totals equal the pack's kept / dropped counts; the SPEC
    audit example (sequential mode: every lag 0)."""
    import synth
    rng = np.random.default_rng(11)
    for _ in range(30):
        G = int(rng.integers(1, 5))
        P = int(rng.integers(1, 9))
        S = 16
        t = 100
        lag_g = rng.integers(-1, 7, P)
        version = np.repeat(t - lag_g, G).astype(np.int64)
        resp = rng.integers(-1, S + 3, P * G).astype(np.int32)
        max_lag, nb = int(rng.integers(0, 4)), int(rng.integers(1, 6))
        h = oracle.staleness_histogram(version, resp, group_size=G, max_len=S, t_train=t, max_lag=max_lag, n_bins=nb)
        exp = np.zeros_like(h)
        for i in range(P * G):
            lag = t - version[i]
            kept = (t - version[(i // G) * G]) <= max_lag
            b = 0 if lag < 0 else (lag + 1 if lag < nb else nb + 1)
            exp[0 if kept else 1, b] += 1
            exp[2 if kept else 3, b] += min(max(int(resp[i]), 0), S)
        np.testing.assert_array_equal(h, exp)
        assert h[0].sum() + h[1].sum() == P * G
    # sequential mode (the Qwen3-4B config, max_lag 0): all kept, all in the lag-0 bin, tokens = pack's n_tokens
    cfg = synth.CONFIGS["qwen3-4b"]
    b = synth.make_batch(cfg, 0, 4 * cfg.G)
    h = oracle.staleness_histogram(b.version, b.resp_len, group_size=cfg.G, max_len=cfg.S, t_train=synth.T_TRAIN,
                                   max_lag=cfg.max_lag, n_bins=4)
    assert h[0, 1] == 4 * cfg.G and h[0].sum() == h[0, 1] and h[1].sum() == 0
    pk = oracle.pack_batch(b.version, b.resp_len, b.action, b.old_logp, b.ref_logp, group_size=cfg.G, max_len=cfg.S,
                           vocab=cfg.V, t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
    assert h[2].sum() == pk.n_tokens


def test_rollout_filter_mode_partial_groups():
    """f3 filter_mode 1: rollouts are kept individually (t_train - v_i <= max_lag), mixed-version groups are not an
    error, n_groups_kept counts groups with a survivor; with uniform group versions it equals filter_mode 0."""
    rng = np.random.default_rng(21)
    G, P, S, V, t = 4, 6, 8, 50, 100
    for trial in range(40):
        version = (t - rng.integers(0, 4, P * G)).astype(np.int64)
        if trial % 4 == 0:
            version = np.repeat(version[::G], G)                    # uniform groups
        L = rng.integers(1, S + 1, P * G).astype(np.int32)
        act = rng.integers(0, V, (P * G, S)).astype(np.int32)
        old = rng.normal(size=(P * G, S)).astype(np.float32)
        ml = int(rng.integers(0, 3))
        pk = oracle.pack_batch(version, L, act, old, None, group_size=G, max_len=S, vocab=V, t_train=t, max_lag=ml,
                               filter_mode=1)
        assert pk.status == 0
        keep = (t - version) <= ml
        np.testing.assert_array_equal(pk.kept_rollout, np.nonzero(keep)[0])
        assert pk.n_groups_kept == len(set((np.nonzero(keep)[0] // G).tolist()))
        exp_act = np.concatenate([act[i, :L[i]] for i in np.nonzero(keep)[0]] + [np.zeros(0, np.int32)])
        np.testing.assert_array_equal(pk.tok_action, exp_act)
        h = oracle.staleness_histogram(version, L, group_size=G, max_len=S, t_train=t, max_lag=ml, n_bins=4,
                                       filter_mode=1)
        assert h[0].sum() == keep.sum() and h[2].sum() == pk.n_tokens
        if trial % 4 == 0:
            pk0 = oracle.pack_batch(version, L, act, old, None, group_size=G, max_len=S, vocab=V, t_train=t,
                                    max_lag=ml)
            np.testing.assert_array_equal(pk0.kept_rollout, pk.kept_rollout)
            np.testing.assert_array_equal(pk0.tok_action, pk.tok_action)
            assert pk0.n_groups_kept == pk.n_groups_kept
        else:
            pk0 = oracle.pack_batch(version, L, act, old, None, group_size=G, max_len=S, vocab=V, t_train=t,
                                    max_lag=ml)
            mixed = any(len(set(version[g * G:(g + 1) * G])) > 1 for g in range(P))
            assert (pk0.status == oracle.DATA_MIXED_GROUP_VERSION) == mixed
