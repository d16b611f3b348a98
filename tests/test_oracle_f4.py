"""Pins of the oracle's f4 loss variants: KL estimators k1/k2/k3, dual clip, per-token
advantages (tok_adv) and per-token loss weights (tok_weight, e.g. sequence-mean aggregation)."""
import math

import numpy as np
import pytest

import oracle
import synth


def _problem(seed=0, n=48, V=300):
    rng = np.random.default_rng(seed)
    z = (rng.normal(size=(n, V)) * 2).astype(np.float32)
    act = rng.integers(0, V, n).astype(np.int32)
    base = oracle.policy_loss(z, act, np.zeros(n, np.float32), None, np.zeros(n, np.int32), np.ones(1, np.float32),
                              n_global=n)
    old = (base.logp + rng.normal(size=n) * 0.3).astype(np.float32)
    ref = (base.logp + rng.normal(size=n) * 0.5).astype(np.float32)
    slot = (np.arange(n) % 6).astype(np.int32)
    adv = np.array([1.0, -0.5, 0.25, -2.0, 0.0, 1.5], np.float32)
    return z, act, old, ref, slot, adv, base


@pytest.mark.parametrize("est", [oracle.KL_K1, oracle.KL_K2, oracle.KL_K3])
def test_kl_estimator_values(est):
    z, act, old, ref, slot, adv, base = _problem()
    n = len(act)
    zero_adv = np.zeros_like(adv)
    out = oracle.policy_loss(z, act, old, ref, slot, zero_adv, n_global=n, kl_coef=1.0, kl_estimator=est)
    x = ref.astype(np.float64) - out.logp
    expect = {oracle.KL_K1: -x, oracle.KL_K2: 0.5 * x * x, oracle.KL_K3: np.exp(x) - x - 1}[est]
    np.testing.assert_allclose(out.loss, expect, rtol=1e-12, atol=1e-15)
    dexpect = {oracle.KL_K1: np.ones_like(x), oracle.KL_K2: -x, oracle.KL_K3: 1 - np.exp(x)}[est]
    np.testing.assert_allclose(out.coef * n, dexpect, rtol=1e-12, atol=1e-15)
    # k2 and k3 are non-negative; k3 >= k2 - O(x^3) near 0; all vanish at ref == logp
    if est != oracle.KL_K1:
        assert np.all(out.loss >= 0)


def test_dual_clip_caps_negative_advantage_loss():
    z, act, old, ref, slot, adv, base = _problem(1)
    n = len(act)
    A = np.full(1, -2.0, np.float32)
    # rho = e^{1.5} = 4.48 > c = 3 : capped at -A c = 6 with zero gradient
    old2 = (base.logp - 1.5).astype(np.float32)
    out = oracle.policy_loss(z, act, old2, None, np.zeros(n, np.int32), A, n_global=n, clip_dual=3.0)
    np.testing.assert_allclose(out.loss, 6.0, rtol=1e-12)
    assert np.all(out.coef == 0) and np.all(out.dlogits == 0) and np.all(out.flags & 1)
    # rho = e^{0.5} = 1.65 < c: dual clip inactive, the PPO branch applies (A < 0: unclipped above 1 - eps)
    old3 = (base.logp - 0.5).astype(np.float32)
    a = oracle.policy_loss(z, act, old3, None, np.zeros(n, np.int32), A, n_global=n, clip_dual=3.0)
    b = oracle.policy_loss(z, act, old3, None, np.zeros(n, np.int32), A, n_global=n)
    np.testing.assert_array_equal(a.loss, b.loss)
    np.testing.assert_array_equal(a.coef, b.coef)


def test_tok_adv_and_tok_weight_reduce_to_the_defaults():
    z, act, old, ref, slot, adv, base = _problem(2)
    n = len(act)
    a = oracle.policy_loss(z, act, old, ref, slot, adv, n_global=n, kl_coef=0.01)
    b = oracle.policy_loss(z, act, old, ref, slot, adv, n_global=n, kl_coef=0.01, tok_adv=adv[slot],
                           tok_weight=np.full(n, 1.0 / n, np.float32))
    np.testing.assert_array_equal(a.loss, b.loss)
    np.testing.assert_allclose(b.coef, a.coef, rtol=1e-7)             # fp32(1/n) vs 1/n
    assert abs(b.stats[10] - a.stats[0] / n) <= 1e-7 * abs(a.stats[0] / n) + 1e-15


def test_sequence_mean_weights_from_lengths():
    """Sequence-mean aggregation: w_t = 1 / (n_seq L_i) -> the step loss is the mean of per-sequence means."""
    cfg = synth.CONFIGS["tiny"]
    b = synth.make_batch(cfg, lengths="ragged")
    pk = oracle.pack_batch(b.version, b.resp_len, b.action, b.old_logp, b.ref_logp, group_size=cfg.G, max_len=cfg.S,
                           vocab=cfg.V, t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
    adv, _ = oracle.group_advantage(b.reward, pk.kept_rollout, group_size=cfg.G)
    L = np.diff(pk.kept_offset)
    w = (1.0 / (pk.n_rollouts_kept * L[pk.tok_slot])).astype(np.float32)
    keys = (pk.kept_rollout[pk.tok_slot].astype(np.int64) * cfg.S
            + (np.arange(pk.n_tokens, dtype=np.int64) - pk.kept_offset[pk.tok_slot]))
    z = synth.logits_rows(keys, pk.tok_action, cfg.V, cfg.seed, "f32")
    out = oracle.policy_loss(z, pk.tok_action, pk.tok_old, pk.tok_ref, pk.tok_slot, adv, n_global=pk.n_tokens,
                             kl_coef=cfg.kl_coef, tok_weight=w)
    per_seq = [out.loss[pk.kept_offset[k]:pk.kept_offset[k + 1]].mean() for k in range(pk.n_rollouts_kept)]
    assert abs(out.stats[10] - np.mean(per_seq)) <= 1e-6 * max(1e-3, abs(np.mean(per_seq)))


@pytest.mark.parametrize("est,dual,seed", [(oracle.KL_K1, 0.0, 0), (oracle.KL_K2, 3.0, 1), (oracle.KL_K3, 2.0, 2)])
def test_finite_differences_variants(est, dual, seed):
    """Central differences (h = 1e-4) of grad_scale * sum_t w_t l_t against the oracle's dlogits, with per-token
    advantages and weights, a KL estimator and a dual clip (SPEC.md :223 style pin)."""
    rng = np.random.default_rng(50 + seed)
    z, act, old, ref, slot, adv, base = _problem(seed, n=24, V=200)
    n = len(act)
    tok_adv = (rng.normal(size=n) * 1.5).astype(np.float32)
    tok_w = (rng.random(n) + 0.5).astype(np.float32) / n
    kw = dict(n_global=n, kl_coef=0.3, kl_estimator=est, clip_dual=dual, tok_adv=tok_adv, tok_weight=tok_w,
              grad_scale=float(n))
    out = oracle.policy_loss(z, act, old, ref, slot, adv, **kw)
    rho = np.exp(out.logp - old.astype(np.float64))
    dmax = np.abs(out.dlogits).max()
    checked = 0
    for _ in range(4000):
        if checked >= 120:
            break
        t = int(rng.integers(0, n))
        if np.min(np.abs(rho[t] - np.array([0.8, 1.2, dual]))) < 1e-2:
            continue
        v = int(act[t]) if rng.random() < 0.2 else int(rng.integers(0, z.shape[1]))
        d = out.dlogits[t, v]
        if abs(d) <= 1e-3 * dmax:
            continue
        row = z[t:t + 1].astype(np.float64)
        args = (act[t:t + 1], old[t:t + 1], ref[t:t + 1], slot[t:t + 1], adv)
        k2 = dict(kw, tok_adv=tok_adv[t:t + 1], tok_weight=tok_w[t:t + 1])
        zp, zm = row.copy(), row.copy()
        zp[0, v] += 1e-4
        zm[0, v] -= 1e-4
        fd = (oracle.scaled_loss(zp, *args, **k2) - oracle.scaled_loss(zm, *args, **k2)) / 2e-4
        assert abs(fd - d) <= 1e-5 * abs(d), (t, v, fd, d)
        checked += 1
    assert checked >= 60


def test_entropy_closed_forms():
    """H_t = -sum p log p: uniform rows give ln V, a row with one unmasked logit gives 0, a two-point row with
    logits (0, d) gives the binary entropy ln(1 + e^d) - d e^d / (1 + e^d)."""
    V = 97
    n = 3
    z = np.zeros((n, V), np.float32)
    z[1, :] = -np.inf
    z[1, 5] = 3.0
    d = 1.75
    z[2, :] = -np.inf
    z[2, 0], z[2, 1] = 0.0, d
    act = np.array([0, 5, 1], np.int32)
    out = oracle.policy_loss(z, act, np.zeros(n, np.float32), None, np.zeros(n, np.int32), np.zeros(1, np.float32),
                             n_global=n, entropy_coef=0.5)
    assert abs(out.entropy[0] - math.log(V)) <= 1e-13
    assert out.entropy[1] == 0.0
    q = math.exp(d) / (1 + math.exp(d))
    assert abs(out.entropy[2] - (-(1 - q) * math.log(1 - q) - q * math.log(q))) <= 1e-14
    # A = 0, no KL: the loss is -eta H
    np.testing.assert_allclose(out.loss, -0.5 * out.entropy, rtol=0, atol=1e-15)   # 0.5 is exact in fp32
    # the masked columns of the one-hot row get an exactly zero gradient
    assert np.all(out.dlogits[1][np.isinf(z[1])] == 0)


def test_entropy_term_is_additive_and_bounded():
    z, act, old, ref, slot, adv, base = _problem(4)
    n = len(act)
    a = oracle.policy_loss(z, act, old, ref, slot, adv, n_global=n, kl_coef=0.01)
    b = oracle.policy_loss(z, act, old, ref, slot, adv, n_global=n, kl_coef=0.01, entropy_coef=0.05)
    assert np.all(b.entropy >= 0) and np.all(b.entropy <= math.log(z.shape[1]) + 1e-12)
    eta = float(np.float32(0.05))                                # the coefficient crosses the ABI as fp32
    np.testing.assert_allclose(b.loss - a.loss, -eta * b.entropy, rtol=1e-12, atol=1e-14)
    np.testing.assert_array_equal(a.coef, b.coef)               # the (delta - p) coefficient is unchanged
    # each gradient row of the entropy part sums to zero: sum_v p_v (log p_v + H) = -H + H
    np.testing.assert_allclose(b.dlogits.sum(axis=1), 0.0, atol=1e-12)


@pytest.mark.parametrize("seed", [0, 1])
def test_finite_differences_entropy(seed):
    """Central differences of grad_scale * sum_t w_t (pg + beta kl - eta H) against dlogits with eta > 0."""
    rng = np.random.default_rng(70 + seed)
    z, act, old, ref, slot, adv, base = _problem(seed, n=16, V=120)
    n = len(act)
    kw = dict(n_global=n, kl_coef=0.2, entropy_coef=0.3, grad_scale=float(n))
    out = oracle.policy_loss(z, act, old, ref, slot, adv, **kw)
    rho = np.exp(out.logp - old.astype(np.float64))
    dmax = np.abs(out.dlogits).max()
    checked = 0
    for _ in range(3000):
        if checked >= 80:
            break
        t = int(rng.integers(0, n))
        if np.min(np.abs(rho[t] - np.array([0.8, 1.2]))) < 1e-2:
            continue
        v = int(act[t]) if rng.random() < 0.2 else int(rng.integers(0, z.shape[1]))
        d = out.dlogits[t, v]
        if abs(d) <= 1e-3 * dmax:
            continue
        row = z[t:t + 1].astype(np.float64)
        args = (act[t:t + 1], old[t:t + 1], ref[t:t + 1], slot[t:t + 1], adv)
        zp, zm = row.copy(), row.copy()
        zp[0, v] += 1e-4
        zm[0, v] -= 1e-4
        fd = (oracle.scaled_loss(zp, *args, **kw) - oracle.scaled_loss(zm, *args, **kw)) / 2e-4
        assert abs(fd - d) <= 1e-5 * abs(d), (t, v, fd, d)
        checked += 1
    assert checked >= 40


@pytest.mark.parametrize("est,dual,eta", [(oracle.KL_K3, 0.0, 0.0), (oracle.KL_K1, 3.0, 0.02), (oracle.KL_K2, 2.0, 0.1)])
def test_loss_from_logp_equals_the_logits_path(est, dual, eta):
    """(4) restated from log-probs (for f1 / f2, which never hold the logits) equals echo_ref_policy_loss's loss,
    flags and coefficient given the same rows."""
    z, act, old, ref, slot, adv, base = _problem(7)
    n = len(act)
    rng = np.random.default_rng(8)
    tok_adv = (rng.normal(size=n)).astype(np.float32)
    w = (rng.random(n) + 0.5).astype(np.float32) / n
    kw = dict(n_global=n, kl_coef=0.05, kl_estimator=est, clip_dual=dual, tok_adv=tok_adv, tok_weight=w,
              grad_scale=3.0, entropy_coef=eta)
    full = oracle.policy_loss(z, act, old, ref, slot, adv, **kw)
    loss, flags, coef = oracle.loss_from_logp(full.logp, old, ref, slot, adv, tok_entropy=full.entropy, **kw)
    np.testing.assert_array_equal(loss, full.loss)
    np.testing.assert_array_equal(flags, full.flags)
    np.testing.assert_array_equal(coef, full.coef)
