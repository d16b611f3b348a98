"""Pins of the oracle's f2 backward ("backward recomputes to give dhidden and dW"):
D = c (delta - p) + e p (log p + H), dhidden = D W, dweight = D^T h for z = h W^T.

None of these re-types the oracle's formula: the finite differences differentiate the logits-path objective
(oracle.scaled_loss, itself pinned by finite differences in test_oracle_loss.py) composed with a numpy matmul; the
identity head reduces to the logits-path gradient of echo_ref_policy_loss; the zero head has a closed form."""
import math

import numpy as np

import oracle


def _bf16(x):
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def _f(b):
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _case(seed, n, d, V, entropy_coef, kl_coef, grad_scale=1.0):
    rng = np.random.default_rng(seed)
    h = _bf16(rng.normal(size=(n, d)))
    w = _bf16(rng.normal(size=(V, d)) * 1.5 / math.sqrt(d))
    act = rng.integers(0, V, n).astype(np.int32)
    logp, _, ent = oracle.lmhead_logp(h, w, act, want_entropy=True)
    old = (logp + rng.normal(size=n) * 0.1).astype(np.float32)   # ratios near 1: most tokens unclipped
    ref = (logp + rng.normal(size=n) * 0.3).astype(np.float32)
    adv = rng.normal(size=4).astype(np.float32)
    slot = rng.integers(0, 4, n).astype(np.int32)
    kw = dict(n_global=float(n), kl_coef=kl_coef, grad_scale=grad_scale, entropy_coef=entropy_coef)
    _, flags, coef = oracle.loss_from_logp(logp, old, ref, slot, adv, tok_entropy=ent, **kw)
    ecoef = np.full(n, float(np.float32(grad_scale)) * float(np.float32(entropy_coef)) / n)  # the oracle's fp32 knobs
    return h, w, act, old, ref, slot, adv, kw, coef, ecoef, flags


def _objective(hf, wf, act, old, ref, slot, adv, kw):
    return oracle.scaled_loss(hf @ wf.T, act, old, ref, slot, adv, **kw)


def test_finite_differences_dhidden_and_dweight():
    """Central differences of J(h, W) = grad_scale sum_t w_t l_t(h W^T) against dhidden and dweight (KL and entropy
    terms on, so every term of D is exercised)."""
    n, d, V = 6, 12, 40
    h, w, act, old, ref, slot, adv, kw, coef, ecoef, flags = _case(0, n, d, V, entropy_coef=0.05, kl_coef=0.1,
                                                                   grad_scale=0.7)
    assert (flags & 1).sum() < n  # some unclipped tokens carry the surrogate's gradient
    dh, dw = oracle.lmhead_backward(h, w, act, coef, ecoef)
    hf, wf = _f(h), _f(w)
    eps = 1e-6
    rng = np.random.default_rng(1)
    for (t, k) in [(int(rng.integers(n)), int(rng.integers(d))) for _ in range(12)]:
        hp, hm = hf.copy(), hf.copy()
        hp[t, k] += eps
        hm[t, k] -= eps
        fd = (_objective(hp, wf, act, old, ref, slot, adv, kw) - _objective(hm, wf, act, old, ref, slot, adv, kw)) / (
            2 * eps)
        assert abs(fd - dh[t, k]) <= 1e-7 + 1e-5 * abs(fd), (t, k, fd, dh[t, k])
    for (v, k) in [(int(rng.integers(V)), int(rng.integers(d))) for _ in range(12)] + [(int(act[0]), 3)]:
        wp, wm = wf.copy(), wf.copy()
        wp[v, k] += eps
        wm[v, k] -= eps
        fd = (_objective(hf, wp, act, old, ref, slot, adv, kw) - _objective(hf, wm, act, old, ref, slot, adv, kw)) / (
            2 * eps)
        assert abs(fd - dw[v, k]) <= 1e-7 + 1e-5 * abs(fd), (v, k, fd, dw[v, k])


def test_identity_head_is_the_logits_path_gradient():
    """W = I (V = d): z = h, so D must equal echo_ref_policy_loss's dlogits on h as bf16 logits, dhidden = D and
    dweight = D^T h."""
    n, d = 9, 48
    rng = np.random.default_rng(2)
    h = _bf16(rng.normal(size=(n, d)) * 2)
    w = _bf16(np.eye(d))
    act = rng.integers(0, d, n).astype(np.int32)
    old = rng.normal(size=n).astype(np.float32) - 3.0
    adv = rng.normal(size=3).astype(np.float32)
    slot = rng.integers(0, 3, n).astype(np.int32)
    out = oracle.policy_loss(h, act, old, None, slot, adv, n_global=n, dtype=oracle.BF16, entropy_coef=0.02,
                             grad_scale=1.3)
    ecoef = np.full(n, float(np.float32(1.3)) * float(np.float32(0.02)) / n)  # fp32 knobs, widened
    dh, dw, dz = oracle.lmhead_backward(h, w, act, out.coef, ecoef, want_dlogits=True)
    np.testing.assert_allclose(dz, out.dlogits, rtol=0, atol=1e-15)
    np.testing.assert_allclose(dh, out.dlogits, rtol=0, atol=1e-15)
    np.testing.assert_allclose(dw, out.dlogits.T @ _f(h), rtol=1e-12, atol=1e-15)


def test_zero_head_closed_form():
    """W = 0: p = 1/V, the entropy term vanishes (log p + H = 0), dhidden = 0 and
    dweight[v] = sum_t c_t (delta_{v, a_t} - 1/V) h_t."""
    n, d, V = 5, 16, 30
    rng = np.random.default_rng(3)
    h = _bf16(rng.normal(size=(n, d)))
    act = rng.integers(0, V, n).astype(np.int32)
    coef = rng.normal(size=n)
    dh, dw = oracle.lmhead_backward(h, np.zeros((V, d), np.uint16), act, coef, np.full(n, 0.3))
    np.testing.assert_array_equal(dh, 0.0)
    expect = np.zeros((V, d))
    for t in range(n):
        expect[act[t]] += coef[t] * _f(h)[t]
        expect -= coef[t] / V * _f(h)[t]
    np.testing.assert_allclose(dw, expect, rtol=1e-12, atol=1e-14)


def test_dweight_columns_sum_to_zero():
    """Every row of D sums to zero (sum_v (delta - p) = 0 and sum_v p (log p + H) = 0), so sum_v dweight[v, :] = 0."""
    h, w, act, *_rest, coef, ecoef, _ = _case(4, 7, 20, 64, entropy_coef=0.1, kl_coef=0.0)
    _, dw, dz = oracle.lmhead_backward(h, w, act, coef, ecoef, want_dlogits=True)
    np.testing.assert_allclose(dz.sum(axis=1), 0.0, atol=1e-15)
    np.testing.assert_allclose(dw.sum(axis=0), 0.0, atol=1e-14)
