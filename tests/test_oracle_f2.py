"""Pins of the oracle's f2 fused LM-head log-prob: z = h W^T, logp = z_a - logsumexp(z)."""
import math

import numpy as np

import oracle


def _bf16(x):
    """Round-to-nearest-even fp32 -> bf16 bit patterns."""
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def _f(b):
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def test_identity_head_reduces_to_token_logp():
    """W = I (V = d): z = h, so the fused log-prob equals the plain log-softmax-and-gather of h as logits."""
    rng = np.random.default_rng(0)
    n, d = 17, 96
    h = _bf16(rng.normal(size=(n, d)) * 3)
    w = _bf16(np.eye(d))
    act = rng.integers(0, d, n).astype(np.int32)
    logp, lse = oracle.lmhead_logp(h, w, act)
    lp2, lse2, _ = oracle.token_logp(h, act, vocab=d, dtype=oracle.BF16)
    np.testing.assert_allclose(logp, lp2, rtol=0, atol=1e-13)
    np.testing.assert_allclose(lse, lse2, rtol=0, atol=1e-13)


def test_zero_head_gives_minus_log_v():
    n, d, V = 5, 64, 1000
    h = _bf16(np.random.default_rng(1).normal(size=(n, d)))
    logp, lse = oracle.lmhead_logp(h, np.zeros((V, d), np.uint16), np.arange(n, dtype=np.int32))
    np.testing.assert_allclose(logp, -math.log(V), rtol=0, atol=1e-13)


def test_brute_force_matmul_and_log_softmax():
    """Small cases against numpy's fp64 matmul followed by the log-softmax formula."""
    rng = np.random.default_rng(2)
    for n, d, V in ((3, 8, 5), (9, 33, 70), (4, 128, 257)):
        h = _bf16(rng.normal(size=(n, d)))
        w = _bf16(rng.normal(size=(V, d)) * 2 / math.sqrt(d))
        act = rng.integers(0, V, n).astype(np.int32)
        z = _f(h) @ _f(w).T
        m = z.max(axis=1, keepdims=True)
        lse = (m + np.log(np.exp(z - m).sum(axis=1, keepdims=True)))[:, 0]
        logp, lse_o = oracle.lmhead_logp(h, w, act)
        np.testing.assert_allclose(lse_o, lse, rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(logp, z[np.arange(n), act] - lse, rtol=1e-13, atol=1e-13)


def test_probabilities_sum_to_one():
    rng = np.random.default_rng(3)
    n, d, V = 2, 64, 300
    h = _bf16(rng.normal(size=(n, d)))
    w = _bf16(rng.normal(size=(V, d)) * 0.3)
    tot = np.zeros(n)
    for a in range(V):
        lp, _ = oracle.lmhead_logp(h, w, np.full(n, a, np.int32))
        tot += np.exp(lp)
    np.testing.assert_allclose(tot, 1.0, rtol=0, atol=1e-12)


def test_entropy_of_the_fused_head():
    """f2 entropy: identity head = the entropy of softmax(h) (the f4 oracle on h as logits); zero head = ln V."""
    rng = np.random.default_rng(5)
    n, d = 7, 64
    h = _bf16(rng.normal(size=(n, d)) * 2)
    act = rng.integers(0, d, n).astype(np.int32)
    _, _, ent = oracle.lmhead_logp(h, _bf16(np.eye(d)), act, want_entropy=True)
    out = oracle.policy_loss(h, act, np.zeros(n, np.float32), None, np.zeros(n, np.int32), np.zeros(1, np.float32),
                             n_global=n, dtype=oracle.BF16, entropy_coef=0.5)
    np.testing.assert_allclose(ent, out.entropy, rtol=0, atol=1e-12)
    _, _, ent0 = oracle.lmhead_logp(h, np.zeros((300, d), np.uint16), act, want_entropy=True)
    np.testing.assert_allclose(ent0, math.log(300), rtol=0, atol=1e-12)
