"""Pins of the oracle's f4 PPO-GAE advantages (rewards / values of PAPER.md :163-164).

Independent formulations: the explicit sum A_t = sum_l (gamma lambda)^l delta_{t+l} (brute force), the
one-step TD error at lambda = 0, the Monte-Carlo return minus the value at gamma = lambda = 1, and returns-to-go
when values are zero."""
import numpy as np
import pytest

import oracle


def _traj(seed, R=6, S=40):
    rng = np.random.default_rng(seed)
    L = rng.integers(1, S + 1, R).astype(np.int32)
    r = rng.normal(size=(R, S)).astype(np.float32)
    v = rng.normal(size=(R, S)).astype(np.float32)
    boot = rng.normal(size=R).astype(np.float32)
    return L, r, v, boot


@pytest.mark.parametrize("gamma,lam", [(0.99, 0.95), (1.0, 1.0), (0.9, 0.0), (0.5, 0.7)])
def test_gae_vs_explicit_sum(gamma, lam):
    L, r, v, boot = _traj(1)
    adv, ret = oracle.gae_advantage(L, r, v, gamma=gamma, lam=lam, bootstrap=boot)
    g, gl = float(np.float32(gamma)), float(np.float32(gamma)) * float(np.float32(lam))
    for i in range(len(L)):
        n = L[i]
        vv = np.append(v[i, :n].astype(np.float64), float(boot[i]))
        delta = r[i, :n].astype(np.float64) + g * vv[1:] - vv[:-1]
        for t in range(n):
            expect = sum(gl ** k * delta[t + k] for k in range(n - t))
            assert abs(adv[i, t] - expect) <= 1e-6 * max(1.0, abs(expect))
            assert abs(ret[i, t] - (expect + vv[t])) <= 1e-6 * max(1.0, abs(expect + vv[t]))
        assert np.all(adv[i, n:] == 0)


def test_gae_special_cases():
    L, r, v, boot = _traj(2)
    # lambda = 0: one-step TD error (bootstrap at the end)
    adv, _ = oracle.gae_advantage(L, r, v, gamma=0.9, lam=0.0, bootstrap=boot)
    for i in range(len(L)):
        n = L[i]
        vn = np.append(v[i, 1:n], boot[i]).astype(np.float64)
        np.testing.assert_allclose(adv[i, :n], r[i, :n] + float(np.float32(0.9)) * vn - v[i, :n], rtol=1e-6, atol=1e-6)
    # gamma = lambda = 1, no bootstrap: Monte-Carlo return-to-go minus the value
    adv, ret = oracle.gae_advantage(L, r, v, gamma=1.0, lam=1.0)
    for i in range(len(L)):
        n = L[i]
        rtg = np.cumsum(r[i, :n][::-1].astype(np.float64))[::-1]
        np.testing.assert_allclose(adv[i, :n], rtg - v[i, :n], rtol=1e-6, atol=1e-5)
        np.testing.assert_allclose(ret[i, :n], rtg, rtol=1e-6, atol=1e-5)
    # zero values: returns are discounted rewards-to-go
    adv, ret = oracle.gae_advantage(L, r, np.zeros_like(v), gamma=0.5, lam=1.0)
    i = 0
    n = L[i]
    expect = [sum(0.5 ** k * float(r[i, t + k]) for k in range(n - t)) for t in range(n)]
    np.testing.assert_allclose(ret[i, :n], expect, rtol=1e-6, atol=1e-6)


def test_pack_carries_aux_payload():
    L, r, v, boot = _traj(3, R=8, S=10)
    version = np.full(8, 1000, np.int64)
    version[4:] = 990                                      # second group stale
    action = np.zeros((8, 10), np.int32)
    aux = np.arange(80, dtype=np.float32).reshape(8, 10)
    pk = oracle.pack_batch(version, L, action, r, None, group_size=4, max_len=10, vocab=5, t_train=1000, max_lag=2,
                           aux=aux)
    expect = np.concatenate([aux[i, :L[i]] for i in range(4)])
    np.testing.assert_array_equal(pk.tok_aux, expect)
