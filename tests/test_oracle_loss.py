"""Pins of the oracle's steps (3)-(5): log-softmax gather, clipped surrogate + KL, dL/dlogits.

(3) closed forms: uniform rows give logp = -ln V (SPEC.md :202; golden logp_closed_forms.json); a single
    spike Delta gives logp = Delta - ln(e^Delta + V - 1) and p > 0.999 at Delta = 20 (SPEC.md :203);
    softmax normalisation to 1e-12 (SPEC.md :204); row-shift invariance; column-permutation equivariance.
(4) old == new => rho = 1 and pg = -A; clip saturation => zero gradient (SPEC.md :219 objective with
    eps 0.2, :243); ref == logp => kl = 0; linearity in beta and grad_scale.
(5) central finite differences of the loss (h = 1e-4) on >= 200 sampled (t, v) of the tiny config,
    relative error <= 1e-5 (SPEC.md :223, :677); row sums of the gradient vanish; sign pattern.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _one(logits, action, old=0.0, ref=None, adv=1.0, **kw):
    logits = np.asarray(logits, np.float32)
    n = logits.shape[0]
    return oracle.policy_loss(logits, np.full(n, action, np.int32) if np.isscalar(action) else action,
                              np.full(n, old, np.float32), None if ref is None else np.full(n, ref, np.float32),
                              np.zeros(n, np.int32), np.array([adv], np.float32), n_global=kw.pop("n_global", 1.0),
                              **kw)


def test_uniform_rows_logp_is_minus_log_v():
    g = json.load(open(os.path.join(GOLD, "logp_closed_forms.json")))
    for e in g["uniform"]:
        V = e["V"]
        for c in [0.0, 3.5, -17.25]:
            out = _one(np.full((1, V), c), action=V // 3)
            assert abs(out.logp[0] + e["minus_logp"]) <= 4e-15
            # closed-form gradient d_v = c (delta - 1/V)
            cc = out.coef[0]
            expect = -cc / V * np.ones(V)
            expect[V // 3] += cc
            np.testing.assert_allclose(out.dlogits[0], expect, rtol=1e-13, atol=1e-18)
    # bf16 input path decodes identically
    out = oracle.policy_loss(np.zeros((1, 1024), np.uint16), np.array([5], np.int32), np.zeros(1, np.float32), None,
                             np.zeros(1, np.int32), np.ones(1, np.float32), n_global=1.0)
    assert abs(out.logp[0] + math.log(1024)) <= 4e-15


def test_spike_closed_form():
    g = json.load(open(os.path.join(GOLD, "logp_closed_forms.json")))["spike"]
    for V, delta in [(1024, 20.0), (1024, 3.0), (151936, 8.0), (50, -2.0)]:
        z = np.zeros((1, V), np.float32)
        z[0, 7] = delta
        out = _one(z, action=7)
        # stable forms of logp_a = Delta - ln(e^Delta + V - 1) and logp_other = -ln(e^Delta + V - 1)
        lse = max(delta, 0.0) + math.log(math.exp(delta - max(delta, 0.0)) + (V - 1) * math.exp(-max(delta, 0.0)))
        # recursive-summation error bound of sum_v exp(z_v - m): (V - 1) u sum|terms|, u = 2^-53
        tol = 4e-15 * max(1.0, abs(delta)) + (V - 1) * 2.0 ** -53 * 2
        assert abs(out.logp[0] - (delta - lse)) <= tol
        out2 = _one(z, action=8)
        assert abs(out2.logp[0] + lse) <= tol
    z = np.zeros((1, g["V_for_p_gt_0999"]), np.float32)
    z[0, 0] = g["delta"]
    assert math.exp(_one(z, action=0).logp[0]) > g["p_min"]


def test_softmax_normalises_and_row_shift_invariance():
    rng = np.random.default_rng(1)
    V = 1024
    z = (rng.normal(size=(4, V)) * 3).astype(np.float32)
    ps = []
    for a in range(0, V, 97):
        ps.append(math.exp(_one(z[:1], action=a).logp[0]))
    full = np.array([math.exp(_one(z[:1], action=a).logp[0]) for a in range(V)])
    assert abs(full.sum() - 1.0) <= 1e-12
    # integer-valued logits + integer shift are exact in fp32
    zi = np.round(z)
    o1 = _one(zi, action=np.array([1, 2, 3, 4], np.int32))
    o2 = _one(zi + 100.0, action=np.array([1, 2, 3, 4], np.int32))
    np.testing.assert_allclose(o1.logp, o2.logp, rtol=0, atol=1e-12)
    np.testing.assert_allclose(o1.dlogits, o2.dlogits, rtol=0, atol=1e-15)



def test_column_permutation_equivariance():
    """(3)-(5) do not depend on the vocabulary's column order (SURVEY.md §8.3 a3 pin): permuting the columns of a row
    (and mapping the action with it) leaves logp, l_t, c_t and the flags unchanged up to the fp64 summation order
    (V u relative) and permutes the gradient the same way.  A kernel or oracle that indexes a column by its tile
    position instead of its vocabulary id (e.g. a wrong action column, an off-by-one tail) breaks this."""
    rng = np.random.default_rng(11)
    n, V = 6, 1031
    z = (rng.normal(size=(n, V)) * 2).astype(np.float32)
    act = rng.integers(0, V, n).astype(np.int32)
    z[np.arange(n), act] += 6.0
    old = (rng.normal(size=n) * 0.3 - 1.0).astype(np.float32)
    ref = (rng.normal(size=n) * 0.3 - 1.0).astype(np.float32)
    slot = np.arange(n, dtype=np.int32) % 3
    adv = np.array([1.25, -0.5, 0.0], np.float32)
    kw = dict(n_global=float(n), kl_coef=0.3, grad_scale=2.0)
    o1 = oracle.policy_loss(z, act, old, ref, slot, adv, **kw)
    for trial in range(3):
        perm = rng.permutation(V)                 # new column j holds old column perm[j]
        inv = np.argsort(perm)
        o2 = oracle.policy_loss(np.ascontiguousarray(z[:, perm]), inv[act].astype(np.int32), old, ref, slot, adv, **kw)
        tol = V * 2.0 ** -53 * 8
        np.testing.assert_allclose(o2.logp, o1.logp, rtol=tol, atol=tol)
        np.testing.assert_allclose(o2.loss, o1.loss, rtol=tol, atol=tol)
        np.testing.assert_allclose(o2.coef, o1.coef, rtol=tol, atol=1e-300)
        np.testing.assert_array_equal(o2.flags, o1.flags)
        np.testing.assert_allclose(o2.dlogits, o1.dlogits[:, perm], rtol=tol, atol=tol * np.abs(o1.coef).max())
    # a wrong action column is visible: the permuted rows with the UNmapped action give different log-probs
    o3 = oracle.policy_loss(np.ascontiguousarray(z[:, perm]), act, old, ref, slot, adv, **kw)
    assert np.max(np.abs(o3.logp - o1.logp)) > 1.0

def test_old_equals_new_gives_unit_ratio():
    cfg = synth.CONFIGS["tiny"]
    rng = np.random.default_rng(2)
    V, n = cfg.V, 64
    z = (rng.normal(size=(n, V)) * 2).astype(np.float32)
    act = rng.integers(0, V, n).astype(np.int32)
    first = oracle.policy_loss(z, act, np.zeros(n, np.float32), None, np.zeros(n, np.int32), np.ones(1, np.float32),
                               n_global=n)
    # feed the policy's own log-probs back as old_logp (fp32 as the ABI stores them)
    adv = np.array([0.75, -1.5], np.float32)
    slot = (np.arange(n) % 2).astype(np.int32)
    out = oracle.policy_loss(z, act, first.logp.astype(np.float32), None, slot, adv, n_global=n)
    rho = np.exp(out.logp - first.logp.astype(np.float32).astype(np.float64))
    assert np.max(np.abs(rho - 1.0)) < 1e-6
    np.testing.assert_allclose(out.loss, -adv[slot].astype(np.float64) * rho, rtol=1e-14)
    np.testing.assert_allclose(out.coef, -adv[slot].astype(np.float64) * rho / n, rtol=1e-14)
    assert not np.any(out.flags)
    # equal lengths and a zero-mean group advantage => L ~ 0 (SPEC.md :214 centering)
    a, _ = oracle.group_advantage(np.array([1, 0, 0, 1], np.float32), np.arange(4, dtype=np.int32), group_size=4)
    slot4 = np.repeat(np.arange(4), n // 4).astype(np.int32)
    out4 = oracle.policy_loss(z, act, first.logp.astype(np.float32), None, slot4, a, n_global=n)
    assert abs(out4.loss.sum() / n) <= 1e-6 * np.abs(out4.loss).sum() / n


@pytest.mark.parametrize("adv,shift", [(1.0, 0.5), (2.0, 0.25), (-1.0, -0.5), (-0.3, -0.3)])
def test_clip_saturation_zeroes_the_gradient(adv, shift):
    rng = np.random.default_rng(4)
    V, n = 512, 8
    z = (rng.normal(size=(n, V))).astype(np.float32)
    act = rng.integers(0, V, n).astype(np.int32)
    base = oracle.policy_loss(z, act, np.zeros(n, np.float32), None, np.zeros(n, np.int32), np.ones(1, np.float32),
                              n_global=n)
    old = (base.logp - shift).astype(np.float32)      # rho = e^shift: > 1.2 or < 0.8
    out = oracle.policy_loss(z, act, old, None, np.zeros(n, np.int32), np.array([adv], np.float32), n_global=n)
    assert np.all(out.flags == 1)
    assert np.all(out.dlogits == 0.0) and np.all(out.coef == 0.0)
    clip = 1.2 if adv > 0 else 0.8
    np.testing.assert_allclose(out.loss, -adv * clip, rtol=1e-6)
    # the other side of the clip range is NOT clipped: gradient flows
    out2 = oracle.policy_loss(z, act, old, None, np.zeros(n, np.int32), np.array([-adv], np.float32), n_global=n)
    assert np.all(out2.flags == 0) and np.all(out2.coef != 0.0)


def test_kl_zero_at_reference_and_linearity():
    rng = np.random.default_rng(6)
    V, n = 256, 16
    z = (rng.normal(size=(n, V)) * 2).astype(np.float32)
    act = rng.integers(0, V, n).astype(np.int32)
    old = (rng.normal(size=n) * 0.05 - 5).astype(np.float32)
    slot = np.zeros(n, np.int32)
    adv = np.array([0.0], np.float32)
    base = oracle.policy_loss(z, act, old, None, slot, adv, n_global=n)
    ref = base.logp.astype(np.float32)
    out = oracle.policy_loss(z, act, old, ref, slot, adv, n_global=n, kl_coef=0.5)
    # ref is the fp32 image of logp: x = ref - logp = O(1e-7) gives kl = x^2/2 + O(x^3), dkl/dlogp = -x + O(x^2)
    x = ref.astype(np.float64) - base.logp
    # (loss = beta * kl since A = 0; exp(x) - x - 1 cancels to ~1 ulp of 1.0 in fp64)
    assert np.all(np.abs(out.loss - 0.5 * x * x / 2) <= np.abs(x) ** 3 + 4.5e-16)
    assert np.all(np.abs(out.coef * n / 0.5 + x) <= x * x + 1e-30)
    # linear in beta (A = 0 isolates the KL term) and in grad_scale
    ref2 = (base.logp + rng.normal(size=n) * 0.3).astype(np.float32)
    o1 = oracle.policy_loss(z, act, old, ref2, slot, adv, n_global=n, kl_coef=0.25)
    o2 = oracle.policy_loss(z, act, old, ref2, slot, adv, n_global=n, kl_coef=0.5)
    o3 = oracle.policy_loss(z, act, old, ref2, slot, adv, n_global=n, kl_coef=0.5, grad_scale=8.0)
    np.testing.assert_allclose(o2.loss, 2 * o1.loss, rtol=1e-14)
    np.testing.assert_allclose(o2.dlogits, 2 * o1.dlogits, rtol=1e-14, atol=1e-300)
    np.testing.assert_array_equal(o3.dlogits, 8 * o2.dlogits)
    # k3 estimator is non-negative (KL-to-reference)
    assert np.all(o1.loss >= 0)


def _tiny_problem(kl_coef, seed):
    cfg = synth.CONFIGS["tiny"]
    b = synth.make_batch(cfg)
    pk = oracle.pack_batch(b.version, b.resp_len, b.action, b.old_logp, b.ref_logp, group_size=cfg.G, max_len=cfg.S,
                           vocab=cfg.V, t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
    adv, _ = oracle.group_advantage(b.reward, pk.kept_rollout, group_size=cfg.G)
    keys = (pk.kept_rollout[pk.tok_slot].astype(np.int64) * cfg.S
            + (np.arange(pk.n_tokens) - pk.kept_offset[pk.tok_slot]))
    z = synth.logits_rows(keys, pk.tok_action, cfg.V, cfg.seed, "f32")
    rng = np.random.default_rng(seed)
    # widen the ratio spread so clipped and unclipped rows, both signs of A, all occur
    old = (pk.tok_old + rng.normal(size=pk.n_tokens) * 0.3).astype(np.float32)
    return cfg, pk, adv, z, old


@pytest.mark.parametrize("kl_coef,seed", [(0.0, 0), (0.5, 1), (0.001, 2)])
def test_finite_differences_tiny(kl_coef, seed):
    cfg, pk, adv, z, old = _tiny_problem(kl_coef, seed)
    n = pk.n_tokens
    out = oracle.policy_loss(z, pk.tok_action, old, pk.tok_ref, pk.tok_slot, adv, n_global=n, kl_coef=kl_coef,
                             grad_scale=float(n))
    rho = np.exp(out.logp - old.astype(np.float64))
    assert (out.flags & 1).any() and (~out.flags & 1).any()
    rng = np.random.default_rng(100 + seed)
    dmax = np.abs(out.dlogits).max()
    checked = 0
    h = 1e-4
    while checked < 200:
        t = int(rng.integers(0, n))
        if np.min(np.abs(rho[t] - np.array([0.8, 1.2]))) < 1e-2:
            continue                                            # stay away from the clip kinks
        v = int(pk.tok_action[t]) if rng.random() < 0.2 else int(rng.integers(0, cfg.V))
        d = out.dlogits[t, v]
        if abs(d) <= 1e-3 * dmax:
            continue
        row = z[t:t + 1].astype(np.float64)
        args = (pk.tok_action[t:t + 1], old[t:t + 1], None if pk.tok_ref is None else pk.tok_ref[t:t + 1],
                np.zeros(1, np.int32), adv[pk.tok_slot[t]:pk.tok_slot[t] + 1])
        kw = dict(n_global=n, kl_coef=kl_coef, grad_scale=float(n))
        zp, zm = row.copy(), row.copy()
        zp[0, v] += h
        zm[0, v] -= h
        fd = (oracle.scaled_loss(zp, *args, **kw) - oracle.scaled_loss(zm, *args, **kw)) / (2 * h)
        assert abs(fd - d) <= 1e-5 * abs(d), (t, v, fd, d)
        checked += 1


def test_gradient_row_sums_and_signs():
    cfg, pk, adv, z, old = _tiny_problem(0.001, 3)
    n = pk.n_tokens
    out = oracle.policy_loss(z, pk.tok_action, old, pk.tok_ref, pk.tok_slot, adv, n_global=n, kl_coef=0.001)
    c = out.coef
    assert np.all(np.abs(out.dlogits.sum(axis=1)) <= 1e-12 * np.abs(c) + 1e-300)
    nz = c != 0
    rows = np.nonzero(nz)[0]
    a = pk.tok_action[rows]
    assert np.all(np.sign(out.dlogits[rows, a]) == np.sign(c[rows]))
    mask = np.ones_like(out.dlogits[rows], bool)
    mask[np.arange(rows.size), a] = False
    assert np.all(np.sign(out.dlogits[rows][mask]).reshape(rows.size, -1) == -np.sign(c[rows])[:, None])


def test_nonfinite_rows_are_flagged_and_masking_is_allowed():
    V = 64
    z = np.zeros((6, V), np.float32)
    z[0, 3] = np.nan
    z[1, :] = -np.inf
    z[2, 5] = np.inf
    z[3, :10] = -np.inf          # masked vocabulary, action unmasked: fine
    z[4, 20] = -np.inf           # masked action: logp = -inf
    act = np.array([0, 0, 0, 30, 20, 1], np.int32)
    old = np.array([0, 0, 0, 0, 0, -100.0], np.float32)   # row 5: rho = e^{~96} overflows fp32
    out = oracle.policy_loss(z, act, old, None, np.zeros(6, np.int32), np.ones(1, np.float32), n_global=6)
    np.testing.assert_array_equal(out.flags >> 1, [1, 1, 1, 0, 1, 1])
    assert abs(out.logp[3] + math.log(V - 10)) < 1e-14
    assert out.stats[4] == 5 and out.stats[8] == 6


def test_stats_vector():
    cfg, pk, adv, z, old = _tiny_problem(0.001, 4)
    n = pk.n_tokens
    out = oracle.policy_loss(z, pk.tok_action, old, pk.tok_ref, pk.tok_slot, adv, n_global=n, kl_coef=0.001)
    rho = np.exp(out.logp - old.astype(np.float64))
    x = pk.tok_ref.astype(np.float64) - out.logp
    assert out.stats[8] == n and out.stats[3] == (out.flags & 1).sum() and out.stats[4] == 0
    np.testing.assert_allclose(out.stats[[0, 1, 2, 7, 9]],
                               [out.loss.sum(), (out.logp - old).sum(), (np.exp(x) - x - 1).sum(), out.logp.sum(),
                                rho.sum()], rtol=1e-12)
    assert out.stats[5] == rho.min() and out.stats[6] == rho.max()


def test_token_logp_closed_forms():
    """f1 forward-only log-probs: uniform rows (-ln V), single spike, all masked but one column (logp = 0)."""
    for V in (1024, 151936):
        z = np.zeros((3, V), np.float32)
        z[1, 5] = 20.0
        z[2, :] = -np.inf
        z[2, 9] = 1.5
        logp, lse, flags = oracle.token_logp(z, np.array([3, 5, 9], np.int32))
        assert abs(logp[0] + math.log(V)) <= 4e-15 and abs(lse[0] - math.log(V)) <= 4e-15
        lse1 = 20.0 + math.log1p((V - 1) * math.exp(-20.0))
        assert abs(logp[1] - (20.0 - lse1)) <= 4e-15 * 20 + (V - 1) * 2.0 ** -52
        assert logp[2] == 0.0 and lse[2] == 1.5
        assert not flags.any()
    z = np.zeros((2, 64), np.float32)
    z[0, 1] = np.nan
    z[1, :] = -np.inf
    _, _, flags = oracle.token_logp(z, np.array([0, 0], np.int32))
    np.testing.assert_array_equal(flags, [2, 2])
