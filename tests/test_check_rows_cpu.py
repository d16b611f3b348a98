"""The dlogits parity bar itself (tests/_util.check_rows), on the CPU: a faithfully rounded copy of the oracle's own
gradient passes it, and plausible kernel mistakes in the bulk of a Qwen-vocabulary row fail it."""
import numpy as np
import pytest

import oracle
import synth
from _util import check_rows, coef_sens, oracle_step, host_rows, pow2_scale_for


def _rne_bf16(x):
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    b = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


@pytest.fixture(scope="module")
def case():
    cfg = synth.CONFIGS["qwen3-4b"]
    b = synth.make_batch(cfg, 0, 2 * cfg.G)
    o = oracle_step(cfg, b)
    rows = np.arange(12)
    z = host_rows(cfg, o.keys[rows], o.pk.tok_action[rows])
    args = (o.pk.tok_action[rows], o.pk.tok_old[rows], o.pk.tok_ref[rows], o.pk.tok_slot[rows], o.adv)
    N = o.pk.n_tokens
    probe = oracle.policy_loss(z, *args, n_global=N, kl_coef=cfg.kl_coef)
    s = pow2_scale_for(np.abs(probe.dlogits).max())
    ref = oracle.policy_loss(z, *args, n_global=N, kl_coef=cfg.kl_coef, grad_scale=s)
    kw = dict(logp_gpu=ref.logp.astype(np.float32), loss_gpu=ref.loss.astype(np.float32), flags_gpu=ref.flags,
              ref=ref, dtype="bf16", old=o.pk.tok_old[rows],
              sens=coef_sens(ref, o.pk.tok_old[rows], o.pk.tok_ref[rows], o.adv[o.pk.tok_slot[rows]], cfg.kl_coef, s,
                             N))
    c = ref.coef[:, None]
    pv = np.where(c != 0, np.abs(ref.dlogits / np.where(c != 0, c, 1.0)), 0.0)
    return ref, kw, pv


def test_faithful_rounding_passes(case):
    ref, kw, _ = case
    check_rows(d_gpu=_rne_bf16(ref.dlogits), label="oracle rounded to bf16", **kw)
    # round toward zero is faithful too (the other bf16 neighbour)
    t = (np.asarray(ref.dlogits, np.float32).view(np.uint32) & 0xFFFF0000).view(np.float32)
    check_rows(d_gpu=t.astype(np.float64), label="oracle truncated to bf16", **kw)


@pytest.mark.parametrize("mutation", ["zero_small", "all_zero", "scale_mid", "fp16_flush", "wrong_sign_small",
                                      "coef_off"])
def test_mutations_fail(case, mutation):
    ref, kw, pv = case
    d = _rne_bf16(ref.dlogits)
    if mutation == "zero_small":          # entries with p_v < 1e-5 dropped: the bulk of every row
        m = np.where(pv < 1e-5, 0.0, d)
    elif mutation == "all_zero":
        m = np.zeros_like(d)
    elif mutation == "scale_mid":         # a relative 2^-6 error (> 1 bf16 ulp) on the entries with p_v >= 1e-4
        m = np.where((pv >= 1e-4) & (pv < 0.5), d * (1 + 2.0 ** -6), d)
    elif mutation == "fp16_flush":        # exp(z - m) cached in fp16 with subnormals flushed (below 2^-14 of the max)
        m = np.where(pv < 2.0 ** -14 * pv.max(axis=1, keepdims=True), 0.0, d)
    elif mutation == "wrong_sign_small":  # a sign slip on the small entries
        m = np.where(pv < 1e-5, -d, d)
    else:                                 # c_t off by a relative 2^-6 in every element
        m = _rne_bf16(ref.dlogits * (1 + 2.0 ** -6))
    with pytest.raises(AssertionError):
        check_rows(d_gpu=m, label=mutation, **kw)
