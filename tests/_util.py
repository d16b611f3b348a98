"""Shared helpers for the parity tests (CUDA path via the C ABI vs. the CPU oracle on the same seeded inputs)."""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

import oracle
import synth


def bf16_ulp(x):
    """ulp of bf16 values (8 significant bits)."""
    x = np.abs(np.asarray(x, np.float64))
    e = np.floor(np.log2(np.maximum(x, 2.0 ** -126)))
    return 2.0 ** (e - 7)


def pow2_scale_for(max_abs_d_at_unit_scale: float) -> float:
    """Power-of-two grad_scale s with max|d| in [0.25, 0.5) (makes the 2e-3 bar meaningful)."""
    if max_abs_d_at_unit_scale == 0:
        return 1.0
    return 2.0 ** (math.floor(math.log2(0.5 / max_abs_d_at_unit_scale)))


@dataclass
class OracleStep:
    pk: oracle.PackOut
    adv: np.ndarray
    adv_stats: np.ndarray
    keys: np.ndarray          # global token key per packed token


def oracle_step(cfg: synth.Config, b: synth.Batch, rollout_base=0) -> OracleStep:
    pk = oracle.pack_batch(b.version, b.resp_len, b.action, b.old_logp, b.ref_logp, group_size=cfg.G, max_len=cfg.S,
                           vocab=cfg.V, t_train=synth.T_TRAIN, max_lag=cfg.max_lag, rollout_base=rollout_base)
    adv, st = oracle.group_advantage(b.reward, pk.kept_rollout, group_size=cfg.G, rollout_base=rollout_base)
    keys = (pk.kept_rollout[pk.tok_slot].astype(np.int64) * cfg.S
            + (np.arange(pk.n_tokens, dtype=np.int64) - pk.kept_offset[pk.tok_slot]))
    return OracleStep(pk, adv, st, keys)


def host_rows(cfg: synth.Config, keys, actions):
    """Logits rows from the numpy twin of the GPU generator: uint16 bf16 bits or float32."""
    return synth.logits_rows(keys, actions, cfg.V, cfg.seed, "bf16" if cfg.dtype == "bf16" else "f32")


def coef_sens(ref: oracle.LossOut, old, tok_ref, adv_tok, kl_coef, grad_scale, n_global=None, tok_weight=None,
              kl_estimator=oracle.KL_K3):
    """(|dc/dlogp|, cmag) per row, from the oracle's fp64 values.

    c_t = s w_t ([unclipped] (-A rho) + beta dkl/dlogp), rho = e^(logp - old)  (echo_ref_policy_loss, SPEC.md :219)
      dc/dlogp = s w_t ([unclipped] (-A rho) + beta d2kl/dlogp2),  d2kl/dlogp2 = e^(ref - logp) (k3), 0 (k1), 1 (k2)
    On a clipped row (oracle flags bit 0: PPO clip or dual clip) the surrogate contributes no gradient, so its term is
    dropped.  cmag = s w_t (|A| rho [unclipped] + beta |dkl/dlogp|) >= |c_t| bounds the terms the fp32 epilogue adds
    (its rounding error is <= 2^-20 cmag)."""
    logp = ref.logp
    rho = np.exp(logp - np.asarray(old, np.float64))
    uncl = (ref.flags & 1) == 0
    A = np.abs(np.asarray(adv_tok, np.float64))
    w = (1.0 / float(n_global)) if tok_weight is None else np.asarray(tok_weight, np.float64)
    sens = np.where(uncl, A * rho, 0.0)
    mag = sens.copy()
    if kl_coef > 0:
        x = np.asarray(tok_ref, np.float64) - logp
        if kl_estimator == oracle.KL_K3:
            sens = sens + kl_coef * np.exp(x)
            mag = mag + kl_coef * np.abs(1.0 - np.exp(x))
        elif kl_estimator == oracle.KL_K2:
            sens = sens + kl_coef
            mag = mag + kl_coef * np.abs(x)
        else:
            mag = mag + kl_coef
    return grad_scale * w * sens, grad_scale * w * mag


def check_rows(*, d_gpu, logp_gpu, loss_gpu, flags_gpu, ref: oracle.LossOut, dtype: str, clip=(0.2, 0.2),
               old=None, sens=None, eslack=None, loss_atol=1e-6, p=None, action=None, label=""):
    """Element-wise parity of a set of rows (SURVEY.md §8.3 tolerances); returns (rows compared, max |err| / |c_t|).

    logp: |d| <= 1e-5 + 1e-6 |logp|;  l_t: rtol 1e-5 (+ loss_atol);  flags equal.
    dlogits, per element (d_ref = c_t (delta_{v,a} - p_v), p_v = exp(z_v - lse) in fp64):
        |d_gpu - d_ref| <= base(d_ref) + 2^-20 cmag_t + dc_t |delta_{v,a} - p_v| + |c_t| p_v dlse_t (+ eslack)
      base = 1 bf16 ulp(d_ref) (faithful rounding: one of the two bf16 neighbours of the exact value) or 1e-5 |d_ref|
      (fp32 logits); dlse_t = |logp_gpu - logp_ref| + 2^-22 (1 + |lse|) is the row's measured log-sum-exp error (z_a
      is exact, so lse errs by what logp errs) plus the rounding of the fp32 exponent arguments (z - lse) log2e, whose
      terms are |lse|-sized; it moves p_v by p_v dlse_t; dc_t = sens_t dlse_t is what that error
      does to c_t through the ratio and the KL term (coef_sens), reaching column v through |delta_{v,a} - p_v| only.
    Consistency (the a5 pin -d/c = exp(z - lse); rows with c_t != 0 and no entropy term): for v != a_t
      with p_v >= 2^-14 max_v p_v,   |(-d_v / c_t) - p_v| <= (2^-7 + dc_t / |c_t| + dlse_t) p_v.
    p / action: the rows' fp64 probabilities and actions; without them (no entropy term) they are recovered from the
    oracle's own gradient, -d_ref / c_t = p_v (v != a) or p_a - 1 (v = a); rows with c_t = 0 take |delta - p| <= 1.
    Rows whose reference ratio sits within 1e-5 of a clip boundary decide "clipped" in different precisions (fp64 vs
    fp32): only logp is compared there.  eslack (per element) widens the bar for the entropy term."""
    logp_gpu = np.asarray(logp_gpu, np.float64)
    lerr = np.abs(logp_gpu - ref.logp)
    assert np.all(lerr <= 1e-5 + 1e-6 * np.abs(ref.logp)), f"logp max err {np.max(lerr)}"
    rho = np.exp(ref.logp - np.asarray(old, np.float64))
    near = (np.abs(rho - (1 - clip[0])) < 1e-5) | (np.abs(rho - (1 + clip[1])) < 1e-5)
    ok = ~near & ((ref.flags & 2) == 0)
    np.testing.assert_array_equal(np.asarray(flags_gpu)[ok], ref.flags[ok])
    loss_gpu = np.asarray(loss_gpu, np.float64)
    lt = loss_atol if np.isscalar(loss_atol) else np.asarray(loss_atol)[ok]
    assert np.all(np.abs(loss_gpu - ref.loss)[ok] <= 1e-5 * np.abs(ref.loss[ok]) + lt), \
        f"loss max err {np.max(np.abs(loss_gpu - ref.loss)[ok])}"
    d = np.asarray(d_gpu, np.float64)[ok]
    dr = ref.dlogits[ok]
    if d.size == 0:
        return 0, 0.0
    c = ref.coef[ok][:, None]
    ca = np.abs(c)
    has_c = ca > 0
    cs = np.where(has_c, c, 1.0)
    # fp32 exponent arguments (z - lse) log2e are formed from |lse|-sized terms: 2^-22 (1 + |lse|) bounds their rounding
    lse_mag = np.abs(ref.lse) if ref.lse is not None else np.abs(ref.logp)
    lse_mag = np.where(np.isfinite(lse_mag), lse_mag, 0.0)
    dlse = (lerr + 2.0 ** -22 * (1 + lse_mag))[ok][:, None]
    if sens is None:
        sens_t, cmag = np.zeros_like(ca), ca
    else:
        sens_t, cmag = (np.asarray(x, np.float64)[ok][:, None] for x in sens)
    dc = sens_t * dlse
    if p is None:
        q = -dr / cs
        onehot = has_c & (q < 0)
        pv = np.where(has_c, np.where(onehot, q + 1.0, q), 0.0)
        dist = np.where(has_c, np.abs(onehot - pv), 1.0)
    else:
        pv = np.asarray(p, np.float64)[ok]
        onehot = np.zeros(pv.shape, bool)
        onehot[np.arange(pv.shape[0]), np.asarray(action)[ok]] = True
        dist = np.abs(onehot - pv)
    base = bf16_ulp(dr) if dtype == "bf16" else 1e-5 * np.abs(dr)
    tol = base + 2.0 ** -20 * cmag + dc * dist + ca * pv * dlse
    if eslack is not None:
        tol = tol + np.asarray(eslack)[ok]
    err = np.abs(d - dr)
    bad = err > tol + 1e-30
    if bad.any():
        r, v = np.nonzero(bad)
        i = np.argmax(err[bad] / tol[bad])
        raise AssertionError(f"dlogits: {bad.sum()} elements out of tolerance; worst row {r[i]} col {v[i]}: "
                             f"gpu {d[r[i], v[i]]!r} ref {dr[r[i], v[i]]!r} c {c[r[i], 0]!r} tol {tol[r[i], v[i]]!r}")
    n_cons = 0
    if eslack is None:
        pmax = np.max(pv, axis=1, keepdims=True)
        sel = has_c & ~onehot & (pv > 0) & (pv >= 2.0 ** -14 * pmax)
        n_cons = int(sel.sum())
        if n_cons:
            ratio = -d / cs
            ctol = (2.0 ** -7 + dc / np.where(has_c, ca, 1.0) + dlse) * pv
            cbad = sel & (np.abs(ratio - pv) > ctol)
            assert not cbad.any(), (f"consistency -d/c vs p: {cbad.sum()} elements off; worst relative "
                                    f"{np.max(np.abs(ratio - pv)[cbad] / pv[cbad]):.3e}")
    rel = float(np.max(np.where(has_c, err / np.where(has_c, ca, 1.0), 0.0)))
    print(f"[check_rows{(' ' + label) if label else ''}] rows {int(ok.sum())}  max|err| {err.max():.3e}  "
          f"max|err|/|c_t| {rel:.3e}  consistency-checked {n_cons}")
    return int(ok.sum()), rel
