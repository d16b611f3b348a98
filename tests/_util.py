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


def coef_slack(ref: oracle.LossOut, old, tok_ref, adv_tok, kl_coef, grad_scale, n_global):
    """Bound on |c_gpu - c_ref| from the fp32 log-prob alone: dc/dlogp = s/N (-A rho [unclipped] - beta e^x),
    x = ref - logp, times |d logp| <= 1e-6 (1 + |logp|) (fp32 log-sum-exp over the row), plus fp32 rounding."""
    rho = np.exp(ref.logp - np.asarray(old, np.float64))
    sens = np.abs(np.asarray(adv_tok, np.float64)) * rho
    if kl_coef > 0:
        sens = sens + kl_coef * np.exp(np.asarray(tok_ref, np.float64) - ref.logp)
    return grad_scale / n_global * sens * 1e-6 * (1 + np.abs(ref.logp)) + 1e-6 * np.abs(ref.coef)


def check_rows(*, d_gpu, logp_gpu, loss_gpu, flags_gpu, ref: oracle.LossOut, dtype: str, clip=(0.2, 0.2),
               old=None, cslack=None, eslack=None, loss_atol=1e-6):
    """Element-wise parity of a set of rows; returns number of gradient rows compared.

    logp: |d| <= 1e-5 + 1e-6 |logp|; l_t: rtol 1e-5 (+1e-6 abs); dlogits (bf16): |d| <= ulp_bf16(d_ref) + 4e-6 |c_t|
    + slack_t (faithful rounding: one of the two bf16 neighbours of the exact value) and the
    north_star bar max|d| <= 2e-3 (checked by the callers at max|d_ref| in [0.25, 0.5));
    (fp32): |d| <= 1e-5 |d_ref| + 4e-6 |c_t| + slack_t, where slack_t (coef_slack) bounds the error the fp32
    log-prob propagates into c_t.  Rows whose reference ratio sits within 1e-5 of a clip boundary decide
    "clipped" in different precisions (fp64 vs fp32): only logp is compared there.  eslack (per element, the
    entropy term's fp32 error bound) and loss_atol widen the bars for the entropy variant.
    """
    logp_gpu = np.asarray(logp_gpu, np.float64)
    assert np.all(np.abs(logp_gpu - ref.logp) <= 1e-5 + 1e-6 * np.abs(ref.logp)), \
        f"logp max err {np.max(np.abs(logp_gpu - ref.logp))}"
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
    c = np.abs(ref.coef[ok])[:, None]
    slack = 0.0 if cslack is None else np.asarray(cslack)[ok][:, None]
    base = bf16_ulp(dr) if dtype == "bf16" else 1e-5 * np.abs(dr)      # faithful bf16 rounding: within 1 ulp
    if eslack is not None:
        slack = slack + np.asarray(eslack)[ok]
    tol = np.broadcast_to(base + 4e-6 * c + slack, d.shape)
    err = np.abs(d - dr)
    bad = err > tol + 1e-30
    if bad.any():
        r, v = np.nonzero(bad)
        i = np.argmax(err[bad] / tol[bad])
        raise AssertionError(f"dlogits: {bad.sum()} elements out of tolerance; worst row {r[i]} col {v[i]}: "
                             f"gpu {d[r[i], v[i]]!r} ref {dr[r[i], v[i]]!r} c {c[r[i], 0]!r} tol {tol[r[i], v[i]]!r}")
    return int(ok.sum()), float(err.max()) if err.size else 0.0
