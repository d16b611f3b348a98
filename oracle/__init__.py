"""CPU oracle for the Echo learner hot path (arXiv 2508.05387) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import this package.  The product package ``paper_2508_05387_b200`` never imports it and the
two share no code.  The arithmetic lives in ``echo_oracle.c`` (plain fp64 C loops, one function per
step of the path, each citing the PAPER.md / SPEC.md passage it follows); this module only builds that
file with gcc and marshals numpy arrays into it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "echo_oracle.c")
_LIB = os.path.join(_HERE, "libecho_oracle.so")

DATA_OK, DATA_FUTURE_VERSION, DATA_MIXED_GROUP_VERSION, DATA_BAD_LENGTH, DATA_BAD_ACTION, DATA_CAPACITY = range(6)
F32, BF16 = 0, 1


def build(force: bool = False) -> str:
    """Compile echo_oracle.c (gcc, -O2, OpenMP, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
                               "-fno-fast-math", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _PackResult(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("first_bad_rollout", ctypes.c_int32),
                ("n_groups_kept", ctypes.c_int32), ("n_rollouts_kept", ctypes.c_int32),
                ("n_tokens", ctypes.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i32, i64, f32, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_double
        _lib.echo_ref_pack_batch.argtypes = [i32, i32, i32, i32, i64, i32, i64, P, P, P, P, P, P, i64,
                                             P, P, P, P, P, P, P, ctypes.POINTER(_PackResult), i32]
        _lib.echo_ref_gae_advantage.argtypes = [i32, i32, P, P, P, P, f32, f32, P, P]
        _lib.echo_ref_gae_advantage.restype = ctypes.c_int
        _lib.echo_ref_pack_batch.restype = ctypes.c_int
        _lib.echo_ref_group_advantage.argtypes = [i32, i32, f32, P, P, i64, P, P, P]
        _lib.echo_ref_group_advantage.restype = ctypes.c_int
        _lib.echo_ref_policy_loss.argtypes = [i64, i32, i64, i32, P, P, P, P, P, P, P, P, f64, f32, f32, f32, f32,
                                              i32, f32, f32, P, P, P, P, P, P, P]
        _lib.echo_ref_policy_loss.restype = ctypes.c_int
        _lib.echo_ref_token_logp.argtypes = [i64, i32, i64, i32, P, P, P, P, P]
        _lib.echo_ref_token_logp.restype = ctypes.c_int
        _lib.echo_ref_scaled_loss.argtypes = [i64, i32, i64, P, P, P, P, P, P, P, P, f64, f32, f32, f32, f32, i32,
                                              f32, f32]
        _lib.echo_ref_scaled_loss.restype = f64
        _lib.echo_ref_csr_from_lengths.argtypes = [i32, P, P, P]
        _lib.echo_ref_csr_from_lengths.restype = ctypes.c_int
        _lib.echo_ref_lmhead_logp.argtypes = [i64, i32, i32, P, P, P, P, P, P]
        _lib.echo_ref_lmhead_logp.restype = ctypes.c_int
        _lib.echo_ref_staleness_histogram.argtypes = [i32, i32, i32, i64, i32, P, P, i32, P, i32]
        _lib.echo_ref_staleness_histogram.restype = ctypes.c_int
        _lib.echo_ref_loss_from_logp.argtypes = [i64, P, P, P, P, P, P, P, P, f64, f32, f32, f32, f32, i32, f32, f32,
                                                 P, P, P]
        _lib.echo_ref_loss_from_logp.restype = ctypes.c_int
        _lib.echo_ref_lmhead_backward.argtypes = [i64, i32, i32, P, P, P, P, P, P, P, P]
        _lib.echo_ref_lmhead_backward.restype = ctypes.c_int
        _lib.echo_ref_set_threads.argtypes = [i32]
        _lib.echo_ref_set_threads.restype = None
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


@dataclass
class PackOut:
    status: int
    first_bad_rollout: int
    n_groups_kept: int
    n_rollouts_kept: int
    n_tokens: int
    kept_rollout: np.ndarray
    kept_offset: np.ndarray
    tok_slot: np.ndarray
    tok_action: np.ndarray
    tok_old: np.ndarray
    tok_ref: np.ndarray | None
    tok_aux: np.ndarray | None = None


def pack_batch(version, resp_len, action, old_logp, ref_logp, *, group_size, max_len, vocab, t_train, max_lag,
               rollout_base=0, token_capacity=None, aux=None, filter_mode=0) -> PackOut:
    """(1) lag filter + pack.  ``action``/``old_logp``/``ref_logp`` are padded ``[R, S]``.  ``filter_mode`` 1 keeps
    rollouts individually (f3 partial groups) instead of whole groups."""
    version = _c(version, np.int64)
    resp_len = _c(resp_len, np.int32)
    R = int(version.shape[0])
    action = _c(action, np.int32).reshape(-1)
    old_logp = _c(old_logp, np.float32).reshape(-1)
    ref_logp = None if ref_logp is None else _c(ref_logp, np.float32).reshape(-1)
    cap = R * max_len if token_capacity is None else int(token_capacity)
    kept_rollout = np.full(R, -1, np.int32)
    kept_offset = np.zeros(R + 1, np.int64)
    n_alloc = max(cap, 1)
    tok_slot = np.zeros(n_alloc, np.int32)
    tok_action = np.zeros(n_alloc, np.int32)
    tok_old = np.zeros(n_alloc, np.float32)
    tok_ref = np.zeros(n_alloc, np.float32) if ref_logp is not None else None
    aux = None if aux is None else _c(aux, np.float32).reshape(-1)
    tok_aux = np.zeros(n_alloc, np.float32) if aux is not None else None
    res = _PackResult()
    rc = lib().echo_ref_pack_batch(R, group_size, max_len, vocab, t_train, max_lag, rollout_base,
                                   _p(version), _p(resp_len), _p(action), _p(old_logp), _p(ref_logp), _p(aux), cap,
                                   _p(kept_rollout), _p(kept_offset), _p(tok_slot), _p(tok_action), _p(tok_old),
                                   _p(tok_ref), _p(tok_aux), ctypes.byref(res), filter_mode)
    if rc != 0:
        raise ValueError(f"echo_ref_pack_batch: invalid argument (rc={rc})")
    n = int(res.n_tokens) if res.n_tokens <= cap else 0
    nk = int(res.n_rollouts_kept)
    return PackOut(int(res.status), int(res.first_bad_rollout), int(res.n_groups_kept), nk, int(res.n_tokens),
                   kept_rollout[:nk].copy(), kept_offset[:nk + 1].copy(), tok_slot[:n].copy(), tok_action[:n].copy(),
                   tok_old[:n].copy(), None if tok_ref is None else tok_ref[:n].copy(),
                   None if tok_aux is None else tok_aux[:n].copy())


def gae_advantage(resp_len, rewards, values, *, gamma, lam, bootstrap=None):
    """f4: PPO-GAE advantages and returns, padded [R, S] float32 (positions >= L left at 0)."""
    rewards = _c(rewards, np.float32)
    values = _c(values, np.float32)
    R, S = rewards.shape
    adv = np.zeros((R, S), np.float32)
    ret = np.zeros((R, S), np.float32)
    rc = lib().echo_ref_gae_advantage(R, S, _p(_c(resp_len, np.int32)), _p(rewards), _p(values),
                                      _p(_c(bootstrap, np.float32)), gamma, lam, _p(adv), _p(ret))
    if rc != 0:
        raise ValueError("echo_ref_gae_advantage: invalid argument")
    return adv, ret


def group_advantage(reward, kept_rollout, *, group_size, eps=1e-8, rollout_base=0, want_f64=False):
    """(2) GRPO advantage per kept rollout slot (fp32) and the 6 advantage statistics (fp64).

    With ``want_f64`` also returns the advantages before their fp32 rounding."""
    reward = _c(reward, np.float32)
    kept_rollout = _c(kept_rollout, np.int32)
    n = int(kept_rollout.shape[0])
    adv = np.zeros(max(n, 1), np.float32)
    adv64 = np.zeros(max(n, 1), np.float64)
    stats = np.zeros(6, np.float64)
    rc = lib().echo_ref_group_advantage(n, group_size, eps, _p(reward), _p(kept_rollout), rollout_base,
                                        _p(adv), _p(adv64), _p(stats))
    if rc != 0:
        raise ValueError("echo_ref_group_advantage: invalid argument")
    if want_f64:
        return adv[:n].copy(), stats, adv64[:n].copy()
    return adv[:n].copy(), stats


@dataclass
class LossOut:
    logp: np.ndarray
    loss: np.ndarray
    flags: np.ndarray
    coef: np.ndarray
    dlogits: np.ndarray | None
    stats: np.ndarray
    entropy: np.ndarray
    lse: np.ndarray | None = None    # log-sum-exp of the row = z_a - logp (z_a decoded exactly from the input row)


KL_K3, KL_K1, KL_K2 = 0, 1, 2


def policy_loss(logits, tok_action, tok_old, tok_ref, tok_slot, adv_slot, *, n_global, vocab=None, dtype=None,
                clip_low=0.2, clip_high=0.2, kl_coef=0.0, grad_scale=1.0, want_dlogits=True, tok_adv=None,
                tok_weight=None, clip_dual=0.0, kl_estimator=KL_K3, entropy_coef=0.0) -> LossOut:
    """(3)-(5) for every row of ``logits``.

    ``logits`` is a 2-D numpy array: float32 (dtype F32) or uint16 bf16 bit patterns (dtype BF16).
    Returns fp64 per-token logp / loss / gradient coefficient, flags, and optional fp64 dlogits.
    """
    if dtype is None:
        dtype = F32 if logits.dtype == np.float32 else BF16
    logits = np.ascontiguousarray(logits)
    assert logits.dtype == (np.float32 if dtype == F32 else np.uint16)
    n, ld = logits.shape
    V = ld if vocab is None else int(vocab)
    tok_action = _c(tok_action, np.int32)
    tok_old = _c(tok_old, np.float32)
    tok_ref = _c(tok_ref, np.float32)
    tok_slot = _c(tok_slot, np.int32)
    adv_slot = _c(adv_slot, np.float32)
    logp = np.zeros(n, np.float64)
    loss = np.zeros(n, np.float64)
    coef = np.zeros(n, np.float64)
    flags = np.zeros(n, np.uint8)
    d = np.zeros((n, V), np.float64) if want_dlogits else None
    tok_adv = _c(tok_adv, np.float32)
    tok_weight = _c(tok_weight, np.float32)
    stats = np.zeros(11, np.float64)
    ent = np.zeros(n, np.float64)
    rc = lib().echo_ref_policy_loss(n, V, ld, dtype, _p(logits), _p(tok_action), _p(tok_old), _p(tok_ref),
                                    _p(tok_slot), _p(adv_slot), _p(tok_adv), _p(tok_weight), float(n_global),
                                    clip_low, clip_high, clip_dual, kl_coef, kl_estimator, grad_scale, entropy_coef,
                                    _p(logp), _p(loss), _p(flags), _p(coef), _p(ent), _p(d), _p(stats))
    if rc != 0:
        raise ValueError("echo_ref_policy_loss: invalid argument")
    za = logits[np.arange(n), np.clip(tok_action, 0, V - 1)] if n else logits[:0, 0]
    za = za.astype(np.float64) if dtype == F32 else (za.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return LossOut(logp, loss, flags, coef, d, stats, ent, za - logp)


def token_logp(logits, tok_action, *, vocab=None, dtype=None):
    """f1: forward-only (logp, lse, flags) per row of ``logits`` (float32 or bf16 bit patterns)."""
    if dtype is None:
        dtype = F32 if logits.dtype == np.float32 else BF16
    logits = np.ascontiguousarray(logits)
    n, ld = logits.shape
    V = ld if vocab is None else int(vocab)
    logp = np.zeros(n, np.float64)
    lse = np.zeros(n, np.float64)
    flags = np.zeros(n, np.uint8)
    rc = lib().echo_ref_token_logp(n, V, ld, dtype, _p(logits), _p(_c(tok_action, np.int32)), _p(logp), _p(lse),
                                   _p(flags))
    if rc != 0:
        raise ValueError("echo_ref_token_logp: invalid argument")
    return logp, lse, flags


def scaled_loss(logits_f64, tok_action, tok_old, tok_ref, tok_slot, adv_slot, *, n_global, clip_low=0.2,
                clip_high=0.2, kl_coef=0.0, grad_scale=1.0, tok_adv=None, tok_weight=None, clip_dual=0.0,
                kl_estimator=KL_K3, entropy_coef=0.0) -> float:
    """grad_scale * sum_t w_t l_t as a function of fp64 logits (for finite differences)."""
    z = np.ascontiguousarray(logits_f64, dtype=np.float64)
    n, V = z.shape
    return float(lib().echo_ref_scaled_loss(n, V, V, _p(z), _p(_c(tok_action, np.int32)), _p(_c(tok_old, np.float32)),
                                            _p(_c(tok_ref, np.float32)), _p(_c(tok_slot, np.int32)),
                                            _p(_c(adv_slot, np.float32)), _p(_c(tok_adv, np.float32)),
                                            _p(_c(tok_weight, np.float32)), float(n_global), clip_low, clip_high,
                                            clip_dual, kl_coef, kl_estimator, grad_scale, entropy_coef))


def csr_from_lengths(lengths):
    """f3: (kept_offset int64[n+1], tok_slot int32[total]) of kept rollouts with these lengths."""
    lengths = _c(lengths, np.int32)
    n = len(lengths)
    off = np.zeros(n + 1, np.int64)
    total = int(np.maximum(lengths, 0).sum())
    slot = np.zeros(max(total, 1), np.int32)
    rc = lib().echo_ref_csr_from_lengths(n, _p(lengths), _p(off), _p(slot))
    if rc != 0:
        raise ValueError("echo_ref_csr_from_lengths: invalid argument")
    return off, slot[:total]


def lmhead_logp(hidden_bf16, weight_bf16, tok_action, want_entropy=False):
    """f2: (logp, lse[, entropy]) of z = hidden @ weight^T (bf16 bit patterns, uint16) at the actions, fp64."""
    h = np.ascontiguousarray(hidden_bf16, np.uint16)
    w = np.ascontiguousarray(weight_bf16, np.uint16)
    n, d = h.shape
    V = w.shape[0]
    assert w.shape[1] == d
    logp = np.zeros(n, np.float64)
    lse = np.zeros(n, np.float64)
    ent = np.zeros(n, np.float64) if want_entropy else None
    rc = lib().echo_ref_lmhead_logp(n, d, V, _p(h), _p(w), _p(_c(tok_action, np.int32)), _p(logp), _p(lse), _p(ent))
    if rc != 0:
        raise ValueError("echo_ref_lmhead_logp: invalid argument")
    return (logp, lse, ent) if want_entropy else (logp, lse)


def staleness_histogram(version, resp_len, *, group_size, max_len, t_train, max_lag, n_bins, filter_mode=0):
    """f3: int64 [4, n_bins + 2] = {kept rollouts, dropped rollouts, kept tokens, dropped tokens} per lag bin
    (bin 0: future versions, 1 + lag for lag < n_bins, n_bins + 1: older)."""
    v = _c(version, np.int64)
    L = _c(resp_len, np.int32)
    h = np.zeros((4, n_bins + 2), np.int64)
    rc = lib().echo_ref_staleness_histogram(len(v), group_size, max_len, t_train, max_lag, _p(v), _p(L), n_bins, _p(h),
                                            filter_mode)
    if rc != 0:
        raise ValueError("echo_ref_staleness_histogram: invalid argument")
    return h


def loss_from_logp(tok_logp, tok_old, tok_ref, tok_slot, adv_slot, *, n_global, clip_low=0.2, clip_high=0.2,
                   kl_coef=0.0, grad_scale=1.0, tok_adv=None, tok_weight=None, clip_dual=0.0, kl_estimator=KL_K3,
                   entropy_coef=0.0, tok_entropy=None):
    """(4) from fp64 log-probs (f1 / f2 outputs): (loss, flags, coef) per token."""
    lp = np.ascontiguousarray(tok_logp, np.float64)
    n = len(lp)
    ent = None if tok_entropy is None else np.ascontiguousarray(tok_entropy, np.float64)
    loss = np.zeros(n, np.float64)
    coef = np.zeros(n, np.float64)
    flags = np.zeros(n, np.uint8)
    rc = lib().echo_ref_loss_from_logp(n, _p(lp), _p(ent), _p(_c(tok_old, np.float32)), _p(_c(tok_ref, np.float32)),
                                       _p(_c(tok_slot, np.int32)), _p(_c(adv_slot, np.float32)),
                                       _p(_c(tok_adv, np.float32)), _p(_c(tok_weight, np.float32)), float(n_global),
                                       clip_low, clip_high, clip_dual, kl_coef, kl_estimator, grad_scale, entropy_coef,
                                       _p(loss), _p(flags), _p(coef))
    if rc != 0:
        raise ValueError("echo_ref_loss_from_logp: invalid argument")
    return loss, flags, coef


def _widen(x):
    """bf16 bit patterns (uint16) -> exact fp64; float arrays -> fp64."""
    x = np.asarray(x)
    if x.dtype == np.uint16:
        return (x.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return np.ascontiguousarray(x, np.float64)


def lmhead_backward(hidden, weight, tok_action, tok_coef, tok_ecoef=None, want_dlogits=False, want_dweight=True):
    """f2 backward: (dhidden [n x d], dweight [V x d][, dlogits [n x V]]) in fp64 for z = hidden @ weight^T, with
    D[t, v] = c_t (delta - p) + e_t p (log p + H).  hidden / weight: bf16 bit patterns (uint16) or floats.
    want_dweight=False skips dweight (None in its place), e.g. for a few rows at a full vocabulary."""
    h = np.ascontiguousarray(_widen(hidden))
    w = np.ascontiguousarray(_widen(weight))
    n, d = h.shape
    V = w.shape[0]
    assert w.shape[1] == d
    dh = np.zeros((n, d), np.float64)
    dw = np.zeros((V, d), np.float64) if want_dweight else None
    dz = np.zeros((n, V), np.float64) if want_dlogits else None
    ec = None if tok_ecoef is None else np.ascontiguousarray(tok_ecoef, np.float64)
    rc = lib().echo_ref_lmhead_backward(n, d, V, _p(h), _p(w), _p(_c(tok_action, np.int32)),
                                        _p(np.ascontiguousarray(tok_coef, np.float64)), _p(ec), _p(dz), _p(dh),
                                        _p(dw))
    if rc != 0:
        raise ValueError("echo_ref_lmhead_backward: invalid argument")
    return (dh, dw, dz) if want_dlogits else (dh, dw)


def set_threads(n: int) -> None:
    """OpenMP thread count of the oracle's row loops (timing only; results do not depend on it)."""
    lib().echo_ref_set_threads(int(n))
