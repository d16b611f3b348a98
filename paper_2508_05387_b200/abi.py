"""ctypes binding of libecho.so -- the C ABI of include/echo.h, same names, argument marshalling only.

Every entry point takes torch tensors (or None for nullable pointers) and forwards their device pointers,
plus the caller's CUDA stream (default: torch's current stream).  No arithmetic of the method happens here:
every step of the path runs in the kernels of libecho.so.  If the library is missing this module raises
at import time -- there is no fallback.
"""
from __future__ import annotations

import ctypes
import os
import struct

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libecho.so")

ECHO_OK, ECHO_ERR_INVALID_ARGUMENT, ECHO_ERR_UNSUPPORTED, ECHO_ERR_CUDA = range(4)
ECHO_F32, ECHO_BF16 = 0, 1
(ECHO_DATA_OK, ECHO_DATA_FUTURE_VERSION, ECHO_DATA_MIXED_GROUP_VERSION, ECHO_DATA_BAD_LENGTH, ECHO_DATA_BAD_ACTION,
 ECHO_DATA_CAPACITY) = range(6)
ECHO_FLAG_CLIPPED, ECHO_FLAG_NONFINITE = 1, 2
ECHO_ALGO_AUTO, ECHO_ALGO_ROW_L2, ECHO_ALGO_QUAD_REG, ECHO_ALGO_QUAD_REG_EXACT, ECHO_ALGO_OCT_REG, ECHO_ALGO_HEX_REG = range(6)
ALGO_NAMES = {"auto": 0, "row_l2": 1, "quad_reg": 2, "quad_reg_exact": 3, "oct_reg": 4, "hex_reg": 5}
PACK_RESULT_BYTES = 32

# kernels launched per call (for the bench's gpu_launches count)
LAUNCHES = {"echo_pack_batch": 3, "echo_group_advantage": 1, "echo_policy_loss_fwd_bwd": 1, "echo_loss_stats": 2,
            "echo_token_logp": 1, "echo_policy_loss_fwd_bwd_v2": 1, "echo_gae_advantage": 1, "echo_csr_from_lengths": 2,
            "echo_lmhead_logp": 2, "echo_staleness_histogram": 1, "echo_pack_batch_v2": 3,
            "echo_loss_from_logp": 1, "echo_lmhead_dlogits": 1, "echo_lmhead_logits": 1}
# echo_lmhead_backward: per chunk 3 libecho kernels (D, dhidden, dweight)
BACKWARD_LAUNCHES_PER_CHUNK = 3
# echo_lmhead_policy_loss_fwd_bwd: per chunk 4 libecho kernels (logits, fused loss, dhidden, dweight)
LMHEAD_LOSS_LAUNCHES_PER_CHUNK = 4

EXPORTS = ("echo_pack_batch", "echo_pack_batch_v2", "echo_group_advantage", "echo_policy_loss_fwd_bwd", "echo_policy_loss_fwd_bwd_ex",
           "echo_policy_loss_launch_shape", "echo_token_logp", "echo_policy_loss_fwd_bwd_v2", "echo_gae_advantage",
           "echo_loss_stats_workspace_bytes", "echo_loss_stats", "echo_csr_from_lengths",
           "echo_lmhead_workspace_bytes", "echo_lmhead_logp", "echo_staleness_histogram", "echo_status_string",
           "echo_abi_version", "echo_loss_from_logp", "echo_lmhead_dlogits", "echo_lmhead_backward",
           "echo_lmhead_logits", "echo_lmhead_policy_loss_fwd_bwd", "echo_gemm_bf16")


ECHO_KL_K3, ECHO_KL_K1, ECHO_KL_K2 = range(3)


class LossConfig(ctypes.Structure):
    """echo_loss_config (include/echo.h)."""
    _fields_ = [("clip_low", ctypes.c_float), ("clip_high", ctypes.c_float), ("clip_dual", ctypes.c_float),
                ("kl_coef", ctypes.c_float), ("grad_scale", ctypes.c_float), ("kl_estimator", ctypes.c_int32),
                ("entropy_coef", ctypes.c_float)]


class EchoError(RuntimeError):
    def __init__(self, fn, status):
        self.status = status
        super().__init__(f"{fn} -> {_lib.echo_status_string(status).decode()}")


def _load(path=LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(f"{path} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    i32, i64, f32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_float
    lib.echo_pack_batch.argtypes = [i32, i32, i32, i32, i64, i32, i64, P, P, P, P, P, P, i64, P, P, P, P, P, P, P, P,
                                    P]
    lib.echo_pack_batch_v2.argtypes = [i32, i32, i32, i32, i64, i32, i64, P, P, P, P, P, P, i64, P, P, P, P, P, P, P,
                                       P, i32, P]
    lib.echo_gae_advantage.argtypes = [i32, i32, P, P, P, P, f32, f32, P, P, P]
    lib.echo_gae_advantage.restype = ctypes.c_int
    lib.echo_group_advantage.argtypes = [i32, i32, f32, P, P, i64, P, P, P, P]
    lib.echo_policy_loss_fwd_bwd.argtypes = [P, i32, i64, i32, i64, P, P, P, P, P, P, f32, f32, f32, f32, P, P, P, P]
    lib.echo_policy_loss_fwd_bwd_ex.argtypes = [P, i32, i64, i32, i64, P, P, P, P, P, P, f32, f32, f32, f32, P, P, P,
                                                i32, P]
    lib.echo_loss_stats.argtypes = [i64, P, P, P, P, P, P, P, P, P]
    lib.echo_policy_loss_launch_shape.argtypes = [i32, i64, i32, i32, P]
    lib.echo_token_logp.argtypes = [P, i32, i64, i32, i64, P, P, P, P, P]
    lib.echo_policy_loss_fwd_bwd_v2.argtypes = [P, i32, i64, i32, i64, P, P, P, P, P, P, P, P,
                                                ctypes.POINTER(LossConfig), P, P, P, P, i32, P]
    lib.echo_policy_loss_fwd_bwd_v2.restype = ctypes.c_int
    lib.echo_token_logp.restype = ctypes.c_int
    lib.echo_policy_loss_launch_shape.restype = ctypes.c_int
    lib.echo_loss_stats_workspace_bytes.argtypes = []
    lib.echo_loss_stats_workspace_bytes.restype = ctypes.c_size_t
    lib.echo_status_string.argtypes = [ctypes.c_int]
    lib.echo_status_string.restype = ctypes.c_char_p
    lib.echo_abi_version.restype = i32
    lib.echo_csr_from_lengths.argtypes = [i32, P, P, P, P]
    lib.echo_staleness_histogram.argtypes = [i32, i32, i32, i64, i32, P, P, i32, P, i32, P]
    lib.echo_lmhead_workspace_bytes.argtypes = [i64, i32]
    lib.echo_lmhead_workspace_bytes.restype = ctypes.c_size_t
    lib.echo_lmhead_logp.argtypes = [P, P, i64, i32, i32, P, P, P, P, P, P]
    lib.echo_loss_from_logp.argtypes = [i64, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P]
    lib.echo_lmhead_dlogits.argtypes = [P, P, i64, i32, i32, P, P, P, P, P, P, i64, P]
    lib.echo_lmhead_backward.argtypes = [P, P, i64, i32, i32, P, P, P, P, P, P, P, i32, P, i64, P]
    lib.echo_lmhead_logits.argtypes = [P, P, i64, i32, i32, P, i64, P]
    lib.echo_gemm_bf16.argtypes = [P, i32, i64, P, i32, i64, i64, i32, i32, P, i64, i32, P]
    lib.echo_lmhead_policy_loss_fwd_bwd.argtypes = [P, P, i64, i32, i32, P, P, P, P, P, P, P, P, P, P, P, P, P, P, P,
                                                    i32, P, i64, P]
    for fn in ("echo_pack_batch", "echo_group_advantage", "echo_policy_loss_fwd_bwd", "echo_policy_loss_fwd_bwd_ex",
               "echo_loss_stats", "echo_policy_loss_fwd_bwd_v2", "echo_csr_from_lengths", "echo_lmhead_logp",
               "echo_staleness_histogram", "echo_pack_batch_v2", "echo_loss_from_logp", "echo_lmhead_dlogits",
               "echo_lmhead_backward", "echo_lmhead_logits", "echo_lmhead_policy_loss_fwd_bwd", "echo_gemm_bf16"):
        getattr(lib, fn).restype = ctypes.c_int
    return lib


_lib = _load()


def _p(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _s(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _check(fn, st):
    if st != ECHO_OK:
        raise EchoError(fn, st)


def echo_abi_version() -> int:
    return _lib.echo_abi_version()


def echo_status_string(status: int) -> str:
    return _lib.echo_status_string(status).decode()


def echo_pack_batch(n_rollouts, group_size, max_len, vocab, t_train, max_lag, rollout_base, version, resp_len, action,
                    old_logp, ref_logp, token_capacity, kept_rollout, kept_offset, tok_slot, tok_action, tok_old,
                    tok_ref, result, stream=None, aux=None, tok_aux=None):
    _check("echo_pack_batch", _lib.echo_pack_batch(
        n_rollouts, group_size, max_len, vocab, t_train, max_lag, rollout_base, _p(version), _p(resp_len), _p(action),
        _p(old_logp), _p(ref_logp), _p(aux), token_capacity, _p(kept_rollout), _p(kept_offset), _p(tok_slot),
        _p(tok_action), _p(tok_old), _p(tok_ref), _p(tok_aux), _p(result), _s(stream)))


ECHO_FILTER_GROUP, ECHO_FILTER_ROLLOUT = 0, 1


def echo_pack_batch_v2(n_rollouts, group_size, max_len, vocab, t_train, max_lag, rollout_base, version, resp_len,
                       action, old_logp, ref_logp, token_capacity, kept_rollout, kept_offset, tok_slot, tok_action,
                       tok_old, tok_ref, result, filter_mode=ECHO_FILTER_GROUP, stream=None, aux=None, tok_aux=None):
    _check("echo_pack_batch_v2", _lib.echo_pack_batch_v2(
        n_rollouts, group_size, max_len, vocab, t_train, max_lag, rollout_base, _p(version), _p(resp_len), _p(action),
        _p(old_logp), _p(ref_logp), _p(aux), token_capacity, _p(kept_rollout), _p(kept_offset), _p(tok_slot),
        _p(tok_action), _p(tok_old), _p(tok_ref), _p(tok_aux), _p(result), filter_mode, _s(stream)))


def echo_gae_advantage(n_rollouts, max_len, resp_len, rewards, values, bootstrap_value, gamma, lam, adv,
                       returns=None, stream=None):
    _check("echo_gae_advantage", _lib.echo_gae_advantage(
        n_rollouts, max_len, _p(resp_len), _p(rewards), _p(values), _p(bootstrap_value), gamma, lam, _p(adv),
        _p(returns), _s(stream)))


def echo_group_advantage(n_rollouts, group_size, eps, reward, kept_rollout, rollout_base, pack, adv_slot, adv_stats,
                         stream=None):
    _check("echo_group_advantage", _lib.echo_group_advantage(
        n_rollouts, group_size, eps, _p(reward), _p(kept_rollout), rollout_base, _p(pack), _p(adv_slot),
        _p(adv_stats), _s(stream)))


def echo_policy_loss_fwd_bwd(logits, dtype, n_rows, vocab, ld, tok_action, tok_old, tok_ref, tok_slot, adv_slot,
                             n_global, clip_low, clip_high, kl_coef, grad_scale, tok_logp, tok_loss, tok_flags,
                             stream=None, algo=None):
    if algo is None:
        _check("echo_policy_loss_fwd_bwd", _lib.echo_policy_loss_fwd_bwd(
            _p(logits), dtype, n_rows, vocab, ld, _p(tok_action), _p(tok_old), _p(tok_ref), _p(tok_slot),
            _p(adv_slot), _p(n_global), clip_low, clip_high, kl_coef, grad_scale, _p(tok_logp), _p(tok_loss),
            _p(tok_flags), _s(stream)))
    else:
        _check("echo_policy_loss_fwd_bwd_ex", _lib.echo_policy_loss_fwd_bwd_ex(
            _p(logits), dtype, n_rows, vocab, ld, _p(tok_action), _p(tok_old), _p(tok_ref), _p(tok_slot),
            _p(adv_slot), _p(n_global), clip_low, clip_high, kl_coef, grad_scale, _p(tok_logp), _p(tok_loss),
            _p(tok_flags), algo, _s(stream)))


def echo_policy_loss_fwd_bwd_v2(logits, dtype, n_rows, vocab, ld, tok_action, tok_old, tok_ref, tok_slot, adv_slot,
                                tok_adv, tok_weight, n_global, cfg: LossConfig, tok_logp, tok_loss, tok_flags,
                                tok_entropy=None, algo=ECHO_ALGO_AUTO, stream=None):
    _check("echo_policy_loss_fwd_bwd_v2", _lib.echo_policy_loss_fwd_bwd_v2(
        _p(logits), dtype, n_rows, vocab, ld, _p(tok_action), _p(tok_old), _p(tok_ref), _p(tok_slot), _p(adv_slot),
        _p(tok_adv), _p(tok_weight), _p(n_global), ctypes.byref(cfg), _p(tok_logp), _p(tok_loss), _p(tok_flags),
        _p(tok_entropy), algo, _s(stream)))


def echo_token_logp(logits, dtype, n_rows, vocab, ld, tok_action, tok_logp, tok_lse=None, tok_flags=None,
                    stream=None):
    _check("echo_token_logp", _lib.echo_token_logp(_p(logits), dtype, n_rows, vocab, ld, _p(tok_action), _p(tok_logp),
                                                   _p(tok_lse), _p(tok_flags), _s(stream)))


def echo_policy_loss_launch_shape(dtype, n_rows, vocab, algo=ECHO_ALGO_AUTO) -> dict:
    buf = (ctypes.c_int32 * 5)()
    _check("echo_policy_loss_launch_shape",
           _lib.echo_policy_loss_launch_shape(dtype, n_rows, vocab, algo, ctypes.cast(buf, ctypes.c_void_p)))
    return dict(zip(("algo", "grid_ctas", "cluster_ctas", "threads", "smem_bytes"), list(buf)))


def echo_csr_from_lengths(n, lengths, kept_offset, tok_slot=None, stream=None):
    _check("echo_csr_from_lengths", _lib.echo_csr_from_lengths(n, _p(lengths), _p(kept_offset), _p(tok_slot),
                                                                _s(stream)))


def echo_staleness_histogram(n_rollouts, group_size, max_len, t_train, max_lag, version, resp_len, n_bins, hist,
                             filter_mode=0, stream=None):
    _check("echo_staleness_histogram", _lib.echo_staleness_histogram(n_rollouts, group_size, max_len, t_train, max_lag,
                                                                      _p(version), _p(resp_len), n_bins, _p(hist),
                                                                      filter_mode, _s(stream)))


def echo_lmhead_workspace_bytes(n_rows, vocab) -> int:
    return int(_lib.echo_lmhead_workspace_bytes(n_rows, vocab))


def echo_lmhead_logp(hidden, weight, n_rows, d, vocab, tok_action, tok_logp, tok_lse, workspace, stream=None,
                     tok_entropy=None):
    _check("echo_lmhead_logp", _lib.echo_lmhead_logp(_p(hidden), _p(weight), n_rows, d, vocab, _p(tok_action),
                                                      _p(tok_logp), _p(tok_lse), _p(tok_entropy), _p(workspace),
                                                      _s(stream)))


def echo_loss_from_logp(n_rows, tok_logp, tok_entropy, tok_old, tok_ref, tok_slot, adv_slot, tok_adv, tok_weight,
                        n_global, cfg: LossConfig, tok_loss, tok_flags, tok_coef, tok_ecoef=None, stream=None):
    _check("echo_loss_from_logp", _lib.echo_loss_from_logp(
        n_rows, _p(tok_logp), _p(tok_entropy), _p(tok_old), _p(tok_ref), _p(tok_slot), _p(adv_slot), _p(tok_adv),
        _p(tok_weight), _p(n_global), ctypes.byref(cfg), _p(tok_loss), _p(tok_flags), _p(tok_coef), _p(tok_ecoef),
        _s(stream)))


def echo_lmhead_dlogits(hidden, weight, n_rows, d, vocab, tok_action, tok_lse, tok_coef, tok_ecoef, tok_entropy,
                        dlogits, ld, stream=None):
    _check("echo_lmhead_dlogits", _lib.echo_lmhead_dlogits(
        _p(hidden), _p(weight), n_rows, d, vocab, _p(tok_action), _p(tok_lse), _p(tok_coef), _p(tok_ecoef),
        _p(tok_entropy), _p(dlogits), ld, _s(stream)))


def echo_lmhead_dlogits_ld(vocab) -> int:
    """Row stride (elements) of echo_lmhead_backward's bf16 D chunk buffer: vocab rounded up to 8."""
    return (vocab + 7) // 8 * 8


def echo_lmhead_backward(hidden, weight, n_rows, d, vocab, tok_action, tok_lse, tok_coef, tok_ecoef, tok_entropy,
                         dhidden, dweight, accumulate, dlogits_ws, chunk_rows, stream=None):
    _check("echo_lmhead_backward", _lib.echo_lmhead_backward(
        _p(hidden), _p(weight), n_rows, d, vocab, _p(tok_action), _p(tok_lse), _p(tok_coef), _p(tok_ecoef),
        _p(tok_entropy), _p(dhidden), _p(dweight), int(accumulate), _p(dlogits_ws), chunk_rows, _s(stream)))


def echo_lmhead_logits(hidden, weight, n_rows, d, vocab, logits, ld, stream=None):
    _check("echo_lmhead_logits", _lib.echo_lmhead_logits(_p(hidden), _p(weight), n_rows, d, vocab, _p(logits), ld,
                                                          _s(stream)))


def echo_lmhead_policy_loss_fwd_bwd(hidden, weight, n_rows, d, vocab, tok_action, tok_old, tok_ref, tok_slot, adv_slot,
                                    tok_adv, tok_weight, n_global, cfg: LossConfig, tok_logp, tok_loss, tok_flags,
                                    tok_entropy, dhidden, dweight, accumulate, logits_ws, chunk_rows, stream=None):
    _check("echo_lmhead_policy_loss_fwd_bwd", _lib.echo_lmhead_policy_loss_fwd_bwd(
        _p(hidden), _p(weight), n_rows, d, vocab, _p(tok_action), _p(tok_old), _p(tok_ref), _p(tok_slot),
        _p(adv_slot), _p(tok_adv), _p(tok_weight), _p(n_global), ctypes.byref(cfg), _p(tok_logp), _p(tok_loss),
        _p(tok_flags), _p(tok_entropy), _p(dhidden), _p(dweight), int(accumulate), _p(logits_ws), chunk_rows,
        _s(stream)))


def echo_gemm_bf16(a, a_mn, lda, b, b_mn, ldb, m, n, k, c, ldc, accumulate=False, stream=None):
    _check("echo_gemm_bf16", _lib.echo_gemm_bf16(_p(a), int(a_mn), lda, _p(b), int(b_mn), ldb, m, n, k, _p(c), ldc,
                                                  int(accumulate), _s(stream)))


def echo_loss_stats_workspace_bytes() -> int:
    return int(_lib.echo_loss_stats_workspace_bytes())


def echo_loss_stats(n_tokens, tok_loss, tok_logp, tok_old, tok_ref, tok_flags, workspace, loss_stats, stream=None,
                    tok_weight=None):
    _check("echo_loss_stats", _lib.echo_loss_stats(
        n_tokens, _p(tok_loss), _p(tok_logp), _p(tok_old), _p(tok_ref), _p(tok_weight), _p(tok_flags), _p(workspace),
        _p(loss_stats), _s(stream)))


def parse_pack_result(raw: bytes) -> dict:
    """Decode the 32-byte echo_pack_result read back from the device."""
    status, first_bad, n_groups, n_rollouts, n_tokens, _ = struct.unpack("<iiiiqq", raw)
    return {"status": status, "first_bad_rollout": first_bad, "n_groups_kept": n_groups,
            "n_rollouts_kept": n_rollouts, "n_tokens": n_tokens}
