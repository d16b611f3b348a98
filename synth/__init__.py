"""Seeded synthetic inputs shared by the oracle side and the CUDA side -- holds NONE of the method's arithmetic.

Everything here is a counter-based random draw (Philox4x32-10) or a fixed workload recipe
(DESIGN.md "Input recipe"); nothing here filters, normalises, log-softmaxes or differentiates.  The
logits generator has a bit-exact CUDA twin in ``synth_gen.cu`` (same counters, same fp32 op order, RNE
to bf16) so that the GPU can produce the 10 GB micro-batches the bench needs while the oracle regenerates
any sampled row on the host.

Workloads follow BASELINE.json ``configs`` and SURVEY.md §8.4:
  * group-major rollouts R = P*G; rewards r_i ~ Bernoulli(p_g), p_g ~ U(0,1) (math-style verifiable
    reward, PAPER.md :359); t_train = 1000; lags per config (tiny fixed [0,1,2,1]; 7B: 38 of 128 groups
    stale by a seeded Fisher-Yates pick);
  * logits z = RNE_bf16(2 * g), g = Irwin-Hall(4) of 16-bit uniforms (integer-exact), plus a spike
    8 + 12u at the sampled action;
  * old_logp = min(0, lhat + N(0, (0.05 (1+lag))^2)), ref_logp = min(0, lhat + N(0, 0.1^2)) with the
    analytic estimate lhat = z_a - ln(V e^{sigma^2/2} + e^{z_a}).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

BASE_SEED = 250805387
T_TRAIN = 1000
SIGMA = 2.0

# Philox stream labels (key word 1)
L_LOGITS, L_ACTION, L_SPIKE, L_REWARD_P, L_REWARD, L_OLD, L_REF, L_LEN, L_LAG = 1, 2, 3, 4, 5, 6, 7, 8, 9

_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = 0x9E3779B9, 0xBB67AE85
_MASK = np.uint64(0xFFFFFFFF)

# fp32 constants of the logits recipe (the CUDA twin uses the same literals)
LOGIT_SCALE = np.float32(SIGMA * math.sqrt(3.0) / 65536.0)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 (Salmon et al., SC'11).  Inputs broadcast; returns 4 uint32 arrays."""
    c = [np.asarray(x, dtype=np.uint64) & _MASK for x in (c0, c1, c2, c3)]
    c = list(np.broadcast_arrays(*c))
    c = [x.copy() for x in c]
    k0 = int(k0) & 0xFFFFFFFF
    k1 = int(k1) & 0xFFFFFFFF
    for r in range(10):
        if r:
            k0 = (k0 + _W0) & 0xFFFFFFFF
            k1 = (k1 + _W1) & 0xFFFFFFFF
        p0 = _M0 * c[0]
        p1 = _M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
    return [x.astype(np.uint32) for x in c]


def _split64(x):
    x = np.asarray(x, dtype=np.int64).astype(np.uint64)
    return x & _MASK, x >> np.uint64(32)


def uniform01(w):
    """24-bit uniform in [0,1) from a uint32 word (exact in fp32)."""
    return (np.asarray(w, np.uint32) >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)


def std_normal(w0, w1):
    """Box-Muller normal from two uint32 words (host-only; float64)."""
    u1 = ((np.asarray(w0, np.uint64) >> np.uint64(11)).astype(np.float64) + 0.5) * 2.0 ** -21
    u2 = (np.asarray(w1, np.uint64).astype(np.float64)) * 2.0 ** -32
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def f32_to_bf16_bits(x):
    """fp32 -> bf16 round-to-nearest-even (finite inputs), as uint16 bit patterns."""
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b):
    return (np.asarray(b, np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def action_of(token_key, vocab, seed):
    """Sampled token id for global token key T = rollout*S + j: floor(w0 * V / 2^32)."""
    lo, hi = _split64(token_key)
    w = philox4x32_10(lo, hi, 0, 0, seed, L_ACTION)[0]
    return ((w.astype(np.uint64) * np.uint64(vocab)) >> np.uint64(32)).astype(np.int32)


def spike_of(token_key, seed):
    """fp32 spike 8 + 12u added to the sampled action's logit."""
    lo, hi = _split64(token_key)
    u = uniform01(philox4x32_10(lo, hi, 0, 0, seed, L_SPIKE)[0])
    return np.float32(8.0) + np.float32(12.0) * u


def _base_logits(token_key, cols, seed):
    """fp32 sigma*g for (token, column) pairs (broadcast)."""
    token_key = np.asarray(token_key, np.int64)
    cols = np.asarray(cols, np.int64)
    lo, hi = _split64(token_key)
    q = (cols >> 1).astype(np.uint64)
    w = philox4x32_10(q, lo, hi, 0, seed, L_LOGITS)
    odd = (cols & 1).astype(bool)
    wa = np.where(odd, w[2], w[0]).astype(np.uint32)
    wb = np.where(odd, w[3], w[1]).astype(np.uint32)
    s = ((wa & 0xFFFF).astype(np.int32) + (wa >> 16).astype(np.int32) + (wb & 0xFFFF).astype(np.int32)
         + (wb >> 16).astype(np.int32) - 131070)
    return s.astype(np.float32) * LOGIT_SCALE


def logits_rows(token_keys, actions, vocab, seed, dtype="bf16"):
    """Host twin of ``synth_fill_logits``: rows [n, vocab] as float32 or bf16 bit patterns (uint16)."""
    token_keys = np.asarray(token_keys, np.int64).reshape(-1)
    actions = np.asarray(actions, np.int32).reshape(-1)
    cols = np.arange(vocab, dtype=np.int64)[None, :]
    z = _base_logits(token_keys[:, None], cols, seed)
    rows = np.arange(token_keys.shape[0])
    z[rows, actions] = z[rows, actions] + spike_of(token_keys, seed)
    if dtype == "bf16":
        return f32_to_bf16_bits(z)
    return z


def action_logit(token_keys, actions, vocab, seed, dtype="bf16"):
    """z[t, a_t] only (what the old/ref log-prob recipe needs), without materialising rows."""
    z = _base_logits(token_keys, actions, seed) + spike_of(token_keys, seed)
    if dtype == "bf16":
        return bf16_bits_to_f32(f32_to_bf16_bits(z)).astype(np.float64)
    return z.astype(np.float64)


@dataclass
class Config:
    name: str
    P: int
    G: int
    S: int
    V: int
    dtype: str           # "f32" | "bf16"
    max_lag: int
    kl_coef: float
    lag_mode: str        # "fixed" | "zero" | "async"
    index: int           # seed offset (BASELINE.json configs order)
    stale_groups: int = 0
    fixed_lags: tuple = ()
    lengths: str = "full"  # "full" | "ragged"

    @property
    def R(self):
        return self.P * self.G

    @property
    def seed(self):
        return BASE_SEED + self.index


CONFIGS = {
    "tiny": Config("tiny", 4, 4, 64, 1024, "f32", 1, 0.001, "fixed", 0, fixed_lags=(0, 1, 2, 1)),
    "qwen3-4b": Config("qwen3-4b", 64, 8, 2048, 151936, "bf16", 0, 0.001, "zero", 1),
    "qwen2.5-7b": Config("qwen2.5-7b", 128, 8, 4096, 152064, "bf16", 2, 0.0, "async", 2, stale_groups=38),
    "qwen3-30b-a3b": Config("qwen3-30b-a3b", 128, 16, 8192, 151936, "bf16", 0, 0.001, "zero", 3),
    "qwen3-32b": Config("qwen3-32b", 256, 8, 4096, 151936, "bf16", 0, 0.001, "zero", 4),
}


def group_lags(cfg: Config, P=None):
    """Per-group lag t_train - version."""
    P = cfg.P if P is None else P
    if cfg.lag_mode == "fixed":
        return np.array([cfg.fixed_lags[g % len(cfg.fixed_lags)] for g in range(P)], np.int64)
    if cfg.lag_mode == "zero":
        return np.zeros(P, np.int64)
    # async: a seeded Fisher-Yates pick of `stale_groups` groups gets lag in {max_lag+1, max_lag+2}
    g = np.arange(P, dtype=np.int64)
    w = philox4x32_10(g, 0, 0, 0, cfg.seed, L_LAG)
    perm = list(range(P))
    for i in range(P - 1, 0, -1):
        j = int(w[0][i]) % (i + 1)
        perm[i], perm[j] = perm[j], perm[i]
    stale = set(perm[:cfg.stale_groups])
    lags = (w[1] % np.uint32(cfg.max_lag + 1)).astype(np.int64)
    for s in stale:
        lags[s] = cfg.max_lag + 1 + int(w[2][s] % np.uint32(2))
    return lags


@dataclass
class Batch:
    """One learner step's rollouts, padded [R, S] per-token arrays (the ABI's input layout)."""
    cfg: Config
    rollout_base: int
    version: np.ndarray     # int64 [R]
    resp_len: np.ndarray    # int32 [R]
    reward: np.ndarray      # float32 [R] (per-rollout return)
    action: np.ndarray      # int32 [R, S]
    old_logp: np.ndarray    # float32 [R, S]
    ref_logp: np.ndarray    # float32 [R, S]
    lag: np.ndarray = field(default=None)


def make_batch(cfg: Config, rollout_lo: int = 0, rollout_hi: int | None = None, lengths: str | None = None,
               want_tokens: bool = True) -> Batch:
    """Rollouts [rollout_lo, rollout_hi) of the config's step (global ids; shard-independent values)."""
    R = cfg.R
    rollout_hi = R if rollout_hi is None else rollout_hi
    lengths = cfg.lengths if lengths is None else lengths
    ids = np.arange(rollout_lo, rollout_hi, dtype=np.int64)
    groups = ids // cfg.G
    lags = group_lags(cfg)[groups]
    version = (T_TRAIN - lags).astype(np.int64)
    wp = philox4x32_10(groups, 0, 0, 0, cfg.seed, L_REWARD_P)[0]
    wr = philox4x32_10(ids, 0, 0, 0, cfg.seed, L_REWARD)[0]
    reward = (uniform01(wr) < uniform01(wp)).astype(np.float32)
    if lengths == "full":
        resp_len = np.full(ids.shape, cfg.S, np.int32)
    else:
        wl = philox4x32_10(ids, 0, 0, 0, cfg.seed, L_LEN)[0]
        resp_len = (1 + ((wl.astype(np.uint64) * np.uint64(cfg.S)) >> np.uint64(32))).astype(np.int32)
    if not want_tokens:
        return Batch(cfg, rollout_lo, version, resp_len, reward, None, None, None, lags)
    keys = (ids[:, None] * cfg.S + np.arange(cfg.S, dtype=np.int64)[None, :]).reshape(-1)
    action = action_of(keys, cfg.V, cfg.seed)
    za = action_logit(keys, action, cfg.V, cfg.seed, "bf16" if cfg.dtype == "bf16" else "f32")
    lhat = za - np.log(cfg.V * math.exp(SIGMA ** 2 / 2.0) + np.exp(za))
    lo, hi = _split64(keys)
    wo = philox4x32_10(lo, hi, 0, 0, cfg.seed, L_OLD)
    wf = philox4x32_10(lo, hi, 0, 0, cfg.seed, L_REF)
    tok_lag = np.repeat(lags, cfg.S).astype(np.float64)
    old = np.minimum(lhat + 0.05 * (1.0 + tok_lag) * std_normal(wo[0], wo[1]), 0.0).astype(np.float32)
    ref = np.minimum(lhat + 0.1 * std_normal(wf[0], wf[1]), 0.0).astype(np.float32)
    n = ids.shape[0]
    return Batch(cfg, rollout_lo, version, resp_len, reward, action.reshape(n, cfg.S), old.reshape(n, cfg.S),
                 ref.reshape(n, cfg.S), lags)
