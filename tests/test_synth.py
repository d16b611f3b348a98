"""The seeded input generator (synth/): counter-based, bit-reproducible, matching its recipe."""
import math

import numpy as np
import pytest
import torch

import synth


def test_philox_known_answers():
    """Philox4x32-10 known-answer vectors (Random123 distribution, kat_vectors: philox4x32 10 rounds)."""
    kat = [
        ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
        ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
        ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
         (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
    ]
    for ctr, key, expect in kat:
        got = tuple(int(x) for x in synth.philox4x32_10(*ctr, *key))
        assert got == expect


def test_bf16_rne_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.normal(size=100000).astype(np.float32) * 10,
                        np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -1.0 - 2 ** -8, 65504.0, 1e-30], np.float32)])
    ours = synth.f32_to_bf16_bits(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(ours, ref)


def test_logits_recipe_moments_and_spike():
    cfg = synth.CONFIGS["qwen3-4b"]
    keys = np.arange(4, dtype=np.int64) * 12345
    act = synth.action_of(keys, cfg.V, cfg.seed)
    rows = synth.logits_rows(keys, act, cfg.V, cfg.seed, "bf16")
    z = synth.bf16_bits_to_f32(rows).astype(np.float64)
    mask = np.ones_like(z, bool)
    mask[np.arange(4), act] = False
    body = z[mask]
    assert abs(body.mean()) < 0.01 and abs(body.std() - synth.SIGMA) < 0.01
    assert np.abs(body).max() <= synth.SIGMA * math.sqrt(3) * 2 + 1e-3   # Irwin-Hall(4) support
    spikes = z[np.arange(4), act]
    assert np.all(spikes > 8 - 7) and np.all(spikes < 20 + 7)
    # row-local: a row depends only on its own key
    again = synth.logits_rows(keys[2:3], act[2:3], cfg.V, cfg.seed, "bf16")
    np.testing.assert_array_equal(again[0], rows[2])
    np.testing.assert_array_equal(synth.action_logit(keys, act, cfg.V, cfg.seed), z[np.arange(4), act])


def test_batch_recipe():
    cfg = synth.CONFIGS["tiny"]
    b = synth.make_batch(cfg)
    assert b.version.tolist() == [1000] * 4 + [999] * 4 + [998] * 4 + [999] * 4
    assert np.all(b.old_logp <= 0) and np.all(b.ref_logp <= 0)          # SPEC.md :41 every logprob <= 0
    assert set(np.unique(b.reward)) <= {0.0, 1.0}
    # shards regenerate identical values
    b2 = synth.make_batch(cfg, 4, 12)
    np.testing.assert_array_equal(b2.action, b.action[4:12])
    np.testing.assert_array_equal(b2.old_logp, b.old_logp[4:12])
    r = synth.make_batch(cfg, lengths="ragged")
    assert r.resp_len.min() >= 1 and r.resp_len.max() <= cfg.S


@pytest.mark.parametrize("G", [4, 8, 16])
def test_zero_variance_fraction(G):
    cfg = synth.Config("x", 4000, G, 1, 8, "f32", 0, 0.0, "zero", 9)
    b = synth.make_batch(cfg, want_tokens=False)
    r = b.reward.reshape(-1, G)
    frac = np.mean(np.all(r == r[:, :1], axis=1))
    assert abs(frac - 2.0 / (G + 1)) < 0.03
