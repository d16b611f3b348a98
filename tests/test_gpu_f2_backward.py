"""GPU parity of the f2 training step through the LM head: echo_loss_from_logp,
echo_lmhead_dlogits (D recomputed on the tensor cores) and echo_lmhead_backward (dhidden, dweight) against the fp64
oracle (oracle.loss_from_logp, oracle.lmhead_backward) on the same seeded inputs, through the C ABI."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from _util import coef_sens

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)


def _bits(t):
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


def _bf(t):
    return (_bits(t).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _case(n, d, V, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    h = torch.randn(n, d, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(V, d, generator=g, device="cuda") * (2.0 / math.sqrt(d))).to(torch.bfloat16)
    act = torch.randint(0, V, (n,), generator=g, device="cuda", dtype=torch.int32)
    return h, w, act


def _coefs(n, seed, lp, eta):
    """Seeded per-token inputs of the backward from the oracle's (4): c_t from oracle.loss_from_logp at the oracle's
    logp with a power-of-two grad_scale putting max|c| in [0.25, 0.5) (so |D| <= 0.5 and the 2e-3 bar is meaningful),
    e_t = grad_scale eta / n; both rounded to fp32 (the ABI's type) and fed to both sides."""
    rng = np.random.default_rng(seed)
    old = (lp + rng.normal(size=n) * 0.2).astype(np.float32)
    adv = rng.normal(size=8).astype(np.float32)
    slot = rng.integers(0, 8, n).astype(np.int32)
    _, _, c1 = oracle.loss_from_logp(lp, old, None, slot, adv, n_global=float(n))
    scale = 2.0 ** math.floor(math.log2(0.5 / max(np.max(np.abs(c1)), 1e-30)))
    _, _, coef = oracle.loss_from_logp(lp, old, None, slot, adv, n_global=float(n), grad_scale=scale)
    c32 = coef.astype(np.float32)
    e32 = np.full(n, np.float32(scale * eta / n), np.float32) if eta > 0 else None
    return c32, e32


# ------------------------------------------------------------------------------------------ (4) from logp
@pytest.mark.parametrize("kl_coef,eta,dual,est,weights", [(0.0, 0.0, 0.0, 0, False), (0.05, 0.0, 3.0, 0, False),
                                                          (0.1, 0.01, 0.0, 1, True), (0.1, 0.02, 2.0, 2, False)])
def test_loss_from_logp_matches_oracle(kl_coef, eta, dual, est, weights):
    from paper_2508_05387_b200 import abi
    n = 5000
    rng = np.random.default_rng(11)
    lp = (-np.abs(rng.normal(size=n)) * 3).astype(np.float32)
    old = (lp + rng.normal(size=n) * 0.3).astype(np.float32)
    ref = (lp + rng.normal(size=n) * 0.3).astype(np.float32)
    ent = np.abs(rng.normal(size=n) * 2).astype(np.float32)
    adv = rng.normal(size=64).astype(np.float32)
    slot = rng.integers(0, 64, n).astype(np.int32)
    wt = (rng.random(n) / n).astype(np.float32) if weights else None
    N = float(n)
    o_loss, o_flags, o_coef = oracle.loss_from_logp(lp.astype(np.float64), old, ref, slot, adv, n_global=N,
                                                    kl_coef=kl_coef, grad_scale=2.0, tok_weight=wt, clip_dual=dual,
                                                    kl_estimator=est, entropy_coef=eta,
                                                    tok_entropy=ent.astype(np.float64))
    c = lambda x: None if x is None else torch.from_numpy(x).cuda()
    loss = torch.empty(n, device="cuda")
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    coef = torch.empty(n, device="cuda")
    ecoef = torch.empty(n, device="cuda")
    ng = torch.tensor([N], dtype=torch.float64, device="cuda")
    cfg = abi.LossConfig(0.2, 0.2, dual, kl_coef, 2.0, est, eta)
    abi.echo_loss_from_logp(n, c(lp), c(ent), c(old), c(ref), c(slot), c(adv), None, c(wt), ng, cfg, loss, flags,
                            coef, ecoef)
    torch.cuda.synchronize()
    g_loss, g_flags, g_coef = loss.cpu().numpy(), flags.cpu().numpy(), coef.cpu().numpy()
    # the clip decision is taken in fp32 on the GPU: allow a flip only within fp32 rounding of a clip boundary
    rho = np.exp(lp.astype(np.float64) - old)
    near = (np.abs(rho - 0.8) < 1e-5) | (np.abs(rho - 1.2) < 1e-5) | (dual > 0) & (np.abs(rho - dual) < 1e-5)
    assert np.all((g_flags == o_flags) | near)
    ok = g_flags == o_flags
    scale = np.maximum(np.abs(o_loss), 1.0)
    assert np.max(np.abs(g_loss - o_loss)[ok] / scale[ok]) <= 1e-5
    cs = np.maximum(np.abs(o_coef), np.max(np.abs(o_coef)) * 1e-3)
    assert np.max(np.abs(g_coef - o_coef)[ok] / cs[ok]) <= 1e-5
    w_t = wt.astype(np.float64) if weights else np.full(n, 1.0 / N)
    np.testing.assert_allclose(ecoef.cpu().numpy(), np.float32(2.0) * w_t * np.float32(eta), rtol=1e-6, atol=0)


def test_loss_from_logp_equals_the_fused_path_bit_for_bit():
    """Same logp in, same scalar arithmetic: the fused kernel's per-token loss and flags on bf16 logits are
    reproduced bit for bit by echo_loss_from_logp fed the fused kernel's own tok_logp / tok_entropy."""
    from paper_2508_05387_b200 import abi
    n, V = 777, 4096
    g = torch.Generator(device="cuda").manual_seed(3)
    logits = (torch.randn(n, V, generator=g, device="cuda") * 2).to(torch.bfloat16)
    act = torch.randint(0, V, (n,), generator=g, device="cuda", dtype=torch.int32)
    old = torch.randn(n, generator=g, device="cuda") - 8.0
    ref = torch.randn(n, generator=g, device="cuda") - 8.0
    adv = torch.randn(16, generator=g, device="cuda")
    slot = torch.randint(0, 16, (n,), generator=g, device="cuda", dtype=torch.int32)
    ng = torch.tensor([float(n)], dtype=torch.float64, device="cuda")
    cfg = abi.LossConfig(0.2, 0.28, 3.0, 0.05, 1.0, abi.ECHO_KL_K3, 0.01)
    lp, loss, ent = (torch.empty(n, device="cuda") for _ in range(3))
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    abi.echo_policy_loss_fwd_bwd_v2(logits, abi.ECHO_BF16, n, V, V, act, old, ref, slot, adv, None, None, ng, cfg, lp,
                                    loss, flags, tok_entropy=ent)
    loss2, coef = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    flags2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    abi.echo_loss_from_logp(n, lp, ent, old, ref, slot, adv, None, None, ng, cfg, loss2, flags2, coef)
    torch.cuda.synchronize()
    assert torch.equal(loss.view(torch.int32), loss2.view(torch.int32))
    assert torch.equal(flags, flags2)


# ------------------------------------------------------------------------------------------ D on the tensor cores
def _d_check(dz_gpu, dz_ref):
    """bf16 output (2^-9 relative rounding) of a value whose inputs carry the fp32-accumulated logit error (~1e-5
    relative in p): |err| <= 2^-8 |D| + 2e-5 max_v |D[t, :]| per element, and 2e-3 absolute with max|D| <= 0.5."""
    row_max = np.max(np.abs(dz_ref), axis=1, keepdims=True)
    err = np.abs(dz_gpu - dz_ref)
    bound = 2.0 ** -8 * np.abs(dz_ref) + 2e-5 * row_max + 1e-30
    assert np.all(err <= bound), np.max(err / bound)
    assert np.max(err) <= 2e-3


@pytest.mark.parametrize("n,d,V,eta", [(128, 64, 256, 0.0), (300, 512, 1000, 0.01), (129, 72, 257, 0.0),
                                       (1, 2560, 4096, 0.02), (700, 256, 5003, 0.0)])
def test_lmhead_dlogits_matches_oracle(n, d, V, eta):
    from paper_2508_05387_b200 import abi
    h, w, act = _case(n, d, V, seed=n * 7 + V)
    hb, wb, a = _bits(h), _bits(w), act.cpu().numpy()
    lp, lse, H = oracle.lmhead_logp(hb, wb, a, want_entropy=True)
    c32, e32 = _coefs(n, n + d, lp, eta=eta)
    _, _, dz_ref = oracle.lmhead_backward(hb, wb, a, c32, e32, want_dlogits=True)
    ld = abi.echo_lmhead_dlogits_ld(V) + 8
    dz = torch.full((n, ld), 7.0, dtype=torch.bfloat16, device="cuda")
    cu = lambda x: None if x is None else torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    abi.echo_lmhead_dlogits(h, w, n, d, V, act, cu(lse), cu(c32), cu(e32), cu(H) if eta > 0 else None, dz, ld)
    torch.cuda.synchronize()
    out = _bf(dz)
    assert np.all(out[:, V:] == 7.0)                                   # columns >= vocab untouched
    _d_check(out[:, :V], dz_ref)


# ------------------------------------------------------------------------------------------ dhidden, dweight
@pytest.mark.parametrize("n,d,V,chunk,eta", [(300, 128, 1000, 128, 0.0), (257, 64, 777, 300, 0.02),
                                             (520, 256, 2048, 200, 0.01), (700, 200, 1500, 700, 0.0)])
def test_lmhead_backward_matches_oracle(n, d, V, chunk, eta):
    """dhidden and dweight (accumulated onto a prefilled buffer) over several chunks with a ragged last chunk.
    Bound: D is bf16 (2^-9 relative) on top of its own ~1e-5 logit error; the GEMMs accumulate in fp32:
    |err| <= 2^-7 (|D| |W|) (resp. |D|^T |h|) + 1e-6 of the row's scale."""
    from paper_2508_05387_b200 import abi
    h, w, act = _case(n, d, V, seed=n + V)
    hb, wb, a = _bits(h), _bits(w), act.cpu().numpy()
    lp, lse, H = oracle.lmhead_logp(hb, wb, a, want_entropy=True)
    c32, e32 = _coefs(n, 5, lp, eta=eta)
    dh_ref, dw_ref, dz_ref = oracle.lmhead_backward(hb, wb, a, c32, e32, want_dlogits=True)
    cu = lambda x: None if x is None else torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
    dh = torch.full((n, d), float("nan"), device="cuda")
    prev = torch.randn(V, d, device="cuda")
    dw = prev.clone()
    ws = torch.empty(chunk * abi.echo_lmhead_dlogits_ld(V), dtype=torch.bfloat16, device="cuda")
    abi.echo_lmhead_backward(h, w, n, d, V, act, cu(lse), cu(c32), cu(e32), cu(H) if eta > 0 else None, dh, dw, 1,
                             ws, chunk)
    torch.cuda.synchronize()
    absD = np.abs(dz_ref)
    bh = 2.0 ** -7 * (absD @ np.abs(_bf(w))) + 1e-6 * np.max(np.abs(dh_ref), axis=1, keepdims=True) + 1e-12
    bw = 2.0 ** -7 * (absD.T @ np.abs(_bf(h))) + 1e-6 * np.max(np.abs(dw_ref)) + 1e-12
    g_dh = dh.cpu().numpy().astype(np.float64)
    g_dw = (dw - prev).cpu().numpy().astype(np.float64)
    assert np.all(np.abs(g_dh - dh_ref) <= bh), np.max(np.abs(g_dh - dh_ref) / bh)
    assert np.all(np.abs(g_dw - dw_ref) <= bw + 1e-6 * np.abs(prev.cpu().numpy())), np.max(np.abs(g_dw - dw_ref) / bw)
    # overwrite mode and determinism
    dw2 = torch.full((V, d), float("nan"), device="cuda")
    dh2 = torch.empty(n, d, device="cuda")
    abi.echo_lmhead_backward(h, w, n, d, V, act, cu(lse), cu(c32), cu(e32), cu(H) if eta > 0 else None, dh2, dw2, 0,
                             ws, chunk)
    torch.cuda.synchronize()
    assert torch.equal(dh, dh2)
    assert np.all(np.abs(dw2.cpu().numpy() - dw_ref) <= bw)


def test_lmhead_backward_edge_cases_and_errors():
    from paper_2508_05387_b200 import abi
    n, d, V = 64, 64, 300
    h, w, act = _case(n, d, V, seed=1)
    f = lambda: torch.zeros(n, device="cuda")
    dh, dw = torch.empty(n, d, device="cuda"), torch.full((V, d), 5.0, device="cuda")
    ws = torch.empty(n * abi.echo_lmhead_dlogits_ld(V), dtype=torch.bfloat16, device="cuda")
    abi.echo_lmhead_backward(h, w, 0, d, V, act, f(), f(), None, None, dh, dw, 1, ws, 16)   # n = 0, accumulate: no-op
    torch.cuda.synchronize()
    assert torch.all(dw == 5.0)
    abi.echo_lmhead_backward(h, w, 0, d, V, act, f(), f(), None, None, dh, dw, 0, ws, 16)   # n = 0, overwrite: zeros
    torch.cuda.synchronize()
    assert torch.all(dw == 0.0)
    with pytest.raises(abi.EchoError):
        abi.echo_lmhead_backward(h, w, n, d, V, act, f(), f(), None, None, dh, dw, 0, ws, 0)   # chunk_rows 0
    with pytest.raises(abi.EchoError):
        abi.echo_lmhead_backward(h, w, n, d, V, act, f(), f(), f(), None, dh, dw, 0, ws, 16)   # ecoef without H
    with pytest.raises(abi.EchoError):
        abi.echo_lmhead_dlogits(h, w, n, d, V, act, f(), f(), None, None, ws, V)               # ld % 8 != 0
    # zero coefficients give a zero gradient
    abi.echo_lmhead_backward(h, w, n, d, V, act, f(), f(), None, None, dh, dw, 0, ws, 16)
    torch.cuda.synchronize()
    assert torch.all(dh == 0) and torch.all(dw == 0)


# ------------------------------------------------------------------------------------------ the step through it
def test_learner_step_loss_from_hidden_recompute_qwen_vocab():
    """LearnerStep.loss_from_hidden at a Qwen vocabulary (d = 2560, V = 151936) over 512 packed tokens in two chunks:
    per-token logp / loss against the oracle chain (lmhead_logp -> loss_from_logp), dhidden on sampled rows against
    oracle.lmhead_backward; dweight's columns sum to ~0 (every row of D sums to zero)."""
    from paper_2508_05387_b200.step import LearnerStep
    cfg = synth.CONFIGS["qwen3-4b"]
    b = synth.make_batch(cfg, 0, cfg.G)
    st = LearnerStep(n_rollouts=cfg.G, group_size=cfg.G, max_len=cfg.S, vocab=cfg.V, dtype=cfg.dtype)
    st.h2d(*[torch.from_numpy(np.ascontiguousarray(x)) for x in (b.version, b.resp_len, b.reward, b.action,
                                                                 b.old_logp, b.ref_logp)])
    info = st.pack(t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
    st.advantage()
    st.reduce_counts()
    n, d, V = 512, 2560, cfg.V
    assert info.n_tokens >= n
    g = torch.Generator(device="cuda").manual_seed(9)
    h = torch.randn(n, d, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(V, d, generator=g, device="cuda") * (2.0 / math.sqrt(d))).to(torch.bfloat16)
    dh = torch.empty(n, d, device="cuda")
    dw = torch.empty(V, d, device="cuda")
    N = info.n_tokens
    st.loss_from_hidden(h, w, 0, dh, dw, accumulate=False, kl_coef=0.01, entropy_coef=0.01, grad_scale=float(N),
                        chunk_rows=256, mode="recompute")
    torch.cuda.synchronize()
    act = st.tok_action[:n].cpu().numpy()
    rows = np.array([0, 1, 255, 256, 400, 511])
    hb, wb = _bits(h[rows]), _bits(w)
    lp, lse, H = oracle.lmhead_logp(hb, wb, act[rows], want_entropy=True)
    slot, adv = st.tok_slot[:n].cpu().numpy()[rows], st.adv_slot.cpu().numpy()
    old, ref = st.tok_old[:n].cpu().numpy()[rows], st.tok_ref[:n].cpu().numpy()[rows]
    o_loss, o_flags, o_coef = oracle.loss_from_logp(lp, old, ref, slot, adv, n_global=float(N), kl_coef=0.01,
                                                    grad_scale=float(N), entropy_coef=0.01, tok_entropy=H)
    g_lp = st.tok_logp[:n].cpu().numpy()[rows]
    assert np.max(np.abs(g_lp - lp)) <= 2e-4
    assert np.max(np.abs(st.tok_loss[:n].cpu().numpy()[rows] - o_loss) / np.maximum(np.abs(o_loss), 1)) <= 1e-3
    e = np.full(len(rows), np.float32(N) * np.float32(0.01) / N)
    dh_ref, _ = oracle.lmhead_backward(hb, wb, act[rows], o_coef, e, want_dweight=False)
    g_dh = dh.cpu().numpy()[rows].astype(np.float64)
    scale = np.max(np.abs(dh_ref), axis=1, keepdims=True)
    assert np.max(np.abs(g_dh - dh_ref) / scale) <= 1e-2, np.max(np.abs(g_dh - dh_ref) / scale)
    col = dw.sum(dim=0).abs().max().item()
    assert col <= 1e-2 * dw.abs().sum(dim=0).max().item()
    assert torch.isfinite(dw).all() and torch.isfinite(dh).all()


# ------------------------------------------------------------------------------------------ chunked: logits + fused loss
def _bf16_rne(x):
    """fp64 -> fp32 -> bf16 (round to nearest even at each step: the GPU's fp32 accumulator -> bf16 store)."""
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def _z_tol(hb, wb):
    """fp32-accumulation bound of the tcgen05 GEMM per element (as _lmhead_tol in test_gpu_parity.py, not doubled)."""
    widen = lambda b: (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    hf, wf = widen(hb), widen(wb)
    return 4 * (hb.shape[1] / 16 + 16) * 2.0 ** -24 * (np.abs(hf) @ np.abs(wf).T), hf, wf


@pytest.mark.parametrize("n,d,V", [(300, 128, 1000), (129, 72, 257), (64, 2560, 4096)])
def test_lmhead_logits_bf16(n, d, V):
    """echo_lmhead_logits: bf16(z) with z = h W^T; each element is the bf16 rounding of a value within the fp32
    accumulation bound of the fp64 product, i.e. one of the (at most two) bf16 values that bracket z +- tol."""
    from paper_2508_05387_b200 import abi
    h, w, _ = _case(n, d, V, seed=V + 1)
    hb, wb = _bits(h), _bits(w)
    tol, hf, wf = _z_tol(hb, wb)
    z = hf @ wf.T
    ld = abi.echo_lmhead_dlogits_ld(V) + 8
    out = torch.full((n, ld), 3.0, dtype=torch.bfloat16, device="cuda")
    abi.echo_lmhead_logits(h, w, n, d, V, out, ld)
    torch.cuda.synchronize()
    g = _bits(out)
    assert np.all(_bf(out)[:, V:] == 3.0)
    gz = _bf(out)[:, :V]
    # |bf16(z_gpu) - z| <= half an ulp of the stored value + the accumulation error of z_gpu (bound doubled, as for logp)
    err = np.abs(gz - z)
    print(f"lmhead_logits n={n} d={d} V={V}: max (err - ulp/2) / tol = {np.max((err - 0.5 * _ulp(gz)) / tol):.3f}")
    assert np.all(err <= 0.5 * _ulp(gz) + 2 * tol), np.max(err / (0.5 * _ulp(gz) + 2 * tol))
    assert (g[:, :V] == _bf16_rne(z)).mean() > 0.99


def _ulp(x):
    """ulp of bf16 values (8 significant bits)."""
    x = np.maximum(np.abs(np.asarray(x, np.float64)), 2.0 ** -126)
    return 2.0 ** (np.floor(np.log2(x)) - 7)


@pytest.mark.parametrize("n,d,V,chunk,eta", [(300, 128, 1000, 128, 0.0), (260, 64, 777, 100, 0.01)])
def test_lmhead_policy_loss_chunked_matches_oracle(n, d, V, chunk, eta):
    """The chunked f2 step (echo_lmhead_policy_loss_fwd_bwd) against the oracle chain on the same bf16-rounded logits:
    oracle.policy_loss on bf16(h W^T) (fp64 from the bf16 values), then dhidden = D W and dweight = D^T h in fp64.
    Tokens whose action logit lies within the GEMM's fp32 error of a bf16 rounding boundary are excluded from the
    per-token comparison (their bf16 logit may legitimately differ by one ulp)."""
    from paper_2508_05387_b200 import abi
    h, w, act = _case(n, d, V, seed=n + 3)
    hb, wb, a = _bits(h), _bits(w), act.cpu().numpy()
    tol, hf, wf = _z_tol(hb, wb)
    z = hf @ wf.T
    zb = _bf16_rne(z)
    amb = _bf16_rne(z - 2 * tol) != _bf16_rne(z + 2 * tol)
    rng = np.random.default_rng(n)
    old = (rng.normal(size=n) - 7.0).astype(np.float32)
    ref = (rng.normal(size=n) - 7.0).astype(np.float32)
    adv = rng.normal(size=16).astype(np.float32)
    slot = rng.integers(0, 16, n).astype(np.int32)
    kl = 0.05
    o = oracle.policy_loss(zb, a, old, ref, slot, adv, n_global=float(n), dtype=oracle.BF16, kl_coef=kl,
                           grad_scale=float(n) / 4, entropy_coef=eta)
    dh_ref, dw_ref = o.dlogits @ wf, o.dlogits.T @ hf
    cu = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    lp, loss, ent = (torch.empty(n, device="cuda") for _ in range(3))
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    dh = torch.empty(n, d, device="cuda")
    dw = torch.empty(V, d, device="cuda")
    ws = torch.empty(chunk * abi.echo_lmhead_dlogits_ld(V), dtype=torch.bfloat16, device="cuda")
    ng = torch.tensor([float(n)], dtype=torch.float64, device="cuda")
    cfg = abi.LossConfig(0.2, 0.2, 0.0, kl, float(n) / 4, abi.ECHO_KL_K3, eta)
    abi.echo_lmhead_policy_loss_fwd_bwd(h, w, n, d, V, act, cu(old), cu(ref), cu(slot), cu(adv), None, None, ng, cfg,
                                        lp, loss, flags, ent, dh, dw, 0, ws, chunk)
    torch.cuda.synchronize()
    # per-token bound: an element whose z lies within the GEMM's error of a bf16 rounding boundary may be stored one
    # ulp away; that moves logp by up to ulp(z_a) at the action and lse by p_v ulp(z_v) elsewhere
    zf = (zb.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    lse = zf[np.arange(n), a] - o.logp
    pz = np.exp(zf - lse[:, None])
    u = _ulp(zf) * amb
    b_lp = 2e-5 + u[np.arange(n), a] + (pz * u).sum(axis=1)
    g_lp = lp.cpu().numpy()
    assert np.all(np.abs(g_lp - o.logp) <= b_lp), np.max(np.abs(g_lp - o.logp) / b_lp)
    # the loss moves with logp at most by |dl/dlogp| <= |A| rho + beta (1 + e^(ref - logp)) (times e^b for rho)
    g_loss = loss.cpu().numpy()
    A = adv[slot].astype(np.float64)
    rho = np.exp(o.logp - old)
    lip = np.abs(A) * rho * np.exp(b_lp) + kl * (1 + np.exp(ref - o.logp) * np.exp(b_lp))
    b_loss = lip * b_lp + 1e-5 * np.maximum(np.abs(o.loss), 1)
    assert np.all(np.abs(g_loss - o.loss) <= b_loss), np.max(np.abs(g_loss - o.loss) / b_loss)
    clean = np.ones(n, bool)
    absD = np.abs(o.dlogits)
    bh = 2.0 ** -7 * (absD @ np.abs(wf)) + 1e-6 * np.max(np.abs(dh_ref)) + 1e-12
    bw = 2.0 ** -7 * (absD.T @ np.abs(hf)) + 1e-6 * np.max(np.abs(dw_ref)) + 1e-12
    g_dh = dh.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(g_dh - dh_ref)[clean] <= bh[clean]), np.max(np.abs(g_dh - dh_ref)[clean] / bh[clean])
    assert np.mean(np.abs(dw.cpu().numpy() - dw_ref) <= bw) > 0.999


def test_learner_step_chunked_equals_unchunked_logits_path():
    """LearnerStep.loss_from_hidden (chunked) at a Qwen vocabulary equals, bit for bit in tok_logp / tok_loss /
    tok_flags, the logits path on the same bf16 logits (echo_lmhead_logits for all rows, then LearnerStep.loss);
    dhidden / dweight equal cuBLAS on that path's gradient chunk by chunk."""
    from paper_2508_05387_b200 import abi
    from paper_2508_05387_b200.step import LearnerStep
    cfg = synth.CONFIGS["qwen3-4b"]
    b = synth.make_batch(cfg, 0, cfg.G)
    st = LearnerStep(n_rollouts=cfg.G, group_size=cfg.G, max_len=cfg.S, vocab=cfg.V, dtype=cfg.dtype)
    st.h2d(*[torch.from_numpy(np.ascontiguousarray(x)) for x in (b.version, b.resp_len, b.reward, b.action,
                                                                 b.old_logp, b.ref_logp)])
    info = st.pack(t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
    st.advantage()
    st.reduce_counts()
    n, d, V = 640, 1024, cfg.V
    g = torch.Generator(device="cuda").manual_seed(4)
    h = torch.randn(n, d, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(V, d, generator=g, device="cuda") * (2.0 / math.sqrt(d))).to(torch.bfloat16)
    dh = torch.empty(n, d, device="cuda")
    dw = torch.empty(V, d, device="cuda")
    st.loss_from_hidden(h, w, 0, dh, dw, accumulate=False, kl_coef=0.01, grad_scale=float(info.n_tokens),
                        chunk_rows=256)
    lp1, loss1, fl1 = st.tok_logp[:n].clone(), st.tok_loss[:n].clone(), st.tok_flags[:n].clone()
    logits = torch.empty(n, V, dtype=torch.bfloat16, device="cuda")
    abi.echo_lmhead_logits(h, w, n, d, V, logits, V)
    st.loss(logits, 0, kl_coef=0.01, grad_scale=float(info.n_tokens))
    torch.cuda.synchronize()
    assert torch.equal(lp1.view(torch.int32), st.tok_logp[:n].view(torch.int32))
    assert torch.equal(loss1.view(torch.int32), st.tok_loss[:n].view(torch.int32))
    assert torch.equal(fl1, st.tok_flags[:n])
    ref_dh = logits.float() @ w.float()
    rel = (dh - ref_dh).abs().max().item() / ref_dh.abs().max().item()
    assert rel < 1e-3, rel


def test_lmhead_policy_loss_edge_cases_and_errors():
    """n_rows = 0 (dweight zeroed or untouched), a single chunk larger than n, argument errors reported before any
    launch."""
    from paper_2508_05387_b200 import abi
    n, d, V = 40, 64, 300
    h, w, act = _case(n, d, V, seed=2)
    z = lambda: torch.zeros(n, device="cuda")
    slot = torch.zeros(n, dtype=torch.int32, device="cuda")
    adv = torch.ones(1, device="cuda")
    ng = torch.tensor([float(n)], dtype=torch.float64, device="cuda")
    cfg = abi.LossConfig(0.2, 0.2, 0.0, 0.0, 1.0, abi.ECHO_KL_K3, 0.0)
    lp, loss = z(), z()
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    dh = torch.empty(n, d, device="cuda")
    dw = torch.full((V, d), 2.0, device="cuda")
    ws = torch.empty(4 * n * abi.echo_lmhead_dlogits_ld(V), dtype=torch.bfloat16, device="cuda")
    args = lambda rows, acc, chunk, c=cfg: (h, w, rows, d, V, act, z(), None, slot, adv, None, None, ng, c, lp, loss,
                                            flags, None, dh, dw, acc, ws, chunk)
    abi.echo_lmhead_policy_loss_fwd_bwd(*args(0, 1, 16))
    torch.cuda.synchronize()
    assert torch.all(dw == 2.0)
    abi.echo_lmhead_policy_loss_fwd_bwd(*args(0, 0, 16))
    torch.cuda.synchronize()
    assert torch.all(dw == 0.0)
    abi.echo_lmhead_policy_loss_fwd_bwd(*args(n, 0, 4 * n))          # one chunk covering everything
    torch.cuda.synchronize()
    assert torch.isfinite(dh).all() and torch.isfinite(dw).all() and torch.isfinite(lp).all()
    for bad in (args(n, 0, 0), args(n, 0, 16, abi.LossConfig(1.5, 0.2, 0.0, 0.0, 1.0, abi.ECHO_KL_K3, 0.0))):
        with pytest.raises(abi.EchoError):
            abi.echo_lmhead_policy_loss_fwd_bwd(*bad)
    with pytest.raises(abi.EchoError):                                  # ld not a multiple of 8
        abi.echo_lmhead_logits(h, w, n, d, V, ws, V)


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("m,n,k", [(256, 256, 64), (300, 200, 1000), (1, 72, 4096), (777, 513, 130),
                                   (300, 200, 16384), (513, 300, 9000)])   # the last two split K (4 and 2 pieces)
@pytest.mark.parametrize("tma_out", [False, True])
@pytest.mark.parametrize("wide", ["0", "1", "1-all-at-once"])
def test_gemm_bf16_all_majors(a_mn, b_mn, m, n, k, tma_out, wide, monkeypatch):
    """echo_gemm_bf16 (the tcgen05 GEMM of the f2 backward) in every operand layout against the fp64 product, within
    the fp32-accumulation bound 4 (K/16 + 16) 2^-24 sum_k |A B|; ragged M / N / K tiles; accumulate and overwrite
    modes; an output row stride that is a multiple of 4 floats takes the TMA store / L2-add epilogue, any other the
    per-thread one.  wide = 1: 256 x 512 units, two TMEM accumulators sharing each A k-block (N tiles paired up, an
    odd last one computed against zero-filled B and not stored); the epilogue releases the two accumulators one by one
    (the default: the next unit's first k-blocks run on accumulator 0 while accumulator 1 drains) or, with
    1-all-at-once (ECHO_GEMM_HALFREL=0), together."""
    monkeypatch.setenv("ECHO_GEMM_WIDE", wide[0])
    monkeypatch.setenv("ECHO_GEMM_HALFREL", "0" if wide.endswith("once") else "1")
    from paper_2508_05387_b200 import abi
    g = torch.Generator(device="cuda").manual_seed(m + n + k + 2 * a_mn + b_mn)
    A = torch.randn(m, k, generator=g, device="cuda").to(torch.bfloat16)
    B = torch.randn(n, k, generator=g, device="cuda").to(torch.bfloat16)
    a_store = (A.t() if a_mn else A).contiguous()
    b_store = (B.t() if b_mn else B).contiguous()
    ld = lambda w: (w + 7) // 8 * 8 + 8                               # row strides: multiples of 8, padded
    a_buf = torch.zeros(a_store.shape[0], ld(a_store.shape[1]), dtype=torch.bfloat16, device="cuda")
    b_buf = torch.zeros(b_store.shape[0], ld(b_store.shape[1]), dtype=torch.bfloat16, device="cuda")
    a_buf[:, :a_store.shape[1]] = a_store
    b_buf[:, :b_store.shape[1]] = b_store
    ldc = (n + 3) // 4 * 4 + 4 if tma_out else n + 3
    prev = torch.randn(m, ldc, generator=g, device="cuda")
    c = prev.clone()
    abi.echo_gemm_bf16(a_buf, a_mn, a_buf.shape[1], b_buf, b_mn, b_buf.shape[1], m, n, k, c, ldc, accumulate=True)
    torch.cuda.synchronize()
    Af, Bf = _bf(A), _bf(B)
    ref = Af @ Bf.T
    bound = 4 * (k / 16 + 16) * 2.0 ** -24 * (np.abs(Af) @ np.abs(Bf).T) + 1e-6 * np.abs(prev[:, :n].cpu().numpy())
    got = (c - prev)[:, :n].cpu().numpy().astype(np.float64)
    assert np.all(np.abs(got - ref) <= bound + 1e-6), np.max(np.abs(got - ref) / (bound + 1e-6))
    assert torch.equal(c[:, n:], prev[:, n:])                          # columns >= n untouched
    c2 = prev.clone()                                                  # deterministic (split-K pieces in fixed order)
    abi.echo_gemm_bf16(a_buf, a_mn, a_buf.shape[1], b_buf, b_mn, b_buf.shape[1], m, n, k, c2, ldc, accumulate=True)
    torch.cuda.synchronize()
    assert torch.equal(c, c2)
    c3 = prev.clone()                                                  # overwrite mode
    abi.echo_gemm_bf16(a_buf, a_mn, a_buf.shape[1], b_buf, b_mn, b_buf.shape[1], m, n, k, c3, ldc, accumulate=False)
    torch.cuda.synchronize()
    got3 = c3[:, :n].cpu().numpy().astype(np.float64)
    bound3 = 4 * (k / 16 + 16) * 2.0 ** -24 * (np.abs(Af) @ np.abs(Bf).T)
    assert np.all(np.abs(got3 - ref) <= bound3 + 1e-6), np.max(np.abs(got3 - ref) / (bound3 + 1e-6))
    assert torch.equal(c3[:, n:], prev[:, n:])


def test_chunked_f4_options_equal_the_logits_path():
    """The chunked step offsets every per-token array per chunk: with per-token advantages and weights, the k2 KL,
    the dual clip and the entropy bonus, its tok_logp / tok_loss / tok_flags / tok_entropy equal (bit for bit) the
    logits path's (echo_lmhead_logits for all rows, then echo_policy_loss_fwd_bwd_v2)."""
    from paper_2508_05387_b200 import abi
    n, d, V, chunk = 1000, 256, 4099, 384
    h, w, act = _case(n, d, V, seed=11)
    g = torch.Generator(device="cuda").manual_seed(12)
    old = torch.randn(n, generator=g, device="cuda") - 8.0
    ref = torch.randn(n, generator=g, device="cuda") - 8.0
    tadv = torch.randn(n, generator=g, device="cuda")
    twt = torch.rand(n, generator=g, device="cuda") / n
    cfg = abi.LossConfig(0.2, 0.28, 3.0, 0.05, 2.0, abi.ECHO_KL_K2, 0.01)
    outs = []
    for path in ("chunked", "logits"):
        lp, loss, ent = (torch.empty(n, device="cuda") for _ in range(3))
        flags = torch.empty(n, dtype=torch.uint8, device="cuda")
        if path == "chunked":
            ws = torch.empty(chunk * abi.echo_lmhead_dlogits_ld(V), dtype=torch.bfloat16, device="cuda")
            dh, dw = torch.empty(n, d, device="cuda"), torch.empty(V, d, device="cuda")
            abi.echo_lmhead_policy_loss_fwd_bwd(h, w, n, d, V, act, old, ref, None, None, tadv, twt, None, cfg, lp,
                                                loss, flags, ent, dh, dw, 0, ws, chunk)
        else:
            ld = abi.echo_lmhead_dlogits_ld(V)
            z = torch.empty(n, ld, dtype=torch.bfloat16, device="cuda")
            abi.echo_lmhead_logits(h, w, n, d, V, z, ld)
            abi.echo_policy_loss_fwd_bwd_v2(z, abi.ECHO_BF16, n, V, ld, act, old, ref, None, None, tadv, twt, None,
                                            cfg, lp, loss, flags, tok_entropy=ent)
        torch.cuda.synchronize()
        outs.append((lp, loss, flags, ent))
    for a, b in zip(*outs):
        assert torch.equal(a.view(torch.uint8), b.view(torch.uint8))


def test_chunked_step_full_size_sampled_outputs():
    """The chunked f2 step at the bench's launch configuration (f2_train_step: 32768 tokens, d = 5120 -- Qwen3-32B's
    hidden size --, V = 151936, 8192-row chunks) against the fp64 oracle on sampled outputs it can compute one by one:
    logp / loss / dhidden of six rows spread over the four chunks (first and last rows of chunks, the last token),
    each row's logits computed in fp64 from the bf16 h and W and rounded like the GPU's fp32 accumulator; and sampled
    dweight entries, sum_t D[t, v] h[t, j] over all 32768 tokens in fp64, from the D that the one-chunk run of the same
    step leaves in its 10 GB buffer (that run's per-token results must equal the chunked run's bit for bit)."""
    from paper_2508_05387_b200 import abi
    n, d, V, chunk = 32768, 5120, 151936, 8192
    h, w, act = _case(n, d, V, seed=2508)
    rng = np.random.default_rng(2508)
    old = (rng.normal(size=n) * 0.3 - 14.0).astype(np.float32)      # ratios around 1: both clip sides populated
    ref = (rng.normal(size=n) * 0.3 - 14.0).astype(np.float32)
    adv = rng.normal(size=4096).astype(np.float32)
    slot = (np.arange(n) // 8).astype(np.int32)                      # 8 tokens per rollout slot
    kl, gs = 0.001, float(n) / 4
    cu = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    ng = torch.tensor([float(n)], dtype=torch.float64, device="cuda")
    cfg = abi.LossConfig(0.2, 0.2, 0.0, kl, gs, abi.ECHO_KL_K3, 0.0)
    ld = abi.echo_lmhead_dlogits_ld(V)
    runs = []
    for ck in (chunk, n):
        lp, loss = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
        flags = torch.empty(n, dtype=torch.uint8, device="cuda")
        dh, dw = torch.empty(n, d, device="cuda"), torch.empty(V, d, device="cuda")
        ws = torch.empty(ck, ld, dtype=torch.bfloat16, device="cuda")
        abi.echo_lmhead_policy_loss_fwd_bwd(h, w, n, d, V, act, cu(old), cu(ref), cu(slot), cu(adv), None, None, ng,
                                            cfg, lp, loss, flags, None, dh, dw, 0, ws, ck)
        torch.cuda.synchronize()
        runs.append((lp, loss, flags, dh, dw, ws))
    (lp, loss, flags, dh, dw, _), (lp1, loss1, flags1, _, _, D_all) = runs
    assert torch.equal(lp.view(torch.int32), lp1.view(torch.int32))
    assert torch.equal(loss.view(torch.int32), loss1.view(torch.int32))
    assert torch.equal(flags, flags1)
    # ---- sampled rows: fp64 logits row by row (W widened block by block), the oracle's (3)-(5), dhidden = D W
    S = np.array([0, 1, chunk - 1, chunk, 2 * chunk + 123, n - 1])
    hb, wb, a = _bits(h[torch.as_tensor(S, device="cuda")]), _bits(w), act.cpu().numpy()[S]
    widen = lambda b: (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    hf = widen(hb)
    z, tol = np.empty((len(S), V)), np.empty((len(S), V))
    blocks = [(v0, min(v0 + 8192, V)) for v0 in range(0, V, 8192)]
    for v0, v1 in blocks:
        wf = widen(wb[v0:v1])
        z[:, v0:v1] = hf @ wf.T
        tol[:, v0:v1] = 4 * (d / 16 + 16) * 2.0 ** -24 * (np.abs(hf) @ np.abs(wf).T)
    zb = _bf16_rne(z)
    # an element whose z lies within the GEMM's fp32 bound of a bf16 rounding boundary may be stored one ulp away (at
    # d = 5120 the worst-case bound makes most elements "ambiguous"; the slack below charges each of them a full ulp)
    amb = _bf16_rne(z - 2 * tol) != _bf16_rne(z + 2 * tol)
    o = oracle.policy_loss(zb, a, old[S], ref[S], slot[S], adv, n_global=float(n), dtype=oracle.BF16, kl_coef=kl,
                           grad_scale=gs)
    zf = (zb.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    r = np.arange(len(S))
    lse = zf[r, a] - o.logp
    pz = np.exp(zf - lse[:, None])
    u = _ulp(zf) * amb
    dlse = (pz * u).sum(axis=1)                                      # what the ambiguous elements can move lse by
    b_lp = 2e-5 + u[r, a] + dlse
    g_lp, g_loss = lp.cpu().numpy()[S], loss.cpu().numpy()[S]
    assert np.all(np.abs(g_lp - o.logp) <= b_lp), np.max(np.abs(g_lp - o.logp) / b_lp)
    A, rho = adv[slot[S]].astype(np.float64), np.exp(o.logp - old[S])
    lip = np.abs(A) * rho * np.exp(b_lp) + kl * (1 + np.exp(ref[S] - o.logp) * np.exp(b_lp))
    b_loss = lip * b_lp + 1e-5 * np.maximum(np.abs(o.loss), 1)
    assert np.all(np.abs(g_loss - o.loss) <= b_loss), np.max(np.abs(g_loss - o.loss) / b_loss)
    # rows whose ratio sits within the logp bound of a clip boundary may legitimately flip branch: excluded
    lr = np.log(rho)
    far = np.minimum(np.abs(lr - math.log(0.8)), np.abs(lr - math.log(1.2))) > 2 * b_lp
    assert far.sum() >= 4
    assert np.array_equal(flags.cpu().numpy()[S][far], o.flags[far])
    # dhidden rows: fp32-accumulation bound (2^-7 of sum |D||W| as in the small-size test) plus what the ambiguous
    # elements and the logp error can move D by: |dc| |delta - p| + |c| p (e^(u + dlse + dlp) - 1)
    sens, _ = coef_sens(o, old[S], ref[S], A, kl, gs, n_global=float(n))
    dlp = np.abs(g_lp - o.logp)
    dh_ref, adw, slack = np.zeros((len(S), d)), np.zeros((len(S), d)), np.zeros((len(S), d))
    for v0, v1 in blocks:
        wf = np.abs(widen(wb[v0:v1]))
        wsg = widen(wb[v0:v1])
        p_blk = pz[:, v0:v1]
        dD = (sens * (dlp + dlse))[:, None] * np.abs((np.arange(v0, v1)[None, :] == a[:, None]) - p_blk) + \
            np.abs(o.coef)[:, None] * p_blk * np.expm1(u[:, v0:v1] + (dlse + dlp)[:, None])
        dh_ref += o.dlogits[:, v0:v1] @ wsg
        adw += np.abs(o.dlogits[:, v0:v1]) @ wf
        slack += dD @ wf
    g_dh = dh[torch.as_tensor(S, device="cuda")].cpu().numpy().astype(np.float64)
    bh = 2.0 ** -7 * adw + slack + 1e-6 * np.max(np.abs(dh_ref)) + 1e-12
    err = np.abs(g_dh - dh_ref)[far]
    assert np.all(err <= bh[far]), np.max(err / bh[far])
    assert np.max(np.abs(dh_ref[far])) > 1e-3                        # the rows carry a real gradient
    print(f"[f2 full size] rows {far.sum()} ambiguous logits {amb.mean():.3f} max|dh err|/bound "
          f"{np.max(err / bh[far]):.3e} max|dh err|/max|dh| {np.max(err) / np.max(np.abs(dh_ref)):.3e}")
    # ---- sampled dweight entries over all four chunks: sum_t D[t, v] h[t, j] in fp64 from the one-chunk run's D
    vs = np.unique(np.concatenate([[0, V - 1, 77777], a, rng.integers(0, V, 6)]))
    js = np.array([0, 1, 2559, d - 1, 777])
    Dv = _bf(D_all[:, torch.as_tensor(vs, device="cuda")].contiguous())          # [n x |vs|]
    hj = _bf(h[:, torch.as_tensor(js, device="cuda")].contiguous())              # [n x |js|]
    dw_ref, adwj = Dv.T @ hj, np.abs(Dv).T @ np.abs(hj)
    g_dw = dw[torch.as_tensor(vs, device="cuda")][:, torch.as_tensor(js, device="cuda")].cpu().numpy()
    bw = 4 * (n / 16 + 16) * 2.0 ** -24 * adwj + 1e-12
    assert np.all(np.abs(g_dw - dw_ref) <= bw), np.max(np.abs(g_dw - dw_ref) / bw)
    assert np.max(np.abs(dw_ref)) > 0


def test_chunked_step_deterministic_and_graph_capturable():
    """The chunked f2 step on libecho's own kernels (no cuBLAS) is bitwise repeatable, and a CUDA graph of it replays
    to the same bits (the fused kernel's row scheduler resets its own counter slot)."""
    from paper_2508_05387_b200 import abi
    n, d, V, chunk = 700, 192, 3001, 256
    h, w, act = _case(n, d, V, seed=21)
    g = torch.Generator(device="cuda").manual_seed(22)
    old = torch.randn(n, generator=g, device="cuda") - 7.0
    slot = torch.zeros(n, dtype=torch.int32, device="cuda")
    adv = torch.randn(1, generator=g, device="cuda")
    ng = torch.tensor([float(n)], dtype=torch.float64, device="cuda")
    cfg = abi.LossConfig(0.2, 0.2, 0.0, 0.0, 4.0, abi.ECHO_KL_K3, 0.0)
    ws = torch.empty(chunk * abi.echo_lmhead_dlogits_ld(V), dtype=torch.bfloat16, device="cuda")

    def bufs():
        return ([torch.empty(n, device="cuda") for _ in range(2)] + [torch.empty(n, dtype=torch.uint8, device="cuda")]
                + [torch.empty(n, d, device="cuda"), torch.empty(V, d, device="cuda")])

    def run(b, stream=None):
        lp, loss, flags, dh, dw = b
        abi.echo_lmhead_policy_loss_fwd_bwd(h, w, n, d, V, act, old, None, slot, adv, None, None, ng, cfg, lp, loss,
                                            flags, None, dh, dw, 0, ws, chunk, stream=stream)

    b1, b2, b3 = bufs(), bufs(), bufs()
    run(b1)
    run(b2)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            run(b3, stream=s)
    graph.replay()
    torch.cuda.synchronize()
    for x, y, z in zip(b1, b2, b3):
        assert torch.equal(x.view(torch.uint8), y.view(torch.uint8))
        assert torch.equal(x.view(torch.uint8), z.view(torch.uint8))


def test_dynamic_schedulers_replay_in_cuda_graphs():
    """f1's one-warp-per-row kernel, the LM head and the backward GEMM take their row / tile counters from per-launch
    slots; launches captured into a CUDA graph draw from a slot range of their own.  One graph holding all
    three, replayed twice with eager launches of the same kernels in between, gives the eager results bit for bit."""
    from paper_2508_05387_b200 import abi
    g = torch.Generator(device="cuda").manual_seed(21)
    n, d, V = 1024, 256, 8200
    ld = (V + 7) // 8 * 8
    z = (torch.randn(n, ld, generator=g, device="cuda") * 2).to(torch.bfloat16)
    act = torch.randint(0, V, (n,), generator=g, device="cuda", dtype=torch.int32)
    h = torch.randn(n, d, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(V, d, generator=g, device="cuda") * (2.0 / math.sqrt(d))).to(torch.bfloat16)
    ws = torch.empty(abi.echo_lmhead_workspace_bytes(n, V) // 4 + 1, dtype=torch.float32, device="cuda")
    outs = lambda: (torch.empty(n, device="cuda"), torch.empty(n, device="cuda"), torch.zeros(n, d, device="cuda"))

    def run(o):
        lp, lm, dh = o
        abi.echo_token_logp(z, abi.ECHO_BF16, n, V, ld, act, lp)
        abi.echo_lmhead_logp(h, w, n, d, V, act, lm, None, ws)
        abi.echo_gemm_bf16(z, 0, ld, w, 1, d, n, d, V, dh, d)   # dhidden-shaped product (K = V)
    eager = outs()
    run(eager)
    torch.cuda.synchronize()
    got = outs()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run(got)                                                # warm-up outside capture
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        run(got)
    for _ in range(2):
        for t in got:
            t.zero_()
        graph.replay()
        run(outs())                                             # eager launches between replays
        torch.cuda.synchronize()
        for a, b in zip(got, eager):
            assert torch.equal(a, b)
