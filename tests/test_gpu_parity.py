"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star, made scale-aware in tests/_util.check_rows): packing and indices bit-exact;
advantages bit-exact; per-token logp |err| <= 1e-5; step loss within 1e-5 relative (of max(|L|, mean|l|));
dlogits within 2e-3 absolute for bf16 at a grad_scale putting max|d| in [0.25, 0.5), and faithful per element.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from _util import check_rows, coef_sens, host_rows, oracle_step, pow2_scale_for

pytestmark = pytest.mark.gpu

ALGOS = {"row_l2": 1, "quad_reg": 2, "quad_reg_exact": 3, "oct_reg": 4}


@pytest.fixture(scope="module", autouse=True)
def _build():
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)


def device_step(cfg, b, rollout_base=0, has_ref=True):
    from paper_2508_05387_b200.step import LearnerStep
    R = b.version.shape[0]
    st = LearnerStep(n_rollouts=R, group_size=cfg.G, max_len=cfg.S, vocab=cfg.V, dtype=cfg.dtype, has_ref=has_ref)
    t = [torch.from_numpy(np.ascontiguousarray(x)) for x in (b.version, b.resp_len, b.reward, b.action, b.old_logp)]
    st.h2d(*t, torch.from_numpy(np.ascontiguousarray(b.ref_logp)) if has_ref else None)
    info = st.pack(t_train=synth.T_TRAIN, max_lag=cfg.max_lag, rollout_base=rollout_base)
    st.advantage()
    st.reduce_counts()
    return st, info


def fill(st, cfg, row0, n_rows, ld=None):
    import synth.gpu as sgpu
    ld = cfg.V if ld is None else ld
    dt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    logits = torch.zeros(n_rows, ld, dtype=dt, device="cuda")
    sgpu.fill_logits(logits, dtype=cfg.dtype, vocab=cfg.V, row0=row0, tok_slot=st.tok_slot, tok_action=st.tok_action,
                     kept_rollout=st.kept_rollout, kept_offset=st.kept_offset, max_len=cfg.S, seed=cfg.seed)
    return logits


def as_oracle_rows(t):
    t = t.cpu()
    return t.view(torch.int16).numpy().view(np.uint16) if t.dtype == torch.bfloat16 else t.numpy()


# ---------------------------------------------------------------------------------------------- generator
def test_gpu_generator_matches_host_twin():
    for name in ("tiny", "qwen2.5-7b"):
        cfg = synth.CONFIGS[name]
        b = synth.make_batch(cfg, 0, 2 * cfg.G)
        st, info = device_step(cfg, b)
        o = oracle_step(cfg, b)
        rows = np.array([0, 1, 7, info.n_tokens - 1])
        logits = fill(st, cfg, 0, info.n_tokens)
        got = as_oracle_rows(logits[torch.from_numpy(rows).cuda()])
        np.testing.assert_array_equal(got, host_rows(cfg, o.keys[rows], o.pk.tok_action[rows]))


# ---------------------------------------------------------------------------------------------- (1) pack
@pytest.mark.parametrize("name,lengths", [("tiny", "full"), ("tiny", "ragged"), ("qwen2.5-7b", "ragged"),
                                          ("qwen3-4b", "full")])
def test_pack_bit_exact(name, lengths):
    cfg = synth.CONFIGS[name]
    b = synth.make_batch(cfg, lengths=lengths)
    st, info = device_step(cfg, b)
    o = oracle_step(cfg, b)
    pk = o.pk
    assert (info.status, info.first_bad_rollout, info.n_groups_kept, info.n_rollouts_kept, info.n_tokens) == \
        (pk.status, pk.first_bad_rollout, pk.n_groups_kept, pk.n_rollouts_kept, pk.n_tokens)
    n, k = pk.n_tokens, pk.n_rollouts_kept
    np.testing.assert_array_equal(st.kept_rollout[:k].cpu().numpy(), pk.kept_rollout)
    np.testing.assert_array_equal(st.kept_offset[:k + 1].cpu().numpy(), pk.kept_offset)
    for gpu, ref in ((st.tok_slot, pk.tok_slot), (st.tok_action, pk.tok_action), (st.tok_old, pk.tok_old),
                     (st.tok_ref, pk.tok_ref)):
        assert gpu[:n].cpu().numpy().tobytes() == ref.tobytes()


def test_pack_exhaustive_lags_and_shards():
    import itertools
    cfg = synth.CONFIGS["tiny"]
    base = synth.make_batch(cfg, lengths="ragged")
    for lags in itertools.product([0, 1, 2], repeat=4):
        b = synth.make_batch(cfg, lengths="ragged")
        b.version = (synth.T_TRAIN - np.repeat(np.array(lags), cfg.G)).astype(np.int64)
        st, info = device_step(cfg, b)
        pk = oracle_step(cfg, b).pk
        assert info.n_tokens == pk.n_tokens and info.n_groups_kept == pk.n_groups_kept
        np.testing.assert_array_equal(st.tok_action[:pk.n_tokens].cpu().numpy(), pk.tok_action)
    # shards with rollout_base give global ids
    for r0, r1 in ((0, 8), (8, 16), (4, 12)):
        b = synth.make_batch(cfg, r0, r1, lengths="ragged")
        st, info = device_step(cfg, b, rollout_base=r0)
        pk = oracle_step(cfg, b, rollout_base=r0).pk
        np.testing.assert_array_equal(st.kept_rollout[:pk.n_rollouts_kept].cpu().numpy(), pk.kept_rollout)
    assert base is not None


def test_pack_errors_and_capacity():
    cfg = synth.CONFIGS["tiny"]
    cases = []
    b = synth.make_batch(cfg); b.version = b.version.copy(); b.version[5] = synth.T_TRAIN + 1; cases.append(b)
    b = synth.make_batch(cfg); b.version = b.version.copy(); b.version[6] -= 1; cases.append(b)
    b = synth.make_batch(cfg); b.resp_len = b.resp_len.copy(); b.resp_len[9] = 0; cases.append(b)
    b = synth.make_batch(cfg); b.action = b.action.copy(); b.action[7, 3] = cfg.V; b.action[13, 0] = -1; cases.append(b)
    b = synth.make_batch(cfg); b.action = b.action.copy(); b.action[8, 1] = cfg.V; cases.append(b)   # dropped: unread
    b = synth.make_batch(cfg); b.version = b.version.copy(); b.version[12] = synth.T_TRAIN + 5
    b.action = b.action.copy(); b.action[1, 0] = -7; cases.append(b)
    for b in cases:
        st, info = device_step(cfg, b)
        pk = oracle_step(cfg, b).pk
        assert (info.status, info.first_bad_rollout) == (pk.status, pk.first_bad_rollout)
    # capacity
    from paper_2508_05387_b200 import abi
    b = synth.make_batch(cfg)
    st, _ = device_step(cfg, b)
    st.cap = 767
    info = st.pack(t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
    assert info.status == abi.ECHO_DATA_CAPACITY and info.n_tokens == 768


# ---------------------------------------------------------------------------------------------- (2) advantage
@pytest.mark.parametrize("name", ["tiny", "qwen2.5-7b", "qwen3-30b-a3b"])
def test_advantage_bit_exact(name):
    cfg = synth.CONFIGS[name]
    b = synth.make_batch(cfg, want_tokens=False)
    S = 4                                            # metadata-only shape: lengths do not affect (2)
    b.action = np.zeros((cfg.R, S), np.int32)
    b.old_logp = np.zeros((cfg.R, S), np.float32)
    b.ref_logp = np.zeros((cfg.R, S), np.float32)
    b.resp_len = np.full(cfg.R, S, np.int32)
    small = synth.Config(cfg.name, cfg.P, cfg.G, S, cfg.V, cfg.dtype, cfg.max_lag, cfg.kl_coef, cfg.lag_mode,
                         cfg.index, cfg.stale_groups, cfg.fixed_lags)
    st, info = device_step(small, b)
    o = oracle_step(small, b)
    assert st.adv_slot[:len(o.adv)].cpu().numpy().tobytes() == o.adv.tobytes()
    assert st.adv_stats.cpu().numpy().tobytes() == o.adv_stats.tobytes()
    # continuous (Sokoban-style) returns, PAPER.md :344 reward structure
    rng = np.random.default_rng(1)
    b.reward = (rng.integers(-2, 3, cfg.R) + 10.0 * (rng.random(cfg.R) < 0.2) - 0.1 * rng.integers(1, 40, cfg.R)
                ).astype(np.float32)
    st, info = device_step(small, b)
    o = oracle_step(small, b)
    assert st.adv_slot[:len(o.adv)].cpu().numpy().tobytes() == o.adv.tobytes()
    assert st.adv_stats.cpu().numpy().tobytes() == o.adv_stats.tobytes()


# ---------------------------------------------------------------------------------------------- (3)-(5)
@pytest.mark.parametrize("kl_coef", [0.0, 0.001, 0.5])
def test_tiny_full_step(kl_coef):
    """configs[0] end to end: every output element vs the oracle (fp32 logits, ROW_L2 kernel)."""
    cfg = synth.CONFIGS["tiny"]
    b = synth.make_batch(cfg)
    st, info = device_step(cfg, b)
    o = oracle_step(cfg, b)
    n = info.n_tokens
    logits = fill(st, cfg, 0, n)
    z = as_oracle_rows(logits)
    probe = oracle.policy_loss(z, o.pk.tok_action, o.pk.tok_old, o.pk.tok_ref, o.pk.tok_slot, o.adv, n_global=n,
                               kl_coef=kl_coef)
    s = pow2_scale_for(np.abs(probe.dlogits).max())
    ref = oracle.policy_loss(z, o.pk.tok_action, o.pk.tok_old, o.pk.tok_ref, o.pk.tok_slot, o.adv, n_global=n,
                             kl_coef=kl_coef, grad_scale=s)
    st.loss(logits, 0, kl_coef=kl_coef, grad_scale=s)
    out = st.finish()
    check_rows(d_gpu=logits.cpu().numpy(), logp_gpu=st.tok_logp[:n].cpu().numpy(),
               loss_gpu=st.tok_loss[:n].cpu().numpy(), flags_gpu=st.tok_flags[:n].cpu().numpy(), ref=ref,
               dtype="f32", old=o.pk.tok_old,
               sens=coef_sens(ref, o.pk.tok_old, o.pk.tok_ref, o.adv[o.pk.tok_slot], kl_coef, s, n))
    L_ref = ref.loss.sum() / n
    assert abs(out["loss"] - L_ref) <= 1e-5 * max(abs(L_ref), np.abs(ref.loss).mean())
    for k, i in (("loss/n_clipped", 3), ("loss/n_nonfinite", 4), ("loss/n_tokens", 8)):
        assert out[k] == ref.stats[i]
    for k, i in (("loss/sum_logp_minus_old", 1), ("loss/sum_kl_k3", 2), ("loss/sum_logp", 7), ("loss/sum_rho", 9),
                 ("loss/rho_min", 5), ("loss/rho_max", 6)):
        assert abs(out[k] - ref.stats[i]) <= 1e-5 * max(1.0, abs(ref.stats[i])), k
    assert out["n_tokens"] == n and out["n_groups_kept"] == 3 and out["n_groups_dropped"] == 1


def _uniform_case(V, dtype, algo):
    from paper_2508_05387_b200 import abi
    n = 6
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    logits = torch.zeros(n, V, dtype=dt, device="cuda")
    logits[1] += 3.5
    logits[2] -= 17.25
    act = torch.tensor([0, 1, V - 1, V // 2, 7, 123], dtype=torch.int32, device="cuda")
    old = torch.zeros(n, dtype=torch.float32, device="cuda")
    slot = torch.zeros(n, dtype=torch.int32, device="cuda")
    adv = torch.ones(1, dtype=torch.float32, device="cuda")
    ng = torch.tensor([float(n)], dtype=torch.float64, device="cuda")
    logp, loss = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    abi.echo_policy_loss_fwd_bwd(logits, abi.ECHO_BF16 if dtype == "bf16" else abi.ECHO_F32, n, V, V, act, old, None,
                                 slot, adv, ng, 0.2, 0.2, 0.0, 1.0, logp, loss, flags, algo=algo)
    return logits, logp.cpu().numpy()


@pytest.mark.parametrize("V,dtype,algo", [(1024, "f32", 1), (151936, "bf16", 1), (151936, "bf16", 2),
                                          (152064, "bf16", 2), (151936, "bf16", 3), (152064, "bf16", 3),
                                          (151936, "bf16", 4), (152064, "bf16", 4)])
def test_uniform_rows_give_minus_log_v(V, dtype, algo):
    """Closed form (SPEC.md :202): uniform logits give logp = -ln V; the GPU is within 2 fp32 ulp."""
    _, logp = _uniform_case(V, dtype, algo)
    target = np.float32(-math.log(V))
    ulp = np.spacing(np.abs(target))
    assert np.all(np.abs(logp - target) <= 2 * ulp), (logp, target)


@pytest.mark.parametrize("algo", [1, 2, 3, 4])
def test_clip_saturation_and_two_call_ratio(algo):
    """old == new (two-call protocol) gives rho = 1 exactly and c = -A s/N; clip saturation zeroes whole rows."""
    cfg = synth.CONFIGS["qwen3-4b"]
    b = synth.make_batch(cfg, 0, 2 * cfg.G)
    st, info = device_step(cfg, b)
    n = 512
    base = fill(st, cfg, 0, n)
    work = base.clone()
    st.loss(work, 0, kl_coef=0.0, algo=algo)
    logp1 = st.tok_logp[:n].clone()
    # call 2: old = logp of call 1
    st.tok_old[:n] = logp1
    work = base.clone()
    st.loss(work, 0, kl_coef=0.0, algo=algo)
    assert torch.equal(st.tok_logp[:n], logp1)                       # deterministic
    adv = st.adv_slot[st.tok_slot[:n].long()]
    assert torch.equal(st.tok_loss[:n], -adv)                        # rho == 1 exactly -> pg = -A
    assert not torch.any(st.tok_flags[:n])
    # clip saturation: A > 0 rows with rho = e^0.5 > 1.2, A < 0 rows with rho = e^-0.5 < 0.8
    sign = torch.sign(adv)
    st.tok_old[:n] = logp1 - 0.5 * sign
    work = base.clone()
    st.loss(work, 0, kl_coef=0.0, algo=algo)
    nz = adv != 0
    assert torch.all(st.tok_flags[:n][nz] == 1)
    assert torch.count_nonzero(work[nz]) == 0


@pytest.mark.parametrize("algo", [1, 2, 3, 4])
def test_determinism_and_microbatch_invariance(algo):
    cfg = synth.CONFIGS["qwen3-4b"]
    b = synth.make_batch(cfg, 0, 2 * cfg.G)
    st, info = device_step(cfg, b)
    n = 700
    base = fill(st, cfg, 0, n)
    a = base.clone()
    st.loss(a, 0, kl_coef=cfg.kl_coef, algo=algo)
    la = st.tok_logp[:n].clone()
    b2 = base.clone()
    st.loss(b2[:333], 0, kl_coef=cfg.kl_coef, algo=algo)             # odd split
    st.loss(b2[333:], 333, kl_coef=cfg.kl_coef, algo=algo)
    assert torch.equal(a.view(torch.int16), b2.view(torch.int16))
    assert torch.equal(la, st.tok_logp[:n])


@pytest.mark.parametrize("name", ["qwen3-4b", "qwen2.5-7b", "qwen3-32b", "qwen3-30b-a3b"])
@pytest.mark.parametrize("algo_name", ["quad_reg", "quad_reg_exact", "oct_reg", "row_l2"])
def test_full_config_sampled_rows(name, algo_name):
    """BASELINE.json full sizes, the bench's micro-batch (32768 rows) and launch configuration: sampled rows
    of the first and the last micro-batch against the oracle, plus the row-sum invariant on every row."""
    cfg = synth.CONFIGS[name]
    algo = ALGOS[algo_name]
    b = synth.make_batch(cfg)
    st, info = device_step(cfg, b)
    o = oracle_step(cfg, b)
    N = info.n_tokens
    assert N == o.pk.n_tokens
    M = 32768
    rng = np.random.default_rng(7)
    for row0 in (0, ((N - 1) // M) * M):
        m = min(M, N - row0)
        logits = fill(st, cfg, row0, m)
        sample = np.unique(np.concatenate([[0, m - 1], rng.integers(0, m, 30)]))
        gl = row0 + sample
        z = host_rows(cfg, o.keys[gl], o.pk.tok_action[gl])
        tr = None if o.pk.tok_ref is None else o.pk.tok_ref[gl]
        probe = oracle.policy_loss(z, o.pk.tok_action[gl], o.pk.tok_old[gl], tr, o.pk.tok_slot[gl], o.adv,
                                   n_global=N, kl_coef=cfg.kl_coef)
        s = pow2_scale_for(np.abs(probe.dlogits).max())
        ref = oracle.policy_loss(z, o.pk.tok_action[gl], o.pk.tok_old[gl], tr, o.pk.tok_slot[gl], o.adv, n_global=N,
                                 kl_coef=cfg.kl_coef, grad_scale=s)
        st.loss(logits, row0, kl_coef=cfg.kl_coef, grad_scale=s, algo=algo)
        idx = torch.from_numpy(sample).cuda()
        d = logits[idx].float().cpu().numpy()
        check_rows(d_gpu=d, logp_gpu=st.tok_logp[gl].cpu().numpy(), loss_gpu=st.tok_loss[gl].cpu().numpy(),
                   flags_gpu=st.tok_flags[gl].cpu().numpy(), ref=ref, dtype=cfg.dtype, old=o.pk.tok_old[gl],
                   sens=coef_sens(ref, o.pk.tok_old[gl], tr, o.adv[o.pk.tok_slot[gl]], cfg.kl_coef, s, N),
                   label=f"{name} {algo_name} row0={row0}")
        assert np.max(np.abs(d - ref.dlogits)) <= 2e-3                 # the north_star bar
        # every row of the micro-batch: |sum_v d| <= 2^-8 |c| (bf16 RNE) + fp32 slack
        rows_sum = logits.float().sum(dim=1).abs()
        logp = st.tok_logp[row0:row0 + m].double()
        rho = torch.exp(logp - st.tok_old[row0:row0 + m].double())
        A = st.adv_slot[st.tok_slot[row0:row0 + m].long()].double()
        kl_term = 0.0
        if cfg.kl_coef > 0:
            kl_term = cfg.kl_coef * (1 - torch.exp(st.tok_ref[row0:row0 + m].double() - logp)).abs()
        cbound = (A.abs() * rho + kl_term) * s / N
        assert torch.all(rows_sum.double() <= 2.0 ** -7 * cbound + 1e-6)
        del logits
    torch.cuda.empty_cache()



@pytest.mark.parametrize("name", ["qwen3-4b", "qwen3-32b"])
def test_token_logp_full_size_sampled_rows(name):
    """f1 at the bench's f1_token_logp launch (the AUTO bf16 kernel, token_logp_warp_kernel, on a 32768-row micro-batch
    of the config's logits): sampled rows of the first and the last micro-batch against the oracle's logp / lse /
    flags; the logits are left bit-for-bit unchanged."""
    from paper_2508_05387_b200 import abi
    cfg = synth.CONFIGS[name]
    b = synth.make_batch(cfg)
    st, info = device_step(cfg, b)
    o = oracle_step(cfg, b)
    N, M = info.n_tokens, 32768
    rng = np.random.default_rng(11)
    for row0 in (0, ((N - 1) // M) * M):
        m = min(M, N - row0)
        logits = fill(st, cfg, row0, m)
        before = logits[-1].clone()
        logp = torch.empty(m, device="cuda")
        lse = torch.empty(m, device="cuda")
        flags = torch.empty(m, dtype=torch.uint8, device="cuda")
        abi.echo_token_logp(logits, abi.ECHO_BF16, m, cfg.V, cfg.V, st.tok_action[row0:], logp, lse, flags)
        torch.cuda.synchronize()
        assert torch.equal(before.view(torch.int16), logits[-1].view(torch.int16))
        sample = np.unique(np.concatenate([[0, m - 1], rng.integers(0, m, 30)]))
        gl = row0 + sample
        z = host_rows(cfg, o.keys[gl], o.pk.tok_action[gl])
        ref_logp, ref_lse, ref_flags = oracle.token_logp(z, o.pk.tok_action[gl], vocab=cfg.V, dtype=oracle.BF16)
        g = torch.from_numpy(sample).cuda()
        assert np.all(np.abs(logp[g].cpu().numpy() - ref_logp) <= 1e-5 + 1e-6 * np.abs(ref_logp))
        assert np.all(np.abs(lse[g].cpu().numpy() - ref_lse) <= 1e-5 + 1e-6 * np.abs(ref_lse))
        np.testing.assert_array_equal(flags[g].cpu().numpy(), ref_flags)
        del logits
    torch.cuda.empty_cache()


@pytest.mark.parametrize("leg", ["entropy", "weights_adv"])
def test_f4_legs_full_size_sampled_rows(leg):
    """The bench's two f4 legs at their launch (AUTO kernel, the Qwen3-32B-shaped batch's first 32768-row micro-batch):
    the entropy bonus (eta = 0.01, tok_entropy written) and per-token advantages + sequence-mean weights; sampled rows
    (first, last, 30 random) against the oracle with the same bars as the small-size variant tests."""
    cfg = synth.CONFIGS["qwen3-32b"]
    b = synth.make_batch(cfg)
    st, info = device_step(cfg, b)
    o = oracle_step(cfg, b)
    N, m = info.n_tokens, 32768
    logits = fill(st, cfg, 0, m)
    rng = np.random.default_rng(5)
    sample = np.unique(np.concatenate([[0, m - 1], rng.integers(0, m, 30)]))
    z = host_rows(cfg, o.keys[sample], o.pk.tok_action[sample])
    args = (o.pk.tok_action[sample], o.pk.tok_old[sample], o.pk.tok_ref[sample], o.pk.tok_slot[sample], o.adv)
    kl, eta = cfg.kl_coef, 0.01
    idx = torch.from_numpy(sample).cuda()
    if leg == "entropy":
        kw = dict(n_global=N, kl_coef=kl, entropy_coef=eta)
        probe = oracle.policy_loss(z, *args, **kw)
        s = pow2_scale_for(np.abs(probe.dlogits).max())
        ref = oracle.policy_loss(z, *args, grad_scale=s, **kw)
        ent = torch.full((m,), float("nan"), device="cuda")
        st.loss(logits, 0, kl_coef=kl, grad_scale=s, entropy_coef=eta, tok_entropy=ent)
        H = ent[idx].cpu().numpy().astype(np.float64)
        _, lse, _ = oracle.token_logp(z, o.pk.tok_action[sample], vocab=cfg.V)
        hbar = 3e-5 * (1 + np.abs(lse) + np.abs(ref.entropy))
        assert np.all(np.abs(H - ref.entropy) <= hbar), np.max(np.abs(H - ref.entropy) / hbar)
        zf = (z.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        p = np.exp(zf - lse[:, None])
        e = s * eta / N
        es = e * p * (np.abs(zf) + np.abs(lse)[:, None] + np.abs(ref.entropy)[:, None] + 1) * 3e-5
        sens = coef_sens(ref, o.pk.tok_old[sample], o.pk.tok_ref[sample], o.adv[o.pk.tok_slot[sample]], kl, s, N)
        extra = dict(eslack=es, loss_atol=1e-6 + eta * hbar, p=p, action=o.pk.tok_action[sample])
    else:
        gen = np.random.default_rng(6)
        tok_adv = (gen.normal(size=N) * 1.5).astype(np.float32)
        L = np.diff(o.pk.kept_offset)
        w = (1.0 / (o.pk.n_rollouts_kept * L[o.pk.tok_slot])).astype(np.float32)
        kw = dict(n_global=N, kl_coef=kl, tok_adv=tok_adv[sample], tok_weight=w[sample])
        probe = oracle.policy_loss(z, *args, **kw)
        s = pow2_scale_for(np.abs(probe.dlogits).max())
        ref = oracle.policy_loss(z, *args, grad_scale=s, **kw)
        st.loss(logits, 0, kl_coef=kl, grad_scale=s, tok_adv=torch.from_numpy(tok_adv).cuda(),
                tok_weight=torch.from_numpy(w).cuda())
        sens = coef_sens(ref, o.pk.tok_old[sample], o.pk.tok_ref[sample], tok_adv[sample], kl, s,
                         tok_weight=w[sample])
        extra = {}
    check_rows(d_gpu=logits[idx].float().cpu().numpy(), logp_gpu=st.tok_logp[idx].cpu().numpy(),
               loss_gpu=st.tok_loss[idx].cpu().numpy(), flags_gpu=st.tok_flags[idx].cpu().numpy(), ref=ref,
               dtype=cfg.dtype, old=o.pk.tok_old[sample], sens=sens, label=f"f4 {leg} full size", **extra)
    del logits
    torch.cuda.empty_cache()


def test_check_rows_rejects_dropped_small_gradients():
    """Mutation test of the dlogits bar: the AUTO kernel's output on sampled Qwen3-4B rows passes check_rows; the same
    output with every entry whose p_v < 1e-5 zeroed (the bulk of a 152k-column row) must fail it, and so must an
    all-zero gradient and one whose entries with p_v >= 1e-4 (non-action) are off by a relative 2^-6 (> 1 bf16 ulp)."""
    cfg = synth.CONFIGS["qwen3-4b"]
    b = synth.make_batch(cfg, 0, 2 * cfg.G)
    st, info = device_step(cfg, b)
    o = oracle_step(cfg, b)
    n = 64
    logits = fill(st, cfg, 0, n)
    z = host_rows(cfg, o.keys[:n], o.pk.tok_action[:n])
    args = (o.pk.tok_action[:n], o.pk.tok_old[:n], o.pk.tok_ref[:n], o.pk.tok_slot[:n], o.adv)
    N = info.n_tokens
    probe = oracle.policy_loss(z, *args, n_global=N, kl_coef=cfg.kl_coef)
    s = pow2_scale_for(np.abs(probe.dlogits).max())
    ref = oracle.policy_loss(z, *args, n_global=N, kl_coef=cfg.kl_coef, grad_scale=s)
    st.loss(logits, 0, kl_coef=cfg.kl_coef, grad_scale=s)                 # AUTO
    d = logits.float().cpu().numpy()
    kw = dict(logp_gpu=st.tok_logp[:n].cpu().numpy(), loss_gpu=st.tok_loss[:n].cpu().numpy(),
              flags_gpu=st.tok_flags[:n].cpu().numpy(), ref=ref, dtype="bf16", old=o.pk.tok_old[:n],
              sens=coef_sens(ref, o.pk.tok_old[:n], o.pk.tok_ref[:n], o.adv[o.pk.tok_slot[:n]], cfg.kl_coef, s, N))
    check_rows(d_gpu=d, label="AUTO unmutated", **kw)
    c = ref.coef[:, None]
    pv = np.where(c != 0, np.abs(ref.dlogits / np.where(c != 0, c, 1.0)), 0.0)
    small = pv < 1e-5
    assert small.mean() > 0.5                                             # the bulk of every row
    for name, mutated in (("p<1e-5 zeroed", np.where(small, 0.0, d)), ("all zero", np.zeros_like(d)),
                          ("x(1+2^-6) where p>=1e-4", np.where((pv >= 1e-4) & (pv < 0.5), d * (1 + 2.0 ** -6), d))):
        with pytest.raises(AssertionError):
            check_rows(d_gpu=mutated, label=name, **kw)

def test_nonfinite_rows_flagged():
    from paper_2508_05387_b200 import abi
    V = 4096
    for dtype, algo in (("bf16", 1), ("bf16", 2), ("bf16", 3), ("bf16", 4), ("f32", 1)):
        dt = torch.bfloat16 if dtype == "bf16" else torch.float32
        z = torch.zeros(6, V, dtype=dt, device="cuda")
        z[0, 3] = float("nan")
        z[1, :] = float("-inf")
        z[2, 5] = float("inf")
        z[3, :10] = float("-inf")
        z[4, 20] = float("-inf")
        act = torch.tensor([0, 0, 0, 30, 20, 1], dtype=torch.int32, device="cuda")
        old = torch.tensor([0, 0, 0, 0, 0, -100.0], device="cuda")
        slot = torch.zeros(6, dtype=torch.int32, device="cuda")
        adv = torch.ones(1, device="cuda")
        ng = torch.tensor([6.0], dtype=torch.float64, device="cuda")
        logp, loss = torch.empty(6, device="cuda"), torch.empty(6, device="cuda")
        flags = torch.empty(6, dtype=torch.uint8, device="cuda")
        abi.echo_policy_loss_fwd_bwd(z, abi.ECHO_BF16 if dtype == "bf16" else abi.ECHO_F32, 6, V, V, act, old, None,
                                     slot, adv, ng, 0.2, 0.2, 0.0, 1.0, logp, loss, flags, algo=algo)
        np.testing.assert_array_equal((flags.cpu().numpy() >> 1) & 1, [1, 1, 1, 0, 1, 1])
        assert abs(logp[3].item() + math.log(V - 10)) < 1e-5


@pytest.mark.parametrize("V,ld,algo", [(1000, 1008, 1), (1001, 1008, 1), (151935, 151936, 1), (151935, 151936, 2),
                                       (40001, 40008, 2), (40001, 40008, 3), (155648, 155648, 2), (33, 40, 2),
                                       (32768, 32768, 3), (151935, 151936, 4), (40001, 40008, 4), (65, 72, 4)])
def test_ragged_vocab_and_padding_untouched(V, ld, algo):
    """V not a multiple of the 8-element vector: tail handling; columns V..ld-1 are never written."""
    from paper_2508_05387_b200 import abi
    n = 37
    rng = np.random.default_rng(V)
    zf = (rng.normal(size=(n, ld)) * 2).astype(np.float32)
    zb = torch.from_numpy(zf).to(torch.bfloat16)
    raw = zb.view(torch.int16).numpy().view(np.uint16)
    act = rng.integers(0, V, n).astype(np.int32)
    act[0] = V - 1
    old = (rng.normal(size=n) * 0.3 - 10).astype(np.float32)
    slot = (np.arange(n) % 4).astype(np.int32)
    adv = np.array([1.0, -0.5, 0.25, -2.0], np.float32)
    ref = oracle.policy_loss(raw[:, :V].copy(), act, old, None, slot, adv, n_global=n, vocab=V, grad_scale=float(n))
    logits = zb.cuda()
    c = lambda x: torch.from_numpy(x).cuda()
    ng = torch.tensor([float(n)], dtype=torch.float64, device="cuda")
    logp, loss = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    abi.echo_policy_loss_fwd_bwd(logits, abi.ECHO_BF16, n, V, ld, c(act), c(old), None, c(slot), c(adv), ng, 0.2, 0.2,
                                 0.0, float(n), logp, loss, flags, algo=algo)
    out = logits.cpu()
    assert torch.equal(out[:, V:].view(torch.int16), zb[:, V:].view(torch.int16))
    check_rows(d_gpu=out[:, :V].float().numpy(), logp_gpu=logp.cpu().numpy(), loss_gpu=loss.cpu().numpy(),
               flags_gpu=flags.cpu().numpy(), ref=ref, dtype="bf16", old=old,
               sens=coef_sens(ref, old, None, adv[slot], 0.0, float(n), n))


def test_abi_argument_errors():
    from paper_2508_05387_b200 import abi
    z = torch.zeros(2, 1000, dtype=torch.bfloat16, device="cuda")
    i = torch.zeros(2, dtype=torch.int32, device="cuda")
    f = torch.zeros(2, device="cuda")
    ng = torch.ones(1, dtype=torch.float64, device="cuda")
    args = lambda **kw: dict(dict(logits=z, dtype=abi.ECHO_BF16, n_rows=2, vocab=1000, ld=1000, tok_action=i,
                                  tok_old=f, tok_ref=None, tok_slot=i, adv_slot=f, n_global=ng, clip_low=0.2,
                                  clip_high=0.2, kl_coef=0.0, grad_scale=1.0, tok_logp=f, tok_loss=f,
                                  tok_flags=torch.zeros(2, dtype=torch.uint8, device="cuda")), **kw)
    with pytest.raises(abi.EchoError):
        abi.echo_policy_loss_fwd_bwd(**args(ld=1001))                 # ld * 2 not a multiple of 16
    with pytest.raises(abi.EchoError):
        abi.echo_policy_loss_fwd_bwd(**args(kl_coef=0.1))             # KL needs tok_ref
    with pytest.raises(abi.EchoError):
        abi.echo_policy_loss_fwd_bwd(**args(dtype=7))
    with pytest.raises(abi.EchoError) as e:
        abi.echo_policy_loss_fwd_bwd(**args(dtype=abi.ECHO_F32, ld=1000), algo=abi.ECHO_ALGO_QUAD_REG)
    assert e.value.status == abi.ECHO_ERR_UNSUPPORTED
    abi.echo_policy_loss_fwd_bwd(**args(n_rows=0))                    # empty micro-batch: no launch, OK


# ---------------------------------------------------------------------------------------------- f1: logp only
@pytest.mark.parametrize("name", ["tiny", "qwen3-4b", "qwen2.5-7b"])
def test_token_logp_forward_only(name):
    """echo_token_logp reads the logits once and matches the oracle's logp / lse; the logits
    are left bit-for-bit unchanged."""
    from paper_2508_05387_b200 import abi
    cfg = synth.CONFIGS[name]
    b = synth.make_batch(cfg, 0, 2 * cfg.G)
    st, info = device_step(cfg, b)
    o = oracle_step(cfg, b)
    n = min(info.n_tokens, 4096)
    logits = fill(st, cfg, 0, n)
    before = logits.clone()
    logp = torch.empty(n, device="cuda")
    lse = torch.empty(n, device="cuda")
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    abi.echo_token_logp(logits, abi.ECHO_BF16 if cfg.dtype == "bf16" else abi.ECHO_F32, n, cfg.V, cfg.V,
                        st.tok_action, logp, lse, flags)
    torch.cuda.synchronize()
    assert torch.equal(before.view(torch.int16) if cfg.dtype == "bf16" else before, 
                       logits.view(torch.int16) if cfg.dtype == "bf16" else logits)
    ref_logp, ref_lse, ref_flags = oracle.token_logp(as_oracle_rows(logits), o.pk.tok_action[:n])
    assert np.max(np.abs(logp.cpu().numpy() - ref_logp)) <= 1e-5 + 1e-6 * np.abs(ref_logp).max()
    assert np.max(np.abs(lse.cpu().numpy() - ref_lse)) <= 1e-5 + 1e-6 * np.abs(ref_lse).max()
    np.testing.assert_array_equal(flags.cpu().numpy(), ref_flags)
    # consistency with the fused kernel's logp on the same rows (a different reduction tree: one warp per row here,
    # so the two agree within the sum of their oracle bounds)
    st.loss(logits, 0, kl_coef=0.0)
    lf = st.tok_logp[:n].double()
    assert torch.all((lf - logp.double()).abs() <= 2e-5 + 2e-6 * lf.abs())


# ---------------------------------------------------------------------------------------------- f4: variants
def test_gae_bit_exact_and_packed_aux():
    """PPO-GAE advantages (echo_gae_advantage) bit-identical to the fp64 oracle; echo_pack_batch carries them."""
    from paper_2508_05387_b200 import abi
    rng = np.random.default_rng(3)
    for R, S in ((16, 64), (512, 2048)):
        L = rng.integers(1, S + 1, R).astype(np.int32)
        r = rng.normal(size=(R, S)).astype(np.float32)
        v = rng.normal(size=(R, S)).astype(np.float32)
        boot = rng.normal(size=R).astype(np.float32)
        ref_adv, ref_ret = oracle.gae_advantage(L, r, v, gamma=0.99, lam=0.95, bootstrap=boot)
        c = lambda x: torch.from_numpy(x).cuda()
        adv = torch.zeros(R, S, device="cuda")
        ret = torch.zeros(R, S, device="cuda")
        abi.echo_gae_advantage(R, S, c(L), c(r), c(v), c(boot), 0.99, 0.95, adv, ret)
        assert adv.cpu().numpy().tobytes() == ref_adv.tobytes()
        assert ret.cpu().numpy().tobytes() == ref_ret.tobytes()
    # packed through echo_pack_batch's aux payload
    cfg = synth.CONFIGS["tiny"]
    b = synth.make_batch(cfg, lengths="ragged")
    aux = rng.normal(size=(cfg.R, cfg.S)).astype(np.float32)
    st, info = device_step(cfg, b)
    from paper_2508_05387_b200 import abi as a2
    tok_aux = torch.zeros(st.cap, device="cuda")
    a2.echo_pack_batch(cfg.R, cfg.G, cfg.S, cfg.V, synth.T_TRAIN, cfg.max_lag, 0, st.version, st.resp_len, st.action,
                       st.old_logp, st.ref_logp, st.cap, st.kept_rollout, st.kept_offset, st.tok_slot, st.tok_action,
                       st.tok_old, st.tok_ref, st.pack_result, aux=torch.from_numpy(aux).cuda(), tok_aux=tok_aux)
    pk = oracle.pack_batch(b.version, b.resp_len, b.action, b.old_logp, b.ref_logp, group_size=cfg.G, max_len=cfg.S,
                           vocab=cfg.V, t_train=synth.T_TRAIN, max_lag=cfg.max_lag, aux=aux)
    assert tok_aux[:pk.n_tokens].cpu().numpy().tobytes() == pk.tok_aux.tobytes()


@pytest.mark.parametrize("name,algo", [("tiny", None), ("qwen3-4b", 2), ("qwen3-4b", 3), ("qwen3-4b", 1)])
@pytest.mark.parametrize("est,dual", [(1, 0.0), (2, 3.0), (0, 2.0)])
def test_loss_variants_v2(name, algo, est, dual):
    """echo_policy_loss_fwd_bwd_v2: per-token advantages, sequence-mean weights, KL estimator, dual clip."""
    from paper_2508_05387_b200 import abi
    cfg = synth.CONFIGS[name]
    b = synth.make_batch(cfg, 0, 2 * cfg.G if name != "tiny" else cfg.R)
    st, info = device_step(cfg, b)
    o = oracle_step(cfg, b)
    n = min(info.n_tokens, 2048)
    rng = np.random.default_rng(est * 10 + int(dual))
    tok_adv = (rng.normal(size=info.n_tokens) * 1.5).astype(np.float32)
    L = np.diff(o.pk.kept_offset)
    w = (1.0 / (o.pk.n_rollouts_kept * L[o.pk.tok_slot])).astype(np.float32)
    old = o.pk.tok_old.copy()
    old[: n // 2] = (old[: n // 2] + rng.normal(size=n // 2) * 1.5).astype(np.float32)   # push some rho past c
    st.tok_old[: info.n_tokens] = torch.from_numpy(old).cuda()
    logits = fill(st, cfg, 0, n)
    z = as_oracle_rows(logits)
    kl = 0.05
    kw = dict(n_global=info.n_tokens, kl_coef=kl, tok_adv=tok_adv[:n], tok_weight=w[:n], clip_dual=dual,
              kl_estimator=est)
    probe = oracle.policy_loss(z, o.pk.tok_action[:n], old[:n], o.pk.tok_ref[:n], o.pk.tok_slot[:n], o.adv, **kw)
    s = pow2_scale_for(np.abs(probe.dlogits).max())
    ref = oracle.policy_loss(z, o.pk.tok_action[:n], old[:n], o.pk.tok_ref[:n], o.pk.tok_slot[:n], o.adv,
                             grad_scale=s, **kw)
    st.loss(logits, 0, kl_coef=kl, grad_scale=s, algo=algo, tok_adv=torch.from_numpy(tok_adv).cuda(),
            tok_weight=torch.from_numpy(w).cuda(), clip_dual=dual, kl_estimator=est)
    rho = np.exp(ref.logp - old[:n].astype(np.float64))
    keep = np.abs(rho - dual) > 1e-5 if dual else np.ones(n, bool)
    sens, cmag = coef_sens(ref, old[:n], o.pk.tok_ref[:n], tok_adv[:n], kl, s, tok_weight=w[:n], kl_estimator=est)
    sub = lambda x: x[keep]
    import copy
    r2 = copy.copy(ref)
    r2.logp, r2.loss, r2.flags, r2.coef, r2.dlogits = (sub(ref.logp), sub(ref.loss), sub(ref.flags), sub(ref.coef),
                                                       ref.dlogits[keep])
    check_rows(d_gpu=logits.float().cpu().numpy()[keep], logp_gpu=sub(st.tok_logp[:n].cpu().numpy()),
               loss_gpu=sub(st.tok_loss[:n].cpu().numpy()), flags_gpu=sub(st.tok_flags[:n].cpu().numpy()), ref=r2,
               dtype=cfg.dtype, old=sub(old[:n]), sens=(sub(sens), sub(cmag)),
               label=f"v2 {name} algo={algo} est={est} dual={dual}")
    if dual:
        assert (ref.flags & 1).any()


@pytest.mark.parametrize("name,algo", [("tiny", None), ("qwen3-4b", None), ("qwen3-4b", 2), ("qwen3-4b", 3),
                                       ("qwen3-4b", 1)])
def test_entropy_bonus_v2(name, algo):
    """f4 entropy bonus through echo_policy_loss_fwd_bwd_v2: per-token entropies, l_t = pg + beta kl - eta H_t and
    the entropy gradient, including rows with masked (-inf) vocabulary columns."""
    from paper_2508_05387_b200 import abi
    cfg = synth.CONFIGS[name]
    b = synth.make_batch(cfg, 0, 2 * cfg.G if name != "tiny" else cfg.R)
    st, info = device_step(cfg, b)
    o = oracle_step(cfg, b)
    n = min(info.n_tokens, 1024)
    logits = fill(st, cfg, 0, n)
    V = cfg.V
    act8 = st.tok_action[:8].long()
    za8 = logits[torch.arange(8, device="cuda"), act8].clone()
    logits[:8, V // 3: V // 3 + 257] = float("-inf")         # masked columns (e.g. a vocabulary mask) ...
    logits[torch.arange(8, device="cuda"), act8] = za8         # ... never the sampled action
    masked = torch.zeros(8, V, dtype=torch.bool, device="cuda")
    masked[:, V // 3: V // 3 + 257] = True
    masked[torch.arange(8, device="cuda"), act8] = False
    z = as_oracle_rows(logits)
    kl, eta = 0.05, 0.01
    args = (o.pk.tok_action[:n], o.pk.tok_old[:n], o.pk.tok_ref[:n], o.pk.tok_slot[:n], o.adv)
    kw = dict(n_global=info.n_tokens, kl_coef=kl, entropy_coef=eta)
    probe = oracle.policy_loss(z, *args, **kw)
    s = pow2_scale_for(np.abs(probe.dlogits).max())
    ref = oracle.policy_loss(z, *args, grad_scale=s, **kw)
    ent = torch.full((st.cap,), float("nan"), device="cuda")
    st.loss(logits, 0, kl_coef=kl, grad_scale=s, algo=algo, entropy_coef=eta, tok_entropy=ent)
    H = ent[:n].cpu().numpy().astype(np.float64)
    _, lse, _ = oracle.token_logp(z, o.pk.tok_action[:n], vocab=V)
    hbar = 3e-5 * (1 + np.abs(lse) + np.abs(ref.entropy))
    assert np.all(np.abs(H - ref.entropy) <= hbar), np.max(np.abs(H - ref.entropy) / hbar)
    zf = (z.astype(np.float64) if cfg.dtype != "bf16" else
          (z.astype(np.uint32) << 16).view(np.float32).astype(np.float64))
    zf = np.where(np.isinf(zf), 0.0, zf)
    p = np.exp(np.where(np.isinf(ref.dlogits), 0.0, zf - lse[:, None]))
    e = s * eta / info.n_tokens
    es = e * p * (np.abs(zf) + np.abs(lse)[:, None] + np.abs(ref.entropy)[:, None] + 1) * 3e-5
    check_rows(d_gpu=logits.float().cpu().numpy(), logp_gpu=st.tok_logp[:n].cpu().numpy(),
               loss_gpu=st.tok_loss[:n].cpu().numpy(), flags_gpu=st.tok_flags[:n].cpu().numpy(), ref=ref,
               dtype=cfg.dtype, old=o.pk.tok_old[:n], eslack=es, loss_atol=1e-6 + eta * hbar,
               sens=coef_sens(ref, o.pk.tok_old[:n], o.pk.tok_ref[:n], o.adv[o.pk.tok_slot[:n]], kl, s, info.n_tokens),
               p=p, action=o.pk.tok_action[:n], label=f"entropy {name} algo={algo}")
    # masked columns: exactly zero gradient
    assert torch.all(logits[:8, :V][masked] == 0)


@pytest.mark.parametrize("n", [0, 1, 7, 1023, 1024, 1025, 5000])
def test_csr_from_lengths_bit_exact(n):
    """f3: echo_csr_from_lengths against the oracle (bit-exact), including zero / negative lengths and n spanning
    several scan blocks."""
    from paper_2508_05387_b200 import abi
    rng = np.random.default_rng(n)
    L = rng.integers(-2, 300, n).astype(np.int32)
    off_ref, slot_ref = oracle.csr_from_lengths(L)
    off = torch.full((n + 1,), -7, dtype=torch.int64, device="cuda")
    slot = torch.full((max(len(slot_ref), 1),), -7, dtype=torch.int32, device="cuda")
    abi.echo_csr_from_lengths(n, torch.from_numpy(L).cuda() if n else None, off, slot)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(off.cpu().numpy(), off_ref)
    np.testing.assert_array_equal(slot[: len(slot_ref)].cpu().numpy(), slot_ref)


def _lmhead_case(n, d, V, seed, device="cuda"):
    g = torch.Generator(device=device).manual_seed(seed)
    h = torch.randn(n, d, generator=g, device=device).to(torch.bfloat16)
    w = (torch.randn(V, d, generator=g, device=device) * (2.0 / math.sqrt(d))).to(torch.bfloat16)
    act = torch.randint(0, V, (n,), generator=g, device=device, dtype=torch.int32)
    return h, w, act


def _lmhead_run(h, w, act):
    from paper_2508_05387_b200 import abi
    n, d = h.shape
    V = w.shape[0]
    ws = torch.empty(abi.echo_lmhead_workspace_bytes(n, V) // 4 + 1, dtype=torch.float32, device="cuda")
    lp = torch.full((n,), float("nan"), device="cuda")
    lse = torch.full((n,), float("nan"), device="cuda")
    abi.echo_lmhead_logp(h, w, n, d, V, act, lp, lse, ws)
    torch.cuda.synchronize()
    return lp.cpu().numpy().astype(np.float64), lse.cpu().numpy().astype(np.float64)


def _lmhead_tol(hb, wb, rows):
    """Bound on the fp32-accumulated logit error: blocked summation (K/16 tensor-core steps of 16 products),
    4 (K/16 + 16) 2^-24 max_v sum_k |h_k W_vk|, doubled for logp = z_a - lse."""
    hf = (hb[rows].astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    wf = (wb.astype(np.uint32) << 16).view(np.float32)
    B = (np.abs(hf).astype(np.float32) @ np.abs(wf).T).max(axis=1).astype(np.float64)
    K = hb.shape[1]
    return 2 * 4 * (K / 16 + 16) * 2.0 ** -24 * B


@pytest.mark.parametrize("n,d,V", [(128, 64, 256), (300, 512, 1000), (129, 72, 257), (1, 2560, 4096),
                                   (700, 256, 5000)])
def test_lmhead_logp_small(n, d, V):
    """f2: the fused LM-head log-prob against the fp64 oracle (every row), ragged token / vocab / K tiles."""
    h, w, act = _lmhead_case(n, d, V, seed=n + d + V)
    lp, lse = _lmhead_run(h, w, act)
    hb = h.cpu().view(torch.int16).numpy().view(np.uint16)
    wb = w.cpu().view(torch.int16).numpy().view(np.uint16)
    lp_ref, lse_ref = oracle.lmhead_logp(hb, wb, act.cpu().numpy())
    tol = _lmhead_tol(hb, wb, np.arange(n))
    print(f"lmhead n={n} d={d} V={V}: max|dlogp| {np.max(np.abs(lp - lp_ref)):.3e}, "
          f"max err/tol {np.max(np.abs(lp - lp_ref) / tol):.3e}")
    assert np.all(np.abs(lse - lse_ref) <= tol), np.max(np.abs(lse - lse_ref) / tol)
    assert np.all(np.abs(lp - lp_ref) <= tol), np.max(np.abs(lp - lp_ref) / tol)
    # regression guard well inside the bound: observed errors are 1e-6 .. 2e-5 (profiles: 100x below tol)
    assert np.max(np.abs(lp - lp_ref)) <= 1e-4 and np.max(np.abs(lse - lse_ref)) <= 1e-4


@pytest.mark.parametrize("n,d", [(4096, 2560), (32768, 5120)])
def test_lmhead_logp_qwen_size_sampled_rows(n, d):
    """f2 at the Qwen3-4B LM-head shape (d = 2560, V = 151936) over 4096 tokens, and at the bench's f2_lmhead_logp
    launch (32768 tokens, d = 5120: Qwen3-32B); sampled rows against the oracle, all rows finite and deterministic
    across two calls."""
    V = 151936
    h, w, act = _lmhead_case(n, d, V, seed=7)
    lp, lse = _lmhead_run(h, w, act)
    lp2, _ = _lmhead_run(h, w, act)
    assert np.array_equal(lp.view(np.uint64), lp2.view(np.uint64))
    assert np.all(np.isfinite(lp)) and np.all(lp <= 0)
    rows = np.unique(np.array([0, 1, 127, 128, 1000, 2047, n // 2 + 255, n - 256, n - 1]))
    hb = h[rows].cpu().view(torch.int16).numpy().view(np.uint16)
    wb = w.cpu().view(torch.int16).numpy().view(np.uint16)
    lp_ref, lse_ref = oracle.lmhead_logp(hb, wb, act.cpu().numpy()[rows])
    tol = _lmhead_tol(hb, wb, np.arange(len(rows)))
    assert np.all(np.abs(lse[rows] - lse_ref) <= tol), np.max(np.abs(lse[rows] - lse_ref) / tol)
    assert np.all(np.abs(lp[rows] - lp_ref) <= tol), np.max(np.abs(lp[rows] - lp_ref) / tol)
    assert np.max(np.abs(lp[rows] - lp_ref)) <= 2e-4


def test_lmhead_logp_edge_cases_and_errors():
    """f2: out-of-range actions give NaN log-probs (finite lse); n_rows = 0 is a no-op; bad arguments are
    reported, not launched."""
    from paper_2508_05387_b200 import abi
    n, d, V = 130, 128, 600
    h, w, act = _lmhead_case(n, d, V, seed=5)
    act[3] = -1
    act[77] = V
    lp, lse = _lmhead_run(h, w, act)
    assert np.isnan(lp[3]) and np.isnan(lp[77]) and np.all(np.isfinite(lse))
    ok = np.ones(n, bool)
    ok[[3, 77]] = False
    assert np.all(np.isfinite(lp[ok]))
    ws = torch.empty(abi.echo_lmhead_workspace_bytes(n, V) // 4 + 1, dtype=torch.float32, device="cuda")
    out = torch.empty(n, device="cuda")
    abi.echo_lmhead_logp(h, w, 0, d, V, act, out, None, ws)                 # n_rows = 0: nothing to do
    for bad in (dict(d=100), dict(d=0), dict(vocab=0)):
        kw = dict(d=d, vocab=V)
        kw.update(bad)
        with pytest.raises(abi.EchoError):
            abi.echo_lmhead_logp(h, w, n, kw["d"], kw["vocab"], act, out, None, ws)
    with pytest.raises(abi.EchoError):                                      # misaligned hidden pointer
        abi.echo_lmhead_logp(h.view(-1)[1:].data_ptr(), w, n - 1, d, V, act, out, None, ws)
    assert abi.echo_lmhead_workspace_bytes(n, V) == (3 * 3 + 1) * n * 4


@pytest.mark.parametrize("d", [2048, 3584, 5120])
def test_lmhead_logp_baseline_hidden_sizes(d):
    """f2 at the other BASELINE.json models' hidden sizes (30B-A3B, 7B, 32B) on a Qwen vocabulary, through the
    LearnerStep API (packed actions); sampled rows against the oracle."""
    cfg = synth.CONFIGS["qwen3-4b"]
    b = synth.make_batch(cfg, 0, cfg.G)
    st, info = device_step(cfg, b)
    n = 384
    g = torch.Generator(device="cuda").manual_seed(d)
    h = torch.randn(n, d, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(cfg.V, d, generator=g, device="cuda") * (2.0 / math.sqrt(d))).to(torch.bfloat16)
    lp = st.token_logp_from_hidden(h, w).cpu().numpy().astype(np.float64)
    rows = np.array([0, 127, 128, 255, 256, 383])
    hb = h[rows].cpu().view(torch.int16).numpy().view(np.uint16)
    wb = w.cpu().view(torch.int16).numpy().view(np.uint16)
    ref, _ = oracle.lmhead_logp(hb, wb, st.tok_action[:n].cpu().numpy()[rows])
    tol = _lmhead_tol(hb, wb, np.arange(len(rows)))
    assert np.all(np.abs(lp[rows] - ref) <= tol) and np.max(np.abs(lp[rows] - ref)) <= 2e-4


def test_fp32_logits_qwen_vocab():
    """fp32 logits at a Qwen vocabulary (the generic row kernel: AUTO's path for fp32) against the oracle."""
    cfg = synth.CONFIGS["qwen3-4b"]
    b = synth.make_batch(cfg, 0, cfg.G)
    st, info = device_step(cfg, b)
    o = oracle_step(cfg, b)
    n = 96
    logits = torch.zeros(n, cfg.V, dtype=torch.float32, device="cuda")
    import synth.gpu as sgpu
    sgpu.fill_logits(logits, dtype="f32", vocab=cfg.V, row0=0, tok_slot=st.tok_slot, tok_action=st.tok_action,
                     kept_rollout=st.kept_rollout, kept_offset=st.kept_offset, max_len=cfg.S, seed=cfg.seed)
    z = logits.cpu().numpy()
    args = (o.pk.tok_action[:n], o.pk.tok_old[:n], o.pk.tok_ref[:n], o.pk.tok_slot[:n], o.adv)
    N = info.n_tokens
    ref = oracle.policy_loss(z, *args, n_global=N, kl_coef=cfg.kl_coef, grad_scale=float(N))
    from paper_2508_05387_b200 import abi
    st.edtype = abi.ECHO_F32                                        # (the LearnerStep was built for bf16 logits)
    st.loss(logits, 0, kl_coef=cfg.kl_coef, grad_scale=float(N))
    check_rows(d_gpu=logits.cpu().numpy(), logp_gpu=st.tok_logp[:n].cpu().numpy(),
               loss_gpu=st.tok_loss[:n].cpu().numpy(), flags_gpu=st.tok_flags[:n].cpu().numpy(), ref=ref,
               dtype="f32", old=o.pk.tok_old[:n],
               sens=coef_sens(ref, o.pk.tok_old[:n], o.pk.tok_ref[:n], o.adv[o.pk.tok_slot[:n]], cfg.kl_coef,
                                 float(N), N))


@pytest.mark.parametrize("name", ["tiny", "qwen2.5-7b"])
def test_staleness_histogram_bit_exact(name):
    """f3: the step's staleness histogram through LearnerStep against the oracle (bit-exact), with ragged
    lengths and stale groups (the 7B config drops 38 of 128 groups)."""
    cfg = synth.CONFIGS[name]
    b = synth.make_batch(cfg, lengths="ragged") if name == "tiny" else synth.make_batch(cfg)
    st, info = device_step(cfg, b)
    for nb in (1, 3, 8):
        h = st.staleness_histogram(t_train=synth.T_TRAIN, max_lag=cfg.max_lag, n_bins=nb).cpu().numpy()
        ref = oracle.staleness_histogram(b.version, b.resp_len, group_size=cfg.G, max_len=cfg.S, t_train=synth.T_TRAIN,
                                         max_lag=cfg.max_lag, n_bins=nb)
        np.testing.assert_array_equal(h, ref)
        assert h[2].sum() == info.n_tokens


def test_rollout_filter_partial_groups_bit_exact():
    """f3 partial groups: per-rollout staleness filter (echo_pack_batch_v2, ECHO_FILTER_ROLLOUT) on groups whose
    rollouts carry different versions; pack, the survivors-only group advantage and the histogram bit-exact."""
    from paper_2508_05387_b200 import abi
    cfg = synth.CONFIGS["qwen2.5-7b"]
    b = synth.make_batch(cfg, 0, 32 * cfg.G, lengths="ragged")
    rng = np.random.default_rng(3)
    b.version = (synth.T_TRAIN - rng.integers(0, 5, len(b.version))).astype(np.int64)   # per-rollout versions
    st = __import__("paper_2508_05387_b200.step", fromlist=["LearnerStep"]).LearnerStep(
        n_rollouts=len(b.version), group_size=cfg.G, max_len=cfg.S, vocab=cfg.V, dtype=cfg.dtype)
    st.h2d(*[torch.from_numpy(np.ascontiguousarray(x)) for x in (b.version, b.resp_len, b.reward, b.action,
                                                                 b.old_logp, b.ref_logp)])
    info = st.pack(t_train=synth.T_TRAIN, max_lag=cfg.max_lag, filter_mode=abi.ECHO_FILTER_ROLLOUT)
    pk = oracle.pack_batch(b.version, b.resp_len, b.action, b.old_logp, b.ref_logp, group_size=cfg.G, max_len=cfg.S,
                           vocab=cfg.V, t_train=synth.T_TRAIN, max_lag=cfg.max_lag, filter_mode=1)
    assert (info.status, info.n_rollouts_kept, info.n_groups_kept, info.n_tokens) == \
        (pk.status, pk.n_rollouts_kept, pk.n_groups_kept, pk.n_tokens) and info.status == 0
    assert 0 < pk.n_rollouts_kept < len(b.version) and pk.n_groups_kept <= 32
    n, nt = pk.n_rollouts_kept, pk.n_tokens
    np.testing.assert_array_equal(st.kept_rollout[:n].cpu().numpy(), pk.kept_rollout)
    np.testing.assert_array_equal(st.kept_offset[:n + 1].cpu().numpy(), pk.kept_offset)
    for a_, b_ in ((st.tok_slot, pk.tok_slot), (st.tok_action, pk.tok_action)):
        np.testing.assert_array_equal(a_[:nt].cpu().numpy(), b_)
    assert st.tok_old[:nt].cpu().numpy().tobytes() == pk.tok_old.tobytes()
    st.advantage()
    adv, stats = oracle.group_advantage(b.reward, pk.kept_rollout, group_size=cfg.G)
    assert st.adv_slot[:n].cpu().numpy().tobytes() == adv.tobytes()
    assert st.adv_stats.cpu().numpy().tobytes() == stats.tobytes()
    h = st.staleness_histogram(t_train=synth.T_TRAIN, max_lag=cfg.max_lag, n_bins=4, filter_mode=1).cpu().numpy()
    ref = oracle.staleness_histogram(b.version, b.resp_len, group_size=cfg.G, max_len=cfg.S, t_train=synth.T_TRAIN,
                                     max_lag=cfg.max_lag, n_bins=4, filter_mode=1)
    np.testing.assert_array_equal(h, ref)
    # the same batch under the whole-group filter is a MIXED_GROUP_VERSION error
    info0 = st.pack(t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
    assert info0.status == abi.ECHO_DATA_MIXED_GROUP_VERSION


def test_loss_kernel_replays_in_a_cuda_graph():
    """The fused kernel captured in a CUDA graph and replayed (twice, on fresh logits) gives the eager results bit
    for bit: the in-order row scheduler's counter slot resets itself at the end of every launch."""
    cfg = synth.CONFIGS["qwen3-4b"]
    b = synth.make_batch(cfg, 0, 2 * cfg.G)
    st, info = device_step(cfg, b)
    n = 4096
    src = fill(st, cfg, 0, n)
    eager = src.clone()
    st.loss(eager, 0, kl_coef=cfg.kl_coef)
    lp_eager = st.tok_logp[:n].clone()
    work = src.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        st.loss(work, 0, kl_coef=cfg.kl_coef, stream=s)          # warm-up outside capture
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    work.copy_(src)
    with torch.cuda.graph(g):
        st.loss(work, 0, kl_coef=cfg.kl_coef)
    for _ in range(2):
        work.copy_(src)
        st.tok_logp.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(work, eager)
        assert torch.equal(st.tok_logp[:n], lp_eager)


@pytest.mark.parametrize("V", [155656, 200003, 262144, 311296])
def test_hex_tile_large_vocabularies(V):
    """ECHO_ALGO_HEX_REG (16-CTA clusters, AUTO past 155648 columns): fwd+bwd, forward-only log-probs and the
    entropy variant on Gemma / Llama-4-class vocabularies against the oracle (sampled rows, ragged V)."""
    import dataclasses
    from paper_2508_05387_b200 import abi
    cfg = dataclasses.replace(synth.CONFIGS["qwen3-4b"], V=V)
    b = synth.make_batch(cfg, 0, cfg.G)
    st, info = device_step(cfg, b)
    o = oracle_step(cfg, b)
    assert abi.echo_policy_loss_launch_shape(abi.ECHO_BF16, 64, V)["algo"] == abi.ECHO_ALGO_HEX_REG
    n = 48
    ld = (V + 7) // 8 * 8
    logits = fill(st, cfg, 0, n, ld=ld)
    z = as_oracle_rows(logits)[:, :V]
    args = (o.pk.tok_action[:n], o.pk.tok_old[:n], o.pk.tok_ref[:n], o.pk.tok_slot[:n], o.adv)
    N = info.n_tokens
    # forward-only log-probs first (read-only)
    lp = torch.empty(n, device="cuda")
    abi.echo_token_logp(logits, abi.ECHO_BF16, n, V, ld, st.tok_action, lp)
    lp_ref, _, _ = oracle.token_logp(z, o.pk.tok_action[:n], vocab=V, dtype=oracle.BF16)
    assert np.all(np.abs(lp.cpu().numpy() - lp_ref) <= 1e-5 + 1e-6 * np.abs(lp_ref))
    probe = oracle.policy_loss(z, *args, n_global=N, kl_coef=cfg.kl_coef)
    s = pow2_scale_for(np.abs(probe.dlogits).max())
    ref = oracle.policy_loss(z, *args, n_global=N, kl_coef=cfg.kl_coef, grad_scale=s)
    work = logits.clone()
    st.loss(work, 0, kl_coef=cfg.kl_coef, grad_scale=s)
    check_rows(d_gpu=work[:, :V].float().cpu().numpy(), logp_gpu=st.tok_logp[:n].cpu().numpy(),
               loss_gpu=st.tok_loss[:n].cpu().numpy(), flags_gpu=st.tok_flags[:n].cpu().numpy(), ref=ref,
               dtype="bf16", old=o.pk.tok_old[:n],
               sens=coef_sens(ref, o.pk.tok_old[:n], o.pk.tok_ref[:n], o.adv[o.pk.tok_slot[:n]], cfg.kl_coef, s, N))
    assert torch.equal(work[:, V:], logits[:, V:])                      # padding untouched
    # entropy variant on the same rows
    eta = 0.01
    ref_e = oracle.policy_loss(z, *args, n_global=N, kl_coef=cfg.kl_coef, grad_scale=s, entropy_coef=eta)
    ent = torch.empty(st.cap, device="cuda")
    work = logits.clone()
    st.loss(work, 0, kl_coef=cfg.kl_coef, grad_scale=s, entropy_coef=eta, tok_entropy=ent)
    H = ent[:n].cpu().numpy().astype(np.float64)
    _, lse, _ = oracle.token_logp(z, o.pk.tok_action[:n], vocab=V, dtype=oracle.BF16)
    hbar = 3e-5 * (1 + np.abs(lse) + np.abs(ref_e.entropy))
    assert np.all(np.abs(H - ref_e.entropy) <= hbar)


@pytest.mark.parametrize("V", [151936, 150001, 32768])
def test_fp32_cluster_tile(V):
    """fp32 logits on the 16-CTA tile (AUTO for fp32, 16384 <= V <= 155648): fwd+bwd, forward-only log-probs and
    the entropy variant against the oracle, ragged V, padding columns untouched."""
    import dataclasses
    from paper_2508_05387_b200 import abi
    cfg = dataclasses.replace(synth.CONFIGS["qwen3-4b"], V=V, dtype="f32")
    b = synth.make_batch(cfg, 0, cfg.G)
    st, info = device_step(cfg, b)
    o = oracle_step(cfg, b)
    assert abi.echo_policy_loss_launch_shape(abi.ECHO_F32, 64, V)["algo"] == abi.ECHO_ALGO_HEX_REG
    n = 40
    ld = (V + 3) // 4 * 4 + 4
    logits = fill(st, cfg, 0, n, ld=ld)
    z = logits[:, :V].cpu().numpy()
    args = (o.pk.tok_action[:n], o.pk.tok_old[:n], o.pk.tok_ref[:n], o.pk.tok_slot[:n], o.adv)
    N = info.n_tokens
    lp = torch.empty(n, device="cuda")
    abi.echo_token_logp(logits, abi.ECHO_F32, n, V, ld, st.tok_action, lp)
    lp_ref, lse, _ = oracle.token_logp(z, o.pk.tok_action[:n], vocab=V, dtype=oracle.F32)
    assert np.all(np.abs(lp.cpu().numpy() - lp_ref) <= 1e-5 + 1e-6 * np.abs(lp_ref))
    ref = oracle.policy_loss(z, *args, n_global=N, kl_coef=cfg.kl_coef, grad_scale=float(N))
    work = logits.clone()
    st.loss(work, 0, kl_coef=cfg.kl_coef, grad_scale=float(N))
    check_rows(d_gpu=work[:, :V].cpu().numpy(), logp_gpu=st.tok_logp[:n].cpu().numpy(),
               loss_gpu=st.tok_loss[:n].cpu().numpy(), flags_gpu=st.tok_flags[:n].cpu().numpy(), ref=ref, dtype="f32",
               old=o.pk.tok_old[:n],
               sens=coef_sens(ref, o.pk.tok_old[:n], o.pk.tok_ref[:n], o.adv[o.pk.tok_slot[:n]], cfg.kl_coef,
                                 float(N), N))
    assert torch.equal(work[:, V:], logits[:, V:])
    eta = 0.02
    ref_e = oracle.policy_loss(z, *args, n_global=N, kl_coef=cfg.kl_coef, grad_scale=float(N), entropy_coef=eta)
    ent = torch.empty(st.cap, device="cuda")
    work = logits.clone()
    st.loss(work, 0, kl_coef=cfg.kl_coef, grad_scale=float(N), entropy_coef=eta, tok_entropy=ent)
    H = ent[:n].cpu().numpy().astype(np.float64)
    hbar = 3e-5 * (1 + np.abs(lse) + np.abs(ref_e.entropy))
    assert np.all(np.abs(H - ref_e.entropy) <= hbar)


def test_fuzz_shapes_and_tiles():
    """Randomised shapes through every tile and dtype: V from 16 to 311296 (ragged, empty high-rank slices), row
    counts below and above the resident clusters, ld padding; sampled rows against the oracle, padding untouched,
    and the AUTO choice reported by echo_policy_loss_launch_shape."""
    import dataclasses
    from paper_2508_05387_b200 import abi
    rng = np.random.default_rng(2026)
    base = synth.CONFIGS["qwen3-4b"]
    cases, used = [], set()
    for i in range(64):
        dtype = "f32" if rng.random() < 0.3 else "bf16"
        vmax = 155648 if dtype == "f32" else 311296
        # half log-uniform over the whole range (row kernel territory below 16384), half in the cluster tiles' range
        V = int(np.exp(rng.uniform(np.log(16), np.log(vmax)))) if i % 2 else int(rng.integers(16384, vmax + 1))
        algo = None
        if dtype == "bf16" and rng.random() < 0.4:
            def ok(a):
                try:
                    abi.echo_policy_loss_launch_shape(abi.ECHO_BF16, 8, V, abi.ALGO_NAMES[a])
                    return True
                except abi.EchoError:
                    return False
            opts = [a for a in ("quad_reg", "quad_reg_exact", "oct_reg", "hex_reg", "row_l2") if ok(a)]
            algo = opts[int(rng.integers(0, len(opts)))]
        cases.append((dtype, V, algo, int(rng.integers(1, 300))))
    for dtype, V, algo_name, n in cases:
        cfg = dataclasses.replace(base, V=V, dtype=dtype)
        b = synth.make_batch(cfg, 0, cfg.G)
        st, info = device_step(cfg, b)
        o = oracle_step(cfg, b)
        n = min(n, info.n_tokens)
        esize = 2 if dtype == "bf16" else 4
        ld = (V + 7) // 8 * 8 + (8 if rng.random() < 0.5 else 0)
        logits = fill(st, cfg, 0, n, ld=ld)
        z = as_oracle_rows(logits)[:, :V]
        rows = np.unique(np.concatenate([[0, n - 1], rng.integers(0, n, 6)]))
        args = (o.pk.tok_action[rows], o.pk.tok_old[rows], o.pk.tok_ref[rows], o.pk.tok_slot[rows], o.adv)
        N = info.n_tokens
        ref = oracle.policy_loss(z[rows], *args, n_global=N, kl_coef=cfg.kl_coef, grad_scale=float(N))
        work = logits.clone()
        algo = None if algo_name is None else abi.ALGO_NAMES[algo_name]
        try:
            st.loss(work, 0, kl_coef=cfg.kl_coef, grad_scale=float(N), algo=algo)
        except abi.EchoError:
            assert algo is not None          # an explicit tile that cannot take this V; AUTO always can
            continue
        torch.cuda.synchronize()
        d = work[torch.from_numpy(rows).cuda(), :V].float().cpu().numpy()
        check_rows(d_gpu=d, logp_gpu=st.tok_logp[rows].cpu().numpy(), loss_gpu=st.tok_loss[rows].cpu().numpy(),
                   flags_gpu=st.tok_flags[rows].cpu().numpy(), ref=ref, dtype=dtype, old=o.pk.tok_old[rows],
                   sens=coef_sens(ref, o.pk.tok_old[rows], o.pk.tok_ref[rows], o.adv[o.pk.tok_slot[rows]],
                                     cfg.kl_coef, float(N), N))
        if ld > V:
            assert torch.equal(work[:, V:], logits[:, V:]), (dtype, V, algo_name)
        used.add((dtype, abi.echo_policy_loss_launch_shape(abi.ECHO_BF16 if dtype == "bf16" else abi.ECHO_F32, n, V,
                                                           algo or 0)["algo"]))
    assert {("bf16", abi.ECHO_ALGO_OCT_REG), ("bf16", abi.ECHO_ALGO_HEX_REG), ("f32", abi.ECHO_ALGO_HEX_REG),
            ("bf16", abi.ECHO_ALGO_ROW_L2), ("f32", abi.ECHO_ALGO_ROW_L2)} <= used, used


@pytest.mark.parametrize("n,d,V", [(300, 512, 1000), (257, 2560, 151936)])
def test_lmhead_entropy(n, d, V):
    """f2 with the entropy output (f4): H_t against the fp64 oracle; logp unchanged by asking for it."""
    from paper_2508_05387_b200 import abi
    h, w, act = _lmhead_case(n, d, V, seed=11 + d)
    ws = torch.empty(abi.echo_lmhead_workspace_bytes(n, V) // 4 + 1, dtype=torch.float32, device="cuda")
    lp = torch.empty(n, device="cuda")
    lp0 = torch.empty(n, device="cuda")
    ent = torch.full((n,), float("nan"), device="cuda")
    lse = torch.empty(n, device="cuda")
    abi.echo_lmhead_logp(h, w, n, d, V, act, lp, lse, ws, tok_entropy=ent)
    abi.echo_lmhead_logp(h, w, n, d, V, act, lp0, None, ws)
    torch.cuda.synchronize()
    assert torch.equal(lp, lp0)
    rows = np.arange(n) if V < 10000 else np.array([0, 1, 128, 255, 256])
    hb = h[torch.from_numpy(rows).cuda()].cpu().view(torch.int16).numpy().view(np.uint16)
    wb = w.cpu().view(torch.int16).numpy().view(np.uint16)
    _, lse_ref, ent_ref = oracle.lmhead_logp(hb, wb, act.cpu().numpy()[rows], want_entropy=True)
    H = ent.cpu().numpy().astype(np.float64)[rows]
    tol = _lmhead_tol(hb, wb, np.arange(len(rows))) + 3e-5 * (1 + np.abs(lse_ref) + np.abs(ent_ref))
    assert np.all(np.abs(H - ent_ref) <= tol), np.max(np.abs(H - ent_ref) / tol)
    assert np.max(np.abs(H - ent_ref)) <= 2e-4


def test_token_logp_fuzz_shapes():
    """f1 (echo_token_logp) over random shapes: bf16 vocabularies from 16 to 311296 (the one-warp-per-row kernel from
    8192 up, ragged V, rows fewer and more than the resident warps, padded ld) and fp32 ones; logp, lse and flags
    against the oracle, the logits untouched."""
    import dataclasses
    from paper_2508_05387_b200 import abi
    rng = np.random.default_rng(4242)
    base = synth.CONFIGS["qwen3-4b"]
    for i in range(24):
        dtype = "f32" if i % 6 == 5 else "bf16"
        V = int(np.exp(rng.uniform(np.log(16), np.log(311296 if dtype == "bf16" else 155648))))
        if i % 3 == 0 and dtype == "bf16":
            V = int(rng.integers(8192, 311297))
        cfg = dataclasses.replace(base, V=V, dtype=dtype)
        b = synth.make_batch(cfg, 0, cfg.G)
        st, info = device_step(cfg, b)
        o = oracle_step(cfg, b)
        n = min(int(rng.integers(1, 3000)), info.n_tokens)
        ld = (V + 7) // 8 * 8 + (8 if i % 2 else 0)
        logits = fill(st, cfg, 0, n, ld=ld)
        before = logits.clone()
        lp = torch.full((n,), float("nan"), device="cuda")
        lse = torch.full((n,), float("nan"), device="cuda")
        flags = torch.full((n,), 7, dtype=torch.uint8, device="cuda")
        abi.echo_token_logp(logits, abi.ECHO_BF16 if dtype == "bf16" else abi.ECHO_F32, n, V, ld, st.tok_action, lp,
                            lse, flags)
        torch.cuda.synchronize()
        assert torch.equal(logits, before)
        rows = np.unique(np.concatenate([[0, n - 1], rng.integers(0, n, 16)]))
        z = as_oracle_rows(logits[torch.from_numpy(rows).cuda()])[:, :V]
        ref_lp, ref_lse, ref_flags = oracle.token_logp(z, o.pk.tok_action[rows], vocab=V)
        g_lp = lp.cpu().numpy()[rows].astype(np.float64)
        g_lse = lse.cpu().numpy()[rows].astype(np.float64)
        assert np.all(np.abs(g_lp - ref_lp) <= 1e-5 + 1e-6 * np.abs(ref_lp)), (dtype, V, n, np.max(np.abs(g_lp - ref_lp)))
        assert np.all(np.abs(g_lse - ref_lse) <= 1e-5 + 1e-6 * np.abs(ref_lse)), (dtype, V, n)
        np.testing.assert_array_equal(flags.cpu().numpy()[rows], ref_flags)
