#!/usr/bin/env python
"""Small invocation of every libecho kernel for compute-sanitizer (one tool per run): tiny fp32 step (row kernel),
a few Qwen-vocab bf16 rows through the quad kernel (both modes) and the forward-only path, ragged vocab."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import synth
    import synth.gpu as sgpu
    from paper_2508_05387_b200 import abi
    from paper_2508_05387_b200.step import LearnerStep
    for name, rows, algos in (("tiny", None, [None]), ("qwen3-4b", 40, [abi.ECHO_ALGO_QUAD_REG,
                                                                        abi.ECHO_ALGO_QUAD_REG_EXACT,
                                                                        abi.ECHO_ALGO_ROW_L2])):
        cfg = synth.CONFIGS[name]
        P = cfg.P if name == "tiny" else 2
        b = synth.make_batch(cfg, 0, P * cfg.G, lengths="ragged")
        st = LearnerStep(n_rollouts=P * cfg.G, group_size=cfg.G, max_len=cfg.S, vocab=cfg.V, dtype=cfg.dtype)
        st.h2d(*[torch.from_numpy(np.ascontiguousarray(x)) for x in (b.version, b.resp_len, b.reward, b.action,
                                                                     b.old_logp, b.ref_logp)])
        info = st.pack(t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
        st.advantage()
        st.reduce_counts()
        n = info.n_tokens if rows is None else min(rows, info.n_tokens)
        dt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
        for algo in algos:
            logits = torch.empty(n, cfg.V, dtype=dt, device="cuda")
            sgpu.fill_logits(logits, dtype=cfg.dtype, vocab=cfg.V, row0=0, tok_slot=st.tok_slot,
                             tok_action=st.tok_action, kept_rollout=st.kept_rollout, kept_offset=st.kept_offset,
                             max_len=cfg.S, seed=cfg.seed)
            lp = torch.empty(n, device="cuda")
            abi.echo_token_logp(logits, st.edtype, n, cfg.V, cfg.V, st.tok_action, lp)
            st.loss(logits, 0, kl_coef=cfg.kl_coef, algo=algo)
        st.finish()
    torch.cuda.synchronize()
    lmhead()
    print("sanitize workload done")


def lmhead():
    """f2 kernels on ragged shapes: fused log-prob (+ entropy), logits store, D recompute, both training-step forms."""
    from paper_2508_05387_b200 import abi
    n, d, V, chunk = 300, 136, 1003, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    h = torch.randn(n, d, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(V, d, generator=g, device="cuda") * 0.2).to(torch.bfloat16)
    act = torch.randint(0, V, (n,), generator=g, device="cuda", dtype=torch.int32)
    ws = torch.empty(abi.echo_lmhead_workspace_bytes(n, V) // 4 + 1, dtype=torch.float32, device="cuda")
    lp, lse, ent, coef, ecoef, loss = (torch.empty(n, device="cuda") for _ in range(6))
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    abi.echo_lmhead_logp(h, w, n, d, V, act, lp, lse, ws, tok_entropy=ent)
    old = lp - 0.1
    adv = torch.randn(8, generator=g, device="cuda")
    slot = torch.randint(0, 8, (n,), generator=g, device="cuda", dtype=torch.int32)
    ng = torch.tensor([float(n)], dtype=torch.float64, device="cuda")
    cfg = abi.LossConfig(0.2, 0.2, 0.0, 0.01, 1.0, abi.ECHO_KL_K3, 0.01)
    abi.echo_loss_from_logp(n, lp, ent, old, old, slot, adv, None, None, ng, cfg, loss, flags, coef, ecoef)
    ld = abi.echo_lmhead_dlogits_ld(V)
    z = torch.empty(n, ld, dtype=torch.bfloat16, device="cuda")
    abi.echo_lmhead_logits(h, w, n, d, V, z, ld)
    abi.echo_lmhead_dlogits(h, w, n, d, V, act, lse, coef, ecoef, ent, z, ld)
    dh = torch.empty(n, d, device="cuda")
    dw = torch.empty(V, d, device="cuda")
    zc = torch.empty(chunk * ld, dtype=torch.bfloat16, device="cuda")
    abi.echo_lmhead_backward(h, w, n, d, V, act, lse, coef, ecoef, ent, dh, dw, 0, zc, chunk)
    abi.echo_lmhead_policy_loss_fwd_bwd(h, w, n, d, V, act, old, old, slot, adv, None, None, ng, cfg, lp, loss, flags,
                                        ent, dh, dw, 1, zc, chunk)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
