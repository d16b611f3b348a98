"""Interleaved A/B of env-var knobs read at launch time by libecho (ECHO_GEMM_MC, ECHO_LM_MC, ECHO_GEMM_GROUP, ...):
each round runs every variant once (CUDA-event timed, median of --reps launches after 2 warm-ups), rounds alternate so
that box clock drift hits every variant alike.  Prints one JSON object with per-variant medians over rounds.

    python tools/ab_env.py --op dh|dw|lm --rows 8192 --d 2560 --variants "ECHO_GEMM_MC=0;ECHO_GEMM_MC=1" --rounds 4

The variant CUBLAS runs the same product in cuBLAS instead (dh / dw: cublasGemmEx with fp32 out, dweight accumulated;
lm / lmlogits: torch.matmul into bf16 logits), interleaved like the others.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--op", default="dh", choices=["dh", "dw", "lm", "lmlogits", "zgemm", "ent", "loss", "logp"])
    ap.add_argument("--config", default="qwen3-32b", help="ent / loss: the BASELINE.json config of the micro-batch")
    ap.add_argument("--rows", type=int, default=8192)
    ap.add_argument("--d", type=int, default=2560)
    ap.add_argument("--vocab", type=int, default=151936)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--variants", required=True, help="';'-separated list of space-separated K=V settings")
    ap.add_argument("--no-flush", action="store_true", help="back-to-back launches (sustained, power-capped clocks)")
    a = ap.parse_args()
    import __graft_entry__
    __graft_entry__.build()
    from paper_2508_05387_b200 import abi
    n, d, V = a.rows, a.d, a.vocab
    ld = (V + 7) // 8 * 8
    g = torch.Generator(device="cuda").manual_seed(0)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    regen = None
    if a.op in ("ent", "loss", "logp"):   # (3)-(5) or f1 on one Qwen-shaped micro-batch (logits regenerated per rep)
        import numpy as np
        import synth
        import synth.gpu as sgpu
        from paper_2508_05387_b200.step import LearnerStep
        cfg = synth.CONFIGS[a.config]
        n_roll = -(-(-(-n // cfg.S)) // cfg.G) * cfg.G
        b = synth.make_batch(cfg, 0, n_roll)
        st = LearnerStep(n_rollouts=n_roll, group_size=cfg.G, max_len=cfg.S, vocab=cfg.V, dtype=cfg.dtype)
        st.h2d(*[torch.from_numpy(np.ascontiguousarray(x)) for x in (b.version, b.resp_len, b.reward, b.action,
                                                                     b.old_logp, b.ref_logp)])
        st.pack(t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
        st.advantage()
        st.reduce_counts()
        V = cfg.V
        ld = (V + 7) // 8 * 8
        logits = torch.empty(n, ld, dtype=torch.bfloat16, device="cuda")
        ent = torch.empty(n, device="cuda")

        def regen():
            sgpu.fill_logits(logits, dtype=cfg.dtype, vocab=V, row0=0, tok_slot=st.tok_slot, tok_action=st.tok_action,
                             kept_rollout=st.kept_rollout, kept_offset=st.kept_offset, max_len=cfg.S, seed=cfg.seed)
        if a.op == "ent":
            fn = lambda: st.loss(logits, 0, kl_coef=cfg.kl_coef, entropy_coef=0.01, tok_entropy=ent)
        elif a.op == "logp":
            from paper_2508_05387_b200 import abi as _abi
            fn = lambda: _abi.echo_token_logp(logits, _abi.ECHO_BF16, n, V, ld, st.tok_action, ent)
        else:
            fn = lambda: st.loss(logits, 0, kl_coef=cfg.kl_coef)
        ref_fn = fn
        flops = (2 * V * 2 + 25) * n   # bytes, for the fused loss ops ("tflops" then reads as GB/s / 1e3)
    elif a.op in ("dh", "dw"):
        D = (torch.randn(n, ld, generator=g, device="cuda") * 1e-3).to(torch.bfloat16)
        W = torch.randn(V, d, generator=g, device="cuda").to(torch.bfloat16)
        h = torch.randn(n, d, generator=g, device="cuda").to(torch.bfloat16)
        dh = torch.empty(n, d, device="cuda")
        dw = torch.zeros(V, d, device="cuda")
        fn = (lambda: abi.echo_gemm_bf16(D, 0, ld, W, 1, d, n, d, V, dh, d)) if a.op == "dh" else \
             (lambda: abi.echo_gemm_bf16(D, 1, ld, h, 1, d, V, d, n, dw, d, accumulate=True))
        import prof_gemm
        lib = prof_gemm.cublas_lib()
        ref_fn = (lambda: prof_gemm.cublas_grads(lib, D, W, h, dh, None, ld, n, d, V, False)) if a.op == "dh" else \
                 (lambda: prof_gemm.cublas_dw(lib, D, h, dw, ld, n, d, V))
        flops = 2.0 * n * d * V
    else:
        h = torch.randn(n, d, generator=g, device="cuda").to(torch.bfloat16)
        w = (torch.randn(V, d, generator=g, device="cuda") * (2.0 / d ** 0.5)).to(torch.bfloat16)
        act = torch.randint(0, V, (n,), generator=g, device="cuda", dtype=torch.int32)
        z = torch.empty(n, ld, dtype=torch.bfloat16, device="cuda")
        ref_fn = lambda: torch.matmul(h, w.t(), out=z[:, :V])
        if a.op == "zgemm":   # the logits product on echo_gemm_bf16 (fp32 out): probes its unit shapes at K = d
            zf = torch.empty(n, ld, device="cuda")
            fn = lambda: abi.echo_gemm_bf16(h, 0, d, w, 0, d, n, V, d, zf, ld)
        elif a.op == "lm":
            ws = torch.empty(abi.echo_lmhead_workspace_bytes(n, V) // 4 + 1, dtype=torch.float32, device="cuda")
            lp = torch.empty(n, device="cuda")
            fn = lambda: abi.echo_lmhead_logp(h, w, n, d, V, act, lp, None, ws)
        else:
            fn = lambda: abi.echo_lmhead_logits(h, w, n, d, V, z, ld)
        flops = 2.0 * n * d * V
    variants = [v.strip() for v in a.variants.split(";")]
    keys = sorted({kv.split("=")[0] for v in variants for kv in v.split() if "=" in kv})
    res = {v: [] for v in variants}
    for rnd in range(a.rounds):
        for v in (variants if rnd % 2 == 0 else variants[::-1]):
            for k in keys:
                os.environ.pop(k, None)
            for kv in v.split():
                if "=" in kv:
                    k, val = kv.split("=")
                    os.environ[k] = val
            run = ref_fn if v == "CUBLAS" else fn
            ts = []
            for r in range(a.reps + 2):
                if regen is not None:
                    regen()
                if not a.no_flush:
                    flush.fill_(float(r))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run()
                e1.record()
                torch.cuda.synchronize()
                if r >= 2:
                    ts.append(e0.elapsed_time(e1))
            res[v].append(statistics.median(ts))
    out = {"op": a.op, "rows": n, "d": d, "vocab": V, "rounds": a.rounds,
           "ms": {v: statistics.median(x) for v, x in res.items()}, "ms_all": res,
           "tflops": {v: flops / statistics.median(x) / 1e9 for v, x in res.items()}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
