"""Interleaved A/B of env-var knobs read at launch time by libecho (ECHO_GEMM_MC, ECHO_LM_MC, ECHO_GEMM_GROUP, ...):
each round runs every variant once (CUDA-event timed, median of --reps launches after 2 warm-ups), rounds alternate so
that box clock drift hits every variant alike.  Prints one JSON object with per-variant medians over rounds.

    python tools/ab_env.py --op dh|dw|lm --rows 8192 --d 2560 --variants "ECHO_GEMM_MC=0;ECHO_GEMM_MC=1" --rounds 4
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--op", default="dh", choices=["dh", "dw", "lm", "lmlogits", "train"])
    ap.add_argument("--rows", type=int, default=8192)
    ap.add_argument("--d", type=int, default=2560)
    ap.add_argument("--vocab", type=int, default=151936)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--variants", required=True, help="';'-separated list of space-separated K=V settings")
    a = ap.parse_args()
    import __graft_entry__
    __graft_entry__.build()
    from paper_2508_05387_b200 import abi
    n, d, V = a.rows, a.d, a.vocab
    ld = (V + 7) // 8 * 8
    g = torch.Generator(device="cuda").manual_seed(0)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    if a.op in ("dh", "dw"):
        D = (torch.randn(n, ld, generator=g, device="cuda") * 1e-3).to(torch.bfloat16)
        W = torch.randn(V, d, generator=g, device="cuda").to(torch.bfloat16)
        h = torch.randn(n, d, generator=g, device="cuda").to(torch.bfloat16)
        dh = torch.empty(n, d, device="cuda")
        dw = torch.zeros(V, d, device="cuda")
        fn = (lambda: abi.echo_gemm_bf16(D, 0, ld, W, 1, d, n, d, V, dh, d)) if a.op == "dh" else \
             (lambda: abi.echo_gemm_bf16(D, 1, ld, h, 1, d, V, d, n, dw, d, accumulate=True))
        flops = 2.0 * n * d * V
    else:
        h = torch.randn(n, d, generator=g, device="cuda").to(torch.bfloat16)
        w = (torch.randn(V, d, generator=g, device="cuda") * (2.0 / d ** 0.5)).to(torch.bfloat16)
        act = torch.randint(0, V, (n,), generator=g, device="cuda", dtype=torch.int32)
        if a.op == "lm":
            ws = torch.empty(abi.echo_lmhead_workspace_bytes(n, V) // 4 + 1, dtype=torch.float32, device="cuda")
            lp = torch.empty(n, device="cuda")
            fn = lambda: abi.echo_lmhead_logp(h, w, n, d, V, act, lp, None, ws)
        else:
            z = torch.empty(n, ld, dtype=torch.bfloat16, device="cuda")
            fn = lambda: abi.echo_lmhead_logits(h, w, n, d, V, z, ld)
        flops = 2.0 * n * d * V
    variants = [v.strip() for v in a.variants.split(";")]
    keys = sorted({kv.split("=")[0] for v in variants for kv in v.split()})
    res = {v: [] for v in variants}
    for rnd in range(a.rounds):
        for v in (variants if rnd % 2 == 0 else variants[::-1]):
            for k in keys:
                os.environ.pop(k, None)
            for kv in v.split():
                k, val = kv.split("=")
                os.environ[k] = val
            ts = []
            for r in range(a.reps + 2):
                flush.fill_(float(r))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
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
