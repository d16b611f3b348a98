"""f2 timing: the fused LM-head log-prob (echo_lmhead_logp) vs the unfused path (cuBLAS bf16 GEMM writing the
[N x V] logits, then echo_token_logp) at a Qwen-shaped LM head.  Prints one JSON object.

    python tools/prof_lmhead.py [--rows 32768 --d 2560 --vocab 151936 --reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=32768)
    ap.add_argument("--d", type=int, default=2560)
    ap.add_argument("--vocab", type=int, default=151936)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-unfused", action="store_true")
    ap.add_argument("--mode", default="logp", choices=["logp", "dlogits", "backward", "logits"],
                    help="logp: echo_lmhead_logp; dlogits: echo_lmhead_dlogits over one chunk of --chunk rows; "
                         "backward: echo_lmhead_backward over --rows in --chunk chunks")
    ap.add_argument("--chunk", type=int, default=8192)
    a = ap.parse_args()
    import __graft_entry__
    __graft_entry__.build()
    from paper_2508_05387_b200 import abi
    n, d, V = a.rows, a.d, a.vocab
    g = torch.Generator(device="cuda").manual_seed(0)
    h = torch.randn(n, d, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(V, d, generator=g, device="cuda") * (2.0 / d ** 0.5)).to(torch.bfloat16)
    act = torch.randint(0, V, (n,), generator=g, device="cuda", dtype=torch.int32)
    ws = torch.empty(abi.echo_lmhead_workspace_bytes(n, V) // 4 + 1, dtype=torch.float32, device="cuda")
    lp = torch.empty(n, device="cuda")
    flops = 2.0 * n * d * V

    def timed(fn):
        ts = []
        for r in range(a.reps + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
        ts.sort()
        return ts[len(ts) // 2]

    out = {"rows": n, "d": d, "vocab": V, "gflop": flops / 1e9, "mode": a.mode}
    if a.mode != "logp":
        ld = abi.echo_lmhead_dlogits_ld(V)
        lse = torch.empty(n, device="cuda")
        abi.echo_lmhead_logp(h, w, n, d, V, act, lp, lse, ws)
        coef = torch.randn(n, generator=g, device="cuda") * 1e-3
        ck = min(a.chunk, n)
        dz = torch.empty(ck, ld, dtype=torch.bfloat16, device="cuda")
        if a.mode == "logits":
            fl = 2.0 * ck * d * V
            ms = timed(lambda: abi.echo_lmhead_logits(h, w, ck, d, V, dz, ld))
            out.update(chunk=ck, logits_ms=ms, logits_tflops=fl / ms / 1e9, logits_store_GBps=ck * V * 2 / ms / 1e6)
        elif a.mode == "dlogits":
            fl = 2.0 * ck * d * V
            ms = timed(lambda: abi.echo_lmhead_dlogits(h, w, ck, d, V, act, lse, coef, None, None, dz, ld))
            out.update(chunk=ck, dlogits_ms=ms, dlogits_tflops=fl / ms / 1e9,
                       dlogits_store_GBps=ck * V * 2 / ms / 1e6)
        else:
            dh = torch.empty(n, d, device="cuda")
            dw = torch.empty(V, d, device="cuda")
            ms = timed(lambda: abi.echo_lmhead_backward(h, w, n, d, V, act, lse, coef, None, None, dh, dw, 0, dz, ck))
            out.update(chunk=ck, backward_ms=ms, backward_tflops_6dV_over_3=2 * flops / ms / 1e9,
                       backward_tflops_executed=3 * flops / ms / 1e9)
        print(json.dumps(out))
        return
    ms = timed(lambda: abi.echo_lmhead_logp(h, w, n, d, V, act, lp, None, ws))
    out["fused_ms"] = ms
    out["fused_tflops"] = flops / ms / 1e9
    if not a.no_unfused:
        ld = (V + 7) // 8 * 8
        logits = torch.empty(n, ld, dtype=torch.bfloat16, device="cuda")
        lp2 = torch.empty(n, device="cuda")
        mm = lambda: torch.matmul(h, w.t(), out=logits[:, :V]) if ld == V else logits[:, :V].copy_(h @ w.t())
        out["cublas_gemm_ms"] = timed(mm)
        out["cublas_tflops"] = flops / out["cublas_gemm_ms"] / 1e9
        mm()
        out["token_logp_ms"] = timed(lambda: abi.echo_token_logp(logits, abi.ECHO_BF16, n, V, ld, act, lp2))
        out["unfused_ms"] = out["cublas_gemm_ms"] + out["token_logp_ms"]
        torch.cuda.synchronize()
        d_ = (lp - lp2).abs().max().item()
        out["max_abs_diff_vs_unfused"] = d_
    print(json.dumps(out))


if __name__ == "__main__":
    main()
