"""Breakdown of the chunked f2 training step (echo_lmhead_policy_loss_fwd_bwd's four launches per chunk, issued one
by one through the ABI with CUDA events between them) in sustained back-to-back operation, with the two backward
GEMMs on libecho's kernel or on cuBLAS (fp32 out, dweight accumulated).  Prints one JSON object (ms per stage, summed
over the chunks of one 32768-token micro-batch, median over reps).

    python tools/prof_f2_step.py [--rows 32768 --d 5120 --chunk 8192 --reps 5]
"""
import argparse
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=32768)
    ap.add_argument("--d", type=int, default=5120)
    ap.add_argument("--vocab", type=int, default=151936)
    ap.add_argument("--chunk", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import __graft_entry__
    __graft_entry__.build()
    from paper_2508_05387_b200 import abi
    import prof_gemm
    lib = prof_gemm.cublas_lib()
    n, d, V, ck = a.rows, a.d, a.vocab, a.chunk
    ld = abi.echo_lmhead_dlogits_ld(V)
    g = torch.Generator(device="cuda").manual_seed(0)
    h = torch.randn(n, d, generator=g, device="cuda").to(torch.bfloat16)
    w = (torch.randn(V, d, generator=g, device="cuda") * (2.0 / math.sqrt(d))).to(torch.bfloat16)
    act = torch.randint(0, V, (n,), generator=g, device="cuda", dtype=torch.int32)
    old = torch.full((n,), -8.0, device="cuda")
    slot = torch.zeros(n, dtype=torch.int32, device="cuda")
    adv = torch.ones(1, device="cuda")
    ng = torch.tensor([float(n)], dtype=torch.float64, device="cuda")
    lp, loss = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    zc = torch.empty(ck, ld, dtype=torch.bfloat16, device="cuda")
    dh = torch.empty(n, d, device="cuda")
    dw = torch.empty(V, d, device="cuda")
    stages = ("logits", "loss", "dhidden", "dweight")
    res = {}
    for arm in ("libecho", "cublas"):
        per = {k: [] for k in stages}
        for r in range(a.reps + 1):
            ev = []
            for r0 in range(0, n, ck):
                rows = min(ck, n - r0)
                e = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
                e[0].record()
                abi.echo_lmhead_logits(h[r0:r0 + rows], w, rows, d, V, zc, ld)
                e[1].record()
                abi.echo_policy_loss_fwd_bwd(zc, abi.ECHO_BF16, rows, V, ld, act[r0:], old[r0:], None, slot[r0:], adv,
                                             ng, 0.2, 0.2, 0.0, 1.0, lp[r0:], loss[r0:], flags[r0:])
                e[2].record()
                if arm == "libecho":
                    abi.echo_gemm_bf16(zc, 0, ld, w, 1, d, rows, d, V, dh[r0:r0 + rows], d)
                    e[3].record()
                    abi.echo_gemm_bf16(zc, 1, ld, h[r0:r0 + rows], 1, d, V, d, rows, dw, d, accumulate=r0 > 0)
                else:
                    prof_gemm.cublas_grads(lib, zc, w, h[r0:r0 + rows], dh[r0:r0 + rows], None, ld, rows, d, V, False)
                    e[3].record()
                    prof_gemm.cublas_dw(lib, zc, h[r0:r0 + rows], dw, ld, rows, d, V, beta_one=r0 > 0)
                e[4].record()
                ev.append(e)
            torch.cuda.synchronize()
            if r == 0:
                continue
            for i, k in enumerate(stages):
                per[k].append(sum(e[i].elapsed_time(e[i + 1]) for e in ev))
        res[arm] = {k: statistics.median(v) for k, v in per.items()}
        res[arm]["total"] = sum(res[arm].values())
    flops6 = 6.0 * n * d * V
    out = {"rows": n, "d": d, "vocab": V, "chunk": ck, "ms": res,
           "tflops_6dV": {k: flops6 / v["total"] / 1e9 for k, v in res.items()},
           "note": "stages are separate launches on one stream (no overlap); dweight overwritten by the first chunk "
                   "(cuBLAS beta = 0) and accumulated by the others"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
