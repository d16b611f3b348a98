"""tcgen05 GEMM (echo_gemm_bf16) vs cuBLAS (torch.matmul) at the f2 backward's shapes:
dhidden = D W ([rows x V] . [V x d]) and dweight = D^T h ([V x rows] . [rows x d]).  Prints one JSON object.

    python tools/prof_gemm.py [--rows 8192 --d 2560 --vocab 151936 --reps 5]
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
    ap.add_argument("--rows", type=int, default=8192)
    ap.add_argument("--d", type=int, default=2560)
    ap.add_argument("--vocab", type=int, default=151936)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import __graft_entry__
    __graft_entry__.build()
    from paper_2508_05387_b200 import abi
    n, d, V = a.rows, a.d, a.vocab
    g = torch.Generator(device="cuda").manual_seed(0)
    D = (torch.randn(n, V, generator=g, device="cuda") * 1e-3).to(torch.bfloat16)
    W = torch.randn(V, d, generator=g, device="cuda").to(torch.bfloat16)
    h = torch.randn(n, d, generator=g, device="cuda").to(torch.bfloat16)
    dh = torch.empty(n, d, device="cuda")
    dw = torch.empty(V, d, device="cuda")
    dh16 = torch.empty(n, d, dtype=torch.bfloat16, device="cuda")
    dw16 = torch.empty(V, d, dtype=torch.bfloat16, device="cuda")
    fl = 2.0 * n * d * V

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

    out = {"rows": n, "d": d, "vocab": V, "gflop_each": fl / 1e9}
    out["dh_tc_ms"] = timed(lambda: abi.echo_gemm_bf16(D, 0, V, W, 1, d, n, d, V, dh, d))
    out["dw_tc_ms"] = timed(lambda: abi.echo_gemm_bf16(D, 1, V, h, 1, d, V, d, n, dw, d))
    out["dh_cublas_ms"] = timed(lambda: torch.matmul(D, W, out=dh16))
    out["dw_cublas_ms"] = timed(lambda: torch.matmul(D.t(), h, out=dw16))
    for k in ("dh_tc", "dw_tc", "dh_cublas", "dw_cublas"):
        out[k + "_tflops"] = fl / out[k + "_ms"] / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
