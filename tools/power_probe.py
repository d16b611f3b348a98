"""Sustained power of the f2 backward GEMMs: each arm (libecho's tcgen05 GEMM or cuBLAS, dhidden / dweight at an
8192-row chunk) runs back to back for --seconds, while NVML samples board power, SM clock and the clock-event reasons.
Prints one JSON object per arm: TFLOP/s from CUDA events over the whole run, median power and clock, the share of
samples with the software power cap active, and joules per PFLOP -- the quantity that decides time once both kernels
sit at the power limit.

    python tools/power_probe.py [--rows 8192 --d 5120 --seconds 4 --arms dh_tc,dh_cublas,dw_tc,dw_cublas]
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

SW_POWER_CAP = 0x4  # nvmlClocksEventReasonSwPowerCap


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=8192)
    ap.add_argument("--d", type=int, default=5120)
    ap.add_argument("--vocab", type=int, default=151936)
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--arms", default="dh_tc,dh_cublas,dw_tc,dw_cublas")
    a = ap.parse_args()
    import __graft_entry__
    __graft_entry__.build()
    from paper_2508_05387_b200 import abi
    import prof_gemm
    import pynvml
    pynvml.nvmlInit()
    nvh = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    n, d, V = a.rows, a.d, a.vocab
    ld = (V + 7) // 8 * 8
    g = torch.Generator(device="cuda").manual_seed(0)
    D = (torch.randn(n, ld, generator=g, device="cuda") * 1e-3).to(torch.bfloat16)
    W = torch.randn(V, d, generator=g, device="cuda").to(torch.bfloat16)
    h = torch.randn(n, d, generator=g, device="cuda").to(torch.bfloat16)
    dh = torch.empty(n, d, device="cuda")
    dw = torch.zeros(V, d, device="cuda")
    lib = prof_gemm.cublas_lib()
    arms = {
        "dh_tc": lambda: abi.echo_gemm_bf16(D, 0, ld, W, 1, d, n, d, V, dh, d),
        "dw_tc": lambda: abi.echo_gemm_bf16(D, 1, ld, h, 1, d, V, d, n, dw, d, accumulate=True),
        "dh_cublas": lambda: prof_gemm.cublas_grads(lib, D, W, h, dh, None, ld, n, d, V, False),
        "dw_cublas": lambda: prof_gemm.cublas_dw(lib, D, h, dw, ld, n, d, V),
    }
    # the LM head's two launches of the f2 paths: logits store (chunked step, 8192 rows) and the fused log-prob
    # (32768 rows), and cuBLAS's bf16 GEMM into the logits buffer for comparison
    w_lm = (torch.randn(V, d, generator=g, device="cuda") * (2.0 / d ** 0.5)).to(torch.bfloat16)
    zc = D  # [n x ld] bf16 buffer
    arms["lm_logits"] = lambda: abi.echo_lmhead_logits(h, w_lm, n, d, V, zc, ld)
    arms["lm_logits_cublas"] = lambda: torch.matmul(h, w_lm.t(), out=zc[:, :V])
    if any(x.startswith("lm_logp") for x in a.arms.split(",")):
        n4 = 4 * n
        h4 = torch.randn(n4, d, generator=g, device="cuda").to(torch.bfloat16)
        act4 = torch.randint(0, V, (n4,), generator=g, device="cuda", dtype=torch.int32)
        ws4 = torch.empty(abi.echo_lmhead_workspace_bytes(n4, V) // 4 + 1, dtype=torch.float32, device="cuda")
        lp4 = torch.empty(n4, device="cuda")
        arms["lm_logp"] = lambda: abi.echo_lmhead_logp(h4, w_lm, n4, d, V, act4, lp4, None, ws4)
    flops_of = {"lm_logp": 2.0 * 4 * n * d * V}
    for name in a.arms.split(","):
        fn = arms[name]
        flops = flops_of.get(name, 2.0 * n * d * V)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        per = time.perf_counter() - t0
        reps = max(8, int(a.seconds / per))
        pw, sm, capped = [], [], []
        stop = threading.Event()

        def sample():
            while not stop.is_set():
                try:
                    pw.append(pynvml.nvmlDeviceGetPowerUsage(nvh) / 1000.0)
                    sm.append(pynvml.nvmlDeviceGetClockInfo(nvh, pynvml.NVML_CLOCK_SM))
                    capped.append(bool(pynvml.nvmlDeviceGetCurrentClocksEventReasons(nvh) & SW_POWER_CAP))
                except Exception:
                    pass
                time.sleep(0.01)

        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps // 4):        # the first quarter settles the power controller; not sampled
            fn()
        e1.record()
        torch.cuda.synchronize()
        th = threading.Thread(target=sample, daemon=True)
        th.start()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        stop.set()
        th.join(timeout=1)
        ms = e0.elapsed_time(e1) / reps
        tfs = flops / ms / 1e9
        p = statistics.median(pw) if pw else None
        print(json.dumps({"arm": name, "rows": n, "d": d, "vocab": V, "reps": reps, "ms": ms, "tflops": tfs,
                          "power_w": p, "sm_mhz": statistics.median(sm) if sm else None,
                          "sw_power_cap_share": (sum(capped) / len(capped)) if capped else None,
                          "samples": len(pw), "joules_per_pflop": (p / tfs * 1e3) if p else None}), flush=True)


if __name__ == "__main__":
    main()
