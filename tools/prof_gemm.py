"""tcgen05 GEMM (echo_gemm_bf16) vs cuBLAS at the f2 backward's shapes:
dhidden = D W ([rows x V] . [V x d]) and dweight (+)= D^T h ([V x rows] . [rows x d]).  Prints one JSON object.

The cuBLAS arm is the fair one: cublasGemmEx on torch's handle with bf16 inputs, fp32 accumulation and the same fp32
outputs as libecho (dweight accumulated, beta = 1, as across the chunks of a training step) -- the calls the training
step made before its backward moved onto libecho's kernels.  NVML SM clock and power are sampled per arm.

    python tools/prof_gemm.py [--rows 8192 --d 2560 --vocab 151936 --reps 5]
"""
import argparse
import ctypes
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402


def cublas_lib():
    import nvidia.cublas  # torch's bundled cuBLAS
    paths = sorted(glob.glob(os.path.join(list(nvidia.cublas.__path__)[0], "lib", "libcublas.so*")))
    lib = ctypes.CDLL(paths[0])
    P, i32 = ctypes.c_void_p, ctypes.c_int
    lib.cublasGemmEx.argtypes = [P, i32, i32, i32, i32, i32, P, P, i32, i32, P, i32, i32, P, P, i32, i32, i32, i32]
    lib.cublasSetStream_v2.argtypes = [P, P]
    return lib


def cublas_grads(lib, D, W, h, dh, dw, ld, rows, d, V, beta_one):
    """The same two products as libecho (column-major views), fp32 out."""
    handle = ctypes.c_void_p(torch.cuda.current_blas_handle())
    lib.cublasSetStream_v2(handle, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    one, zero = ctypes.c_float(1.0), ctypes.c_float(0.0)
    BF, F32, C32, DEF = 14, 0, 68, -1
    st = lib.cublasGemmEx(handle, 0, 0, d, rows, V, ctypes.byref(one), W.data_ptr(), BF, d, D.data_ptr(), BF, ld,
                          ctypes.byref(zero), dh.data_ptr(), F32, d, C32, DEF)
    assert st == 0, st
    if dw is not None:
        st = lib.cublasGemmEx(handle, 0, 1, d, V, rows, ctypes.byref(one), h.data_ptr(), BF, d, D.data_ptr(), BF, ld,
                              ctypes.byref(one if beta_one else zero), dw.data_ptr(), F32, d, C32, DEF)
        assert st == 0, st


def cublas_dw(lib, D, h, dw, ld, rows, d, V, beta_one=True):
    handle = ctypes.c_void_p(torch.cuda.current_blas_handle())
    lib.cublasSetStream_v2(handle, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    one, zero = ctypes.c_float(1.0), ctypes.c_float(0.0)
    st = lib.cublasGemmEx(handle, 0, 1, d, V, rows, ctypes.byref(one), h.data_ptr(), 14, d, D.data_ptr(), 14, ld,
                          ctypes.byref(one if beta_one else zero), dw.data_ptr(), 0, d, 68, -1)
    assert st == 0, st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=8192)
    ap.add_argument("--d", type=int, default=2560)
    ap.add_argument("--vocab", type=int, default=151936)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="", help="comma list of arms: dh_tc,dw_tc,dh_cublas,dw_cublas,dh_bf16,dw_bf16")
    a = ap.parse_args()
    import __graft_entry__
    __graft_entry__.build()
    from paper_2508_05387_b200 import abi
    n, d, V = a.rows, a.d, a.vocab
    ld = (V + 7) // 8 * 8
    g = torch.Generator(device="cuda").manual_seed(0)
    D = (torch.randn(n, ld, generator=g, device="cuda") * 1e-3).to(torch.bfloat16)
    W = torch.randn(V, d, generator=g, device="cuda").to(torch.bfloat16)
    h = torch.randn(n, d, generator=g, device="cuda").to(torch.bfloat16)
    dh = torch.empty(n, d, device="cuda")
    dw = torch.zeros(V, d, device="cuda")
    fl = 2.0 * n * d * V
    lib = cublas_lib()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")

    from _clock import Clock
    clocks = {}

    def timed(fn, key=None):
        ts = []
        with Clock() as ck:
            _timed(fn, ts)
        if key:
            clocks[key] = ck.summary()
        ts.sort()
        return ts[len(ts) // 2]

    def _timed(fn, ts):
        for r in range(a.reps + 2):
            flush.fill_(float(r))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(e0.elapsed_time(e1))

    arms = {
        "dh_tc": lambda: abi.echo_gemm_bf16(D, 0, ld, W, 1, d, n, d, V, dh, d),
        "dw_tc": lambda: abi.echo_gemm_bf16(D, 1, ld, h, 1, d, V, d, n, dw, d, accumulate=True),
        "dh_cublas": lambda: cublas_grads(lib, D, W, h, dh, None, ld, n, d, V, False),
        "dw_cublas": lambda: cublas_dw(lib, D, h, dw, ld, n, d, V),
    }
    only = [x for x in a.only.split(",") if x]
    out = {"rows": n, "d": d, "vocab": V, "gflop_each": fl / 1e9,
           "cublas": "cublasGemmEx bf16 in, fp32 compute and out (dweight beta = 1)"}
    for k, fn in arms.items():
        if only and k not in only:
            continue
        out[k + "_ms"] = timed(fn, k)
        out[k + "_tflops"] = fl / out[k + "_ms"] / 1e9
    for p in ("dh", "dw"):
        if f"{p}_tc_ms" in out and f"{p}_cublas_ms" in out:
            out[f"{p}_tc_vs_cublas"] = out[f"{p}_cublas_ms"] / out[f"{p}_tc_ms"]
    out["clocks"] = clocks
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
