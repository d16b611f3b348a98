"""Build + ctypes binding of synth_gen.cu (the GPU logits generator; test/bench infrastructure)."""
from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "synth_gen.cu")
LIB = os.path.join(_HERE, "libechosynth.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(_SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P, i32, i64, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
        _lib.synth_fill_logits.argtypes = [P, i32, i64, i32, i64, i64, P, P, P, P, i32, u32, P]
        _lib.synth_fill_logits.restype = ctypes.c_int
    return _lib


def fill_logits(logits, *, dtype, vocab, row0, tok_slot, tok_action, kept_rollout, kept_offset, max_len, seed,
                stream=None):
    """Write rows [row0, row0 + logits.shape[0]) of the packed batch into the device tensor ``logits``."""
    import torch
    n_rows, ld = logits.shape
    s = torch.cuda.current_stream().cuda_stream if stream is None else stream
    rc = lib().synth_fill_logits(logits.data_ptr(), 1 if dtype == "bf16" else 0, n_rows, vocab, ld, row0,
                                 tok_slot.data_ptr(), tok_action.data_ptr(), kept_rollout.data_ptr(),
                                 kept_offset.data_ptr(), max_len, seed & 0xFFFFFFFF, s)
    if rc != 0:
        raise RuntimeError(f"synth_fill_logits: CUDA error {rc}")
