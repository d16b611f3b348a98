"""HBM probes at the kernel's footprint (32768 x 151936 bf16 = 9.96 GB, read + write in place): torch elementwise
ops with different access patterns, to bound what an in-place read-modify-write stream can reach on this box.

    python tools/bw_probe.py [rows] [vocab]
"""
import json
import sys

import torch


def timeit(fn, reps=5, warmup=2, flush=None):
    ts = []
    for r in range(warmup + reps):
        if flush is not None:
            flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if r >= warmup:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    V = int(sys.argv[2]) if len(sys.argv) > 2 else 151936
    x = torch.randn(rows, V, device="cuda", dtype=torch.bfloat16)
    n = x.numel()
    rw = 2 * n * 2
    flush = torch.empty(64 << 20, device="cuda", dtype=torch.float32)
    out = {"rows": rows, "V": V, "probes": {}}
    y = torch.empty_like(x)
    probes = {
        "mul_1.0_inplace": (lambda: x.mul_(1.0), rw),
        "mul_1.0001_inplace": (lambda: x.mul_(1.0001), rw),
        "neg_inplace": (lambda: x.neg_(), rw),
        "copy_to_other": (lambda: y.copy_(x), rw),
        "fill_write_only": (lambda: x.fill_(0.5), n * 2),
        "amax_read_only": (lambda: x.amax(), n * 2),
    }
    for name, (fn, nbytes) in probes.items():
        ms = timeit(fn, flush=flush)
        out["probes"][name] = {"ms": round(ms, 4), "GBps": round(nbytes / ms / 1e6, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
