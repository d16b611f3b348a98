#!/usr/bin/env python
"""Per-phase timing of the fused policy-loss kernels from in-kernel clock64 stamps (diagnostic build).

Builds libecho_trace.so (-DECHO_TRACE), runs one Qwen-shaped micro-batch per algorithm, and prints the mean
cycles per row spent in each phase of CTAs 0..63: 0->1 pass 1a (ring -> registers), 1->2 max + pass 1b,
2->3 first barrier, 3->4 merge / exchange / epilogue, 4->5 pass 2, 5->0' loop overhead.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "paper_2508_05387_b200"))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--algos", default="quad_reg,quad_reg_exact")
    ap.add_argument("--rows", type=int, default=32768)
    args = ap.parse_args()
    import _build
    import __graft_entry__
    __graft_entry__.build()
    trace_lib = _build.build(trace=True)
    import ctypes
    from paper_2508_05387_b200 import abi
    abi._lib = abi._load(trace_lib)
    abi._lib.echo_trace_set.argtypes = [ctypes.c_void_p, ctypes.c_int32]
    import synth
    import synth.gpu as sgpu
    from paper_2508_05387_b200.step import LearnerStep

    cfg = synth.CONFIGS["qwen3-4b"]
    n_roll = -(-args.rows // cfg.S)
    n_roll = -(-n_roll // cfg.G) * cfg.G
    b = synth.make_batch(cfg, 0, n_roll)
    st = LearnerStep(n_rollouts=n_roll, group_size=cfg.G, max_len=cfg.S, vocab=cfg.V, dtype=cfg.dtype)
    st.h2d(*[torch.from_numpy(np.ascontiguousarray(x)) for x in (b.version, b.resp_len, b.reward, b.action,
                                                                 b.old_logp, b.ref_logp)])
    info = st.pack(t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
    st.advantage()
    st.reduce_counts()
    M = min(args.rows, info.n_tokens)
    logits = torch.empty(M, cfg.V, dtype=torch.bfloat16, device="cuda")
    rows_cap = 1024
    trace = torch.zeros(64 * rows_cap * 16, dtype=torch.int64, device="cuda")
    out = {}
    for name in args.algos.split(","):
        algo = abi.ALGO_NAMES[name]
        for rep in range(2):
            sgpu.fill_logits(logits, dtype=cfg.dtype, vocab=cfg.V, row0=0, tok_slot=st.tok_slot,
                             tok_action=st.tok_action, kept_rollout=st.kept_rollout, kept_offset=st.kept_offset,
                             max_len=cfg.S, seed=cfg.seed)
            trace.zero_()
            abi._lib.echo_trace_set(trace.data_ptr(), rows_cap)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st.loss(logits, 0, kl_coef=cfg.kl_coef, algo=algo)
            e1.record()
            torch.cuda.synchronize()
            abi._lib.echo_trace_set(None, 0)
        t = trace.view(64, rows_cap, 16).cpu().numpy().astype(np.float64)
        valid = (t[:, :, 0] > 0) & (t[:, :, 5] > 0)
        ph = {}
        for k, lab in ((1, "pass1a"), (2, "max+pass1b"), (3, "barrier1"), (4, "merge+epilogue"), (5, "pass2")):
            d = (t[:, :, k] - t[:, :, k - 1])[valid]
            ph[lab] = float(d.mean())
        if (t[:, :, 6] > 0).any():
            ph["merge:before_send"] = float((t[:, :, 6] - t[:, :, 3])[valid].mean())
            ph["merge:wait_peers"] = float((t[:, :, 7] - t[:, :, 6])[valid].mean())
            ph["merge:after_wait"] = float((t[:, :, 4] - t[:, :, 7])[valid].mean())
        if (t[:, :, 12] > 0).any():
            for lab, k0, k1 in (("1a:wait_full", 0, 8), ("1a:lds", 8, 9), ("1a:consumed+tma", 9, 10),
                                ("1b:exp_loop", 10, 11), ("1b:warp_reduce", 11, 2), ("merge:cta_reduce", 3, 12),
                                ("merge:send", 12, 6)):
                ph[lab] = float((t[:, :, k1] - t[:, :, k0])[valid].mean())
        nxt = (t[:, 1:, 0] - t[:, :-1, 5])[valid[:, 1:] & valid[:, :-1]]
        ph["loop"] = float(nxt.mean()) if nxt.size else 0.0
        rowt = (t[:, 1:, 0] - t[:, :-1, 0])[valid[:, 1:] & valid[:, :-1]]
        ph["row_total"] = float(rowt.mean()) if rowt.size else 0.0
        out[name] = {"ms": e0.elapsed_time(e1), "cycles_per_row": ph,
                     "rows_per_cta": float(valid.sum(axis=1).mean())}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
