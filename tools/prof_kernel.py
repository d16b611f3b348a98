#!/usr/bin/env python
"""Kernel-level timing of echo_policy_loss_fwd_bwd on one Qwen-shaped micro-batch (for ncu and tuning).

Generates M packed rows of a BASELINE.json config with the synthetic generator, flushes L2, and times each
requested algorithm with CUDA events over --reps launches (logits regenerated before every launch).  Also times
two plain in-place/copy streams over the same bytes (torch ops) as the achievable-bandwidth reference.
Prints one JSON object.  Under ncu use --reps 1 --warmup 1 and -k regex:policy_loss.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen3-4b")
    ap.add_argument("--rows", type=int, default=32768)
    ap.add_argument("--algos", default="quad_reg,quad_reg_exact,row_l2")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--streams", action="store_true", help="also time torch in-place / copy streams")
    ap.add_argument("--dtype", default=None, choices=[None, "bf16", "f32"], help="override the config's logits dtype")
    ap.add_argument("--vocab", type=int, default=None, help="override the config's vocabulary size")
    ap.add_argument("--entropy", type=float, default=0.0, help="f4 entropy bonus eta (> 0: the entropy variant)")
    args = ap.parse_args()

    import __graft_entry__
    __graft_entry__.build()
    import synth
    import synth.gpu as sgpu
    from paper_2508_05387_b200 import abi
    from paper_2508_05387_b200.step import LearnerStep

    cfg = synth.CONFIGS[args.config]
    if args.vocab:
        import dataclasses
        cfg = dataclasses.replace(cfg, V=args.vocab)
    dt = args.dtype or cfg.dtype
    n_roll = -(-args.rows // cfg.S)
    n_roll = -(-n_roll // cfg.G) * cfg.G
    b = synth.make_batch(cfg, 0, n_roll)
    st = LearnerStep(n_rollouts=n_roll, group_size=cfg.G, max_len=cfg.S, vocab=cfg.V, dtype=dt)
    st.h2d(*[torch.from_numpy(np.ascontiguousarray(x)) for x in (b.version, b.resp_len, b.reward, b.action,
                                                                 b.old_logp, b.ref_logp)])
    info = st.pack(t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
    st.advantage()
    st.reduce_counts()
    M = min(args.rows, info.n_tokens)
    ld = (cfg.V + 7) // 8 * 8
    esize = 2 if dt == "bf16" else 4
    logits = torch.empty(M, ld, dtype=torch.bfloat16 if dt == "bf16" else torch.float32, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    bpt = 2 * cfg.V * esize + 21 + (4 if cfg.kl_coef > 0 else 0)
    names = abi.ALGO_NAMES
    ent = torch.empty(M, dtype=torch.float32, device="cuda")
    out = {"config": cfg.name, "rows": M, "bytes_per_token": bpt, "algos": {}}

    def regen():
        sgpu.fill_logits(logits, dtype=dt, vocab=cfg.V, row0=0, tok_slot=st.tok_slot, tok_action=st.tok_action,
                         kept_rollout=st.kept_rollout, kept_offset=st.kept_offset, max_len=cfg.S, seed=cfg.seed)
        flush.fill_(1.0)

    for name in args.algos.split(","):
        algo = names[name]
        shape = abi.echo_policy_loss_launch_shape(abi.ECHO_BF16 if dt == "bf16" else abi.ECHO_F32, M, cfg.V, algo)
        times = []
        for r in range(args.warmup + args.reps):
            regen()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if args.entropy > 0:
                st.loss(logits, 0, kl_coef=cfg.kl_coef, algo=algo, entropy_coef=args.entropy, tok_entropy=ent)
            else:
                st.loss(logits, 0, kl_coef=cfg.kl_coef, algo=algo)
            e1.record()
            torch.cuda.synchronize()
            if r >= args.warmup:
                times.append(e0.elapsed_time(e1))
        ms = float(np.median(times))
        out["algos"][name] = {"ms": ms, "ms_all": times, "GBps": bpt * M / ms / 1e6, "shape": shape}

    if args.streams:
        x = logits.view(-1)
        for label, fn in (("inplace_mul", lambda: x.mul_(1.0)), ("copy", lambda: flush2.copy_(x))):
            if label == "copy":
                flush2 = torch.empty_like(x)
            ts = []
            for r in range(args.warmup + args.reps):
                flush.fill_(2.0)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                if r >= args.warmup:
                    ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            out["algos"][label] = {"ms": ms, "GBps": 2 * x.numel() * 2 / ms / 1e6}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
