#!/usr/bin/env python
"""Benchmark of one Echo learner step (BASELINE.json metric: policy-loss fwd+bwd tokens/s and % of HBM roofline).

A step = the whole hot path over one batch of the workload on every rank: H2D of the rank's rollouts (e2e only),
(1) pack + the one 32-byte D2H that sizes the logits, (2) GRPO advantage, all-reduce of counts, then for each
micro-batch of M packed rows the fused (3)-(5) kernel over [M x V] bf16 logits in place, the statistics
reduction and its all-reduce, and the D2H of the step statistics.  The logits of each micro-batch are written
by the synthetic generator (the stand-in for the model's LM-head forward, which in a trainer produces them on
the device) OUTSIDE the timed segments, followed by a 256 MB write that flushes L2, so each kernel starts cold.

value      = kept tokens of all ranks / max-over-ranks device time of the path (inputs resident in HBM)
e2e.value  = the same through the public step API with pinned host inputs copied H2D and the statistics read
             back inside the timed region (generator time subtracted, it is not part of the method)

  python bench.py [--gpus N --steps K --warmup W] [--config qwen3-32b] [--algo auto|quad_reg|quad_reg_exact|row_l2]
  python bench.py --impl reference ...      # the CPU oracle arm (rank 0 only)

With --gpus N > 1 and no torchrun environment (WORLD_SIZE unset) the script re-executes itself under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU, NCCL).  N > 1 defaults to strong scaling
(BASELINE.json configs[4]: one Qwen3-32B-shaped batch split by rollout group over the ranks).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "policy-loss fwd+bwd tokens/sec and % HBM roofline at 1/2/4/8 B200"
DEFAULT_CONFIG = "qwen3-32b"     # BASELINE.json configs[4]: the north_star's target batch (fits one GPU: 8.4 M tokens
                                 # streamed in 32768-row micro-batches), swept over 1/2/4/8 GPUs by strong scaling
L2_FLUSH_BYTES = 256 << 20
# LM-head hidden sizes of the BASELINE.json models (f2: the fused LM-head log-prob is measured at this shape)
HIDDEN = {"tiny": 64, "qwen3-4b": 2560, "qwen2.5-7b": 3584, "qwen3-30b-a3b": 2048, "qwen3-32b": 5120}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="echo", choices=["echo", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--algo", default="auto", choices=["auto", "row_l2", "quad_reg", "quad_reg_exact", "oct_reg", "hex_reg"])
    ap.add_argument("--micro-batch", type=int, default=32768)
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N > 1: strong = one batch split over the ranks (default, BASELINE.json configs[4]); "
                         "weak = one batch per rank")
    ap.add_argument("--balance", action="store_true",
                    help="f3: token-balanced resharding of the kept rollouts after the stale filter (N > 1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-f2", action="store_true", help="skip the f2 fused LM-head measurement")
    ap.add_argument("--no-f2-train", action="store_true", help="skip the f2 training-step measurement")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU-oracle sample duration")
    return ap.parse_args()


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, D2D copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def measured_bf16_peak(sustained=False):
    """Dense bf16 tensor peak: MEASURED_PEAKS.json bf16_tflops (cuBLAS 8192^3, burst: a kernel timed alone) or
    bf16_tflops_sustained (back to back for 4 s, power-capped clocks)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    key = "bf16_tflops_sustained" if sustained else "bf16_tflops"
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)[key]), f"measured (MEASURED_PEAKS.json {key}, cuBLAS)"
    return 2250.0, "fallback (nominal dense bf16)"


def bytes_per_token(V, esize, kl):
    """Algorithmic HBM bytes per packed token of the fused kernel: read the logits row once,
    write the gradient row once, plus per-token metadata (action 4, old 4, slot 4, [ref 4], logp 4, loss 4,
    flags 1).  The adv_slot table is a few KB and stays in cache."""
    return 2 * V * esize + 21 + (4 if kl else 0)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ================================================================================= the CPU oracle (baseline arm)
def oracle_rate(cfg, rank_batch, n_tokens_total, target_s, threads=None):
    """Time the oracle (as it stands) on a bounded sample of the workload on this host's cores: the full pack +
    advantage of the batch, and the fused loss on a row sample sized to ~target_s.  Returns a dict."""
    cores = len(os.sched_getaffinity(0)) if threads is None else int(threads)
    # torchrun exports OMP_NUM_THREADS=1; the oracle is timed on all of this host's cores (read when the OpenMP
    # runtime starts, i.e. when the oracle library is first loaded)
    os.environ["OMP_NUM_THREADS"] = str(cores)
    import oracle
    import synth
    oracle.set_threads(cores)
    b = rank_batch
    t0 = time.perf_counter()
    pk = oracle.pack_batch(b.version, b.resp_len, b.action, b.old_logp, b.ref_logp, group_size=cfg.G, max_len=cfg.S,
                           vocab=cfg.V, t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
    adv, _ = oracle.group_advantage(b.reward, pk.kept_rollout, group_size=cfg.G)
    t_meta = time.perf_counter() - t0
    keys = (pk.kept_rollout[pk.tok_slot].astype(np.int64) * cfg.S
            + (np.arange(pk.n_tokens, dtype=np.int64) - pk.kept_offset[pk.tok_slot]))

    # a pool of sampled rows (numpy twin of the GPU generator; generation is not timed), evaluated repeatedly
    # until ~target_s of oracle time: the oracle's cost per row does not depend on the values
    rng = np.random.default_rng(0)
    pool = rng.integers(0, pk.n_tokens, 16 * cores)   # >= one 16-row OpenMP chunk (schedule(dynamic, 16)) per thread
    z = synth.logits_rows(keys[pool], pk.tok_action[pool], cfg.V, cfg.seed, "bf16" if cfg.dtype == "bf16" else "f32")
    tr = None if pk.tok_ref is None else pk.tok_ref[pool]
    t_loss, rows = 0.0, 0
    while t_loss < target_s or rows == 0:
        t = time.perf_counter()
        oracle.policy_loss(z, pk.tok_action[pool], pk.tok_old[pool], tr, pk.tok_slot[pool], adv,
                           n_global=pk.n_tokens, kl_coef=cfg.kl_coef)
        t_loss += time.perf_counter() - t
        rows += len(pool)
    per_row = t_loss / rows
    step_s = t_meta + per_row * n_tokens_total
    return {"tokens_per_s": n_tokens_total / step_s, "rows": rows, "t_loss": t_loss, "t_meta": t_meta,
            "cores": cores, "per_row_s": per_row, "step_s": step_s}


def reference_arm(args):
    """--impl reference: the CPU oracle on the box's host cores, rank 0 only.  Loads oracle/ and synth/ only (never
    the product library).  Each step is one bounded sample of the workload: pack + advantage of the whole batch and
    the fused loss on a row sample of ~--cpu-seconds; ms_per_step is that sample's measured wall time, `value` the
    whole-batch rate it implies (N / (t_meta + N t_row)), and the extrapolated full-batch step is reported apart."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synth
    cfg, config = run_config(synth.CONFIGS[args.config], args, args.gpus)
    b = synth.make_batch(cfg)
    n_tok = _kept_tokens(cfg, b)
    budget = max(2.0, min(args.cpu_seconds, 150.0 / max(1, args.steps + args.warmup)))
    results = []
    for i in range(args.warmup + args.steps):
        r = oracle_rate(cfg, b, n_tok, budget)
        if i >= args.warmup:
            results.append(r)
    v = statistics.median([r["tokens_per_s"] for r in results])
    r = results[-1]
    sample = (f"pack+advantage of the full {cfg.name} batch ({cfg.R} rollouts) + fused loss on {r['rows']} sampled "
              f"rows (V={cfg.V}; a pool of {16 * r['cores']} generated rows evaluated repeatedly, ~{budget:.0f} s); "
              f"value = N / (t_meta + N * t_row)")
    sample_ms = [1e3 * (x["t_meta"] + x["t_loss"]) for x in results]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.median(sample_ms),
            "ms_per_step_is": "measured wall time of one bounded oracle sample (pack + advantage of the full batch, "
                              "fused loss on the sampled rows)",
            "extrapolated_full_step_ms": 1e3 * statistics.median([x["step_s"] for x in results]),
            "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": r["cores"], "kind": "oracle", "sample": sample,
                             "cpu_model": _cpu_model()},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_config(base, args, world):
    """The workload as both arms report it (identical dicts: the driver compares them)."""
    cfg = scaled_config(base, args, world)
    return cfg, {"workload": cfg.name, "prompts": cfg.P, "group_size": cfg.G, "seq_len": cfg.S, "vocab": cfg.V,
                 "max_lag": cfg.max_lag, "kl_coef": cfg.kl_coef, "parallelism": f"dp{world}",
                 "scaling": args.scaling if world > 1 else "n/a (1 GPU)", "micro_batch_rows": args.micro_batch,
                 "l2": "inputs >> L2 (10 GB micro-batches) + 256 MB L2 flush after each generator launch"}


def scaled_config(base, args, world):
    """Weak scaling: one BASELINE batch per rank (global batch world x P prompts); strong: one batch in total."""
    import synth
    if args.scaling == "weak" and world > 1:
        return synth.Config(base.name, base.P * world, base.G, base.S, base.V, base.dtype, base.max_lag, base.kl_coef,
                            base.lag_mode, base.index, base.stale_groups * world, base.fixed_lags, base.lengths)
    return base


def _kept_tokens(cfg, b):
    import synth
    keep = (synth.T_TRAIN - b.version) <= cfg.max_lag
    return int(b.resp_len[keep].sum())


# ================================================================================= the B200 arm
def main_echo(args):
    import torch
    import torch.distributed as dist

    from paper_2508_05387_b200 import abi
    from paper_2508_05387_b200.parallel import init_from_env, shard_groups
    from paper_2508_05387_b200.step import LearnerStep
    import synth
    import synth.gpu as sgpu

    rank, world = init_from_env("nccl")
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch with torchrun, or let bench.py "
                         f"re-execute itself under torchrun by leaving WORLD_SIZE unset)")
    base = synth.CONFIGS[args.config]
    cfg, config = run_config(base, args, world)
    g0, g1 = shard_groups(cfg.P, world, rank)
    r0, r1 = g0 * cfg.G, g1 * cfg.G
    b = synth.make_batch(cfg, r0, r1)
    kl = cfg.kl_coef > 0
    host = {k: torch.from_numpy(np.ascontiguousarray(getattr(b, k))).pin_memory()
            for k in ("version", "resp_len", "reward", "action", "old_logp", "ref_logp")}
    st = LearnerStep(n_rollouts=r1 - r0, group_size=cfg.G, max_len=cfg.S, vocab=cfg.V, dtype=cfg.dtype,
                     has_ref=True, device=dev)
    M = args.micro_batch
    ld = (cfg.V + 7) // 8 * 8
    logits = torch.empty(M, ld, dtype=torch.bfloat16 if cfg.dtype == "bf16" else torch.float32, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    algo = None if args.algo == "auto" else abi.ALGO_NAMES[args.algo]
    stream = torch.cuda.current_stream()

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    plans = []

    def align():
        """Untimed rank alignment before each collective.  The synthetic logits generator (the LM-head stand-in,
        excluded from the timed work) runs ~7x longer per micro-batch than the loss kernel, so without this a rank
        with fewer tokens would wait inside the next collective for the other ranks' generator time.  With it,
        each rank's timed work is its own path work, and value = max over ranks of that."""
        if world > 1:
            torch.cuda.synchronize()
            dist.barrier()

    def one_step(record):
        t0 = ev()
        h2d = st.h2d(host["version"], host["resp_len"], host["reward"], host["action"], host["old_logp"],
                     host["ref_logp"])
        t1 = ev()
        info = st.pack(t_train=synth.T_TRAIN, max_lag=cfg.max_lag, rollout_base=r0)
        assert info.status == 0, info
        st.advantage()
        ta = ev()
        align()      # untimed: ranks enter the collectives together (see align)
        tb = ev()
        st.reduce_counts()
        if args.balance:
            plans.append(st.rebalance())
        t2 = ev()
        gens, kers = [], []
        N = st.pack_info.n_tokens
        for row0 in range(0, N, M):
            m = min(M, N - row0)
            ga = ev()
            sgpu.fill_logits(logits[:m], dtype=cfg.dtype, vocab=cfg.V, row0=row0, tok_slot=st.tok_slot,
                             tok_action=st.tok_action, kept_rollout=st.kept_rollout, kept_offset=st.kept_offset,
                             max_len=cfg.S, seed=cfg.seed)
            flush.fill_(float(row0))
            gb = ev()
            st.loss(logits[:m], row0, kl_coef=cfg.kl_coef, grad_scale=1.0, algo=algo)
            kb = ev()
            gens.append((ga, gb))
            kers.append((gb, kb))
        t3 = ev()
        align()
        t3b = ev()
        st.finish(read_back=False)
        t4 = ev()
        st.stats_host[:9].copy_(st.stats1, non_blocking=True)
        st.stats_host[9:].copy_(st.loss_stats, non_blocking=True)
        t5 = ev()
        torch.cuda.synchronize()
        if not record:
            return None
        el = lambda a, b_: a.elapsed_time(b_)
        gen_ms = sum(el(a, b_) for a, b_ in gens)
        ker = [el(a, b_) for a, b_ in kers]
        waits = el(ta, tb) + el(t3, t3b)
        return {"e2e_ms": el(t0, t5) - gen_ms - waits, "dev_ms": el(t1, ta) + el(tb, t2) + sum(ker) + el(t3b, t4),
                "kernel_ms": ker,
                "n_tokens": N, "h2d": h2d, "d2h": abi.PACK_RESULT_BYTES + st.stats_host.numel() * 8,
                "nonfinite": float(st.stats_host[9 + 4]),
                "loss": float(st.stats_host[9]) / max(float(st.stats_host[0]), 1.0)}   # sum l (all ranks) / N_global

    for _ in range(args.warmup):
        one_step(False)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = st.launches
    recs = [one_step(True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = st.launches - launches0

    dev_ms = sum(r["dev_ms"] for r in recs)
    e2e_ms = sum(r["e2e_ms"] for r in recs)
    toks = sum(r["n_tokens"] for r in recs)
    kern = [k for r in recs for k in r["kernel_ms"]]
    full = [k for r in recs for k, n in zip(r["kernel_ms"], _mb_sizes(r["n_tokens"], M)) if n == M]
    agg = torch.tensor([dev_ms, e2e_ms, float(toks), float(sum(r["nonfinite"] for r in recs))], dtype=torch.float64,
                       device=dev)
    if world > 1:
        mx = agg[:2].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = agg[2:].clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        agg = torch.cat([mx, sm])
    dev_ms, e2e_ms, toks_all, nonfinite = agg.tolist()
    if rank != 0:
        if world > 1:
            dist.barrier()
        return
    peak, peak_src = measured_peak()
    esize = 2 if cfg.dtype == "bf16" else 4
    bpt = bytes_per_token(cfg.V, esize, kl)
    avg_full = statistics.mean(full) if full else statistics.mean(kern)
    achieved = bpt * M / (avg_full * 1e-3) / 1e9
    traffic = _ncu_traffic(args)
    line = {
        "metric": METRIC, "value": toks_all / (dev_ms * 1e-3), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
        "config": config,
        "run": {"tokens_per_step": int(toks_all / args.steps), "algo": args.algo, "balance": bool(args.balance)},
        "clocks": clk,
        "e2e": {"value": toks_all / (e2e_ms * 1e-3), "unit": "tokens/s",
                "h2d_bytes_per_step": recs[0]["h2d"], "d2h_bytes_per_step": recs[0]["d2h"]},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src, "bytes_per_token": bpt,
                     "kernel": "echo_policy_loss_fwd_bwd", "kernel_ms_avg": avg_full,
                     "kernel_share_of_step": sum(kern) / sum(r["dev_ms"] for r in recs),
                     "frac_of_8TBps_nominal": achieved / 8000.0,
                     "kernel_ms_p10_p50_p90": _pct(full or kern, (10, 50, 90)),
                     "kernel_launches_timed": len(full or kern),
                     "fwd_bwd_only_tokens_per_s": M / (statistics.median(full or kern) * 1e-3) * world},
        "nonfinite_tokens": nonfinite,
        "loss": recs[-1]["loss"],
    }
    # forward-only log-probs over the same micro-batch (read-only: half the traffic)
    f1 = []
    f1_lp = torch.empty(M, dtype=torch.float32, device=dev)
    for r in range(6):
        sgpu.fill_logits(logits, dtype=cfg.dtype, vocab=cfg.V, row0=0, tok_slot=st.tok_slot, tok_action=st.tok_action,
                         kept_rollout=st.kept_rollout, kept_offset=st.kept_offset, max_len=cfg.S, seed=cfg.seed)
        flush.fill_(float(r))
        a0 = ev()
        abi.echo_token_logp(logits, st.edtype, M, cfg.V, ld, st.tok_action, f1_lp)
        a1 = ev()
        torch.cuda.synchronize()
        if r >= 2:
            f1.append(a0.elapsed_time(a1))
    f1_ms = statistics.median(f1)
    f1_bpt = cfg.V * esize + 4 + 4    # read the row once + action in + logp out
    line["f1_token_logp"] = {"ms_per_micro_batch": f1_ms, "tokens_per_s_per_gpu": M / (f1_ms * 1e-3),
                             "achieved_GBps": f1_bpt * M / (f1_ms * 1e-3) / 1e9, "bytes_per_token": f1_bpt,
                             "frac": f1_bpt * M / (f1_ms * 1e-3) / 1e9 / peak}
    # SURVEY.md §8.6 f4 loss variants on the same micro-batch: the entropy bonus (eta = 0.01, per-token entropies
    # written) and per-token advantages + sequence-mean weights (PPO-GAE style advantages, w_t = 1 / (n_seq L_i))
    ent = torch.empty(M, dtype=torch.float32, device=dev)
    gen4 = torch.Generator(device=dev).manual_seed(cfg.seed + 4)
    tok_adv = torch.randn(st.cap, generator=gen4, device=dev)
    n_seq = max(1, st.pack_info.n_rollouts_kept)
    tok_w = torch.full((st.cap,), 1.0 / (n_seq * cfg.S), dtype=torch.float32, device=dev)
    legs = {"f4_entropy": (dict(entropy_coef=0.01, tok_entropy=ent), bpt + 4,
                           "entropy bonus eta = 0.01 with tok_entropy written (+4 B/token)"),
            "f4_weights_adv": (dict(tok_adv=tok_adv, tok_weight=tok_w), bpt + 4,
                               "per-token advantages + sequence-mean weights (tok_adv and tok_weight read instead "
                               "of tok_slot: +4 B/token)")}
    plain_gbps = achieved
    for key, (kw, leg_bpt, what) in legs.items():
        ts = []
        for r in range(6):
            sgpu.fill_logits(logits, dtype=cfg.dtype, vocab=cfg.V, row0=0, tok_slot=st.tok_slot,
                             tok_action=st.tok_action, kept_rollout=st.kept_rollout, kept_offset=st.kept_offset,
                             max_len=cfg.S, seed=cfg.seed)
            flush.fill_(float(r))
            a0 = ev()
            st.loss(logits, 0, kl_coef=cfg.kl_coef, grad_scale=1.0, algo=algo, **kw)
            a1 = ev()
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(a0.elapsed_time(a1))
        ms = statistics.median(ts)
        gbps = leg_bpt * M / (ms * 1e-3) / 1e9
        line[key] = {"ms_per_micro_batch": ms, "tokens_per_s_per_gpu": M / (ms * 1e-3), "achieved_GBps": gbps,
                     "bytes_per_token": leg_bpt, "frac": gbps / peak, "vs_plain_fused_GBps": gbps / plain_gbps,
                     "variant": what}
    del ent, tok_adv, tok_w
    # the LM head fused with the log-prob (tensor-core bound), same micro-batch of tokens, against
    # the unfused path (cuBLAS GEMM into the logits buffer, then echo_token_logp)
    if cfg.dtype == "bf16" and not args.no_f2:
        hd = HIDDEN.get(base.name, 2560)
        gen = torch.Generator(device=dev).manual_seed(cfg.seed)
        hid = torch.randn(M, hd, generator=gen, device=dev).to(torch.bfloat16)
        wgt = (torch.randn(cfg.V, hd, generator=gen, device=dev) * (2.0 / hd ** 0.5)).to(torch.bfloat16)
        ws2 = torch.empty(abi.echo_lmhead_workspace_bytes(M, cfg.V) // 4 + 1, dtype=torch.float32, device=dev)
        lp2 = torch.empty(M, dtype=torch.float32, device=dev)
        f2, f2u = [], []
        for r in range(5):
            flush.fill_(float(r))
            a0 = ev()
            abi.echo_lmhead_logp(hid, wgt, M, hd, cfg.V, st.tok_action, lp2, None, ws2)
            a1 = ev()
            flush.fill_(float(r))
            b0 = ev()
            torch.matmul(hid, wgt.t(), out=logits[:, :cfg.V])
            abi.echo_token_logp(logits, st.edtype, M, cfg.V, ld, st.tok_action, f1_lp)
            b1 = ev()
            torch.cuda.synchronize()
            if r >= 2:
                f2.append(a0.elapsed_time(a1))
                f2u.append(b0.elapsed_time(b1))
        f2_ms, f2u_ms = statistics.median(f2), statistics.median(f2u)
        fl = 2.0 * M * hd * cfg.V
        pk = measured_bf16_peak()
        line["f2_lmhead_logp"] = {
            "ms_per_micro_batch": f2_ms, "tokens_per_s_per_gpu": M / (f2_ms * 1e-3), "hidden": hd,
            "roofline": {"bound": "tensor", "achieved": fl / (f2_ms * 1e-3) / 1e12, "peak": pk[0], "unit": "TFLOP/s",
                         "frac": fl / (f2_ms * 1e-3) / 1e12 / pk[0], "peak_source": pk[1],
                         "frac_of_sustained": fl / (f2_ms * 1e-3) / 1e12 / measured_bf16_peak(sustained=True)[0],
                         "flops_per_token": 2.0 * hd * cfg.V},
            "unfused_ms": f2u_ms, "unfused": "torch.matmul (cuBLAS bf16) into the logits buffer + echo_token_logp",
            "speedup_vs_unfused": f2u_ms / f2_ms}
        del ws2
        # f2 training step through the LM head (LearnerStep.loss_from_hidden), every GEMM on libecho's tcgen05 kernels,
        # against two comparison arms that call cuBLAS from this script (bench tooling only, not the library): the
        # chunked step with cuBLAS dhidden / dweight (fp32 out, dweight accumulated -- what the library did in round
        # 1) and the unfused step (cuBLAS logits into a full buffer, the fused loss kernel in place, cuBLAS backward)
        if not args.no_f2_train:
            chunk = 8192
            ldz = abi.echo_lmhead_dlogits_ld(cfg.V)
            dh = torch.empty(M, hd, dtype=torch.float32, device=dev)
            dw = torch.empty(cfg.V, hd, dtype=torch.float32, device=dev)
            dh_u = torch.empty(M, hd, dtype=torch.bfloat16, device=dev)
            dw_u = torch.empty(cfg.V, hd, dtype=torch.bfloat16, device=dev)
            zc = torch.empty(M, ldz, dtype=torch.bfloat16, device=dev)
            scratch = {}
            kl = cfg.kl_coef

            def chunked_cublas_backward(chunk=chunk):
                for r0 in range(0, M, chunk):
                    rows = min(chunk, M - r0)
                    z = zc[:rows]
                    abi.echo_lmhead_logits(hid[r0:r0 + rows], wgt, rows, hd, cfg.V, z, ldz)
                    st.loss(z, r0, kl_coef=kl, grad_scale=1.0)
                    D = z[:, :cfg.V]
                    torch.mm(D, wgt, out_dtype=torch.float32, out=dh[r0:r0 + rows])
                    if r0 == 0:
                        torch.mm(D.t(), hid[r0:r0 + rows], out_dtype=torch.float32, out=dw)
                    else:
                        torch.addmm(dw, D.t(), hid[r0:r0 + rows], out_dtype=torch.float32, out=dw)

            t2 = {"chunked": [], "chunked_16384": [], "chunked_32768": [], "recompute": [],
                  "chunked_cublas_backward": [], "chunked_cublas_backward_32768": [], "unfused_cublas": []}
            for r in range(5):
                for mode in t2:
                    flush.fill_(float(r))
                    a0 = ev()
                    if mode.startswith("chunked_") and mode[8:].isdigit():   # larger chunks: bigger GEMMs, bigger buffer
                        st.loss_from_hidden(hid, wgt, 0, dh, dw, accumulate=False, kl_coef=kl, grad_scale=1.0,
                                            chunk_rows=int(mode[8:]), scratch=scratch, mode="chunked")
                    elif mode in ("chunked", "recompute"):
                        st.loss_from_hidden(hid, wgt, 0, dh, dw, accumulate=False, kl_coef=kl, grad_scale=1.0,
                                            chunk_rows=chunk, scratch=scratch, mode=mode)
                    elif mode == "chunked_cublas_backward":
                        chunked_cublas_backward()
                    elif mode == "chunked_cublas_backward_32768":
                        chunked_cublas_backward(M)
                    else:
                        torch.matmul(hid, wgt.t(), out=logits[:, :cfg.V])
                        st.loss(logits, 0, kl_coef=kl, grad_scale=1.0)
                        torch.matmul(logits[:, :cfg.V], wgt, out=dh_u)     # dh = D W, dW = D^T h (bf16 outputs)
                        torch.matmul(logits[:, :cfg.V].t(), hid, out=dw_u)
                    a1 = ev()
                    torch.cuda.synchronize()
                    if r >= 2:
                        t2[mode].append(a0.elapsed_time(a1))
            ms = {k: statistics.median(v) for k, v in t2.items()}
            t2_ms = ms["chunked"]
            fl6 = 6.0 * M * hd * cfg.V
            line["f2_train_step"] = {
                "ms_per_micro_batch": t2_ms, "tokens_per_s_per_gpu": M / (t2_ms * 1e-3), "hidden": hd,
                "mode": "chunked (echo_lmhead_policy_loss_fwd_bwd)", "chunk_rows": chunk,
                "chunk_buffer_GB": chunk * cfg.V * 2 / 1e9,
                "roofline": {"bound": "tensor", "achieved": fl6 / (t2_ms * 1e-3) / 1e12, "peak": pk[0],
                             "unit": "TFLOP/s", "frac": fl6 / (t2_ms * 1e-3) / 1e12 / pk[0], "peak_source": pk[1],
                             "frac_of_sustained": fl6 / (t2_ms * 1e-3) / 1e12 / measured_bf16_peak(sustained=True)[0],
                             "flops_per_token": 6.0 * hd * cfg.V},
                "gemms": "logits GEMM, fused loss, dhidden and dweight all on libecho's kernels (tcgen05, no cuBLAS)",
                "chunk_rows_sweep_ms": {"8192": t2_ms, "16384": ms["chunked_16384"], "32768": ms["chunked_32768"]},
                "recompute_ms": ms["recompute"],
                "recompute": "echo_lmhead_logp + echo_loss_from_logp + echo_lmhead_backward (D recomputed: 8 d V "
                             "flops per token)",
                "chunked_cublas_backward_ms": ms["chunked_cublas_backward"],
                "chunked_cublas_backward": "comparison: the same chunked step with dhidden / dweight in cuBLAS "
                                           "(torch.mm / addmm, fp32 out, dweight accumulated)",
                "vs_chunked_cublas_backward": ms["chunked_cublas_backward"] / t2_ms,
                "chunked_cublas_backward_32768_ms": ms["chunked_cublas_backward_32768"],
                "chunked_32768_vs_cublas_backward_32768": ms["chunked_cublas_backward_32768"] / ms["chunked_32768"],
                "unfused_ms": ms["unfused_cublas"],
                "unfused": f"comparison: cuBLAS logits ({M * cfg.V * 2 / 1e9:.1f} GB buffer) + echo_policy_loss_fwd_bwd "
                           "in place + cuBLAS dh, dW (bf16 out)",
                "speedup_vs_unfused": ms["unfused_cublas"] / t2_ms}
            del dh, dw, dh_u, dw_u, scratch, zc
        del hid, wgt
    if plans:
        line["run"]["tokens_per_rank_before"] = plans[-1]["tokens_before"]
        line["run"]["tokens_per_rank_after"] = plans[-1]["tokens_after"]
    if world == 1 and not args.no_cpu_baseline:
        r = oracle_rate(cfg, b, toks_all / args.steps, args.cpu_seconds)
        r1 = oracle_rate(cfg, b, toks_all / args.steps, args.cpu_seconds / 4, threads=1)
        line["cpu_baseline"] = {
            "single_thread_tokens_per_s": r1["tokens_per_s"],
            "value": r["tokens_per_s"], "unit": "tokens/s", "cores": r["cores"], "kind": "oracle",
            "cpu_model": _cpu_model(),
            "sample": f"pack+advantage of the full batch + fused loss on {r['rows']} rows (a pool of {16 * r['cores']} sampled rows, repeated) "
                      f"({r['t_loss']:.1f} s); step extrapolated as t_meta + N * t_row"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()


def _pct(xs, ps):
    xs = sorted(xs)
    return [xs[min(len(xs) - 1, int(round(p / 100 * (len(xs) - 1))))] for p in ps]


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _mb_sizes(N, M):
    return [min(M, N - r) for r in range(0, N, M)]


def _ncu_traffic(args):
    """dram bytes per launch from the committed ncu --set full capture of this workload, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(f"{args.config}/{args.algo}") or d.get(args.config)
        return None if e is None else e.get("bytes_per_launch_at_M32768")
    except Exception:
        return None


def _reexec_under_torchrun(args):
    """--gpus N > 1 without a torchrun environment: run N ranks (one per GPU) of this same command line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    print(f"bench.py: re-executing under torchrun ({args.gpus} ranks)", file=sys.stderr, flush=True)
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.impl == "reference":
        # the oracle arm builds and loads oracle/ and synth/ only -- never the product library
        import oracle
        oracle.build()
        reference_arm(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _reexec_under_torchrun(args)
    # rank count visible in the NCCL init log (the driver counts ranks from it), on stderr so stdout keeps the JSON
    if os.environ.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
        os.environ["NCCL_DEBUG"] = "INFO"
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    import __graft_entry__
    __graft_entry__.build()
    main_echo(args)
    try:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()
    except Exception:
        pass


if __name__ == "__main__":
    main()
