"""Multi-GPU check of f3 token-balanced resharding (run under torchrun, NCCL):

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
        tools/check_rebalance.py [--config qwen2.5-7b] [--scaling strong]

Every rank runs the same step twice on its shard of the batch: as packed, and after LearnerStep.rebalance().
Rank 0 checks that the per-token log-probs and losses of every global token (keyed by rollout id and
position) are bit-identical between the two runs, that the all-reduced statistics agree, and that the
rebalanced token counts are within one rollout of N_global / W.  Prints one JSON line (tokens per rank before
and after, max/mean imbalance) and exits non-zero on a mismatch.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="qwen2.5-7b")
    ap.add_argument("--micro-batch", type=int, default=32768)
    ap.add_argument("--max-rows", type=int, default=0, help="score only the first rows of each rank (0 = all)")
    args = ap.parse_args()
    import __graft_entry__
    __graft_entry__.build()
    import synth
    import synth.gpu as sgpu
    from paper_2508_05387_b200.parallel import init_from_env, shard_groups
    from paper_2508_05387_b200.step import LearnerStep

    rank, world = init_from_env("nccl")
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    cfg = synth.CONFIGS[args.config]
    g0, g1 = shard_groups(cfg.P, world, rank)
    r0, r1 = g0 * cfg.G, g1 * cfg.G
    b = synth.make_batch(cfg, r0, r1)
    st = LearnerStep(n_rollouts=r1 - r0, group_size=cfg.G, max_len=cfg.S, vocab=cfg.V, dtype=cfg.dtype, device=dev)
    M = args.micro_batch
    logits = torch.empty(M, (cfg.V + 7) // 8 * 8, dtype=torch.bfloat16, device=dev)

    def run(balance):
        st.h2d(*[torch.from_numpy(np.ascontiguousarray(getattr(b, k)))
                 for k in ("version", "resp_len", "reward", "action", "old_logp", "ref_logp")])
        info = st.pack(t_train=synth.T_TRAIN, max_lag=cfg.max_lag, rollout_base=r0)
        assert info.status == 0, info
        st.advantage()
        st.reduce_counts()
        plan = None
        if balance:
            extra = st.tok_old[: st.pack_info.n_tokens].clone()      # an extra per-token array rides along
            plan = st.rebalance(extra_tokens=[extra])
            assert torch.equal(plan["extra"][0], st.tok_old[: st.pack_info.n_tokens]), "extra_tokens mismatch"
        N = st.pack_info.n_tokens if not args.max_rows else min(args.max_rows, st.pack_info.n_tokens)
        for row0 in range(0, N, M):
            m = min(M, N - row0)
            sgpu.fill_logits(logits[:m], dtype=cfg.dtype, vocab=cfg.V, row0=row0, tok_slot=st.tok_slot,
                             tok_action=st.tok_action, kept_rollout=st.kept_rollout, kept_offset=st.kept_offset,
                             max_len=cfg.S, seed=cfg.seed)
            st.loss(logits[:m], row0, kl_coef=cfg.kl_coef)
        out = st.finish() if not args.max_rows else None
        n_r, n_t = st.pack_info.n_rollouts_kept, st.pack_info.n_tokens
        off = st.kept_offset[: n_r + 1].cpu().numpy()
        kr = st.kept_rollout[:n_r].cpu().numpy().astype(np.int64)
        slot = np.repeat(np.arange(n_r), np.diff(off))
        keys = (kr[slot] * cfg.S + (np.arange(n_t) - off[slot]))[:N]
        return plan, out, keys, st.tok_logp[:N].cpu().numpy().copy(), st.tok_loss[:N].cpu().numpy().copy()

    plan0, out0, k0, lp0, ls0 = run(False)
    plan1, out1, k1, lp1, ls1 = run(True)
    gathered = [None] * world
    dist.all_gather_object(gathered, (k0, lp0, ls0, k1, lp1, ls1))
    ok = True
    line = {}
    if rank == 0:
        K0 = np.concatenate([g[0] for g in gathered]); K1 = np.concatenate([g[3] for g in gathered])
        o0, o1 = np.argsort(K0), np.argsort(K1)
        same_keys = np.array_equal(K0[o0], K1[o1]) if not args.max_rows else True
        if not args.max_rows:
            lp_eq = np.array_equal(np.concatenate([g[1] for g in gathered])[o0].view(np.uint32),
                                   np.concatenate([g[4] for g in gathered])[o1].view(np.uint32))
            ls_eq = np.array_equal(np.concatenate([g[2] for g in gathered])[o0].view(np.uint32),
                                   np.concatenate([g[5] for g in gathered])[o1].view(np.uint32))
            s0, s1 = np.array([out0[k] for k in sorted(out0)]), np.array([out1[k] for k in sorted(out1)])
            stats_close = bool(np.allclose(s0, s1, rtol=1e-9, atol=1e-9))
        else:
            lp_eq = ls_eq = stats_close = True
        after, before = plan1["tokens_after"], plan1["tokens_before"]
        Ng = sum(after)
        bound_ok = max(after) <= Ng / world + cfg.S
        ok = same_keys and lp_eq and ls_eq and stats_close and bound_ok
        line = {"check": "f3 rebalance", "config": cfg.name, "world": world, "ok": bool(ok),
                "tokens_before": before, "tokens_after": after,
                "imbalance_before": max(before) / (Ng / world), "imbalance_after": max(after) / (Ng / world),
                "same_tokens": bool(same_keys), "logp_bit_identical": bool(lp_eq), "loss_bit_identical": bool(ls_eq),
                "stats_close": stats_close}
        print(json.dumps(line), flush=True)
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.broadcast(flag, 0)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if int(flag) else 1)


if __name__ == "__main__":
    main()
