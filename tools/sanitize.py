#!/usr/bin/env python
"""Small invocation of every libecho kernel for compute-sanitizer (one tool per run): tiny fp32 step (row kernel),
a few Qwen-vocab bf16 rows through the quad kernel (both modes) and the forward-only path, ragged vocab."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import synth
    import synth.gpu as sgpu
    from paper_2508_05387_b200 import abi
    from paper_2508_05387_b200.step import LearnerStep
    for name, rows, algos in (("tiny", None, [None]), ("qwen3-4b", 40, [abi.ECHO_ALGO_QUAD_REG,
                                                                        abi.ECHO_ALGO_QUAD_REG_EXACT,
                                                                        abi.ECHO_ALGO_ROW_L2])):
        cfg = synth.CONFIGS[name]
        P = cfg.P if name == "tiny" else 2
        b = synth.make_batch(cfg, 0, P * cfg.G, lengths="ragged")
        st = LearnerStep(n_rollouts=P * cfg.G, group_size=cfg.G, max_len=cfg.S, vocab=cfg.V, dtype=cfg.dtype)
        st.h2d(*[torch.from_numpy(np.ascontiguousarray(x)) for x in (b.version, b.resp_len, b.reward, b.action,
                                                                     b.old_logp, b.ref_logp)])
        info = st.pack(t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
        st.advantage()
        st.reduce_counts()
        n = info.n_tokens if rows is None else min(rows, info.n_tokens)
        dt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
        for algo in algos:
            logits = torch.empty(n, cfg.V, dtype=dt, device="cuda")
            sgpu.fill_logits(logits, dtype=cfg.dtype, vocab=cfg.V, row0=0, tok_slot=st.tok_slot,
                             tok_action=st.tok_action, kept_rollout=st.kept_rollout, kept_offset=st.kept_offset,
                             max_len=cfg.S, seed=cfg.seed)
            lp = torch.empty(n, device="cuda")
            abi.echo_token_logp(logits, st.edtype, n, cfg.V, cfg.V, st.tok_action, lp)
            st.loss(logits, 0, kl_coef=cfg.kl_coef, algo=algo)
        st.finish()
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
