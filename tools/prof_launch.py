"""Host-side cost of one small echo_policy_loss_fwd_bwd call (64 Qwen-vocab rows): wall time per call over a
back-to-back loop, i.e. launch overhead through the C ABI.  Prints one JSON object."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import __graft_entry__
    __graft_entry__.build()
    import synth
    from paper_2508_05387_b200.step import LearnerStep
    cfg = synth.CONFIGS["qwen3-4b"]
    b = synth.make_batch(cfg, 0, cfg.G)
    st = LearnerStep(n_rollouts=cfg.G, group_size=cfg.G, max_len=cfg.S, vocab=cfg.V, dtype=cfg.dtype)
    st.h2d(*[torch.from_numpy(np.ascontiguousarray(getattr(b, k)))
             for k in ("version", "resp_len", "reward", "action", "old_logp", "ref_logp")])
    st.pack(t_train=synth.T_TRAIN, max_lag=cfg.max_lag)
    st.advantage()
    st.reduce_counts()
    n = 64
    logits = torch.randn(n, cfg.V, device="cuda").to(torch.bfloat16)
    for _ in range(20):
        st.loss(logits, 0, kl_coef=cfg.kl_coef)
    torch.cuda.synchronize()
    reps = 2000
    t0 = time.perf_counter()
    for _ in range(reps):
        st.loss(logits, 0, kl_coef=cfg.kl_coef)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(json.dumps({"host_us_per_call": 1e6 * (t1 - t0) / reps, "wall_us_per_call": 1e6 * (t2 - t0) / reps}))


if __name__ == "__main__":
    main()
