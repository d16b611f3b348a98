"""f1 timing: echo_token_logp (forward-only log-probs) on one Qwen-shaped micro-batch (L2 flushed per launch)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402


def main():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2508_05387_b200 import abi
    n, V = 32768, 151936
    g = torch.Generator(device="cuda").manual_seed(0)
    logits = (torch.randn(n, V, generator=g, device="cuda") * 2).to(torch.bfloat16)
    act = torch.randint(0, V, (n,), generator=g, device="cuda", dtype=torch.int32)
    lp = torch.empty(n, device="cuda")
    flush = torch.empty(64 << 20, device="cuda")
    ts = []
    for r in range(8):
        flush.fill_(float(r))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        abi.echo_token_logp(logits, abi.ECHO_BF16, n, V, V, act, lp)
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(json.dumps({"token_logp_ms": ts[len(ts) // 2], "all": ts, "GBps": n * (2 * V + 8) / ts[len(ts) // 2] / 1e6}))


if __name__ == "__main__":
    main()
