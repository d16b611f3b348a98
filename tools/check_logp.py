"""f1 sanity for A/B builds: echo_token_logp against the fused kernel's tok_logp on the same bf16 logits
(different launch shapes, same quantity): prints the max |difference| and the f1 time."""
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
    n, V = 4096, 151936
    g = torch.Generator(device="cuda").manual_seed(1)
    logits = (torch.randn(n, V, generator=g, device="cuda") * 2).to(torch.bfloat16)
    act = torch.randint(0, V, (n,), generator=g, device="cuda", dtype=torch.int32)
    lp = torch.empty(n, device="cuda")
    lse = torch.empty(n, device="cuda")
    abi.echo_token_logp(logits, abi.ECHO_BF16, n, V, V, act, lp, lse)
    old = torch.zeros(n, device="cuda")
    slot = torch.zeros(n, dtype=torch.int32, device="cuda")
    adv = torch.ones(1, device="cuda")
    ng = torch.tensor([float(n)], dtype=torch.float64, device="cuda")
    lp2, loss = torch.empty(n, device="cuda"), torch.empty(n, device="cuda")
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    abi.echo_policy_loss_fwd_bwd(logits.clone(), abi.ECHO_BF16, n, V, V, act, old, None, slot, adv, ng, 0.2, 0.2, 0.0,
                                 1.0, lp2, loss, flags)
    torch.cuda.synchronize()
    print(json.dumps({"max_abs_diff_logp": (lp - lp2).abs().max().item(), "finite": bool(torch.isfinite(lp).all())}))


if __name__ == "__main__":
    main()
