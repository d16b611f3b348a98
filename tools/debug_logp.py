"""Debug: f1 warp kernel vs cluster tile vs oracle at large vocabularies; prints the worst rows."""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import __graft_entry__
    __graft_entry__.build()
    import oracle
    import synth
    from paper_2508_05387_b200 import abi
    from test_gpu_parity import device_step, fill, as_oracle_rows
    from _util import oracle_step
    for V in (200003, 311296, 262144, 151936):
        cfg = dataclasses.replace(synth.CONFIGS["qwen3-4b"], V=V)
        b = synth.make_batch(cfg, 0, cfg.G)
        st, info = device_step(cfg, b)
        o = oracle_step(cfg, b)
        n = 48
        ld = (V + 7) // 8 * 8
        logits = fill(st, cfg, 0, n, ld=ld)
        z = as_oracle_rows(logits)[:, :V]
        res = {}
        for env in ("0", "1"):
            os.environ["ECHO_LOGP_CLUSTER"] = env
            lp = torch.full((n,), float("nan"), device="cuda")
            lse = torch.full((n,), float("nan"), device="cuda")
            abi.echo_token_logp(logits, abi.ECHO_BF16, n, V, ld, st.tok_action, lp, lse)
            torch.cuda.synchronize()
            res[env] = (lp.cpu().numpy().astype(np.float64), lse.cpu().numpy().astype(np.float64))
        lp_ref, lse_ref, _ = oracle.token_logp(z, o.pk.tok_action[:n], vocab=V, dtype=oracle.BF16)
        for env, (lp, lse) in res.items():
            err = np.abs(lp - lp_ref)
            i = int(np.nanargmax(err))
            print(f"V={V} cluster={env}: max|dlogp| {np.nanmax(err):.3e} row {i} nan {int(np.isnan(lp).sum())} "
                  f"lse {lse[i]:.6f} ref {lse_ref[i]:.6f} logp {lp[i]:.6f} ref {lp_ref[i]:.6f} a {o.pk.tok_action[i]}")


if __name__ == "__main__":
    main()
