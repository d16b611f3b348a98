"""Summarise the ncu outputs of tools/gpu_round.sh into profiles/.

    python tools/ncu_summary.py TAG [--src gpurun_out] [--dst profiles]

Reads  SRC/TAG_launches.csv  (ncu --metrics gpu__time_duration.sum --csv over bench.py)
       SRC/TAG_kernel.ncu-rep (ncu --set full of one fused-kernel launch)
Writes DST/TAG_ncu_launches.csv, DST/TAG_launch_summary.md, DST/TAG_kernel.ncu-rep,
       DST/TAG_ncu_kernel_details.csv, DST/TAG_ncu_kernel_metrics.json, and the DRAM traffic per launch into
       DST/ncu_traffic.json (read by bench.py for roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import os
import shutil
import subprocess

METRICS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum",
]
STALLS = ["wait", "barrier", "selected", "no_instructions", "not_selected", "short_scoreboard", "math_pipe_throttle",
          "long_scoreboard", "mio_throttle", "branch_resolving", "membar", "dispatch_stall", "lg_throttle", "sleeping",
          "drain", "imc_miss", "tex_throttle", "misc"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def launch_summary(src_csv, dst_md):
    lines = open(src_csv).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        ns *= {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r["Metric Unit"], 1)
        tot[r["Kernel Name"]] += ns
        cnt[r["Kernel Name"]] += 1
    all_ns = sum(tot.values())
    echo_ns = sum(v for k, v in tot.items() if "echo::" in k)
    out = ["# ncu launch list (bench.py --steps 1 --warmup 1 --no-cpu-baseline, cold/serialised per-launch times, us)", "",
           "| kernel | launches | total us | share of all | share of libecho |", "|---|---|---|---|---|"]
    for k, v in tot.most_common():
        mine = f"{100 * v / echo_ns:.2f}%" if "echo::" in k else "—"
        out.append(f"| `{k[:70]}` | {cnt[k]} | {v / 1e3:.1f} | {100 * v / all_ns:.2f}% | {mine} |")
    # the learner steps alone: every launch before the first forward-only (logp-mode, `, 2>`) launch, which starts
    # the f1 / f2 side measurements bench.py runs after its timed steps
    ids = []
    for r in rows:
        if r["Metric Name"] == "gpu__time_duration.sum":
            ids.append((int(r["ID"]), r["Kernel Name"], r["Metric Value"], r["Metric Unit"]))
    ids.sort()
    cut = next((i for i, (_, k, _, _) in enumerate(ids)
                if "token_logp_warp" in k or ("policy_loss" in k and ", 2>" in k)), len(ids))
    st, sc = collections.Counter(), collections.Counter()
    for _, k, v, u in ids[:cut]:
        ns = float(v.replace(",", "")) * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(u, 1)
        st[k] += ns
        sc[k] += 1
    step_echo = sum(v for k, v in st.items() if "echo::" in k)
    out += ["", "## Learner steps only (launches before the post-step f1 / f2 measurements; warm-up + timed steps)", "",
            "| kernel | launches | total us | share of libecho in the steps |", "|---|---|---|---|"]
    for k, v in st.most_common():
        if "echo::" in k:
            out.append(f"| `{k[:70]}` | {sc[k]} | {v / 1e3:.1f} | {100 * v / step_echo:.2f}% |")
    open(dst_md, "w").write("\n".join(out) + "\n")


def kernel_metrics(rep, dst_json, dst_details):
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    m = {w: [vals[hdr.index(w)], units[hdr.index(w)]] for w in METRICS if w in hdr}
    st = {}
    for s in STALLS:
        key = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
        if key in hdr:
            st[s] = float(vals[hdr.index(key)].replace(",", ""))
    if st:
        tot = sum(st.values())
        m["stall_share_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])
                                if 100 * v / tot >= 1.0}
    json.dump(m, open(dst_json, "w"), indent=1)
    open(dst_details, "w").write(ncu("-i", rep, "--page", "details", "--csv"))
    return m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--src", default="gpurun_out")
    ap.add_argument("--dst", default="profiles")
    ap.add_argument("--workload", default="qwen3-32b")
    ap.add_argument("--rows", type=int, default=32768)
    a = ap.parse_args()
    t = a.tag
    shutil.copy(os.path.join(a.src, f"{t}_launches.csv"), os.path.join(a.dst, f"{t}_ncu_launches.csv"))
    launch_summary(os.path.join(a.src, f"{t}_launches.csv"), os.path.join(a.dst, f"{t}_launch_summary.md"))
    rep = os.path.join(a.dst, f"{t}_kernel.ncu-rep")
    shutil.copy(os.path.join(a.src, f"{t}_kernel.ncu-rep"), rep)
    m = kernel_metrics(rep, os.path.join(a.dst, f"{t}_ncu_kernel_metrics.json"),
                       os.path.join(a.dst, f"{t}_ncu_kernel_details.csv"))
    gb = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}
    rd = float(m["dram__bytes_read.sum"][0]) * gb[m["dram__bytes_read.sum"][1]]
    wr = float(m["dram__bytes_write.sum"][0]) * gb[m["dram__bytes_write.sum"][1]]
    path = os.path.join(a.dst, "ncu_traffic.json")
    tr = json.load(open(path)) if os.path.exists(path) else {}
    tr[f"{a.workload}/auto"] = {f"bytes_per_launch_at_M{a.rows}": int(rd + wr), "kernel": m["Kernel Name"][0],
                                "source": f"profiles/{t}_ncu_kernel_metrics.json: dram__bytes_read.sum + "
                                          "dram__bytes_write.sum (ncu --set full, 1 launch)"}
    json.dump(tr, open(path, "w"), indent=1)
    print(json.dumps(m, indent=1))
    # the f2 captures (tensor-core kernels): the fused LM-head log-prob and the logits-store GEMM of the chunked step
    for name in ("f1", "f2", "f2_logits", "gemm_dh", "gemm_dw"):
        src = os.path.join(a.src, f"{t}_{name}.ncu-rep")
        if not os.path.exists(src):
            continue
        rep = src
        if not name.startswith("gemm"):   # the GEMM reports stay in the scratch dir (size); their metrics are kept
            rep = os.path.join(a.dst, f"{t}_{name}.ncu-rep")
            shutil.copy(src, rep)
        raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
        hdr, units, vals = raw[0], raw[1], raw[2]
        keys = METRICS + ["sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
                          "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
                          "lts__t_bytes.sum", "sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_active"]
        mm = {w: [vals[hdr.index(w)], units[hdr.index(w)]] for w in keys if w in hdr}
        mm.update({h: [vals[i], units[i]] for i, h in enumerate(hdr) if "tensor" in h and "pct" in h})
        st = {}
        for stall in STALLS:
            key = f"smsp__average_warps_issue_stalled_{stall}_per_issue_active.ratio"
            if key in hdr:
                st[stall] = float(vals[hdr.index(key)].replace(",", "") or 0)
        if st and sum(st.values()) > 0:
            tot = sum(st.values())
            mm["stall_share_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])
                                     if 100 * v / tot >= 1.0}
        json.dump(mm, open(os.path.join(a.dst, f"{t}_ncu_{name}_metrics.json"), "w"), indent=1)
        print(name, json.dumps(mm, indent=1))


if __name__ == "__main__":
    main()
