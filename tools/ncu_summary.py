"""Summarise an ncu report (or a --metrics launch-list CSV) for profiles/.

    python tools/ncu_summary.py gpurun_out/fwd_jit1.ncu-rep profiles/r1_fwd_jit.md --title "..."
    python tools/ncu_summary.py --launches gpurun_out/launches.csv profiles/r1_launches.md
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe % of peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % of peak"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active % (per SMSP)"),
    ("sm__inst_executed.sum.per_cycle_active", "warp-instructions / cycle (all SMs)"),
    ("sm__inst_executed.sum", "warp-instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % of peak"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall: wait / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall: short scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall: not selected / issue"),
    ("smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio", "stall: no instruction / issue"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall: long scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall: math pipe throttle / issue"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        kernels.append(d)
    return kernels


def summarise(path, dst, title):
    ks = raw(path)
    lines = [f"# {title}", "", f"Source: `{path}` (ncu --set full --clock-control none), "
             f"{len(ks)} kernel(s) captured.", ""]
    js = []
    for d in ks:
        name = d.get("Kernel Name", ("?", ""))[0]
        lines += [f"## `{name[:120]}`", "", "| metric | value |", "|---|---|"]
        rec = {"kernel": name}
        for key, label in KEYS:
            if key in d:
                v, u = d[key]
                lines.append(f"| {label} (`{key}`) | {v} {u} |")
                rec[key] = v
        js.append(rec)
        lines.append("")
    with open(dst, "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(dst.rsplit(".", 1)[0] + ".json", "w") as f:
        json.dump(js, f, indent=1)


def launches(path, dst, title):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = {}
    cnt = {}
    for r in rows[start + 1:]:
        if len(r) <= max(ki, vi):
            continue
        k = r[ki].split("(")[0][:80]
        tot[k] = tot.get(k, 0.0) + float(r[vi].replace(",", ""))
        cnt[k] = cnt.get(k, 0) + 1
    s = sum(tot.values())
    lines = [f"# {title}", "", f"Source: `{path}` (ncu --metrics gpu__time_duration.sum; cold-cache, "
             "serialised: compare shares, not absolutes).", "",
             "| kernel | launches | total | share |", "|---|---|---|---|"]
    for k in sorted(tot, key=lambda x: -tot[x]):
        lines.append(f"| `{k}` | {cnt[k]} | {tot[k]:.1f} | {100 * tot[k] / s:.1f}% |")
    with open(dst, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("dst")
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--launches", action="store_true")
    a = ap.parse_args()
    (launches if a.launches else summarise)(a.src, a.dst, a.title)
