"""Summarise ncu captures into profiles/ (tracked).

    python tools/ncu_summary.py <report.ncu-rep> <round-tag> <workload> [kernel]
    python tools/ncu_summary.py --launches <launches.csv> <round-tag>

Writes profiles/<tag>_<kernel>_<workload>_{details,raw}.csv and merges the key
counters into profiles/ncu_summary.json, which bench.py reads for `traffic`.
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "ipc_active": "sm__inst_executed.avg.per_cycle_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex_throughput_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smem_wavefront_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "warp_inst": "smsp__inst_executed.sum",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm_cycles_active_avg": "sm__cycles_active.avg",
    "sm_cycles_active_max": "sm__cycles_active.max",
    "registers": "launch__registers_per_thread",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
         "s": 1e3}


def ncu_page(rep, page):
    return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], check=True,
                          capture_output=True, text=True).stdout


def summarise(rep, tag, workload, kernel="k_sieve"):
    raw = ncu_page(rep, "raw")
    det = ncu_page(rep, "details")
    base = f"{tag}_{kernel}_{workload}"
    open(os.path.join(PROF, base + "_raw.csv"), "w").write(raw)
    open(os.path.join(PROF, base + "_details.csv"), "w").write(det)
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {n: (un, val) for n, un, val in zip(h, u, v)}
    out = {}
    for k, m in KEYS.items():
        if m not in d:
            continue
        un, val = d[m]
        try:
            x = float(val.replace(",", ""))
        except ValueError:
            continue
        if k.startswith("dram") or k == "duration_ms":
            x *= SCALE.get(un, 1)
        out[k] = x
    out["dram_bytes"] = out.get("dram_read", 0) + out.get("dram_write", 0)
    out["report"] = os.path.basename(rep)
    out["round"] = tag
    path = os.path.join(PROF, "ncu_summary.json")
    allj = json.load(open(path)) if os.path.exists(path) else {}
    allj.setdefault(kernel, {})[workload] = out
    json.dump(allj, open(path, "w"), indent=1, sort_keys=True)
    print(json.dumps(out, indent=1))


def launches(path, tag):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        k = r[ki].split("(")[0].replace("cgpu::<unnamed>::", "").replace("void ", "")
        x = float(r[vi].replace(",", "")) * {"ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6}.get(r[ui], 1)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += x
    tot = sum(a[1] for a in agg.values())
    lines = [f"# ncu launch list ({os.path.basename(path)}), per-kernel totals, cold-cache serialised",
             f"{'kernel':62s} {'launches':>8s} {'total_us':>12s} {'share':>7s}"]
    for k, (n, t) in agg.items():
        lines.append(f"{k[:62]:62s} {n:8d} {t:12.1f} {100 * t / tot:6.1f}%")
    txt = "\n".join(lines) + "\n"
    open(os.path.join(PROF, f"{tag}_launches_summary.txt"), "w").write(txt)
    subprocess.run(["cp", path, os.path.join(PROF, f"{tag}_launches.csv")], check=True)
    print(txt)


if __name__ == "__main__":
    os.makedirs(PROF, exist_ok=True)
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        summarise(*sys.argv[1:])
