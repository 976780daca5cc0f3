#!/usr/bin/env python3
"""Summarise ncu evidence into profiles/ (run here, on the CPU box).

  python scripts/ncu_summary.py gpurun_out/launches.csv gpurun_out/decode_full.ncu-rep r01

writes profiles/<tag>_launches.csv (copy), profiles/<tag>_ncu_summary.md and
profiles/ncu_summary.json (read by bench.py for roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smsp__inst_executed.sum",
    "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e-6, "us": 1e-6, "ns": 1e-9, "ms": 1e-3,
         "msecond": 1e-3, "nsecond": 1e-9, "second": 1.0}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
    per = collections.OrderedDict()
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "")
        per.setdefault(name, []).append(float(r[14].replace(",", "")))
    return per


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    res = []
    for r in rows[2:]:
        d = {"kernel": r[idx["Kernel Name"]]}
        for m in METRICS:
            if m in idx:
                v = r[idx[m]].replace(",", "")
                try:
                    d[m] = float(v) * SCALE.get(units[idx[m]], 1.0)
                except ValueError:
                    d[m] = v
        res.append(d)
    return res


def main():
    lpath, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    os.makedirs(PROF, exist_ok=True)
    shutil.copy(lpath, os.path.join(PROF, f"{tag}_launches.csv"))
    per = launches(lpath)
    fr = full(rep)
    lines = [f"# ncu summary ({tag})", "",
             "Command: `ncu --metrics gpu__time_duration.sum --clock-control none` over one "
             "`bench.py --profile` step (cold, serialised launches) and one "
             "`ncu --set full` capture of the first two K2 launches (layer 0 FP16, FP8). "
             "In --profile mode the kv_append launches are the 32-layer prefill (setup); the "
             "decode step itself is one fused paged_decode launch per layer and model.", "",
             "## Launch list (per kernel family)", "",
             "| kernel | launches | mean us | min us | max us | share of listed time |",
             "|---|---|---|---|---|---|"]
    tot = sum(sum(v) for v in per.values())
    for k, v in per.items():
        lines.append(f"| `{k}` | {len(v)} | {sum(v)/len(v)/1e3:.2f} | {min(v)/1e3:.2f} | "
                     f"{max(v)/1e3:.2f} | {sum(v)/tot:.1%} |")
    lines += ["", "## Full capture", ""]
    summary = {}
    for d in fr:
        lines.append(f"### `{d['kernel'][:90]}`")
        lines.append("")
        for m in METRICS:
            if m in d:
                lines.append(f"- {m}: {d[m]:.4g}" if isinstance(d[m], float) else f"- {m}: {d[m]}")
        rb, wb = d.get("dram__bytes_read.sum", 0.0), d.get("dram__bytes_write.sum", 0.0)
        dur = d.get("gpu__time_duration.sum", 0.0)
        lines.append(f"- DRAM traffic per launch: {(rb + wb)/1e6:.2f} MB; "
                     f"DRAM GB/s (cold, under ncu): {(rb + wb)/dur/1e9:.0f}")
        lines.append("")
        key = "decode_fp16" if "<0," in d["kernel"] or "(int)0," in d["kernel"] else (
            "decode_fp8" if "<1," in d["kernel"] or "(int)1," in d["kernel"] else d["kernel"])
        summary[key] = {"kernel": d["kernel"], "dram_bytes_per_launch": rb + wb,
                        "duration_s": dur, "tag": tag}
    open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    json.dump(summary, open(os.path.join(PROF, "ncu_summary.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
