#!/usr/bin/env python3
"""Summarise one `ncu --set full --import-source on` capture into markdown
(run here on the CPU box): headline metrics, issue-stall reasons, and the SASS
opcode mix weighted by executed instructions.

  python scripts/ncu_kernel_summary.py gpurun_out/int4_full.ncu-rep profiles/r01_int4_ncu.md "title"
"""
import collections, csv, io, subprocess, sys

rep, out, title = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Issue Slots Busy",
        "Executed Ipc Active", "Achieved Occupancy", "Active Warps Per Scheduler",
        "Eligible Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Registers Per Thread", "Executed Instructions", "L2 Hit Rate", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block"]
lines = [f"# {title}", "", f"Source: `{rep}` (ncu --set full --clock-control none --import-source on; "
         "times under ncu are cold-cache and serialised).", ""]
rows = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
hdr = rows[0]
seen = collections.OrderedDict()
for r in rows[1:]:
    d = dict(zip(hdr, r))
    k = (d.get("Kernel Name", "")[:60], d.get("ID", ""))
    if d.get("Metric Name") in WANT:
        seen.setdefault(k, []).append((d["Metric Name"], d["Metric Value"], d.get("Metric Unit", "")))
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
rh = raw[0]
for ki, (k, ms) in enumerate(seen.items()):
    lines += [f"## `{k[0]}` (launch id {k[1]})", "", "| metric | value |", "|---|---|"]
    lines += [f"| {n} | {v} {u} |" for n, v, u in ms]
    if ki + 2 < len(raw):
        d = dict(zip(rh, raw[ki + 2]))
        st = []
        for h in rh:
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    v = float(d[h].replace(",", ""))
                except ValueError:
                    continue
                if v > 0.05:
                    st.append((v, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        for h in ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                  "dram__bytes_read.sum", "dram__bytes_write.sum"):
            if h in d:
                lines.append(f"| {h} | {d[h]} |")
        lines += ["", "Issue-stall reasons (warps stalled per issued instruction):", ""]
        lines += [f"- {n}: {v:.2f}" for v, n in sorted(st, reverse=True)]
    lines.append("")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
if len(src) > 2:
    h = src[1]
    i_s, i_e = h.index("Source"), h.index("Instructions Executed")
    op = collections.Counter()
    tot = 0
    for r in src[2:]:
        try:
            e = int(r[i_e])
        except (ValueError, IndexError):
            continue
        t = r[i_s].split()
        if not t:
            continue
        o = (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]
        op[o] += e
        tot += e
    lines += [f"SASS opcode mix of the first captured kernel ({tot} warp instructions):", "",
              "| opcode | share |", "|---|---|"]
    lines += [f"| {o} | {100 * c / tot:.1f} % |" for o, c in op.most_common(16)]
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:60]))
