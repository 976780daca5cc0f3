#!/usr/bin/env python3
"""Summarise the r02 ncu evidence (scripts/gpu_profile.sh) into profiles/:
the c4 launch list (per kernel family), one --set full capture per K2 / K1
format at the c4 shape, and profiles/ncu_summary.json keyed
'<workload>_decode_<fmt>' / '<workload>_k1_<fmt>' (bench.py reads
roofline.traffic from it).  Run here, on the CPU box:

  python scripts/ncu_profiles_r02.py gpurun_out r02
"""
import collections, csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
FMTS = ["fp16", "fp8", "int8", "int4"]
MET = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__warps_active.avg.per_cycle_active",
       "smsp__warps_eligible.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
       "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct"]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e-6, "nsecond": 1e-9, "us": 1e-6, "ns": 1e-9, "ms": 1e-3,
         "msecond": 1e-3, "second": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    r = rows[2]
    d = {"kernel": r[idx["Kernel Name"]]}
    for m in MET:
        if m in idx:
            try:
                d[m] = float(r[idx[m]].replace(",", "")) * SCALE.get(units[idx[m]], 1.0)
            except ValueError:
                pass
    return d


def main():
    src, tag = sys.argv[1], sys.argv[2]
    lines = [f"# {tag}: ncu evidence at the c4 shape (bench.py --profile)", "",
             "Launch list: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
             "--clock-control none` over `bench.py --profile` (admission K1 of the four models' prompts, then "
             "eager decode steps at B = 64: one fused K1+K2 launch + merge per layer and model).  Cold, "
             "serialised launches: shares and traffic, never bench values.", "",
             "| kernel | launches | mean us | share of listed time | DRAM MB per launch |", "|---|---|---|---|---|"]
    per = collections.OrderedDict()
    for r in csv.reader(open(os.path.join(src, "launches_c4.csv"))):
        if len(r) > 14 and r[12] in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"):
            k = (r[4].split("(")[0].replace("void ", ""), r[0])
            per.setdefault(k, {})[r[12]] = float(r[14].replace(",", "")) * SCALE.get(r[13], 1.0)
    fam = collections.OrderedDict()
    for (name, _), d in per.items():
        fam.setdefault(name, []).append(d)
    tot = sum(d.get("gpu__time_duration.sum", 0) for v in fam.values() for d in v)
    for name, v in fam.items():
        t = [d.get("gpu__time_duration.sum", 0) for d in v]
        b = [d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in v]
        lines.append(f"| `{name}` | {len(v)} | {sum(t)/len(t)*1e6:.2f} | {sum(t)/tot:.1%} | {sum(b)/len(b)/1e6:.1f} |")
    lines += ["", "## Full captures (first launch of each format; `ncu --set full`)", "",
              "| capture | kernel | us | DRAM MB | DRAM % peak | issue active % | warps active / eligible per scheduler | regs |",
              "|---|---|---|---|---|---|---|---|"]
    summary = {}
    for kind in ("decode", "k1"):
        for f in FMTS:
            rep = os.path.join(src, f"c4_{kind}_{f}.ncu-rep")
            if not os.path.exists(rep):
                continue
            d = raw(rep)
            by = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
            dur = d.get("gpu__time_duration.sum", 0)
            lines.append(f"| c4_{kind}_{f} | `{d['kernel'][:60]}` | {dur*1e6:.2f} | {by/1e6:.1f} | "
                         f"{d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                         f"{d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                         f"{d.get('smsp__warps_active.avg.per_cycle_active', 0):.2f} / "
                         f"{d.get('smsp__warps_eligible.avg.per_cycle_active', 0):.2f} | "
                         f"{d.get('launch__registers_per_thread', 0):.0f} |")
            summary[f"c4_{kind}_{f}"] = {"kernel": d["kernel"], "dram_bytes_per_launch": by, "duration_s": dur,
                                         "tag": tag}
    open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    old = {}
    p = os.path.join(PROF, "ncu_summary.json")
    if os.path.exists(p):
        old = json.load(open(p))
    old.update(summary)
    json.dump(old, open(p, "w"), indent=1)
    import shutil
    shutil.copy(os.path.join(src, "launches_c4.csv"), os.path.join(PROF, f"{tag}_launches_c4.csv"))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
