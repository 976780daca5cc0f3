"""Static SASS census of a kernel's loops (design probe): for each backward
branch with > 50 instructions in its body, the opcode histogram.
usage: python scripts/sass_loops.py <lib.so> <mangled-name-substring>"""
import re, subprocess, sys
from collections import Counter
lib, pat = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ins = []
    for l in f.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    print(name, len(ins), "instructions")
    for i, (a, s) in enumerate(ins):
        if "BRA" not in s:
            continue
        mm = re.search(r"0x([0-9a-f]+)", s.split("BRA")[1])
        if not mm:
            continue
        tgt = int(mm.group(1), 16)
        if tgt < a and tgt in addr:
            body = ins[addr[tgt]:i + 1]
            if len(body) > 50 and len(body) < int(sys.argv[3] if len(sys.argv) > 3 else 700):
                c = Counter((x.split()[1] if x.startswith("@") else x.split()[0]).split(".")[0] for _, x in body)
                print(f"  loop {tgt:#x}-{a:#x}: {len(body)} instr", dict(c.most_common(14)))
