#!/usr/bin/env python3
"""SURVEY.md 8f rank 1, closed: re-runs the reference's acceptance criteria 8
and 9 (acceptance_test.cpp:465-506) with the decode cost's per-cached-token
term replaced by this repo's measured K1+K2 cost (oracle/ref_calib.cpp links
the unmodified reference simulator).  Reads a fit written by
scripts/calibrate_decode_cost.py (default: the newest profiles/*decode_cost_fit.json),
writes profiles/<round>_calibrated_acceptance.json.  Needs /root/reference
(run here, not on the GPU box).

  python scripts/calibrated_acceptance.py [fit.json] [out.json]
"""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
fit_path = sys.argv[1] if len(sys.argv) > 1 else sorted(glob.glob(os.path.join(ROOT, "profiles", "*decode_cost_fit.json")))[-1]
out_path = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "r02_calibrated_acceptance.json")
subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
fits = json.load(open(fit_path))["fits"]
eps = {k: v["decode_cost"]["epsilon_s_per_cached_token"] for k, v in fits.items()}
# kv_bits 8 in the reference scenarios is the paper's FP8 KV (vLLM fp8)
args = [eps["FP16"], eps["FP8_E4M3"], eps["INT4"], 32]
p = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_calib"), "/root/reference/proj/scenarios",
                    *map(str, args)], capture_output=True, text=True, check=True)
res = json.loads(p.stdout)
res["fit"] = os.path.relpath(fit_path, ROOT)
res["epsilon_s_per_cached_token_32_layers"] = {"fp16": args[0], "kv8 (fp8)": args[1], "kv4": args[2]}
res["note"] = ("scenario gamma/delta kept (weight GEMMs, outside this path); epsilon replaced by the "
               "measured B200 attention+append cost scaled to each model's num_layers; shipped value 1e-9")
json.dump(res, open(out_path, "w"), indent=1)
print(json.dumps(res, indent=1))
