#!/usr/bin/env python3
"""One line per bench log: it/s, ms/step, roofline frac, per-kernel ms per step."""
import json
import sys

for f in sys.argv[1:]:
    line = None
    for ln in open(f):
        if ln.startswith("{"):
            line = json.loads(ln)
    if line is None:
        print(f, "NO JSON:", open(f).read()[-400:].replace("\n", " | "))
        continue
    d = line
    ks = {k: round(v["ms_per_launch"] * v["launches"] / d["steps"], 4) for k, v in (d.get("kernels") or {}).items()}
    roof = d.get("roofline") or {}
    print(f.split("/")[-1], d["config"].get("method"), f"{d['value']:.1f} it/s", f"{d['ms_per_step']:.3f} ms",
          "frac", round(roof.get("frac") or 0, 3), "step_frac", round(d.get("step_frac_of_peak") or 0, 3),
          "sm", (d.get("clocks") or {}).get("sm_mhz"), ks)
