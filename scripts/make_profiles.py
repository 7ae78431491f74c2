#!/usr/bin/env python
"""Turns one gpurun session's raw ncu output (gpurun_out/) into the committed
evidence under profiles/<tag>/:

  launches_c<N>.md     -- every launch of the `ncu --metrics gpu__time_duration.sum`
                          pass, aggregated per kernel (count, mean, share)
  <report>.txt         -- key counters + top stalls of each `ncu --set full` report
  ncu_summary.json     -- per config: DRAM bytes per launch of the SpMM kernel
                          (read by bench.py as roofline.traffic)
  bench_*.json         -- the bench lines of the same session

    python scripts/make_profiles.py r01 [gpurun_out]
"""
from __future__ import annotations

import collections
import csv
import json
import os
import re
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from ncu_summary import KEYS, raw  # noqa: E402

UNIT_US = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h, d = rows[0], rows[1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in d:
        if r[ui] not in UNIT_US:
            continue
        agg.setdefault(r[ki], []).append(float(r[vi].replace(",", "")) * UNIT_US[r[ui]])
    tot = sum(sum(v) for v in agg.values()) or 1.0
    out = ["| kernel | launches | mean us | min us | max us | share of GPU time |", "|---|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k[:110]}` | {len(v)} | {sum(v) / len(v):.2f} | {min(v):.2f} | {max(v):.2f} | "
                   f"{sum(v) / tot:.3f} |")
    return "\n".join(out) + "\n", agg


def main():
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    dst = os.path.join(ROOT, "profiles", tag)
    os.makedirs(dst, exist_ok=True)
    summary = {}
    for f in sorted(os.listdir(src)):
        p = os.path.join(src, f)
        if f.startswith("launches_") and f.endswith(".csv"):
            md, _ = launches(p)
            cmdlog = p.replace("launches_", "ncu_launch_").replace(".csv", ".log")
            hdr = f"# {f} -- ncu --metrics gpu__time_duration.sum --clock-control none\n\n"
            hdr += ("Cold-cache, serialised per-launch times (compare shares, not absolutes). "
                    "Includes the CSR builds, the e2e (chunked) launches and torch's input "
                    "generation of the bench run.\n\n")
            with open(os.path.join(dst, f.replace(".csv", ".md")), "w") as o:
                o.write(hdr + md)
            shutil.copy(p, os.path.join(dst, f))
            if os.path.exists(cmdlog):
                shutil.copy(cmdlog, os.path.join(dst, os.path.basename(cmdlog)))
        elif f.endswith(".ncu-rep"):
            res = raw(p)
            lines = []
            name = f.replace(".ncu-rep", "")
            mt = re.match(r"prof_(\w+?)_c(\d+)(?:_b(\d+))?$", name)
            for ri, r in enumerate(res):
                lines.append(f"== {r['kernel']}")
                for k in KEYS:
                    if k in r:
                        lines.append(f"   {k:70s} {r[k][0]:>16s} {r[k][1]}")
                lines.append(f"   top stalls (pc sampling share): {r['top_stalls']}")
                rd = float(r["dram__bytes_read.sum"][0].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[r["dram__bytes_read.sum"][1]]
                wr = float(r["dram__bytes_write.sum"][0].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[r["dram__bytes_write.sum"][1]]
                summary[f"{name}#{ri}"] = {"kernel": r["kernel"], "dram_read_bytes": rd, "dram_write_bytes": wr,
                                 "role": mt.group(1) if mt else None,
                                 "config": int(mt.group(2)) if mt else None,
                                 "batch": int(mt.group(3)) if mt and mt.group(3) else None,
                                 "dram_bytes_per_launch": rd + wr,
                                 "duration_us": float(r["gpu__time_duration.sum"][0].replace(",", "")) *
                                 UNIT_US.get(r["gpu__time_duration.sum"][1], 1.0),
                                 "source": f"profiles/{tag}/{name}.txt"}
            with open(os.path.join(dst, f.replace(".ncu-rep", ".txt")), "w") as o:
                o.write(f"# ncu --set full --clock-control none --import-source on ({f})\n")
                o.write("\n".join(lines) + "\n")
        elif f.startswith("bench") and f.endswith(".log"):
            with open(p) as fh:
                js = [ln for ln in fh if ln.startswith("{")]
            if js:
                with open(os.path.join(dst, f.replace(".log", ".json")), "w") as o:
                    o.write(js[-1])
        elif f in ("pytest_gpu.log", "smoke.log", "status.txt", "exp.txt"):
            shutil.copy(p, os.path.join(dst, f))
    with open(os.path.join(dst, "ncu_summary.json"), "w") as o:
        json.dump(summary, o, indent=1)
    if summary:  # bench.py reads roofline.traffic from the newest pass
        with open(os.path.join(ROOT, "profiles", "LATEST"), "w") as o:
            o.write(os.path.basename(dst.rstrip("/")) + "\n")
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
