#!/usr/bin/env python
"""Kernel-choice evidence table: the ncu --set full counters of each A/B pair
captured by scripts/gpu_choices.sh (one JSON per capture, written by
ncu_summary.py --json), as profiles/<tag>/choices.md.

    python scripts/choices_table.py gpurun_out/choices profiles/r01_choices
"""
import json
import os
import shutil
import sys

NOTES = {
    "Band apply blocking, config 3 (two-kernel form, apply alone)":
        "V=16 feeds up to 3 x 4 outputs from each 16-byte shared load and moves 6 % fewer DRAM bytes "
        "(64-row tiles halve the row halo); it runs one CTA per SM (7.8 % warps active) and is issue-bound "
        "('selected'), the V=8 form waits on memory ('long_scoreboard') with 3x the warps. Bench: 404 -> 380 us.",
    "Check + apply, config 3":
        "The fused kernel streams the matrix inside the apply: 2.18 GB in 353 us (6.2 TB/s), against "
        "18.7 us of check + 365 us of apply; the fixup pass only reads the 8 KB of segment flags.",
    "CSR build write-back, config 3 (block build)":
        "80 MB of output stays in L2 (only ~22 MB reach DRAM during the kernel): latency/issue-bound "
        "('barrier'); the bulk store still saves the per-thread store instructions (24.9 -> 21.5 us).",
    "CSR build, config 4":
        "The TMA bulk store is the difference (4.8 -> 6.3 TB/s, 0.98 of the copy peak); with it the block "
        "kernel also beats the warp-local one, so it is the default for every k.",
    "Latency SpMV staging, config 2 (one image, cold)":
        "All three are latency-bound near 9-10 us (long_scoreboard); the staged kernels coalesce the "
        "matrix (10.7 vs 23.6 sectors per request) and, PDL-chained, win where it matters: the DenseNet "
        "table (profiles/r01l) and the warm 3.0 us chained SpMV.",
    "Band check, config 4":
        "1.66 GB read in 230 us: 7.2 TB/s, above the copy kernel's read+write rate (read-only traffic).",
}

PAIRS = [
    ("Band apply blocking, config 3 (two-kernel form, apply alone)",
     [("apply_v16", "V=16 rows x 4 cols, 64-row tiles (kept)"), ("apply_v8", "V=8 x 4, 32-row tiles")]),
    ("Check + apply, config 3",
     [("fused", "fused check-and-apply + fixup (kept)"), ("check_c3", "separate check kernel (+ the apply above)")]),
    ("CSR build write-back, config 3 (block build)",
     [("build3_bulk", "TMA bulk store (kept)"), ("build3_stg", "16-byte st.global")]),
    ("CSR build, config 4",
     [("build4_block_bulk", "block scan, bulk store (kept)"), ("build4_warp_bulk", "warp-local, bulk store"),
      ("build4_block_stg", "block scan, 16-byte st.global")]),
    ("Latency SpMV staging, config 2 (one image, cold)",
     [("spmv_lsu", "per-lane 16-byte loads (kept)"), ("spmv_bulk", "cp.async.bulk by one lane"),
      ("spmv_plain", "thread per row, no staging")]),
    ("Band check, config 4", [("check_c4", "one warp per segment, 3 bulk copies (kept)")]),
]


def num(rec, key):
    v = rec.get(key)
    if not v:
        return None
    try:
        return float(v[0].replace(",", ""))
    except ValueError:
        return None


def to_us(rec):
    v, u = rec["gpu__time_duration.sum"]
    v = float(v.replace(",", ""))
    return v * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1.0)


def to_bytes(rec, key):
    v, u = rec[key]
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(dst, exist_ok=True)
    out = ["# Kernel choices and their ncu evidence (`ncu --set full --clock-control none`, one launch each)",
           "",
           "Each section is an A/B pair captured by `scripts/gpu_choices.sh` on one B200; DRAM GB/s = "
           "(dram__bytes_read + dram__bytes_write) / gpu__time_duration of that launch (cold, serialised, "
           "so it differs from the bench's back-to-back numbers). The raw per-capture summaries are next "
           "to this file (`*.txt`).", ""]
    for title, items in PAIRS:
        out += [f"## {title}", "",
                "| variant | kernel | us | DRAM MB | DRAM GB/s | L2 hit % | sectors/req (global ld) | "
                "issue active % | warps active % | top stall |",
                "|---|---|---|---|---|---|---|---|---|---|"]
        for name, label in items:
            p = os.path.join(src, name + ".json")
            if not os.path.exists(p):
                out.append(f"| {label} | (missing) | | | | | | | | |")
                continue
            for rec in json.load(open(p)):
                us = to_us(rec)
                mb = (to_bytes(rec, "dram__bytes_read.sum") + to_bytes(rec, "dram__bytes_write.sum")) / 1e6
                sec, req = num(rec, "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"), num(
                    rec, "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")
                spr = f"{sec / req:.1f}" if sec and req else "-"
                stall = rec["top_stalls"][0] if rec.get("top_stalls") else ("-", 0)
                kname = rec["kernel"].split("(")[0].replace("void ", "")[:60]
                out.append(f"| {label} | `{kname}` | {us:.1f} | {mb:.1f} | {mb / 1e3 / (us * 1e-6):.0f} | "
                           f"{num(rec, 'lts__t_sector_hit_rate.pct') or 0:.1f} | {spr} | "
                           f"{num(rec, 'smsp__issue_active.avg.pct_of_peak_sustained_active') or 0:.1f} | "
                           f"{num(rec, 'sm__warps_active.avg.pct_of_peak_sustained_active') or 0:.1f} | "
                           f"{stall[0]} {stall[1]:.2f} |")
        if title in NOTES:
            out += ["", NOTES[title]]
        out.append("")
    with open(os.path.join(dst, "choices.md"), "w") as f:
        f.write("\n".join(out))
    for fn in os.listdir(src):
        if fn.endswith(".txt") or fn.endswith(".json"):
            shutil.copy(os.path.join(src, fn), os.path.join(dst, fn))


if __name__ == "__main__":
    main()
