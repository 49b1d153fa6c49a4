"""Summarise ncu evidence into profiles/ (committed; gpurun_out/ is scratch).

    python tools/profile_summary.py <tag> [--full rep.ncu-rep] [--launches launches.csv]

Writes profiles/<tag>_kernels.md (per-kernel metrics, stall breakdown, top
source lines) and profiles/<tag>_kernels.json (machine-readable; bench.py
reads the dram traffic per launch from the newest one), plus
profiles/<tag>_launches.md (share of device time per kernel from the
serialised cold-cache launch list).
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct_peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_pct"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block", "smem_per_block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_shared_mem", "occ_limit_smem"),
    ("launch__occupancy_limit_registers", "occ_limit_regs"),
    ("smsp__inst_executed.sum", "inst_executed"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_float(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return None


def summarize_full(rep):
    hdr, units, rows = raw(rep)
    per = defaultdict(list)
    for r in rows:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").strip()
        d = {}
        for m, short in METRICS:
            if m in hdr:
                val = to_float(r[hdr.index(m)])
                u = units[hdr.index(m)]
                if val is not None and u in ("Kbyte", "Mbyte", "Gbyte", "byte"):
                    val *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
                if val is not None and u == "us" and short == "duration":
                    val *= 1e3  # -> ns
                if val is not None and u == "ms" and short == "duration":
                    val *= 1e6
                d[short] = val
        stalls = {}
        for i, h in enumerate(hdr):
            if "pcsamp_warps_issue_stalled" in h and "not_issued" not in h:
                v = to_float(r[i])
                if v:
                    stalls[h.split("stalled_")[1]] = v
        tot = sum(stalls.values()) or 1.0
        d["stalls_pct"] = {k: round(100 * v / tot, 1)
                           for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]}
        per[name].append(d)
    out = {}
    for name, ds in per.items():
        avg = {}
        for k in ds[0]:
            if k == "stalls_pct":
                avg[k] = ds[0][k]
            else:
                vals = [x[k] for x in ds if x.get(k) is not None]
                avg[k] = sum(vals) / len(vals) if vals else None
        avg["captures"] = len(ds)
        if avg.get("dram_read") is not None:
            avg["dram_traffic_bytes"] = avg["dram_read"] + (avg.get("dram_write") or 0)
        out[name] = avg
    return out


def hot_lines(rep, kernel, top=10):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_hot.py"), rep, kernel,
                        str(top)], capture_output=True, text=True)
    return r.stdout


def summarize_launches(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        v = to_float(r[vi])
        if v is None:
            continue
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "").strip()
        agg[name][0] += 1
        agg[name][1] += v * scale
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--full")
    ap.add_argument("--launches")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.full:
        s = summarize_full(a.full)
        json.dump(s, open(os.path.join(PROF, f"{a.tag}_kernels.json"), "w"), indent=1)
        with open(os.path.join(PROF, f"{a.tag}_kernels.md"), "w") as f:
            f.write(f"# {a.tag}: ncu --set full summary\n\nSource: `{os.path.basename(a.full)}` "
                    "(ncu --set full --clock-control none --import-source on; times are "
                    "serialised replays, use them for shares and counters, not as bench "
                    f"values).\n{a.note}\n\n")
            for name, d in s.items():
                f.write(f"## {name}\n\n| metric | value |\n|---|---|\n")
                for k, v in d.items():
                    if k == "stalls_pct":
                        continue
                    if isinstance(v, float):
                        v = f"{v:,.3f}" if abs(v) < 1e4 else f"{v:,.0f}"
                    f.write(f"| {k} | {v} |\n")
                f.write("\nwarp-stall sample shares: " +
                        ", ".join(f"{k} {v}%" for k, v in d["stalls_pct"].items()) + "\n\n")
                f.write("hottest source lines (stall samples):\n\n```\n" +
                        hot_lines(a.full, name) + "```\n\n")
    if a.launches:
        agg = summarize_launches(a.launches)
        tot = sum(v[1] for v in agg.values()) or 1.0
        with open(os.path.join(PROF, f"{a.tag}_launches.md"), "w") as f:
            f.write(f"# {a.tag}: kernel launch list (ncu --metrics gpu__time_duration.sum "
                    "--clock-control none)\n\nCold-cache, serialised per-launch device times; "
                    "compare SHARES, not absolutes.\n{}\n\n| kernel | launches | total us | "
                    "share |\n|---|---|---|---|\n".format(a.note))
            for name, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
                f.write(f"| {name} | {n} | {us:,.1f} | {100 * us / tot:.1f}% |\n")
    print("wrote profiles for", a.tag)


if __name__ == "__main__":
    main()
