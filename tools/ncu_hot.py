"""Aggregate ncu warp-stall samples per CUDA source line.

    python tools/ncu_hot.py report.ncu-rep <kernel-regex> [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, agg, src = None, None, {}, {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue
        try:
            v = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        key = (fname, int(r[0]))
        agg[key] = agg.get(key, 0.0) + v
        src.setdefault(key, r[1].strip()[:100])
    tot = sum(agg.values()) or 1.0
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"{100 * v / tot:5.1f}%  {k[0]}:{k[1]:<5d} {src[k]}")


if __name__ == "__main__":
    main()
