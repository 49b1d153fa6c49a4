"""Executed instructions per CUDA source line from an ncu report.

    python tools/ncu_inst.py report.ncu-rep <kernel-regex> [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, agg, src, fname = None, {}, {}, None
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
        col = None
        for name in ("Instructions Executed",):
            if name in hdr:
                col = hdr.index(name)
                break
        if col is None:
            continue
        try:
            v = float(r[col] or 0)
        except ValueError:
            continue
        key = (fname, int(r[0]))
        agg[key] = agg.get(key, 0.0) + v
        src.setdefault(key, r[1].strip()[:90])
    tot = sum(agg.values()) or 1.0
    print(f"total {tot:.4g}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"{100 * v / tot:5.1f}% {v:10.4g}  {k[0]}:{k[1]:<5d} {src[k]}")


if __name__ == "__main__":
    main()
