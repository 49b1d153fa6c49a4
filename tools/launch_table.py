"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_table.py launches.csv [--md]
"""
import collections
import csv
import sys


def table(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr, d = None, collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("(anonymous namespace)::", "")
        d[name].append(float(r[hdr.index("Metric Value")].replace(",", "")))
    tot = sum(sum(v) for v in d.values()) or 1.0
    return [(k, len(v), sum(v) / len(v) / 1e3, sum(v) / 1e6, 100 * sum(v) / tot)
            for k, v in sorted(d.items(), key=lambda x: -sum(x[1]))]


if __name__ == "__main__":
    md = "--md" in sys.argv
    if md:
        print("| kernel | launches | mean us | total ms | share |\n|---|---|---|---|---|")
    for k, n, mean, total, share in table(sys.argv[1]):
        print(f"| {k} | {n} | {mean:.1f} | {total:.2f} | {share:.1f}% |" if md else
              f"{k:45s} n={n:6d} mean={mean:9.1f}us total={total:8.2f}ms {share:5.1f}%")
