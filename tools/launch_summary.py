"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel:
    python tools/launch_summary.py gpurun_out/launches.csv [top]
Per-launch times are serialised and cold-cache: compare SHARES, not absolutes."""
import collections
import csv
import re
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h, data = rows[0], rows[1:]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for x in data:
        name = re.sub(r"\(.*", "", x[ik]).replace("void ", "").replace("unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(x[iv])
    tot = sum(v[1] for v in agg.values())
    print(f"{len(data)} launches, {tot / 1e6:.3f} ms of kernel time (serialised)\n")
    print("| kernel | launches | ms | share |")
    print("|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"| `{k}` | {v[0]} | {v[1] / 1e6:.3f} | {100 * v[1] / tot:.1f}% |")


if __name__ == "__main__":
    main()
