"""Per-class kernel time shares and DRAM traffic from an ncu launch list taken with
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv
Usage: python tools/traffic_summary.py launches.csv [out.json]
Prints a markdown table per kernel class (launches, serialised ms and share, mean DRAM
bytes per launch) and writes {class: mean DRAM bytes per launch} for bench.py's
roofline.traffic. ncu times are cold-cache and serialised: compare SHARES, not absolutes."""
import collections
import csv
import json
import re
import sys


def klass(name):
    n = name.replace("(int)", "").replace("(bool)", "")
    m = re.search(r"gemm_tc_kernel<(\d+), (\d+), (\w+), (\w+), (\d+), (\d+)[,>]", n)
    if m:
        mode = int(m.group(6))
        return {0: "gemm_tc", 1: "sample", 2: "lm_rows", 3: "lm_rows", 4: "sample"}[mode]
    if "gemm_tc2_kernel" in n:
        return "gemm_tc"
    for key, cls in (("attn_decode", "attn_decode"), ("attn_fwd", "attn_fwd"), ("attn_bwd", "attn_bwd"),
                     ("sample_scan", "sample"), ("embed_", "embed"), ("DeviceRadixSort", "embed"), ("lse_reduce", "lm_rows"), ("optimizer_k", "optimizer"),
                     ("gemm_simt", "gemm_simt"), ("colsum", "colsum"), ("kv_append", "kv_append"),
                     ("attn_bwd_dot", "attn_bwd"), ("pack_dqkv", "attn_bwd"), ("pack_batch_rows", "pack")):
        if key in n:
            return cls
    return "other"


def main():
    path = sys.argv[1]
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.reader(lines))
    h, data = rows[0], rows[1:]
    ii, ik, im, iv = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = collections.defaultdict(dict)
    names = {}
    for r in data:
        per[r[ii]][r[im]] = float(r[iv].replace(",", ""))
        names[r[ii]] = r[ik]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, mets in per.items():
        c = klass(names[i])
        a = agg[c]
        a[0] += 1
        a[1] += mets.get("gpu__time_duration.sum", 0.0)
        a[2] += mets.get("dram__bytes_read.sum", 0.0) + mets.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values())
    print(f"{len(per)} launches, {tot / 1e6:.3f} ms of kernel time (serialised)\n")
    print("| class | launches | ms | share | mean DRAM bytes / launch |")
    print("|---|---|---|---|---|")
    out = {}
    for c, (n, ns, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {c} | {n} | {ns / 1e6:.3f} | {100 * ns / max(tot, 1):.1f}% | {b / n:.4g} |")
        out[c] = b / n
    if len(sys.argv) > 2:
        json.dump(out, open(sys.argv[2], "w"), indent=1)


if __name__ == "__main__":
    main()
