"""DRAM traffic of the dominant kernel class at the C2 (Qwen2.5-0.5B) shapes, for bench.py's
roofline.traffic. Run under ncu (one process, one GPU):

  ncu --kernel-name regex:gemm_tc --metrics gpu__time_duration.sum,dram__bytes_read.sum,\\
      dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic.csv \\
      python tools/traffic_c2.py run
  python tools/traffic_c2.py summarize gpurun_out/traffic.csv > profiles/ncu_traffic_c2.json

`run` launches each shape twice through dashcu_selftest_gemm_timed (warm-up + 1); the
summary keeps the second launch and sets its DRAM bytes against the algorithmic bytes
(A + B read once, C written once; fp32 C for the accumulate / residual shapes)."""
import csv
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

# (name, M, N, K, a_kmajor, b_kmajor, epi, bytes per C element) -- epi 0 bf16 out, 3 fp32 += , 4 fp32 resid
SHAPES = [("fwd_w1", 36832, 4864, 896, 1, 1, 1, 2), ("fwd_w2_res", 36832, 896, 4864, 1, 1, 4, 10),
          ("dec_w1", 4096, 4864, 896, 1, 1, 1, 2), ("dec_w2_res", 4096, 896, 4864, 1, 1, 4, 10),
          ("wgrad_w1", 4864, 896, 36832, 0, 0, 3, 8), ("dgrad_w1_res", 36832, 896, 4864, 1, 0, 4, 10)]


def run():
    import paper_2505_17218_b200 as D
    L = D.lib()
    L.dashcu_selftest_gemm_timed.argtypes = [C.c_void_p] + [C.c_int] * 7 + [C.POINTER(C.c_double)]
    ctx = D.Context(0)
    for name, M, N, K, ak, bk, epi, _ in SHAPES:
        ms = C.c_double(0)
        assert L.dashcu_selftest_gemm_timed(ctx.h, M, N, K, ak, bk, epi, 1, C.byref(ms)) == 0


def summarize(path):
    rows = [r for r in csv.reader(open(path))]
    hdr = next(r for r in rows if r and r[0] == "ID")
    per = {}
    for r in rows:
        if len(r) != len(hdr) or r[0] == "ID":
            continue
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3}.get(d["Metric Unit"], 1)
        per.setdefault(int(d["ID"]), {})[d["Metric Name"]] = v * scale
    ids = sorted(per)
    out = {"shapes": []}
    for i, (name, M, N, K, ak, bk, epi, cb) in enumerate(SHAPES):
        m = per[ids[2 * i + 1]]   # the timed launch (the first one is the warm-up)
        dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        alg = 2.0 * (M * K + N * K) + cb * M * N
        out["shapes"].append({"shape": f"{name} M{M} N{N} K{K}", "dram_bytes": dram, "alg_bytes": alg,
                              "ratio": dram / alg, "ms": m["gpu__time_duration.sum"] * 1e3})
    top = out["shapes"][0]
    out["gemm_tc"] = {k: top[k] for k in ("shape", "dram_bytes", "alg_bytes")}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    run() if sys.argv[1] == "run" else summarize(sys.argv[2])
