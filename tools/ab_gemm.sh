#!/bin/bash
# Same-box A/B of a GEMM environment switch: tools/ab_gemm.sh VAR "v0 v1" shape...
# (box-to-box variance is 10-30 %, so both arms run back to back in one call); value "-" = unset
VAR=$1; VALS=$2; shift 2
for v in $VALS; do
  if [ "$v" = "-" ]; then env -u $VAR timeout 120 python tools/gemm_bench.py "$@" > gpurun_out/ab_$v.log
  else env $VAR=$v timeout 120 python tools/gemm_bench.py "$@" > gpurun_out/ab_$v.log; fi
done
python - "$VALS" <<'PY'
import json, sys
vals = sys.argv[1].split()
runs = [[json.loads(l) for l in open(f"gpurun_out/ab_{v}.log")] for v in vals]
for rows in zip(*runs):
    print(f"{rows[0]['shape']:14s} " + "  ".join(f"{v}: {r['tflops']:7.1f}" for v, r in zip(vals, rows)) +
          f"  ratio {rows[-1]['tflops'] / rows[0]['tflops']:.3f}")
PY
