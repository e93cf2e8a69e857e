#!/bin/bash
# Same-box A/B/C of the current build against two variant libraries (libdashcu_alt.so,
# libdashcu_alt2.so): bench.py alternating, one JSON summary per run.
ARGS=${ARGS:-"--prompts 256 --steps 1 --warmup 3 --no-cpu-baseline"}
L=$PWD/paper_2505_17218_b200/lib
P='import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], round(d["value"]), round(d["phases_ms"]["sample_ms"]), round(d["phases_ms"]["accumulate_ms"]), d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"]) for k, v in d.get("kernel_classes", {}).items() if k in ("attn_decode", "gemm_tc")})'
for i in 1 2; do
  python bench.py $ARGS | python3 -c "$P" BASE
  DASHCU_LIB_PATH=$L/libdashcu_alt.so python bench.py $ARGS | python3 -c "$P" ALT
  DASHCU_LIB_PATH=$L/libdashcu_alt2.so python bench.py $ARGS | python3 -c "$P" ALT2
done
