#!/bin/bash
# Same-box A/B of the current build against a variant library built with different flags
# (paper_2505_17218_b200/lib/libdashcu_alt.so, DASHCU_LIB_PATH): bench.py alternating.
ARGS=${ARGS:-"--prompts 128 --steps 2 --warmup 2 --no-cpu-baseline"}
ALT=$PWD/paper_2505_17218_b200/lib/libdashcu_alt.so
P='import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], round(d["value"]), round(d["phases_ms"]["sample_ms"]), round(d["phases_ms"]["accumulate_ms"]), d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"]) for k, v in d["kernel_classes"].items()})'
for i in 1 2 3; do
  DASHCU_LIB_PATH=$ALT python bench.py $ARGS | python3 -c "$P" ALT
  python bench.py $ARGS | python3 -c "$P" NEW
done
