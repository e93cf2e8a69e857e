#!/bin/bash
# Same-box A/B of the current tree against a previous build copied into ab/<name>/ (its own
# bench.py + package + lib): python bench.py with the same arguments, alternating.
OLD=${OLD:-ab/r1}
ARGS=${ARGS:-"--prompts 128 --steps 2 --warmup 2 --no-cpu-baseline"}
P='import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], round(d["value"]), round(d["phases_ms"]["sample_ms"]), round(d["phases_ms"]["accumulate_ms"]), d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"]) for k, v in d["kernel_classes"].items()})'
for i in 1 2; do
  (cd $OLD && python bench.py $ARGS) | python3 -c "$P" OLD
  python bench.py $ARGS | python3 -c "$P" NEW
done
