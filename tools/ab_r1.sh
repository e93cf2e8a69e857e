#!/bin/bash
# Same-box A/B of the current tree against a previous build copied into ab/<name>/ (its own
# bench.py + package + lib): python bench.py with the same arguments, alternating.
set -e
OLD=${OLD:-ab/r1}
ARGS=${ARGS:-"--prompts 128 --steps 2 --warmup 2 --no-cpu-baseline"}
for i in 1 2; do
  (cd $OLD && python bench.py $ARGS) | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('OLD', round(d['value']), d['phases_ms']['sample_ms'], d['phases_ms']['accumulate_ms'], d['clocks']['sm_mhz'])"
  python bench.py $ARGS | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('NEW', round(d['value']), d['phases_ms']['sample_ms'], d['phases_ms']['accumulate_ms'], d['clocks']['sm_mhz'])"
done
