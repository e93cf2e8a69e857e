#!/bin/bash
# Same-box A/B of environment switches on one C2 training micro-batch (tools/train_bench.py):
#   tools/ab_train.sh "ENV=a ENV2=b" "ENV=c" ...   ("" = defaults); REPS runs per arm
for arm in "$@"; do
  for r in $(seq ${REPS:-2}); do
    echo -n "[$arm] "; env $arm REPS=2 timeout 300 python tools/train_bench.py | head -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('accumulate_ms', round(d['accumulate_ms_unprofiled'], 2))"
  done
done
