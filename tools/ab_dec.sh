#!/bin/bash
# Same-box A/B of the decode phase (tools/sample_bench.py) between the current build and
# paper_2505_17218_b200/lib/libdashcu_alt.so (and _alt2.so if present): C2 shape (SIZE /
# PROMPTS override, STEPS decode steps) and the 32-row GRPO micro-batch (4 prompts, 64 steps).
ALT=$PWD/paper_2505_17218_b200/lib/libdashcu_alt.so
ALT2=$PWD/paper_2505_17218_b200/lib/libdashcu_alt2.so
P='import json,sys; d=json.loads(sys.stdin.readline()); c=d["classes"]; print(sys.argv[1], round(d["sample_ms_unprofiled"], 2), {k: round(v["ms"], 2) for k, v in c.items()})'
for i in 1 2; do
  for arm in ALT NEW $([ -f $ALT2 ] && echo ALT2); do
    L=""; [ $arm = ALT ] && L=$ALT; [ $arm = ALT2 ] && L=$ALT2
    echo -n "${SIZE:-0.5b} "; DASHCU_LIB_PATH=$L PROMPTS=${PROMPTS:-512} python tools/sample_bench.py ${STEPS:-256} | python3 -c "$P" $arm
    [ -z "$NO_SMALL" ] && { echo -n "small "; DASHCU_LIB_PATH=$L PROMPTS=4 python tools/sample_bench.py 64 | python3 -c "$P" $arm; }
  done
done
true
