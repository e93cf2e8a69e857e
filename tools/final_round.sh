#!/bin/bash
# End-of-round measurement pass (GPU box, repo root): the bench lines of BASELINE configs
# 1-3 (C2 with the CPU baseline, C3, C4), an unprofiled C2 line (graphs on), and the
# configs[4] DASH-vs-GRPO sweep. Outputs under gpurun_out/final_*.
set -u
O=gpurun_out
mkdir -p $O
timeout 1500 python bench.py > $O/final_c2.json 2> $O/final_c2.err
timeout 900 python bench.py --no-profile --no-cpu-baseline > $O/final_c2_noprof.json 2> $O/final_c2_noprof.err
timeout 1500 python bench.py --config c3 --no-cpu-baseline > $O/final_c3.json 2> $O/final_c3.err
timeout 1500 python bench.py --config c4 --no-cpu-baseline > $O/final_c4.json 2> $O/final_c4.err
timeout 2400 python tools/sweep_c5.py --interleaved 64,256 --prompts 4,64,256,512 --taus off,0.1,0.3 \
  > $O/final_c5.log 2> $O/final_c5.err
echo done
