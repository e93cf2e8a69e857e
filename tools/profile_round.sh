#!/bin/bash
# Evidence pass for profiles/ (run on the GPU box from the repo root; 1 GPU):
#   1. per-shape CUDA-event breakdowns of one C2 micro-batch and a few C2 decode steps
#   2. the ncu launch list of a full bench step (mini config: same kernels, fewer decode steps)
#   3. ncu --set full of the LM-head sampling GEMM and the top training GEMM
# Every ncu pass runs only after the same command exited 0 without ncu.
set -u
O=gpurun_out
mkdir -p $O
TAG=${1:-r1}
timeout 300 python tools/train_bench.py > $O/train_keys_$TAG.log 2>&1 || exit 1
timeout 300 python tools/sample_bench.py 8 > $O/sample_keys_$TAG.log 2>&1 || exit 1
timeout 600 python bench.py --config mini --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_mini_$TAG.log 2>&1 || exit 1
L=$(python -c "import json;print(json.loads(open('$O/bench_mini_$TAG.log').read().strip().splitlines()[-1])['gpu_launches'])")
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s $((3 * L)) -c $L --csv \
  --log-file $O/launches_mini_$TAG.csv python bench.py --config mini --steps 1 --warmup 3 --no-cpu-baseline \
  > $O/ncu_launches_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:gemm_tc_kernelILi256ELi4ELb1ELb1ELi8ELi1E -s 2 -c 1 -o $O/prof_sample_$TAG -f \
  python tools/sample_bench.py 4 > $O/ncu_sample_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:gemm_tc -s 30 -c 3 -o $O/prof_train_gemm_$TAG -f \
  python tools/train_bench.py 8 > $O/ncu_train_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:attn_bwd_tc -s 2 -c 1 -o $O/prof_attn_bwd_$TAG -f \
  python tools/train_bench.py 8 > $O/ncu_attn_bwd_$TAG.log 2>&1
echo done
