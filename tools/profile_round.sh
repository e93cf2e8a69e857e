#!/bin/bash
# Evidence pass for profiles/ (run on the GPU box from the repo root; 1 GPU):
#   1. per-shape CUDA-event breakdowns of one C2 micro-batch and a few C2 decode steps
#   2. the ncu launch list (+ DRAM bytes) of one full bench step (mini config: same
#      kernels as C2, fewer decode steps) -> per-class shares and bench roofline.traffic
#   3. ncu --set full of the top kernels: LM-head sampling GEMM, a training GEMM, the
#      tcgen05 attention forward / backward and the decode attention
# Every ncu pass runs only after the same command exited 0 without ncu.
set -u
O=gpurun_out
mkdir -p $O
TAG=${1:-r1}
timeout 300 python tools/train_bench.py > $O/train_keys_$TAG.log 2>&1 || exit 1
timeout 300 python tools/sample_bench.py 8 > $O/sample_keys_$TAG.log 2>&1 || exit 1
timeout 600 python bench.py --config mini --steps 1 --warmup 3 --no-cpu-baseline > $O/bench_mini_$TAG.log 2>&1 || exit 1
L=$(python -c "import json;print(json.loads(open('$O/bench_mini_$TAG.log').read().strip().splitlines()[-1])['gpu_launches'])")
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -s $((3 * L + 200)) -c $L --csv --log-file $O/launches_mini_$TAG.csv \
  python bench.py --config mini --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_launches_$TAG.log 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base mangled -f"
REPS=1 timeout 600 $NCU -k regex:gemm_tc_kernelILi256ELi4ELb1ELb1ELi8ELi1E -s 2 -c 1 -o $O/prof_sample_$TAG \
  python tools/sample_bench.py 4 > $O/ncu_sample_$TAG.log 2>&1
REPS=1 timeout 600 $NCU -k regex:gemm_tc2_kernel -s 40 -c 2 -o $O/prof_train_gemm_$TAG \
  python tools/train_bench.py 32 > $O/ncu_train_$TAG.log 2>&1
REPS=1 timeout 600 $NCU -k regex:attn_bwd_tc5 -s 2 -c 1 -o $O/prof_attn_bwd_$TAG python tools/train_bench.py 32 \
  > $O/ncu_attn_bwd_$TAG.log 2>&1
REPS=1 timeout 600 $NCU -k regex:attn_fwd_tc5 -s 2 -c 1 -o $O/prof_attn_fwd_$TAG python tools/train_bench.py 32 \
  > $O/ncu_attn_fwd_$TAG.log 2>&1
timeout 600 $NCU -k regex:attn_decode -s 60 -c 1 -o $O/prof_attn_decode_$TAG python tools/sample_bench.py 4 \
  > $O/ncu_attn_decode_$TAG.log 2>&1
# the sampling GEMM's DRAM traffic (no logits store) and the chosen-slice recompute, C2 decode
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled \
  -k regex:"gemm_tc_kernel<\\(int\\)256, \\(int\\)4," -s 4 -c 4 --csv --log-file $O/sample_traffic_$TAG.csv \
  python tools/sample_bench.py 4 > $O/ncu_sample_traffic_$TAG.log 2>&1
echo done
