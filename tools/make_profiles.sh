#!/bin/bash
# Turn one profiling pass (tools/profile_round.sh TAG on the GPU box, results merged into
# gpurun_out/) into the tracked summaries under profiles/ (run here, no GPU needed).
set -eu
TAG=${1:-r1}
O=gpurun_out
P=profiles
mkdir -p $P
python tools/traffic_summary.py $O/launches_mini_$TAG.csv $P/${TAG}_traffic_mini.json > $P/${TAG}_launch_list.md
for k in sample train_gemm attn_bwd attn_fwd attn_decode; do
  [ -f $O/prof_${k}_$TAG.ncu-rep ] && python tools/ncu_summary.py $O/prof_${k}_$TAG.ncu-rep > $P/${TAG}_ncu_${k}.md
done
cp $O/train_keys_$TAG.log $P/${TAG}_train_microbatch_shapes.txt
cp $O/sample_keys_$TAG.log $P/${TAG}_decode_step_shapes.txt
echo "profiles for $TAG written"
