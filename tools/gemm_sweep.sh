# decode-step GEMM shapes (C2, M 4096) under each tile choice (KNOB_GEMM_PAIR): model, forced
# 256x256 / 256x128 / 256x224 pairs, single-CTA
for pair in 0 1 2 3 -1; do
  echo "== GEMM_PAIR=$pair"
  DASHCU_GEMM_PAIR=$pair python tools/gemm_bench.py dec_qkv dec_w1_tanh dec_w2_res dec_wo_res dec_w1 dec_w2
done
