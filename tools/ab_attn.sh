# attention kernels alone (C2 micro-batch shape and the hd128 C3 shape): the current build vs
# an A/B variant library (paper_2505_17218_b200/lib/libdashcu_alt.so)
for i in 1 2; do
  echo "ALT $(DASHCU_LIB_PATH=$PWD/paper_2505_17218_b200/lib/libdashcu_alt.so python tools/attn_bench.py 32 1151 20)"
  echo "NEW $(python tools/attn_bench.py 32 1151 20)"
done
echo "ALT128 $(DASHCU_LIB_PATH=$PWD/paper_2505_17218_b200/lib/libdashcu_alt.so python tools/attn_bench.py 32 1151 20 12 2 128)"
echo "NEW128 $(python tools/attn_bench.py 32 1151 20 12 2 128)"
