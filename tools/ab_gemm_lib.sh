S="wgrad_w1 wgrad_qkv wgrad_wo wgrad_lm"
P='import json,sys
for l in sys.stdin:
    d=json.loads(l); print(sys.argv[1], d["shape"], round(d["ms"]*1e3,1), round(d["tflops"]))'
for i in 1 2; do
python tools/gemm_bench.py $S | python3 -c "$P" NEW
DASHCU_LIB_PATH=$PWD/paper_2505_17218_b200/lib/libdashcu_alt.so python tools/gemm_bench.py $S | python3 -c "$P" ALT
done
DASHCU_LIB_PATH=$PWD/paper_2505_17218_b200/lib/libdashcu_alt.so python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2
