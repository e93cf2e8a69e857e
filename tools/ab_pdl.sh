P='import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], round(d["value"]), round(d["phases_ms"]["sample_ms"]), round(d["phases_ms"]["accumulate_ms"]), d["clocks"]["sm_mhz"], {k: round(v["ms_per_step"]) for k, v in d["kernel_classes"].items()})'
A="--prompts 128 --steps 2 --warmup 2 --no-cpu-baseline"
for i in 1 2; do
python bench.py $A | python3 -c "$P" PDL0
DASHCU_PDL=1 python bench.py $A | python3 -c "$P" PDL1
done
