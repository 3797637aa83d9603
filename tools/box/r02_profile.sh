mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_full.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/launches_c5_full.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pull -s 3 -c 1 -o gpurun_out/c5_bgk_f32_L512 python bench.py --L 512 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c5.log 2>&1; echo "ncu full rc=$?"
bash tools/all_configs.sh; cat gpurun_out/all_configs.jsonl | python -c "
import json,sys
for l in sys.stdin:
    if not l.startswith('{'): continue
    d=json.loads(l); c=d['config']
    print(c['workload'][:3], c['arith'], c['layout'][:3], round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), c['kernel'])"
