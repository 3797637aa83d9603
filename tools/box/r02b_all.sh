mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gputest_full.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/gputest_full.log | tail -10
bash tools/all_configs.sh
DLB_VEC=1 timeout 400 python bench.py --no-cpu --no-e2e 2>/dev/null | tail -1 >> gpurun_out/all_configs.jsonl
DLB_POROUS_COMPACT=1 timeout 400 python bench.py --config c4 --no-cpu --no-e2e 2>/dev/null | tail -1 >> gpurun_out/all_configs.jsonl
python -c "
import json
for l in open('gpurun_out/all_configs.jsonl'):
    if not l.startswith('{'): continue
    d=json.loads(l); c=d['config']
    print(c['workload'][:3], c['arith'], c['layout'][:3], round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['gpu_launches'], c['kernel'])"
