mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/gputest_full.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/gputest_full.log | tail -10
timeout 600 python __graft_entry__.py --smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_full.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "launch list rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1])
print(round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks'], d['e2e']['value'], d['cpu_baseline']['value'])"
