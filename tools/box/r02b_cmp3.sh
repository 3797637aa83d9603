mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_porous_compact.py tests/test_full_parity.py -q -m gpu -x -k "compact or c4" > gpurun_out/gputest_cmp.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/gputest_cmp.log | tail -15
for v in 1 0; do DLB_POROUS_COMPACT=$v timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e 2>gpurun_out/c4_cmp$v.err | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('compact=$v', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['config']['kernel'])"; done
