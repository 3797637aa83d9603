mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_porous_compact.py tests/test_gpu_parity.py tests/test_full_parity.py -q -m gpu -x -k "masked or segment or porous or sphere or compact or skip or c4" > gpurun_out/gt4.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/gt4.log
for v in 1 0 1 0; do DLB_SEG_PACK=$v timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pack=$v', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"; done
