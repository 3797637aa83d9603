mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_porous_compact.py tests/test_gpu_parity.py tests/test_full_parity.py tests/test_ragged.py tests/test_dolb_capi.py -q -m gpu -x > gpurun_out/gt2.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/gt2.log | tail -8
for v in 1 0; do DLB_DENSE_SEG=$v timeout 600 python bench.py --config c4 --porous dense --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('denseseg=$v', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['gpu_launches'], d['config']['kernel'])"; done
