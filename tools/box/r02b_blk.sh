mkdir -p gpurun_out
for b in 256 128 256 128; do for p in masked dense; do DLB_SEG_BLOCK=$b timeout 600 python bench.py --config c4 --porous $p --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('block=$b $p', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"; done; done
