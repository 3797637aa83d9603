mkdir -p gpurun_out
for c in c2 c1 c3 c5; do for t in 128 64; do DLB_PULL_THREADS=$t timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c threads=$t', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"; done; done
for t in 128 64; do DLB_PULL_THREADS=$t timeout 600 python bench.py --layout aa --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c5 AA threads=$t', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"; done
