mkdir -p gpurun_out
for v in 0 1; do for a in 2 4; do DLB_BLOCK_1D=$v DLB_BLOCK_AHEAD=$a timeout 600 python bench.py --L 256 --steps 3 --warmup 3 --no-cpu --e2e-L 512 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('1d=$v ahead=$a e2e', round(d['e2e']['value'],1))"; done; done
