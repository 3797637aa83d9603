mkdir -p gpurun_out
for c in 16 32 64 128; do DLB_BLOCK_CHUNKS=$c timeout 600 python bench.py --L 256 --steps 3 --warmup 3 --no-cpu --e2e-L 512 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('chunks=$c e2e', round(d['e2e']['value'],1))"; done
