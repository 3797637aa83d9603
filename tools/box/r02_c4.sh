mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "segment or masked or porous or skip or config4 or registry" > gpurun_out/gputest_c4.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/gputest_c4.log | tail -20
for v in 1 0; do DLB_FLUID_SEGMENTS=$v timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/c4_fs$v.json 2>gpurun_out/c4_fs$v.err; python -c "
import json; d=json.load(open('gpurun_out/c4_fs$v.json')); c=d['config']
print('fluidseg=$v', round(d['value']), 'frac', round(d['roofline']['frac'],3), c['kernel'], 'alg bytes', c.get('algorithmic_bytes_per_step'), 'per fluid', round(c['mlups_per_fluid_cell']))"; done
timeout 900 ncu --set full --clock-control none -k regex:k_seg -c 2 -o gpurun_out/c4_segbb_L256 python bench.py --config c4 --L 256 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_c4.log 2>&1; echo "ncu rc=$?"
