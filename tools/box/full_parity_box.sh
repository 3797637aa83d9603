set -x
nproc; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
mkdir -p gpurun_out
timeout 2400 python tools/full_parity_gpu.py > gpurun_out/gpu_full.log 2>&1 &
GP=$!
timeout 2700 python tests/golden/make_golden_box.py > gpurun_out/golden_box.log 2>&1
echo "golden rc=$?"
wait $GP
echo "gpu rc=$?"
tail -5 gpurun_out/gpu_full.log gpurun_out/golden_box.log
