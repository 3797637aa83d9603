#!/bin/bash
# c4 porous variants: dense / masked (compacted segments, ballot) at several skip granularities / lists
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "masked or sparse or skip" > gpurun_out/c4_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c4_pytest.log
for gb in 32 64 128; do
  DLB_SKIP_GROUP_BYTES=$gb timeout 300 python bench.py --config c4 --porous masked --no-cpu --steps 5 --warmup 3 > gpurun_out/c4_seg_$gb.json 2> gpurun_out/c4_seg_$gb.err
done
DLB_MASKED_COMPACT=0 timeout 300 python bench.py --config c4 --porous masked --no-cpu --steps 5 --warmup 3 > gpurun_out/c4_masked_32.json 2> gpurun_out/c4_masked_32.err
