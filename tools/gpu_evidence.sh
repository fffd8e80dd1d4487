#!/bin/bash
# The round's closing evidence without profiling: smoke, pytest -m gpu, every
# bench line (tools/gpu_bench_all.sh), config 5 at the per-rank path counts of
# 2/4/8 GPUs (strong-scaling shares measured on one GPU), the reference
# calibrator on the GPU gradient. Usage: tools/gpu_evidence.sh
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt
nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
bash tools/gpu_bench_all.sh
for p in 33554432 16777216 8388608; do
  timeout 300 python bench.py --paths $p --no-cpu-baseline --no-alt-method > gpurun_out/bench_share_$p.json 2> gpurun_out/bench_share_$p.err
done
[ -x examples/calibrate_gpu ] && timeout 600 examples/calibrate_gpu tests/golden/heston_calibrate.json > gpurun_out/calibrate_gpu.json 2>&1
