#!/bin/bash
# One gpurun session: smoke, tests, every bench line (+ the reference arm),
# then the ncu evidence (tools/gpu_profile.sh: launch list, --set full
# captures exported as text / gzipped CSV, census). Usage: tools/gpu_round.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt
nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --precision fp32 --no-cpu-baseline > gpurun_out/bench_cfg5_fp32.json 2> gpurun_out/bench_cfg5_fp32.err
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
bash tools/gpu_profile.sh $TAG > gpurun_out/${TAG}_profile.log 2>&1
