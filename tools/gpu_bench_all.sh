#!/bin/bash
# The bench lines of one round (no profiling): cfg5 fp64 (default), reference arm, fp32, cfg1-4
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --precision fp32 --no-cpu-baseline > gpurun_out/bench_cfg5_fp32.json 2> gpurun_out/bench_cfg5_fp32.err
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 python -m pytest tests/test_bench_gpu.py -q > gpurun_out/pytest_bench.log 2>&1; tail -1 gpurun_out/pytest_bench.log
