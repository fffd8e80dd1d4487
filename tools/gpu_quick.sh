#!/bin/bash
# Quick GPU check: pytest -m gpu, smoke, per-config timings.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python tools/quick_time.py cfg1 cfg2 cfg3 2>&1 | tail -4
timeout 300 python bench.py --no-cpu-baseline --steps 3 2>&1 | tail -1 | cut -c1-400
