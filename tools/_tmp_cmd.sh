timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_full.log 2>&1; tail -3 gpurun_out/gpu_full.log
python tools/host_overhead.py > gpurun_out/ho.log 2>&1
python bench.py --config cfg1 --steps 3 --warmup 3 --no-alt-method --no-cpu-baseline > gpurun_out/b1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launch_cfg1.csv python bench.py --config cfg1 --steps 2 --warmup 3 --no-alt-method --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
