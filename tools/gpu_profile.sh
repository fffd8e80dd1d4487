#!/bin/bash
# ncu evidence for profiles/: (1) the launch list of the default bench command,
# (2) --set full captures of both Heston passes on cfg3 at 2^20 paths with and
# without the draw store (the regimes of cfg5's chunks on one GPU) and of the
# fp32 variant, (3) the executed-instruction census of every config's pass
# kernels. Usage: tools/gpu_profile.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out /tmp/ncu
# .ncu-rep files stay on the box (/tmp/ncu; gpurun copies back <= 64 MiB):
# their raw and source pages come back as gzipped CSV, plus ncu_summary.py text
summ() {  # summ NAME PATHS
  python tools/ncu_summary.py full /tmp/ncu/$1.ncu-rep $2 > gpurun_out/$1_summary.txt 2>&1
  ncu -i /tmp/ncu/$1.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/$1_raw.csv.gz
  ncu -i /tmp/ncu/$1.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/$1_sass.csv.gz
  ncu -i /tmp/ncu/$1.ncu-rep --page source --csv --print-source cuda 2>/dev/null | gzip > gpurun_out/$1_cuda.csv.gz
}
M=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fp32_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum
CMD="python bench.py --steps 2 --warmup 3 --no-alt-method --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain_bench.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_cfg5.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
PCMD="python tools/profile_case.py --config cfg3 --paths 1048576"
for z in 0 1; do
  LTG_ZSTORE=$z $PCMD > gpurun_out/${TAG}_plain_z$z.log 2>&1 && \
    LTG_ZSTORE=$z timeout 900 ncu --set full --import-source on --clock-control none -k regex:heston_pass -c 2 \
      --metrics $M -o /tmp/ncu/${TAG}_cfg3_z$z -f $PCMD > gpurun_out/${TAG}_ncu_cfg3_z$z.log 2>&1
  summ ${TAG}_cfg3_z$z 1048576
done
P32="python tools/profile_case.py --config cfg3 --paths 1048576 --precision fp32"
for z in 0 1; do
  LTG_ZSTORE=$z $P32 > gpurun_out/${TAG}_plain_f32_z$z.log 2>&1 && \
    LTG_ZSTORE=$z timeout 900 ncu --set full --import-source on --clock-control none -k regex:heston_pass -c 2 \
      --metrics $M -o /tmp/ncu/${TAG}_cfg3f32_z$z -f $P32 > gpurun_out/${TAG}_ncu_cfg3f32_z$z.log 2>&1
  summ ${TAG}_cfg3f32_z$z 1048576
done
for spec in "cfg1 65536 fp64" "cfg2 262144 fp64" "cfg4 262144 fp64" "cfg2 262144 fp32" "cfg1 65536 fp32"; do
  set -- $spec
  P2="python tools/profile_case.py --config $1 --paths $2 --precision $3"
  for z in 0 1; do
    LTG_ZSTORE=$z $P2 > gpurun_out/${TAG}_plain_$1_$3_z$z.log 2>&1 && \
      LTG_ZSTORE=$z timeout 600 ncu --clock-control none -k regex:pass -c 2 --metrics $M --csv \
        --log-file gpurun_out/${TAG}_census_$1_$3_z$z.csv $P2 > gpurun_out/${TAG}_ncu_census_$1_$3_z$z.log 2>&1
  done
done
du -sh gpurun_out; ls -la gpurun_out | grep ${TAG}
