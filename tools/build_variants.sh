#!/bin/bash
# Build engine variants with different register budgets into _lib/variants/<name>.so
# usage: tools/build_variants.sh "5 4" "6 5" ...
set -e
cd "$(dirname "$0")/../paper_1901_04200_b200/csrc"
OUT=../_lib/variants; mkdir -p $OUT/obj
for v in "$@"; do
  set -- $v; name=p$1_$2${3:+_$3}
  extra="-DLTG_P1_MINB=$1 -DLTG_P2_MINB=$2 $4"
  for f in heston reduce probe; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off -I. -I../../include $extra -c $f.cu -o $OUT/obj/${name}_$f.o
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/$name.so $OUT/obj/${name}_heston.o $OUT/obj/${name}_reduce.o $OUT/obj/${name}_probe.o ../_lib/obj/engine.o ../_lib/obj/host_libm.o -ldl
  echo built $OUT/$name.so
done
