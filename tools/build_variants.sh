#!/bin/bash
# Build engine variants into _lib/variants/<name>.so
# usage: tools/build_variants.sh "name P1MINB P2MINB [extra nvcc flags...]" ...
set -e
cd "$(dirname "$0")/../paper_1901_04200_b200/csrc"
OUT=../_lib/variants; mkdir -p $OUT/obj
make -s -C . >/dev/null
for v in "$@"; do
  set -- $v; name=$1; p1=$2; p2=$3; shift 3; extra="$*"
  for f in heston basket reduce probe; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off -I. -I../../include -DLTG_P1_MINB=$p1 -DLTG_P2_MINB=$p2 $extra -Xptxas -v -c $f.cu -o $OUT/obj/${name}_$f.o 2> $OUT/obj/${name}_$f.log &
  done
  # (the host side too: a flag may change a shared struct's layout)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off -I. -I../../include $extra -c engine.cpp -o $OUT/obj/${name}_engine.o &
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/$name.so $OUT/obj/${name}_heston.o $OUT/obj/${name}_basket.o $OUT/obj/${name}_reduce.o $OUT/obj/${name}_probe.o $OUT/obj/${name}_engine.o ../_lib/obj/host_libm.o -ldl
  echo "built $name: $(grep -h registers $OUT/obj/${name}_heston.log | awk '{print $5}' | tr '\n' ' ') spill: $(grep -h spill $OUT/obj/${name}_heston.log | awk '{s+=$5} END {print s}')"
done
