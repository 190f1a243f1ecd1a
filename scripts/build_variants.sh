#!/bin/bash
# build library variants for A/B: scripts/build_variants.sh name "EXTRA flags" [name "flags" ...]
# -> build/var_<name>/libjh_hstu.so
cd "$(dirname "$0")/../paper_2508_04711_b200/csrc"
while [ $# -ge 2 ]; do
  n=$1; f=$2; shift 2
  mkdir -p ../../build/var_$n
  make -j8 OUT=../../build/var_$n/libjh_hstu.so OBJDIR=../../build/var_$n/obj EXTRA="$f" > ../../build/var_$n/build.log 2>&1 || { echo "build $n failed"; tail -5 ../../build/var_$n/build.log; exit 1; }
  echo "built $n ($f)"
done
