#!/bin/bash
# A/B of library builds on config(s): gpurun -- 'bash tools/gpu_ab_lib.sh <tag> "<libs>" <cfgs...>'
# (libs: names under abtmp/ without the libmr3_ prefix; the first is the reference output)
set -u
TAG=$1; LIBS=$2; shift 2
O=gpurun_out
mkdir -p $O
for c in "$@"; do
  first=""
  for rep in 1 2; do
    for L in $LIBS; do
      [ -z "$first" ] && first=$L
      ref=""
      [ "$L" != "$first" ] && ref=/tmp/ab_${TAG}_c${c}_${first}.npz
      timeout 600 python tools/ab_lib.py abtmp/libmr3_$L.so $c 3 /tmp/ab_${TAG}_c${c}_$L.npz $ref >> $O/${TAG}_ab.log 2>&1
      echo "config $c lib $L exit $?" >> $O/${TAG}_ab.log
    done
  done
done
