#!/bin/bash
# A/B of a parameter on configs: gpurun -- 'bash tools/gpu_ab.sh <tag> <PARAM> <v1> <v2> <cfgs...>'
set -u
TAG=$1; PARAM=$2; V1=$3; V2=$4; shift 4
O=gpurun_out
mkdir -p $O
for c in "$@"; do
  timeout 600 python tools/ab_param.py $c $PARAM $V1 $V2 3 >> $O/${TAG}_ab.log 2>&1
  echo "config $c exit $?" >> $O/${TAG}_ab.log
done
