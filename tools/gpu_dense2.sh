#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
timeout 600 python tools/probe_dense2.py 4096 > $O/dense2_probe.log 2>&1; echo "exit $?" >> $O/dense2_probe.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/dense2_launches.csv python tools/probe_dense.py 2048 > $O/dense2_ncu.log 2>&1; echo "ncu exit $?" >> $O/dense2_ncu.log
