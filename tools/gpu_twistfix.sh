#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
timeout 300 python tools/probe_twist.py tools/data/dense_T_d.npy tools/data/dense_T_e.npy > $O/twist5.log 2>&1
timeout 600 python tools/probe_dense.py 4096 > $O/twist5_dense.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "default_needs_no or rare_paths or config5 or config3 or newton_path or small_random" > $O/twist5_pytest.log 2>&1; echo "pytest exit $?" >> $O/twist5_pytest.log
timeout 600 python bench.py --other-configs=1,2,3,4 --emulate-world= --no-zstore --no-e2e --no-cpu --dense= > $O/twist5_bench.json 2> $O/twist5_bench.err
