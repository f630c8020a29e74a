#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "chunk or glued or small_random or config1 or rare_paths or split or fp32 or newton or index_and" > $O/r02j_pytest.log 2>&1
echo "pytest exit $?" >> $O/r02j_pytest.log
bash tools/gpu_ab.sh r02j GROUPS 0 8 4 3 2 1
