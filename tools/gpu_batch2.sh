#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "chunk or glued or small_random or config1 or rare_paths or split or fp32" > $O/r02h_pytest.log 2>&1
echo "pytest exit $?" >> $O/r02h_pytest.log
bash tools/gpu_ab.sh r02h RQI_CHUNK 0 8192 4 3 2 1
