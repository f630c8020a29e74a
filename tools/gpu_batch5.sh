#!/bin/bash
O=gpurun_out
./tools/micro/fp64tp > $O/fp64tp.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "glued or newton or chunk or config3 or config4" > $O/r02m_pytest.log 2>&1
echo "pytest exit $?" >> $O/r02m_pytest.log
bash tools/gpu_ab.sh r02m RQI_FB 1 0 3 4
