#!/bin/bash
O=gpurun_out
python tools/dbg_chunk.py 3 > $O/dbgc3b.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "chunk or glued or small_random or config1 or rare_paths or split or fp32 or rqi_fb" > $O/r02i_pytest.log 2>&1
echo "pytest exit $?" >> $O/r02i_pytest.log
bash tools/gpu_ab.sh r02i RQI_CHUNK 0 8192 4 3
