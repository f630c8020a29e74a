#!/bin/bash
# NEXT-1b / NEXT-3 checks: the relax + absgap GPU tests, A/B of MR3_RELAX on the configs
set -u
O=gpurun_out; mkdir -p $O
TAG=${1:-relax}
shift || true
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "relaxed_isolation or absolute_gap" > $O/${TAG}_pytest.log 2>&1; echo "pytest exit $?" >> $O/${TAG}_pytest.log
bash tools/gpu_ab.sh $TAG RELAX 0 0.5 "$@"
