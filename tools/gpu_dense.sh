#!/bin/bash
# dense pipeline (NEXT-4): GPU tests and a timing probe
set -u
O=gpurun_out; mkdir -p $O
TAG=${1:-dense}
timeout 1200 python -m pytest tests/test_dense_gpu.py -q -x --durations=10 > $O/${TAG}_pytest.log 2>&1; echo "pytest exit $?" >> $O/${TAG}_pytest.log
timeout 600 python tools/probe_dense.py > $O/${TAG}_probe.log 2>&1; echo "probe exit $?" >> $O/${TAG}_probe.log
