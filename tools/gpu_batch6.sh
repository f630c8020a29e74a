#!/bin/bash
O=gpurun_out
timeout 1700 python -m pytest tests -m gpu -v -x --durations=40 -k "glued or newton or chunk or config3 or config4" > $O/r02n_pytest.log 2>&1
echo "pytest exit $?" >> $O/r02n_pytest.log
