set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_dense_gpu.py -q -x > $O/dense5_pytest.log 2>&1; echo "pytest exit $?" >> $O/dense5_pytest.log
timeout 600 python tools/probe_dense.py 1024 2048 4096 > $O/dense5_probe.log 2>&1
timeout 900 python bench.py --other-configs= --emulate-world= --no-zstore --no-e2e > $O/dense5_bench.json 2> $O/dense5_bench.err; echo "bench exit $?" >> $O/dense5_bench.err
