set -u
O=gpurun_out; mkdir -p $O
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "async" 2>&1 | grep -i "assert\|passed\|failed" | tail -3; done
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests.log
