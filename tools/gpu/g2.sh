set -x
timeout 2400 python -m pytest tests/test_ties.py tests/test_gpu_windows.py -m gpu -x -q -s > gpurun_out/g2_pytest.log 2>&1; echo "pytest rc=$?"
