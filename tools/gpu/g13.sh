set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_long.py -m gpu -x -q > gpurun_out/g13_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python tools/kprof.py --config 5 --warmup 5 --steps 20 > gpurun_out/g13_kprof.log 2>&1
MRLBM_K8_THREAD=1 timeout 300 python tools/kprof.py --config 5 --warmup 5 --steps 20 > gpurun_out/g13_kprof_thread.log 2>&1
timeout 300 python tools/kprof.py --config 5 --warmup 3000 --steps 20 > gpurun_out/g13_kprof_dev.log 2>&1
