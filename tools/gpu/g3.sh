set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_long.py tests/test_ties.py -m gpu -x -q > gpurun_out/g3_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python tools/kprof.py --config 5 --warmup 5 --steps 20 > gpurun_out/g3_kprof.log 2>&1
MRLBM_K8_WARP=1 timeout 300 python tools/kprof.py --config 5 --warmup 5 --steps 20 > gpurun_out/g3_kprof_k8warp.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/g3_bench.log 2>&1; echo "bench rc=$?"
