set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_long.py tests/test_ties.py -m gpu -x -q > gpurun_out/g4_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python tools/kprof.py --config 5 --warmup 5 --steps 20 > gpurun_out/g4_kprof.log 2>&1
timeout 600 ncu --profile-from-start off --set full --import-source on -k regex:"k_stream_fallback|k_stream_collide" -c 6 --launch-skip 12 -o gpurun_out/g4_k8_mode2 python tools/window.py 5 10 > gpurun_out/g4_ncu.log 2>&1; echo "ncu rc=$?"
