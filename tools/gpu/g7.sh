set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_long.py tests/test_ties.py -m gpu -x -q > gpurun_out/g8_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python tools/kprof.py --config 5 --warmup 5 --steps 20 > gpurun_out/g8_kprof.log 2>&1
timeout 300 python tools/kprof.py --config 5 --warmup 3000 --steps 20 > gpurun_out/g8_kprof_dev.log 2>&1
timeout 900 ncu --profile-from-start off --set full -k regex:"k_stream_fallback|k_virtual" -c 11 --launch-skip 165 -o gpurun_out/g8_step20 python tools/window.py 5 17 > gpurun_out/g8_ncu.log 2>&1; echo "ncu rc=$?"
bash tools/gpu/ncu_export.sh gpurun_out/g8_step20.ncu-rep k_stream_fallback
