set -x
nproc; lscpu | grep "Model name"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/g1_bench.log 2>&1; echo "bench rc=$?"
timeout 300 python tools/kprof.py --config 5 --warmup 5 --steps 20 > gpurun_out/g1_kprof_w5.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g1_window_w5k20.csv python tools/window.py 5 20 > gpurun_out/g1_ncu_window.log 2>&1; echo "ncu rc=$?"
