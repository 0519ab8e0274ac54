set -x
nproc; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/g15_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g15_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/g15_bench.log 2>&1; echo "bench rc=$?"
timeout 300 python tools/kprof.py --config 5 --warmup 5 --steps 20 > gpurun_out/g15_kprof.log 2>&1
timeout 300 python tools/kprof.py --config 5 --warmup 200 --steps 20 > gpurun_out/g15_kprof_settled.log 2>&1
timeout 300 python tools/kprof.py --config 5 --warmup 3000 --steps 20 > gpurun_out/g15_kprof_dev.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g15_window_w5k20.csv python tools/window.py 5 20 > gpurun_out/g15_ncu_window.log 2>&1; echo "ncu rc=$?"
python tools/launch_window.py gpurun_out/g15_window_w5k20.csv > gpurun_out/g15_window_summary.txt
gzip -f gpurun_out/g15_window_w5k20.csv
