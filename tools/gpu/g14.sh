set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/g14_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g14_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/g14_bench.log 2>&1; echo "bench rc=$?"
timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/g14_bench_ref.log 2>&1; echo "ref rc=$?"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g14_window_w5k20.csv python tools/window.py 5 20 > gpurun_out/g14_ncu_window.log 2>&1; echo "ncu rc=$?"
python tools/launch_window.py gpurun_out/g14_window_w5k20.csv > gpurun_out/g14_window_summary.txt
gzip -f gpurun_out/g14_window_w5k20.csv
