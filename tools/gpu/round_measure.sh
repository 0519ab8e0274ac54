#!/bin/bash
# Round measurement on the GPU box: gpu tests, bench (product + reference arm), warm per-kernel
# times of the three regimes, ncu launch list of the driver window (W=5, K=20).
# usage: tools/gpu/round_measure.sh TAG
TAG=$1
python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_gputests.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench exit $?" >> gpurun_out/${TAG}_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
for w in 5 200 3000; do python tools/kprof.py --warmup $w --steps 20 > gpurun_out/${TAG}_kprof_w$w.txt 2>&1; done
python tools/window.py 5 20 > gpurun_out/${TAG}_window.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${TAG}_window_w5k20_launches.csv \
    python tools/window.py 5 20 > gpurun_out/${TAG}_window_ncu.log 2>&1
python tools/window_summary.py gpurun_out/${TAG}_window_w5k20_launches.csv 5 "driver window (W=5, K=20), config 5 at J=12, $TAG" > gpurun_out/${TAG}_window_w5k20_summary.txt 2>&1
gzip -f gpurun_out/${TAG}_window_w5k20_launches.csv
tail -2 gpurun_out/${TAG}_gputests.log; head -c 600 gpurun_out/${TAG}_bench.json; echo; tail -3 gpurun_out/${TAG}_bench.err; head -5 gpurun_out/${TAG}_window_w5k20_summary.txt
# ncu --set full of the window's dominant kernels at step 15 (summaries only; the reports stay in /tmp)
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"k_stream_fallback|k_stream_collide|k_virtual|k_transfer|k_details|k_project|k_fallback_v" \
    -o /tmp/${TAG}_win15_full -f python tools/window.py 15 1 > gpurun_out/${TAG}_win15_ncu.log 2>&1
python tools/ncu_summary.py /tmp/${TAG}_win15_full.ncu-rep > gpurun_out/${TAG}_win15_ncu_summary.txt 2>&1
# the 3D engine: per-kernel times and an ncu --set full of one step at J=8
MRLBM_E3_PROF=1 python tools/window3d.py 30 20 > gpurun_out/${TAG}_d3q6_prof.txt 2>&1
ncu --set full --clock-control none --profile-from-start off -k regex:"k3_stream_collide|k3_recon|k3_need_seed|k3_transfer|k3_details" \
    -o /tmp/${TAG}_d3q6_full -f python tools/window3d.py 30 1 > gpurun_out/${TAG}_d3q6_ncu.log 2>&1
python tools/ncu_summary.py /tmp/${TAG}_d3q6_full.ncu-rep > gpurun_out/${TAG}_d3q6_ncu_summary.txt 2>&1
tail -14 gpurun_out/${TAG}_d3q6_prof.txt
