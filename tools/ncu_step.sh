#!/bin/bash
# On the GPU box: bench once without ncu (must exit 0), then the ncu launch list of the same command.
# usage: tools/ncu_step.sh TAG [extra bench args]
set -e
TAG=$1; shift
python bench.py --steps 1 --warmup 12 --no-cpu --no-steady "$@" > gpurun_out/bench_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 12 --no-cpu --no-steady "$@" > gpurun_out/ncu_$TAG.log 2>&1
python tools/launch_summary.py gpurun_out/launches_$TAG.csv 12 | head -20
