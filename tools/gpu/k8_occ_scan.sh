#!/bin/bash
# K8 thread-kernel register budget scan (resident blocks per SM): graph ms/step and K8 times per regime
for occ in 4 5 6; do
  for w in 5 200 3000; do
    echo "== MRLBM_K8_OCC=$occ warmup=$w"
    MRLBM_K8_OCC=$occ python tools/kprof.py --warmup $w --steps 20 | grep -E "^graph|k_stream_fallback(_long)? +[0-9]"
  done
done
