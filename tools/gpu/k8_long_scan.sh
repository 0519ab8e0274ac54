#!/bin/bash
# K8 long-rim threshold scan: graph ms/step and the K8 kernel times per regime
for gap in 0 4 5 6; do
  for w in 5 200 3000; do
    echo "== MRLBM_K8_LONG_GAP=$gap warmup=$w"
    MRLBM_K8_LONG_GAP=$gap python tools/kprof.py --warmup $w --steps 20 | grep -E "^graph|k_stream_fallback(_long)? +[0-9]"
  done
done
