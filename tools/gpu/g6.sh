set -x
timeout 900 ncu --profile-from-start off --set full -k regex:"k_stream_fallback|k_virtual|k_stream_collide" -c 16 --launch-skip 240 -o gpurun_out/g6_step20 python tools/window.py 5 17 > gpurun_out/g6_ncu.log 2>&1; echo "ncu rc=$?"
bash tools/gpu/ncu_export.sh gpurun_out/g6_step20.ncu-rep k_stream_fallback
MRLBM_K8_WARP=1 timeout 900 ncu --profile-from-start off --set full -k regex:"k_stream_fallback" -c 1 --launch-skip 15 -o gpurun_out/g6_step20_k8warp python tools/window.py 5 17 > gpurun_out/g6_ncu2.log 2>&1; echo "ncu rc=$?"
bash tools/gpu/ncu_export.sh gpurun_out/g6_step20_k8warp.ncu-rep
ls -la gpurun_out
