set -x
timeout 1500 ncu --profile-from-start off --set full --import-source on --clock-control none -o gpurun_out/g16_step14 python tools/window.py 14 1 > gpurun_out/g16_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/g16_step14.ncu-rep --page raw --csv > gpurun_out/g16_step14_raw.csv 2>/dev/null
ncu -i gpurun_out/g16_step14.ncu-rep --page source --csv --kernel-name regex:"k_stream_fallback_t" --print-source sass > gpurun_out/g16_k8_sass.csv 2>/dev/null
ncu -i gpurun_out/g16_step14.ncu-rep --page details --csv --kernel-name regex:"k_stream_fallback_t" > gpurun_out/g16_k8_details.csv 2>/dev/null
gzip -f gpurun_out/g16_*.csv
rm -f gpurun_out/g16_step14.ncu-rep
timeout 1200 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_case.py > gpurun_out/g16_memcheck.log 2>&1; echo "memcheck rc=$?"
timeout 1200 compute-sanitizer --tool racecheck python tools/sanitize_case.py > gpurun_out/g16_racecheck.log 2>&1; echo "racecheck rc=$?"
timeout 1200 compute-sanitizer --tool initcheck python tools/sanitize_case.py > gpurun_out/g16_initcheck.log 2>&1; echo "initcheck rc=$?"
