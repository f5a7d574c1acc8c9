mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_bm_twc --launch-skip 2 -c 2 -o gpurun_out/twc -f python bench.py --app sssp --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ablation --no-configs --no-heavy --extra "" > gpurun_out/twc.log 2>&1; echo "rc=$?"
ncu -i gpurun_out/twc.ncu-rep --page details --csv > gpurun_out/twc_details.csv 2>/dev/null
ncu -i gpurun_out/twc.ncu-rep --page source --csv --print-source sass > gpurun_out/twc_src.csv 2>/dev/null
ncu -i gpurun_out/twc.ncu-rep --page raw --csv > gpurun_out/twc_raw.csv 2>/dev/null
rm -f gpurun_out/twc.ncu-rep
ls -la gpurun_out/twc*
