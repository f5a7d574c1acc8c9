#!/usr/bin/env bash
# One GPU-box pass: build check, GPU parity tests, smoke, bench line, ncu launch
# list and one full ncu capture of the dominant kernel.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
     --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra "" --no-ablation \
     > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_bm_large_pipe} -c ${NCOUNT:-9} \
     -o gpurun_out/${TAG}_prof -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra "" --no-ablation \
     > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
