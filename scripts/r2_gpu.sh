#!/usr/bin/env bash
# Round-2 GPU pass: default bench line, ncu launch list of the headline, and
# full ncu captures of the exact pr kernel (k_prx, relabeled rmat24 rounds)
# and of k_bm_twc (sssp rmat24).  Outputs under gpurun_out/${TAG}_*.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r2k}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 1500 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/${TAG}_bench.json
FAST="--steps 1 --warmup 2 --no-e2e --no-cpu-baseline --extra '' --no-ablation --no-configs --no-heavy"
if [ "${NCU:-1}" = 1 ]; then
  eval timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
     --log-file gpurun_out/${TAG}_launches.csv python bench.py $FAST > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  eval timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_prx --launch-skip 360 -c 2 \
     -o gpurun_out/${TAG}_prx_prof -f python bench.py --app pr $FAST > gpurun_out/${TAG}_ncu_prx.log 2>&1; echo "ncu prx rc=$?"
  eval timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bm_twc --launch-skip 18 -c 9 \
     -o gpurun_out/${TAG}_twc_prof -f python bench.py $FAST > gpurun_out/${TAG}_ncu_twc.log 2>&1; echo "ncu twc rc=$?"
fi
