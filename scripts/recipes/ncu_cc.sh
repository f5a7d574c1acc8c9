# ncu --set full of the cc workloads' dominant kernels after the dense round 0
FAST="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --extra '' --no-ablation --no-configs --no-heavy"
H="--probs 0.8,0.1,0.05,0.05"
mkdir -p gpurun_out/ncu
cap() {  # tag kernel_regex count skip workload bench-args
  eval timeout 900 ncu --set full --clock-control none -k regex:$2 -c $3 --launch-skip $4 -o gpurun_out/$1_prof -f python bench.py $6 $FAST > gpurun_out/$1_ncu.log 2>&1; echo "$1 rc=$?"
  python scripts/ncu_summary.py $1 --workload $5 > /dev/null 2>&1; echo "$1 summary rc=$?"
  cp profiles/$1_ncu.json gpurun_out/ncu/ 2>/dev/null
  rm -f gpurun_out/$1_prof.ncu-rep
}
cap r2aq_cc24 "k_bm_twc" 3 0 cc/rmat24 "--app cc"
cap r2aq_cc25 "k_bm_large_pipe" 3 0 cc/rmat25 "--app cc --scale 25"
cap r2aq_hcc "k_bm_lb" 3 0 cc/heavy24 "--app cc $H"
cp profiles/ncu_summary.json gpurun_out/ncu/ncu_summary.json
