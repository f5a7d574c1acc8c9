# relabel parity tests + hot-set size sweep (SG_HOT_K) on rmat24; outputs in gpurun_out/
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "relabel or larger_scale" > gpurun_out/relabel_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/relabel_tests.log
for K in ${KS:-off default}; do
  if [ "$K" = default ]; then timeout 300 python scripts/hotk_sweep.py ${SCALE:-24} >> gpurun_out/hotk.jsonl 2>>gpurun_out/hotk.err
  else SG_HOT_K=$K timeout 300 python scripts/hotk_sweep.py ${SCALE:-24} >> gpurun_out/hotk.jsonl 2>>gpurun_out/hotk.err; fi
done
cat gpurun_out/hotk.jsonl
