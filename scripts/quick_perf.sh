#!/usr/bin/env bash
# Quick GPU iteration: parity subset, headline bench line (no configs /
# ablations), ncu launch list of one SSSP run.  Outputs gpurun_out/${TAG}_*.
set -u
mkdir -p gpurun_out
TAG=${TAG:-q}
export CUDA_DEVICE_MAX_CONNECTIONS=32
if [ "${TESTS:-1}" = 1 ]; then
  timeout 900 python -m pytest ${TESTSEL:-tests/test_gpu_parity.py tests/test_gpu_scale.py} -x -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
fi
FAST="--no-cpu-baseline --no-ablation --no-configs --no-heavy"
timeout 600 python bench.py --steps ${STEPS:-10} --warmup 3 $FAST ${BENCHARGS:-} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/${TAG}_bench.json").read().strip().splitlines()[-1])
print("value", round(d["value"],1), "ms", round(d["ms_per_step"],3), "loop_frac", d["roofline"] and round(d["roofline"]["loop_frac"],3), "frac", d["roofline"] and round(d["roofline"]["frac"],3), "e2e", d["e2e"] and round(d["e2e"]["value"],2))
print({k:(v["launches"], round(v["ms"],3)) for k,v in d["kernel_ms"].items()})
for k,v in d.get("apps",{}).items(): print(k, v.get("gteps"), v.get("ms_per_step"), v.get("labels_match"), v.get("roofline",{}).get("loop_frac"))
PY
if [ "${NCU:-1}" = 1 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
     --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 2 --no-e2e $FAST --extra "" > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
fi
