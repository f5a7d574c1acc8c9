#!/usr/bin/env bash
# BASELINE.json configs C3-C5 on one B200 (C2 = the default bench line).
# Output: gpurun_out/${TAG}_configs.jsonl (one bench JSON line per config).
set -u
mkdir -p gpurun_out
out=gpurun_out/${TAG:-cfg}_configs.jsonl
: > $out
run() {
  timeout ${TO:-900} python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline --no-e2e --extra "" "$@" \
    >> $out 2>> gpurun_out/${TAG:-cfg}_configs.err
  echo "rc=$? $*"
}
# CONFIGS: ';'-separated bench argument lists (default: C3-C5)
IFS=';' read -ra LIST <<< "${CONFIGS:---app cc --scale 25;--app pr --scale 25;--app pr --scale 25 --uniform;--app bfs --scale 27;--app kcore --scale 27}"
for c in "${LIST[@]}"; do
  run $c
done
python - "$out" <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    d = json.loads(ln)
    ab = d.get("ablation_alb_vs_twc", {})
    print(d["config"]["workload"], round(d["value"], 1), "GTEPS", round(d["ms_per_step"], 2), "ms",
          {k: round(v["alb_over_twc"], 3) for k, v in ab.items()})
PY
