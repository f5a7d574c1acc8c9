#!/usr/bin/env bash
mkdir -p gpurun_out
for b in 0 -1 4194304 8388608 11534336 16777216 0; do
  timeout 900 python bench.py --app pr --scale 25 --uniform --pr-block $b --steps 2 --warmup 2 --no-cpu-baseline --no-ablation --no-configs --no-heavy --extra "" --no-e2e > gpurun_out/prb.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/prb.json').read().strip().splitlines()[-1]);print('block $b', round(d['value'],1), round(d['ms_per_step'],1), d['labels']['labels_match'], round(d['roofline']['frac'],3))"
done
