for S in -1 4194304 5592406 8388608 11184811 16777216; do
  for U in "" "--uniform"; do
    python bench.py --app pr --scale 25 $U --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --extra= --no-ablation --pr-block $S 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$S', '$U', round(d['value'],1), round(d['ms_per_step'],1), d['config']['rounds'])"
  done
done
