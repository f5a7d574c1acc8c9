# pr source-block size sweep (bench --pr-block S, vertices per block; -1 = no tiling)
# usage: SCALE=25 UNI="--uniform" bash scripts/pr_block_sweep.sh  -> one line per S
for S in ${SIZES:--1 4194304 8388608 11184811 16777216}; do
  python bench.py --app pr --scale ${SCALE:-25} ${UNI:-} --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --extra= --no-ablation --pr-block $S 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'S': $S, 'args': '${UNI:-}', 'gteps': round(d['value'],1), 'ms': round(d['ms_per_step'],1), 'rounds': d['config']['rounds']}))"
done
