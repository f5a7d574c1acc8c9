for args in "--scale 25" "--scale 25 --uniform" "--scale 24" "--scale 24 --uniform"; do
  python bench.py --app pr $args --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --extra= --no-ablation 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$args', round(d['value'],1), round(d['ms_per_step'],1), d['config']['rounds'], {k: round(v['ms'],1) for k,v in d['kernel_ms'].items()})"
done
