export CUDA_DEVICE_MAX_CONNECTIONS=32
for app in ${APPS:-sssp bfs cc pr kcore}; do
for mode in ${MODES:-"" "--peer"}; do
timeout 600 python bench.py --app $app --steps 5 --warmup 3 --no-cpu-baseline --no-ablation --no-configs --no-heavy --extra "" $mode > gpurun_out/peer1_$app.json 2>gpurun_out/peer1.err; echo "rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/peer1_$app.json").read().strip().splitlines()[-1])
print("$app", "$mode" or "sg_run", round(d["value"],1), round(d["ms_per_step"],3), d["labels"].get("labels_match"), "e2e", d["e2e"] and round(d["e2e"]["value"],2), d["config"]["parallelism"][:40])
PY
done; done
