export CUDA_DEVICE_MAX_CONNECTIONS=32
mkdir -p gpurun_out
for app in sssp bfs; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --app $app --steps 3 --warmup 3 --no-cpu-baseline --no-ablation --no-configs --no-heavy > gpurun_out/two_rank_$app.json 2> gpurun_out/two_rank_$app.err; echo "$app rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/two_rank_$app.json').read().strip().splitlines()[-1]);print(d['config']['workload'],d['n_gpus'],round(d['value'],1),round(d['ms_per_step'],2),d['labels'],d.get('e2e'))"
done
