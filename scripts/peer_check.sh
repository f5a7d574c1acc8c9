#!/usr/bin/env bash
# GPU pass for the NVLink peer transport: its GPU tests, the full GPU suite,
# and bench.py under torchrun with 2 ranks (on one GPU the ranks share it:
# a functional check of the N>1 path, not a scaling number).
set -u
mkdir -p gpurun_out
TAG=${TAG:-r2p}
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
for app in ${APPS:-sssp bfs cc pr kcore}; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 \
    --master-port=29533 bench.py --gpus 2 --steps 2 --warmup 1 --scale ${SCALE:-20} --app $app \
    > gpurun_out/${TAG}_bench2_${app}.json 2> gpurun_out/${TAG}_bench2_${app}.err
  echo "bench2 $app rc=$?"; head -c 700 gpurun_out/${TAG}_bench2_${app}.json; echo
done
