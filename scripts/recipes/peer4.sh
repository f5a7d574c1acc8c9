export CUDA_DEVICE_MAX_CONNECTIONS=32
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_peer.py -x -q -m gpu > gpurun_out/peer2_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/peer2_pytest.log
MODES="--peer" APPS="${APPS:-kcore}" bash scripts/recipes/peer1.sh
for app in ${NCUAPPS:-kcore}; do
SG_PEER_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/peerncu_$app.csv python bench.py --app $app --peer --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-ablation --no-configs --no-heavy --extra "" > gpurun_out/peerncu_$app.log 2>&1; echo "$app ncu rc=$?"
done
