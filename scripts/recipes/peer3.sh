export CUDA_DEVICE_MAX_CONNECTIONS=32
mkdir -p gpurun_out
T='tests/test_gpu_peer.py::test_peer_ranks_as_threads'
for i in 1 2; do timeout 600 python -m pytest "$T" -x -q -m gpu -k "False and bfs and rmat12" > gpurun_out/peer3_new_$i.log 2>&1; echo "new $i rc=$?"; tail -n 1 gpurun_out/peer3_new_$i.log; done
timeout 1500 python -m pytest tests/test_gpu_peer.py -x -q -m gpu > gpurun_out/peer2_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/peer2_pytest.log
SG_PEER_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/peerncu_launches.csv python bench.py --app ${APP:-sssp} --peer --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-ablation --no-configs --no-heavy --extra "" > gpurun_out/peerncu.log 2>&1; echo "rc=$?"
