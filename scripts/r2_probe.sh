mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | head -20
free -g
./scripts/micro/seqsum > gpurun_out/r2_seqsum.jsonl 2>&1; cat gpurun_out/r2_seqsum.jsonl
timeout 300 python scripts/host_probe.py > gpurun_out/r2_host_probe.json 2>&1; cat gpurun_out/r2_host_probe.json
