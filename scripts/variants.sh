#!/usr/bin/env bash
# Run the bench for several library builds (SIMTGRAPH_CUDA_LIB) and apps.
# usage: VARIANTS="base var_ku8 ..." APPS="sssp bfs" TAG=x bash scripts/variants.sh
set -u
mkdir -p gpurun_out
out=gpurun_out/${TAG:-var}_variants.jsonl
: > $out
for v in ${VARIANTS:-base}; do
  if [ "$v" = base ]; then lib=paper_1911_09135_b200/_lib/libsimtgraph_cuda.so; else lib=paper_1911_09135_b200/_lib/$v/libsimtgraph_cuda.so; fi
  for app in ${APPS:-sssp}; do
    for sched in ${SCHEDS:-alb}; do
      line=$(SIMTGRAPH_CUDA_LIB=$lib timeout 600 python bench.py --app $app --sched $sched --scale ${SCALE:-24} --steps ${STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline --extra "" --no-ablation ${EXTRA:-} 2>>gpurun_out/${TAG:-var}_variants.err)
      python -c "
import json,sys
d=json.loads(sys.argv[1]); k=d.get('kernel_ms',{})
print(json.dumps({'variant':sys.argv[2],'app':sys.argv[3],'sched':sys.argv[4],'gteps':round(d['value'],1),'ms':round(d['ms_per_step'],3),'kernels':{n:round(x['ms'],3) for n,x in k.items()}}))" "$line" $v $app $sched | tee -a $out
    done
  done
done
