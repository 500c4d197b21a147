#!/bin/bash
# Fig. 11-style ablation on real B200s: for each failure count and
# micro-batch count, the same workload under (i) coupled 1F1B (the paper's DeepSpeed
# baseline), (ii) Decoupled BackProp with a global optimizer barrier and (iii) Decoupled
# BackProp + Staggered Optimizer.  One JSON line per run in gpurun_out/ablation/.
#   tools/ablation.sh NGPUS "M_LIST" "FAILURE_LIST"
N=${1:-4}
MS=${2:-"1 2 4"}
FS=${3:-"0 1"}
mkdir -p gpurun_out/ablation
port=29600
for m in $MS; do
  for f in $FS; do
    for plan in coupled no-stagger staggered; do
      flag=""
      [ "$plan" = coupled ] && flag="--coupled"
      [ "$plan" = no-stagger ] && flag="--no-stagger"
      port=$((port + 1))
      out=gpurun_out/ablation/n${N}_m${m}_f${f}_${plan}.json
      timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port $port bench.py --gpus $N --steps 5 --warmup 3 --microbatches $m --failures $f $flag \
        --no-e2e --no-cpu-baseline > ${out%.json}.log 2>&1
      grep '"metric"' ${out%.json}.log > $out
      python -c "import json;d=json.load(open('$out'));print('$plan m=$m f=$f', round(d['value']), round(d['ms_per_step'],2), d['predicted_period_units'])" 2>/dev/null || echo "$plan m=$m f=$f FAILED"
    done
  done
done
