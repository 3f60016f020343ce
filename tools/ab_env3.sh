#!/bin/bash
# tools/ab_env3.sh N RATE ROUNDS "ENV1;ENV2;..." : ms_per_step per env setting, interleaved rounds
N=$1; R=$2; ROUNDS=$3; IFS=';' read -ra ENVS <<< "$4"
for round in $(seq $ROUNDS); do
  for e in "${ENVS[@]}"; do
    ms=$(env $( [ "$e" = "-" ] || echo $e ) timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
         --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 30 --warmup 5 \
         --rate $R --nccl 0 2>&1 | grep -o '"ms_per_step": [0-9.]*' | cut -d' ' -f2)
    echo "[$e] $ms"
  done
done
