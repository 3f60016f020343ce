#!/bin/bash
# tools/ab_env.sh N RATE "ENV1;ENV2;..." lib1 lib2 ...: ms_per_step per (env setting, lib), two rounds.
# ENVk is a space-separated list of VAR=value (or "-" for none).
N=$1; R=$2; IFS=';' read -ra ENVS <<< "$3"; shift 3
for round in 1 2; do
  for e in "${ENVS[@]}"; do
    for lib in "$@"; do
      ms=$(env $( [ "$e" = "-" ] || echo $e ) HCCX_LIB=$(realpath $lib) timeout 300 python -m torch.distributed.run \
           --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py \
           --gpus $N --steps 20 --warmup 5 --rate $R --nccl 0 2>&1 | grep -o '"ms_per_step": [0-9.]*')
      echo "N=$N r=$R [$e] $lib $ms"
    done
  done
done
