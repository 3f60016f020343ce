#!/bin/bash
# tools/ab_steps.sh N RATE "S1 S2 ..." lib1 lib2 ...: ms_per_step for each (step size, lib), two rounds
N=$1; R=$2; SS=$3; shift 3
for round in 1 2; do
  for S in $SS; do
    for lib in "$@"; do
      if [ "$S" = auto ]; then unset HCCX_STEP_SEGS; else export HCCX_STEP_SEGS=$S; fi
      ms=$(HCCX_LIB=$(realpath $lib) timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
           --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 20 --warmup 5 \
           --rate $R --nccl 0 2>&1 | grep -o '"ms_per_step": [0-9.]*')
      echo "N=$N r=$R S=$S $lib $ms"
    done
  done
done
unset HCCX_STEP_SEGS
