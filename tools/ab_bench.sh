#!/bin/bash
# A/B of libhccx builds on the same box: tools/ab_bench.sh N RATE lib1 lib2 ...
# (interleaved, two rounds; prints ms_per_step per lib)
N=$1; R=$2; shift 2
for round in 1 2; do
  for lib in "$@"; do
    ms=$(HCCX_LIB=$(realpath $lib) timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
         --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 20 --warmup 5 \
         --rate $R --nccl 0 2>&1 | grep -o '"ms_per_step": [0-9.]*')
    echo "N=$N r=$R $lib $ms"
  done
done
