#!/usr/bin/env bash
# tools/ab_libs.sh P N lib1 lib2 ...: fused allreduce ms per library build,
# alternating the builds over two rounds (tools/nvl_ab.py, one process each).
P=$1; N=$2; shift 2
for round in 1 2; do
  for lib in "$@"; do
    r=$(HCCX_LIB=$(realpath $lib) timeout 300 torchrun --nproc-per-node $P --master-addr 127.0.0.1 \
        --master-port $((29700 + RANDOM % 200)) tools/nvl_ab.py $N 3 2>&1 | grep median)
    echo "round $round $lib: $r"
  done
done
