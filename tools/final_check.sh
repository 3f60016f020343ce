#!/usr/bin/env bash
# Round-end pass on one box: the full GPU suite, smoke(), and the bench lines
# of both arms at N = 1 and N = every GPU count up to the box's (self-launched).
#   tools/final_check.sh <tag>
set -u
tag="${1:-final}"
mkdir -p gpurun_out
ng=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
for n in 1 2 4 8; do
  [ "$n" -le "$ng" ] || continue
  python bench.py --impl reference --gpus $n > gpurun_out/${tag}_ref_n$n.json 2> gpurun_out/${tag}_ref_n$n.err
  python bench.py --gpus $n > gpurun_out/${tag}_bench_n$n.json 2> gpurun_out/${tag}_bench_n$n.err
done
SMALL_SIZES=4096,65536,262144,1048576 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 tools/nvl_small.py > gpurun_out/${tag}_small_p2.log 2>&1
python -m pytest tests -m gpu -x -q --timeout 1200 > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
true
