#!/usr/bin/env bash
# One GPU-box pass used during development: virtual-rank parity, multi-process
# NVLink parity, bench at N = 2 and N = the box's GPU count, CTA-0 traces.
#   tools/gpu_check.sh <tag> [tests...]
set -u
tag="${1:-dev}"; shift || true
mkdir -p gpurun_out
export HCCX_TIMEOUT_MS=${HCCX_TIMEOUT_MS:-10000}
ng=$(nvidia-smi -L | wc -l)
python -m pytest ${@:-tests/test_fused_virtual_gpu.py tests/test_nvlink_gpu.py} -x -q --timeout 900 > gpurun_out/${tag}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
python bench.py --gpus 2 > gpurun_out/${tag}_bench_n2.json 2> gpurun_out/${tag}_bench_n2.err
if [ "$ng" -ge 4 ]; then python bench.py --gpus 4 > gpurun_out/${tag}_bench_n4.json 2> gpurun_out/${tag}_bench_n4.err; fi
TRACE_N=67108864 torchrun --nproc-per-node $([ "$ng" -ge 4 ] && echo 4 || echo 2) --master-addr 127.0.0.1 --master-port 29611 tools/nvl_trace.py > gpurun_out/${tag}_trace.log 2>&1
for f in gpurun_out/acc_r*_ar.txt; do mv "$f" "gpurun_out/${tag}_$(basename $f)"; done
true
