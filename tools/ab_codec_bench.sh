#!/usr/bin/env bash
# tools/ab_codec_bench.sh lib1 lib2 ...: bench.py N=1 (codec round trip) per
# library build, two alternating rounds; prints value / compress / decompress.
for round in 1 2; do
  for lib in "$@"; do
    HCCX_LIB=$(realpath $lib) python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('round $round $lib', d['value'], d['detail']['compress_ms'], d['detail']['decompress_ms'], d['roofline']['frac'], d['parity']['payload_bit_exact'])"
  done
done
