#!/bin/bash
# Development tool (GPU box): bench.py lines (no e2e / CPU baseline) for every
# variants/<name>/ library, fp64 and fp32.
cd "$(dirname "$0")/.."
N=paper_2303_09523_b200/_native
cp $N/libvolkrig_b200.so /tmp/vk_keep.so
for d in variants/*/; do
  v=$(basename $d)
  cp $d/libvolkrig_b200.so $N/libvolkrig_b200.so
  for acc in fp64 fp32; do
    timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --accum $acc 2>/dev/null | \
      python -c "import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v', '$acc', round(d['ms_per_step'],4), 'pred', round(d['roofline']['launch_ms'],4), 'frac', round(d['roofline']['frac'],4), 'pipe', round(d['pipelined']['ms_per_step'],4))"
  done
done
cp /tmp/vk_keep.so $N/libvolkrig_b200.so
