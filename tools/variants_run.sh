#!/bin/bash
# Development tool (GPU box): time every variants/<name>/libvolkrig_b200.so
# with tools/stage_time.py; the in-tree library is restored afterwards.
cd "$(dirname "$0")/.."
N=paper_2303_09523_b200/_native
cp $N/libvolkrig_b200.so /tmp/vk_keep.so
for d in variants/*/; do
  v=$(basename $d)
  [ -f $d/libvolkrig_b200.so ] || continue
  cp $d/libvolkrig_b200.so $N/libvolkrig_b200.so
  VK_VARIANT=$v timeout 300 python tools/stage_time.py ${1:-C4} ${2:-20}
done
cp /tmp/vk_keep.so $N/libvolkrig_b200.so
