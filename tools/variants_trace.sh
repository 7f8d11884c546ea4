#!/bin/bash
# Development tool (GPU box): chain traces of every variants/<name>/ library
# (slowest fit completion after the fork, 3 runs each) plus stage times.
cd "$(dirname "$0")/.."
N=paper_2303_09523_b200/_native
cp $N/libvolkrig_b200.so /tmp/vk_keep.so
for d in variants/*/; do
  v=$(basename $d)
  cp $d/libvolkrig_b200.so $N/libvolkrig_b200.so
  for i in 1 2 3; do
    VK_CHAIN_TRACE=1 timeout 300 python tools/chain_timeline.py ${1:-C4} > /tmp/tr.log 2>&1
    n=$(grep -n "fork at" /tmp/tr.log | tail -1 | cut -d: -f1)
    echo "$v run $i: $(tail -n +$n /tmp/tr.log | head -1) slowest $(tail -n +$n /tmp/tr.log | grep chain | awk '{print $8}' | sort -n | tail -1)"
  done
  VK_VARIANT=$v timeout 300 python tools/stage_time.py ${1:-C4} 20
done
cp /tmp/vk_keep.so $N/libvolkrig_b200.so
