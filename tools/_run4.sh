for c in 6 10 15 22; do for g in "15,9,6,4" "5,5,5,15"; do
  echo "cap $c guide $g"; VK_FT_CAP=$c VK_FT_GUIDE=$g timeout 300 python tools/stage_time.py C4 20 2>&1 | tail -1 | cut -c118-140
done; done
