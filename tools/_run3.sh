R=gpurun_out/s4f; mkdir -p $R
timeout 1200 python -m pytest tests -m gpu -x -q > $R/gputests.log 2>&1; echo tests rc=$?; tail -3 $R/gputests.log
for c in C4 C5 C2; do timeout 300 python tools/stage_time.py $c 20 2>&1 | tail -1 | cut -c1-220; done
