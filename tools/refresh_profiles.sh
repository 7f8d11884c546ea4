# One GPU call that refreshes the round's bench lines and launch lists
# (profiles/ gets the copies; gpurun_out/ is scratch).
set -u
O=gpurun_out/refresh
mkdir -p $O
python bench.py > $O/bench_fp64.jsonl 2> $O/bench_fp64.err
python bench.py --accum fp32 --no-cpu-baseline > $O/bench_fp32.jsonl 2> $O/bench_fp32.err
python bench.py --accum fixed --no-cpu-baseline > $O/bench_fixed.jsonl 2> $O/bench_fixed.err
for c in C2 C3 C5; do python bench.py --config $c --no-cpu-baseline --no-e2e --no-pipelined > $O/bench_${c}_fp64.jsonl 2>/dev/null; done
for c in C3 C5; do python bench.py --config $c --accum fp32 --no-cpu-baseline --no-e2e --no-pipelined > $O/bench_${c}_fp32.jsonl 2>/dev/null; done
# launch lists (ncu only after the same command exited 0 without it)
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-pipelined"
$CMD --serial > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_serial.csv $CMD --serial > $O/ncu_serial.log 2>&1
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_chained.csv $CMD > $O/ncu_chained.log 2>&1
echo bench+launches done
# one full ncu capture per prediction mode (traffic, pipes, stalls) and of
# the stage kernels (solve / fit / bins / pair draw / stats)
NCMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-pipelined --serial"
for m in fp64 fp32; do
  ncu --set full --clock-control none --import-source on -k regex:predict_fast_kernel -s 2 -c 1 \
    -o $O/predict_$m $NCMD --accum $m > $O/ncu_predict_$m.log 2>&1
done
ncu --set full --clock-control none --import-source on -k "regex:(solve|fit|bins|pair_draw|plane_stats)_kernel" \
  -s 10 -c 5 -o $O/stages $NCMD > $O/ncu_stages.log 2>&1
echo ncu done
