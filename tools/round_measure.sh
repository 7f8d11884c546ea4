#!/bin/bash
# Round measurement pass on the GPU box (development tool): the default bench
# line, the reference arm, the mode lines, the other configs, the launch list
# of the bench command and ncu --set full captures of the prediction and fit
# kernels.  Everything lands in gpurun_out/$1/.
cd "$(dirname "$0")/.."
R=gpurun_out/${1:-r02}; mkdir -p $R
python bench.py --steps 20 --warmup 5 > $R/bench_default.jsonl 2> $R/bench_default.err
python bench.py --impl reference --steps 3 --warmup 3 > $R/bench_reference.jsonl 2> $R/bench_reference.err
for m in "--variance" "--drift constant" "--values normalized" "--accum fp32"; do
  n=$(echo $m | tr -d ' -'); python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $m > $R/bench_$n.jsonl 2> $R/bench_$n.err
done
for c in C1 C2 C3 C5; do
  python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $R/bench_$c.jsonl 2> $R/bench_$c.err
done
python bench.py --config C3 --accum fp32 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $R/bench_C3fp32.jsonl 2> $R/bench_C3fp32.err
python bench.py --config C5 --accum fp32 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $R/bench_C5fp32.jsonl 2> $R/bench_C5fp32.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $R/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-pipelined > $R/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:predict_fast_kernel -s 1 -c 1 -o $R/predict \
  python tools/fit_profile_run.py C4 > $R/ncu_predict.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fit_kernel -c 1 -o $R/fit \
  python tools/fit_profile_run.py C4 > $R/ncu_fit.log 2>&1
ncu --set full --clock-control none -k regex:"solve_kernel|plane_stats|npsum_warp|binsq|binsum|pair_draw" -c 12 -o $R/stages \
  python tools/fit_profile_run.py C4 > $R/ncu_stages.log 2>&1
echo done
