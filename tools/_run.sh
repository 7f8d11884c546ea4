python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
python bench.py --steps 50 --warmup 3 --no-e2e --no-cpu-baseline --no-pipelined > gpurun_out/b64.json 2>/dev/null
echo "C4 fp64: $(grep -o '"ms_per_step": [0-9.]*\|"solve": [0-9.]*' gpurun_out/b64.json | head -2 | tr '\n' ' ')"
for c in C2 C3; do
python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --no-pipelined --config $c > gpurun_out/bc.json 2>/dev/null
echo "$c fp64: $(grep -o '"ms_per_step": [0-9.]*\|"solve": [0-9.]*' gpurun_out/bc.json | head -2 | tr '\n' ' ')"
done
