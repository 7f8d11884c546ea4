for cc in 0 8 3 2; do
VK_CHAIN_CHUNK=$cc python bench.py --steps 40 --warmup 3 --no-e2e --no-cpu-baseline --no-pipelined > gpurun_out/b64.json 2>/dev/null
echo "chunk $cc: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/b64.json | head -1)"
done
for cc in 0 8; do
VK_CHAIN_CHUNK=$cc VK_DIAG_SKIP=3 python bench.py --steps 40 --warmup 3 --no-e2e --no-cpu-baseline --no-pipelined > gpurun_out/b64.json 2>/dev/null
echo "chunk $cc skip fit+solve: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/b64.json | head -1)"
done
