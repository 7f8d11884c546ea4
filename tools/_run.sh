for v in 0 1; do
touch paper_2303_09523_b200/csrc/vk_predict.cu
VK_NVCC_EXTRA="-DVK_FT_F32_MINB3=$v" python paper_2303_09523_b200/build.py > /dev/null 2>&1
for c in C4; do
python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --no-pipelined --config $c --accum fp32 > gpurun_out/b32.json 2>/dev/null
echo "minb3 $v $c fp32: $(grep -o '"launch_ms": [0-9.]*\|"frac": [0-9.]*\|"ms_per_step": [0-9.]*' gpurun_out/b32.json | head -3 | tr '\n' ' ')"
done
done
