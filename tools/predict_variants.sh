# Tuning sweep of the streaming kernel's compile-time shape (COLS WARPS TY MINB).
for cfg in "${@:-4 8 32 2}"; do
  set -- $cfg
  touch paper_2303_09523_b200/csrc/vk_predict.cu
  VK_NVCC_EXTRA="-DVK_FT_COLS=$1 -DVK_FT_WARPS=$2 -DVK_FT_TY=$3 -DVK_FT_MINB=$4" python paper_2303_09523_b200/build.py > /dev/null 2>&1
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var.log 2>&1
  echo "cfg $cfg: $(grep -o '"launch_ms": [0-9.]*' gpurun_out/var.log) $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/var.log)"
done
