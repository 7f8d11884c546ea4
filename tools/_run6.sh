for i in 1 2; do timeout 300 python tools/stage_time.py C4 20 2>&1 | tail -1 | cut -c118-150; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -2
