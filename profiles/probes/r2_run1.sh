set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -m gpu 2>&1 | tail -15
timeout 1200 python -m pytest tests -q -m gpu -x --deselect tests/test_gpu_configs.py 2>&1 | tail -8
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.err; tail -2 gpurun_out/r2_bench0.err
