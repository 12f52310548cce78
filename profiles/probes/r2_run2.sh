set -x
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -x -q -m gpu -k "standard or baseline or bad_row" 2>&1 | tail -6
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; tail -3 gpurun_out/r2_bench1.err
timeout 300 python profiles/probes/std_probe.py
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2_std.csv python profiles/probes/std_probe.py > /dev/null 2>&1
python profiles/summarize.py launches gpurun_out/launches_r2_std.csv gpurun_out/launches_r2_std.md; head -30 gpurun_out/launches_r2_std.md
