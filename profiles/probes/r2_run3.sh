# full GPU suite + default bench after the kernel-variant prune
set -x
timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -8
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err; tail -3 gpurun_out/r2_bench3.err
python -c "import json; d=json.load(open('gpurun_out/r2_bench3.json')); print(d['value'], d['e2e']['value'], d['e2e']['wire']['value'], d['bit_exact_vs_reference'], d['latency_ms_single_individual'], d['standard_algorithm']['ms'])"
