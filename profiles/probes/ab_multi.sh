# multi-way A/B: each setting in $VARS (space-separated env assignments, ',' joins several) on the default bench (value only), $REPS rounds + a parity subset
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "${PT_K:-key_switch_variants or production or sum_all}" > gpurun_out/ab_pytest.log 2>&1; echo rc=$? >> gpurun_out/ab_pytest.log
for rep in $(seq ${REPS:-2}); do for v in ${VARS:-X=0}; do
  env ${v//,/ } timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-latency --no-baseline ${BENCH_ARGS:-} > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],1), d['client_roundtrip']['decrypted_equals_integer_product'], round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['digits_avg_launch_ms'],3))" >> gpurun_out/ab.log 2>&1 || tail -3 gpurun_out/ab.err >> gpurun_out/ab.log
done; done
