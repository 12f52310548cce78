mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "chunk_products or mask_table or production" > gpurun_out/dr_pytest.log 2>&1; echo rc=$? >> gpurun_out/dr_pytest.log
for v in 0 1 0 1; do
  HEI_DOT_ROWS=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/dr_$v.json 2>gpurun_out/dr_$v.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/dr_$v.json').read().strip().splitlines()[-1]);print('dot_rows=$v', round(d['value'],1), d['client_roundtrip']['decrypted_equals_integer_product'])" >> gpurun_out/dr.log 2>&1
done
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-baseline --no-latency"
HEI_PROFILE_STEPS=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dr.csv $CMD > /dev/null 2>&1
