# A/B of the full-batch key switch: shared-memory accumulators (0) vs TMEM
# (2: 2 CTAs/SM, 3: 3 CTAs/SM 8-slot rounds, 4: 3 CTAs/SM 4-slot rounds)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "key_switch_variants or sum_all_slots or production" > gpurun_out/kst_pytest.log 2>&1; echo rc=$? >> gpurun_out/kst_pytest.log
for v in ${KS_VARIANTS:-0 3 4 3 4}; do
  HEI_KS_TMEM=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/kst$v.json 2>gpurun_out/kst$v.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/kst$v.json').read().strip().splitlines()[-1]);print('tmem=$v', round(d['value'],1), d['client_roundtrip']['decrypted_equals_integer_product'], round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['digits_avg_launch_ms'],3), round(d['int_roofline']['frac'],3))" >> gpurun_out/kst.log 2>&1
done
