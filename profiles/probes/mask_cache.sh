# mask table A/B + parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "mask_table or production or stream" > gpurun_out/mc_pytest.log 2>&1; echo rc=$? >> gpurun_out/mc_pytest.log
for v in 0 1 0 1; do
  HEI_MASK_CACHE=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/mc_$v.json 2>gpurun_out/mc_$v.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/mc_$v.json').read().strip().splitlines()[-1]);print('mask_cache=$v', round(d['value'],1), d['client_roundtrip']['decrypted_equals_integer_product'])" >> gpurun_out/mc.log 2>&1
done
HEI_MASK_CACHE=1 timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/mc_c5.json 2>gpurun_out/mc_c5.err
python -c "import json,sys;d=json.loads(open('gpurun_out/mc_c5.json').read().strip().splitlines()[-1]);print('c5 mask_cache=1', round(d['value'],1), d['client_roundtrip']['decrypted_equals_integer_product'])" >> gpurun_out/mc.log 2>&1
