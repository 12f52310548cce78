# N = 16384 half-ring key switch: parity subset, then C5 with HEI_KS14_HALF=1 vs 0
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "n16384 or 16384 or c5 or gemv_variants" > gpurun_out/c5h_pytest.log 2>&1; echo rc=$? >> gpurun_out/c5h_pytest.log
for v in ${VARS:-HEI_KS14_HALF=1 HEI_KS14_HALF=0}; do
  env ${v//,/ } timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/c5h.json 2>gpurun_out/c5h.err
  python -c "import json;d=json.loads(open('gpurun_out/c5h.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],1), d['client_roundtrip']['decrypted_equals_integer_product'], round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['digits_avg_launch_ms'],3), d['int_roofline']['frac'])" >> gpurun_out/c5h.log 2>&1 || tail -5 gpurun_out/c5h.err >> gpurun_out/c5h.log
done
