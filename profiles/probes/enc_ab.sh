mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "baseline or encode or encrypt or keygen" > gpurun_out/enc_pytest.log 2>&1; echo rc=$? >> gpurun_out/enc_pytest.log
for rep in 1 2; do for v in ${VARS:-HEI_ENC_MINB=2 HEI_ENC_MINB=3}; do
  env ${v//,/ } timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-latency > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);s=d['standard_algorithm'];print('$v', round(d['value'],1), round(s['ms'],2), round(s['client_encrypt']['ms'],2), d['client_roundtrip']['decrypted_equals_integer_product'])" >> gpurun_out/enc_ab.log 2>&1 || tail -3 gpurun_out/ab.err >> gpurun_out/enc_ab.log
done; done
