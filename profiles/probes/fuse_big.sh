# A/B: separate digit kernel (0) vs next-digit INTT fused into the TMEM key switch (1)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "key_switch_variants" > gpurun_out/fb_pytest.log 2>&1; echo rc=$? >> gpurun_out/fb_pytest.log
for v in 0 1 0 1; do
  HEI_FUSE_BIG=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/fb$v.json 2>gpurun_out/fb$v.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/fb$v.json').read().strip().splitlines()[-1]);print('fuse_big=$v', round(d['value'],1), d['client_roundtrip']['decrypted_equals_integer_product'], round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['digits_avg_launch_ms'],3))" >> gpurun_out/fb.log 2>&1
done
