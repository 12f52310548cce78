mkdir -p gpurun_out
for v in "${ENV_A:-X=0}" "${ENV_B:-X=1}"; do
  env $v timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/c5ab.json 2>gpurun_out/c5ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/c5ab.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],1), d['client_roundtrip']['decrypted_equals_integer_product'], round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['digits_avg_launch_ms'],3))" >> gpurun_out/c5ab.log 2>&1
done
