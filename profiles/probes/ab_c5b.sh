# C5 A/B of two library builds (1 timed step each, twice) + N=16384 parity on B
mkdir -p gpurun_out
HEI_LIB_PATH=abl/lib_b.so timeout 900 python -m pytest tests -m gpu -q -x -k "16384 or c5 or half" 2>&1 | tail -1
for rep in 1 2; do for v in a b; do
  HEI_LIB_PATH=abl/lib_$v.so timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/ab5.json 2>gpurun_out/ab5.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab5.json').read().strip().splitlines()[-1]);print('$v c5', round(d['value'],1), d['client_roundtrip']['decrypted_equals_integer_product'], round(d['roofline'].get('avg_launch_ms'),3), round(d['roofline'].get('digits_avg_launch_ms'),3))"
done; done
