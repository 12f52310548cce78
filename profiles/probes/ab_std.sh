# A/B of two library builds on the standard algorithm (C3), client encryption and the C3 latency
mkdir -p gpurun_out
HEI_LIB_PATH=abl/lib_b.so timeout 1200 python -m pytest tests -m gpu -q -x -k "${PT_K:-baseline or standard or encrypt or ntt or weights or coeff or wire or keygen or decrypt}" 2>&1 | tail -1
for rep in 1 2; do for v in a b; do
  HEI_LIB_PATH=abl/lib_$v.so timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);s=d['standard_algorithm'];print('$v c4', round(d['value'],1), 'std ms', round(s['ms'],2), s['bit_exact_vs_reference'], 'enc ms', round(s['client_encrypt']['ms'],2), 'lat', round(d['latency_single_individual']['ms'],4), 'keygen', round(d['client_roundtrip']['keygen_ms'],1))"
done; done
