# A/B of two library builds: parity subset on B, C4 value + C3 latency, then C5 (1 step)
mkdir -p gpurun_out
HEI_LIB_PATH=abl/lib_b.so timeout 1200 python -m pytest tests -m gpu -q -x -k "${PT_K:-fold or galois or configs or key_switch}" 2>&1 | tail -1
for rep in 1 2; do for v in a b; do
  HEI_LIB_PATH=abl/lib_$v.so timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$v c4', round(d['value'],1), d.get('bit_exact_vs_reference'), 'ks', round(d['roofline']['avg_launch_ms'],3), 'dig', round(d['roofline']['digits_avg_launch_ms'],3))"
  HEI_LIB_PATH=abl/lib_$v.so timeout 300 python profiles/probes/latency_probe3.py 2>&1 | head -1 | sed "s/^/$v /"
done; done
for v in a b; do
  HEI_LIB_PATH=abl/lib_$v.so timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/ab5.json 2>gpurun_out/ab5.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab5.json').read().strip().splitlines()[-1]);print('$v c5', round(d['value'],1), d.get('bit_exact_vs_reference'), d['client_roundtrip']['decrypted_equals_integer_product'])"
done
