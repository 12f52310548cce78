# A/B of two builds of the product library (abl/lib_a.so vs abl/lib_b.so):
# GPU parity tests on B, then C4 value and C3 latency for both, interleaved.
mkdir -p gpurun_out
: > gpurun_out/ab_lib.log
if [ -n "${PT_K:-}" ]; then
  HEI_LIB_PATH=abl/lib_b.so timeout 1200 python -m pytest tests -m gpu -q -x -k "$PT_K" > gpurun_out/ab_pytest.log 2>&1; echo rc=$? >> gpurun_out/ab_pytest.log
  tail -2 gpurun_out/ab_pytest.log >> gpurun_out/ab_lib.log
fi
for rep in 1 2; do for v in a b; do
  HEI_LIB_PATH=abl/lib_$v.so timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$v c4', round(d['value'],1), d['client_roundtrip']['decrypted_equals_integer_product'], d.get('bit_exact_vs_reference'), 'ks', round(d['roofline']['avg_launch_ms'],3), 'dig', round(d['roofline']['digits_avg_launch_ms'],3))" >> gpurun_out/ab_lib.log 2>&1
  HEI_LIB_PATH=abl/lib_$v.so timeout 300 python profiles/probes/latency_probe3.py 2>&1 | sed "s/^/$v /" >> gpurun_out/ab_lib.log
done; done
cat gpurun_out/ab_lib.log
