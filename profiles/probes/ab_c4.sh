# A/B of two library builds (abl/lib_a.so, abl/lib_b.so) on C4 only: parity subset on B, then 3 alternating reps
mkdir -p gpurun_out
HEI_LIB_PATH=abl/lib_b.so timeout 1200 python -m pytest tests -m gpu -q -x -k "${PT_K:-fold or galois or configs or key_switch}" 2>&1 | tail -1
for rep in 1 2 3; do for v in a b; do
  HEI_LIB_PATH=abl/lib_$v.so timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$v c4', round(d['value'],1), d.get('bit_exact_vs_reference'), 'ks', round(d['roofline']['avg_launch_ms'],3), 'dig', round(d['roofline']['digits_avg_launch_ms'],3))"
done; done
