# A/B of two library builds: fold/parity GPU tests on B, C4 value, C3/R=2 latency, standard algorithm at C3
mkdir -p gpurun_out
HEI_LIB_PATH=abl/lib_b.so timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for rep in 1 2; do for v in a b; do
  HEI_LIB_PATH=abl/lib_$v.so timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-latency > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$v c4', round(d['value'],1), d.get('bit_exact_vs_reference'), 'std_ms', round(d['standard_algorithm']['ms'],2))"
  HEI_LIB_PATH=abl/lib_$v.so timeout 300 python profiles/probes/latency_probe3.py 2>&1 | sed "s/^/$v /"
done; done
