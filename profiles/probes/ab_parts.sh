# C4 value vs the number of concurrent fold slices (HEI_FOLD_PARTS)
mkdir -p gpurun_out
for rep in 1 2; do for v in 2 3 4; do
  HEI_FOLD_PARTS=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('parts=$v c4', round(d['value'],1), d.get('bit_exact_vs_reference'))"
done; done
