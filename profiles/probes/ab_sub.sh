# C4 value vs full-batch sub-slicing (HEI_SUBSLICE pairs per digit+key-switch pair of launches)
mkdir -p gpurun_out
HEI_SUBSLICE=128 timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -k "c4" 2>&1 | tail -1
for rep in 1 2; do for v in 0 64 128 256; do
  HEI_SUBSLICE=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('sub=$v c4', round(d['value'],1), d.get('bit_exact_vs_reference'))"
done; done
