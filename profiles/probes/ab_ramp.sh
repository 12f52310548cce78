# C4 e2e vs the first host-buffer chunk size (HEI_E2E_RAMP)
mkdir -p gpurun_out
for rep in 1 2; do for v in 8 16 32 4; do
  HEI_E2E_RAMP=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-latency --no-baseline --no-wire > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('ramp=$v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['parity'].get('e2e_packed_equals_reference'))"
done; done
