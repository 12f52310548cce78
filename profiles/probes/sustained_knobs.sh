# Concurrency knobs under the sustained power cap (100-step C4 runs)
mkdir -p gpurun_out
run() {
  env "$@" timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$*', 'c4', round(d['value'],1), d.get('bit_exact_vs_reference'), 'mhz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'))"
}
for rep in 1 2; do
  run HEI_X=0
  run HEI_TWO_STREAMS=0
  run HEI_FOLD_PARTS=3
  run HEI_FOLD_PARTS=4
  run HEI_KS_CARVE=-1
done
