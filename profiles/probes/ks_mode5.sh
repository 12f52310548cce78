# Key-switch block-order experiment under the sustained power cap (100-step runs; abl/lib_mode.so = HEAD + ks_mode.patch)
mkdir -p gpurun_out
run() {
  env "$@" HEI_LIB_PATH=abl/lib_mode.so timeout 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$*', 'c4', round(d['value'],1), d.get('bit_exact_vs_reference'), 'mhz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'))"
}
for rep in 1 2; do
  run HEI_KS_MODE=0
  run HEI_KS_MODE=1
  run HEI_KS_MODE=3
  run HEI_KS_MODE=1 HEI_TWO_STREAMS=0
done
