# Key-switch experiment at HEAD (library built with profiles/probes/ks_mode.patch as abl/lib_mode.so)
mkdir -p gpurun_out
run() {
  env "$@" HEI_LIB_PATH=abl/lib_mode.so timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$*', 'c4', round(d['value'],1), d.get('bit_exact_vs_reference'), 'ks', round(d['roofline']['avg_launch_ms'],3), 'mhz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'))"
}
for rep in 1 2 3; do
  run HEI_KS_MODE=0
  run HEI_KS_MODE=3
  run HEI_KS_MODE=3 HEI_TWO_STREAMS=0
done
