# Key-switch experiment, part 3: more reps of the four candidates (10 timed steps each)
mkdir -p gpurun_out
run() {
  env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$*', 'c4', round(d['value'],1), d.get('bit_exact_vs_reference'), 'mhz', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'))"
}
nvidia-smi -q -d POWER | grep -i "limit\|draw" | head -8
for rep in 1 2; do
  run HEI_KS_MODE=0
  run HEI_KS_MODE=0 HEI_KS_CARVE=43
  run HEI_KS_MODE=3 HEI_KS_CARVE=43
  run HEI_KS_MODE=3 HEI_KS_CARVE=43 HEI_TWO_STREAMS=0
done
