# Key-switch experiment: HEI_KS_MODE (bit 0 prime-major blocks, bit 1 keys/digits past L1) x HEI_KS_CARVE
mkdir -p gpurun_out
run() {
  env "$@" timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$*', 'c4', round(d['value'],1), d.get('bit_exact_vs_reference'), 'ks', round(d['roofline']['avg_launch_ms'],3), 'dig', round(d['roofline']['digits_avg_launch_ms'],3))"
}
for rep in 1 2; do
  run HEI_KS_MODE=0
  run HEI_KS_MODE=0 HEI_KS_CARVE=43
  run HEI_KS_MODE=1
  run HEI_KS_MODE=2
  run HEI_KS_MODE=3
  run HEI_KS_MODE=3 HEI_KS_CARVE=43
  run HEI_KS_MODE=1 HEI_KS_CARVE=43
done
