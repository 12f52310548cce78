# cluster-fused key switch (HEI_KS_CLUSTER=1) vs the two-kernel path: parity, then C4 A/B
mkdir -p gpurun_out
HEI_KS_CLUSTER=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -x -k "fold_paths or c4 or counters" 2>&1 | tail -2
for rep in 1 2; do for v in 0 1; do
  HEI_KS_CLUSTER=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('cluster=$v c4', round(d['value'],1), d.get('bit_exact_vs_reference'), 'ks', round(d['roofline']['avg_launch_ms'],3), 'dig', round(d['roofline']['digits_avg_launch_ms'],3))" 2>&1 | tail -1
done; done
