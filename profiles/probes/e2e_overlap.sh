# e2e overlap A/B: consecutive host-buffer chunks concurrent (default) vs serialised
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu2.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu2.log
for v in 1 0 1 0; do
  HEI_E2E_OVERLAP=$v timeout 300 python bench.py --no-cpu-baseline --no-latency --no-baseline > gpurun_out/e2e_ov$v.json 2>/dev/null
  python -c "import json,sys;d=json.loads(open('gpurun_out/e2e_ov$v.json').read().strip().splitlines()[-1]);print('ov=$v', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['wire']['value'],1))" >> gpurun_out/e2e_ov.log
done
for d in 2 3 4 6 8; do
  HEI_E2E_DIV=$d timeout 300 python bench.py --no-cpu-baseline --no-latency --no-baseline --no-wire > gpurun_out/e2e_d$d.json 2>/dev/null
  python -c "import json,sys;d=json.loads(open('gpurun_out/e2e_d$d.json').read().strip().splitlines()[-1]);print('div=$d', round(d['value'],1), round(d['e2e']['value'],1))" >> gpurun_out/e2e_ov.log
done
