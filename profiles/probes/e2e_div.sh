# e2e (host-buffer C ABI path) vs HEI_E2E_DIV on the default C4 bench
mkdir -p gpurun_out
for rep in 1 2; do for v in ${VARS:-HEI_E2E_DIV=4 HEI_E2E_DIV=2 HEI_E2E_DIV=8}; do
  env $v timeout 300 python bench.py --no-cpu-baseline --no-latency --no-baseline > gpurun_out/e2e.json 2>gpurun_out/e2e.err
  python -c "import json;d=json.loads(open('gpurun_out/e2e.json').read().strip().splitlines()[-1]);print('$v', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['wire']['value'],1))" >> gpurun_out/e2e.log 2>&1 || tail -3 gpurun_out/e2e.err >> gpurun_out/e2e.log
done; done
