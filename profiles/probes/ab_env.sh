# env A/B on the C3 latency (same library): ENV_A vs ENV_B, plus fold-path parity under ENV_B
mkdir -p gpurun_out
env ${ENV_B} timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fold_paths or production" 2>&1 | tail -1
for rep in 1 2 3 4; do for v in "${ENV_A}" "${ENV_B}"; do
  env $v timeout 300 python profiles/probes/latency_probe3.py 2>&1 | sed "s/^/$v /"
done; done
