# C1-C3 bench lines with a timed region long enough for nvidia-smi clock samples
mkdir -p gpurun_out
TAG=${1:-r01c}
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo rc=$? >> gpurun_out/smoke_$TAG.log
for c in c1 c2 c3; do
  timeout 600 python bench.py --config $c --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
done
