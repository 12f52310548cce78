# Round-end evidence at HEAD (run from the repo root on the GPU box).
mkdir -p gpurun_out
TAG=${1:-r01e}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo rc=$? >> gpurun_out/smoke_$TAG.log
bash profiles/capture.sh $TAG > gpurun_out/capture_$TAG.log 2>&1
for c in c1 c2 c3; do
  timeout 600 python bench.py --config $c --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
done
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline --no-latency --no-baseline > gpurun_out/bench_${TAG}_c5.json 2> gpurun_out/bench_${TAG}_c5.err
HEI_PROFILE_STEPS=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_c5.csv python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-baseline --no-latency > /dev/null 2>&1
echo done
