mkdir -p gpurun_out
TAG=r01d
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo rc=$? >> gpurun_out/smoke_$TAG.log
bash profiles/capture.sh $TAG > gpurun_out/capture_$TAG.log 2>&1
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline --no-latency --no-baseline > gpurun_out/bench_${TAG}_c5.json 2> gpurun_out/bench_${TAG}_c5.err
echo done
