# Refresh every committed bench line and the ncu evidence (run from the repo root on the GPU box).
mkdir -p gpurun_out
TAG=${1:-r01c}
bash profiles/capture.sh $TAG > gpurun_out/capture_$TAG.log 2>&1
for c in c1 c2 c3; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
done
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline --no-latency --no-baseline > gpurun_out/bench_${TAG}_c5.json 2> gpurun_out/bench_${TAG}_c5.err
echo done
