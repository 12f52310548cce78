#!/bin/bash
# Measurement recipe for the committed profiles/ evidence (run on the GPU box
# from the repo root): bench lines first, then the ncu launch list and one
# `--set full` capture of the fold kernels, each ncu pass only after the same
# command has exited 0 without ncu. Outputs go to gpurun_out/.
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_${TAG}_c4.json 2> gpurun_out/bench_${TAG}_c4.err || exit 1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-baseline --no-latency"
$CMD > gpurun_out/plain.json 2>/dev/null || exit 2
HEI_PROFILE_STEPS=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_c4.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_rot_keyswitch_[st]|k_rot_digits_f" -s 60 -c 2 \
    -o gpurun_out/full_${TAG}_c4 $CMD > gpurun_out/ncu_full.log 2>&1
python profiles/probes/latency_probe2.py > /dev/null 2>&1 || exit 3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_latency.csv \
    env HEI_NO_GRAPHS=1 python profiles/probes/latency_probe2.py > /dev/null 2>&1
echo done
