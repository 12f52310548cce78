#!/bin/bash
# Round-2 evidence (run from the repo root on the GPU box): tests, smoke,
# bench lines for C1-C5 and the reference arm, then the ncu launch lists and
# `--set full` captures, each ncu pass only after the same command has exited
# 0 without ncu. Outputs go to gpurun_out/ (summarised into profiles/ by
# profiles/summarize.py).
set -u
T=r02
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$T.log 2>&1; echo rc=$? >> gpurun_out/pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo rc=$? >> gpurun_out/smoke_$T.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${T}_c4.json 2> gpurun_out/bench_${T}_c4.err || exit 1
for c in c1 c2 c3; do
  timeout 600 python bench.py --config $c --steps 1000 --warmup 20 --no-cpu-baseline > gpurun_out/bench_${T}_$c.json 2> gpurun_out/bench_${T}_$c.err
done
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline --no-latency --no-baseline > gpurun_out/bench_${T}_c5.json 2> gpurun_out/bench_${T}_c5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${T}_ref.json 2> gpurun_out/bench_${T}_ref.err
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-baseline --no-latency"
$CMD > gpurun_out/plain.json 2>/dev/null || exit 2
HEI_PROFILE_STEPS=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${T}_c4.csv $CMD > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_rot_keyswitch_t|k_rot_digits_f" -s 60 -c 2 \
    -o gpurun_out/full_${T}_c4 $CMD > gpurun_out/ncu_full_c4.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_chunk_dot_rows|k_mask_acc_c" -s 4 -c 2 \
    -o gpurun_out/full_${T}_c4_hbm $CMD > gpurun_out/ncu_full_hbm.log 2>&1
python profiles/probes/latency_probe2.py > /dev/null 2>&1 || exit 3
HEI_NO_GRAPHS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${T}_latency.csv \
    python profiles/probes/latency_probe2.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_rot_keyswitch_w2" -s 30 -c 2 \
    -o gpurun_out/full_${T}_w2 python profiles/probes/latency_probe2.py > gpurun_out/ncu_full_w2.log 2>&1
C5="python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-baseline --no-latency"
HEI_PROFILE_STEPS=1 timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${T}_c5.csv $C5 > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_rot_keyswitch_h|k_rot_digits_h" -s 60 -c 2 \
    -o gpurun_out/full_${T}_c5 $C5 > gpurun_out/ncu_full_c5.log 2>&1
echo done
