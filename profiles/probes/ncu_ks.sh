mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-baseline --no-latency"
$CMD > gpurun_out/plain.json 2>/dev/null || exit 2
ncu --set full --clock-control none --import-source on -k regex:"k_rot_keyswitch_t" -s 30 -c 1 -o gpurun_out/full_kst $CMD > gpurun_out/ncu_kst.log 2>&1
