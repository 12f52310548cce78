# ncu --set full of the C5 half-ring kernels and of C4's HBM-bound kernels (chunk products, mask/pack)
mkdir -p gpurun_out
C5="python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-baseline --no-latency"
C4="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-baseline --no-latency"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_rot_keyswitch_h|k_rot_digits_h" -s 40 -c 2 \
    -o gpurun_out/full_r01_c5 $C5 > gpurun_out/ncu_c5.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_chunk_dot_rows|k_mask_acc_c" -c 2 \
    -o gpurun_out/full_r01_c4_hbm $C4 > gpurun_out/ncu_c4hbm.log 2>&1
echo done
