# A/B of two library builds on the chunk-product kernel: parity subset on B, launch times from a short ncu list, C4 value
mkdir -p gpurun_out
HEI_LIB_PATH=abl/lib_b.so timeout 1200 python -m pytest tests -m gpu -q -x -k "configs or random or shapes or chunk or coeff or weights" 2>&1 | tail -1
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-baseline --no-latency"
for v in a b; do
  HEI_LIB_PATH=abl/lib_$v.so HEI_PROFILE_STEPS=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:"k_chunk_dot_rows|k_mask_acc_c" --log-file gpurun_out/dot_$v.csv $CMD > /dev/null 2>&1
  echo "$v: $(grep "k_chunk_dot_rows\|k_mask_acc_c" gpurun_out/dot_$v.csv | awk -F'","' '{print $(NF-2), $NF}' | tr '\n' ' ')"
done
for rep in 1 2 3; do for v in a b; do
  HEI_LIB_PATH=abl/lib_$v.so timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$v c4', round(d['value'],1), d.get('bit_exact_vs_reference'))"
done; done
