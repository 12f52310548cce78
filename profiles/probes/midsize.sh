# mid-size batches: shared-memory vs TMEM key switch (fused next digit below 592 blocks)
mkdir -p gpurun_out
for r in 2 3 4 6 8 16; do for v in 0 4; do
  HEI_KS_TMEM=$v timeout 300 python bench.py --rows $r --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/mid_$r_$v.json 2>/dev/null
  python -c "import json,sys;d=json.loads(open('gpurun_out/mid_$r_$v.json').read().strip().splitlines()[-1]);print('rows=$r tmem=$v', round(d['value'],1), round(d['ms_per_step'],3), d['client_roundtrip']['decrypted_equals_integer_product'])" >> gpurun_out/mid.log 2>&1
done; done
