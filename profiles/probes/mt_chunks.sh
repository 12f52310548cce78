# Standard algorithm (C3) vs the number of mt19937_64 chunk generators per branch (HEI_MT_CHUNKS, default 128)
mkdir -p gpurun_out
for rep in 1 2; do for v in 128 256 512 1024 2048; do
  HEI_MT_CHUNKS=$v timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-latency > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);s=d['standard_algorithm'];print('chunks $v std ms', round(s['ms'],2), s['bit_exact_vs_reference'], 'enc ms', round(s['client_encrypt']['ms'],2), 'keygen', round(d['client_roundtrip']['keygen_ms'],1))"
done; done
