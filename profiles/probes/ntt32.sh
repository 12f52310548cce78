# 32-residue transforms: parity, then C5 / C4 A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ntt32 or n16384 or ntt_bit_exact" > gpurun_out/n32_pytest.log 2>&1; echo rc=$? >> gpurun_out/n32_pytest.log
grep -q "rc=0" gpurun_out/n32_pytest.log || exit 1
for v in 0 1; do
  HEI_NTT32=$v timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/n32_c5_$v.json 2>gpurun_out/n32_c5_$v.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/n32_c5_$v.json').read().strip().splitlines()[-1]);print('c5 ntt32=$v', round(d['value'],1), d['client_roundtrip']['decrypted_equals_integer_product'], round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['digits_avg_launch_ms'],3))" >> gpurun_out/n32.log 2>&1
done
for v in 0 2; do
  HEI_NTT32=$v timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-latency --no-baseline > gpurun_out/n32_c4_$v.json 2>gpurun_out/n32_c4_$v.err
  python -c "import json,sys;d=json.loads(open('gpurun_out/n32_c4_$v.json').read().strip().splitlines()[-1]);print('c4 ntt32=$v', round(d['value'],1), d['client_roundtrip']['decrypted_equals_integer_product'], round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['digits_avg_launch_ms'],3))" >> gpurun_out/n32.log 2>&1
done
