# Session-2 status at HEAD: full GPU test suite, smoke, default bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s2_pytest.log 2>&1; echo rc=$? >> gpurun_out/s2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2_smoke.log 2>&1; echo rc=$? >> gpurun_out/s2_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err; echo rc=$? >> gpurun_out/s2_bench.err
tail -3 gpurun_out/s2_pytest.log; tail -2 gpurun_out/s2_smoke.log; tail -2 gpurun_out/s2_bench.err
