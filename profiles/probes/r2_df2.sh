# dataflow v2 (K + RD tasks): parity, C3 latency, task trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fold_paths" > gpurun_out/df2_pytest.log 2>&1; echo rc=$? >> gpurun_out/df2_pytest.log
tail -2 gpurun_out/df2_pytest.log
HEI_DATAFLOW=1 timeout 300 python profiles/probes/latency_probe3.py 2>&1 | sed "s/^/df2 /"
HEI_DATAFLOW=1 timeout 300 python profiles/probes/df_trace.py 2>&1 | sed "s/^/df2 /"
HEI_DATAFLOW=0 timeout 300 python profiles/probes/latency_probe3.py 2>&1 | sed "s/^/graph /"
