# half-ring dataflow: parity, then C3 latency at 1..4 resident CTAs per SM
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fold_paths" 2>&1 | tail -1
for k in 4 3 2 1; do
  HEI_DF_PER_SM=$k HEI_DATAFLOW=1 timeout 300 python profiles/probes/latency_probe3.py 2>&1 | sed "s/^/per_sm=$k /"
done
HEI_DF_PER_SM=2 HEI_DATAFLOW=1 timeout 300 python profiles/probes/df_trace.py 2>&1 | grep -v rotation | sed "s/^/per_sm=2 /"
