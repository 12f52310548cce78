mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "split_key_switch or production_c1" > gpurun_out/ls_pytest.log 2>&1; echo rc=$? >> gpurun_out/ls_pytest.log
for v in "HEI_SPLIT=0" "HEI_SPLIT=2" "HEI_SPLIT=1"; do
  echo "$v $(env $v python profiles/probes/latency_probe.py 2>&1 | tail -1)" >> gpurun_out/lat_split.log
done
HEI_SPLIT=2 HEI_NO_GRAPHS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_split2.csv python profiles/probes/latency_probe2.py > /dev/null 2>&1
