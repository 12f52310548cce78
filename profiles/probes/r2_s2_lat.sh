# Latency-path evidence: warm per-launch timing, dataflow task trace, and an
# ncu --set full capture of the w2 latency key switch (C3 shape).
mkdir -p gpurun_out
timeout 300 python profiles/probes/latency_probe3.py > gpurun_out/lat_probe.log 2>&1; echo rc=$? >> gpurun_out/lat_probe.log
HEI_DATAFLOW=1 timeout 300 python profiles/probes/latency_probe3.py >> gpurun_out/lat_probe.log 2>&1
timeout 300 python profiles/probes/latency_probe2.py > gpurun_out/lat_probe2.log 2>&1
HEI_DATAFLOW=1 timeout 300 python profiles/probes/df_trace.py > gpurun_out/df_trace.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rot_keyswitch_w2" -s 30 -c 2 \
   -o gpurun_out/full_w2 python profiles/probes/latency_probe2.py > gpurun_out/ncu_w2.log 2>&1
HEI_NO_GRAPHS=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lat.csv \
   python profiles/probes/latency_probe2.py > /dev/null 2>&1
cat gpurun_out/lat_probe.log gpurun_out/lat_probe2.log gpurun_out/df_trace.log; tail -3 gpurun_out/ncu_w2.log
