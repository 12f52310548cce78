# compute-sanitizer passes over the smoke test (tiny ring + N = 8192 production
# kernels incl. the full-batch TMEM key switch): shared-memory races
# (racecheck, incl. the warp-barrier NTT exchange), barrier misuse
# (synccheck) and out-of-bounds accesses (memcheck)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/san_$tool.log
done
