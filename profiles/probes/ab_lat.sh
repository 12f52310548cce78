# A/B of two library builds on the single-individual latency (C3) only, plus fold-path parity on B
mkdir -p gpurun_out
HEI_LIB_PATH=abl/lib_b.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fold_paths or production" 2>&1 | tail -1
for rep in 1 2 3; do for v in a b; do
  HEI_LIB_PATH=abl/lib_$v.so HEI_DATAFLOW=0 timeout 300 python profiles/probes/latency_probe3.py 2>&1 | sed "s/^/$v /"
done; done
