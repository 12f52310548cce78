set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fold_paths or c1_shape or graph_replay or wire_path_byte or random_shapes" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_configs.py -q -m gpu -x -k "c1 or c2 or c3" 2>&1 | tail -3
python profiles/probes/df_trace.py
timeout 300 python profiles/probes/latency_probe3.py
