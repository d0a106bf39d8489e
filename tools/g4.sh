O=gpurun_out; mkdir -p $O
timeout 900 python tools/accuracy_precise.py 32 36 40 > $O/g4_precise.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_dense_real.py tests/test_gpu_batch.py tests/test_gpu_edges.py tests/test_gpu_configs.py -m gpu -q > $O/g4_pytest.txt 2>&1
