O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dense_real.py tests/test_gpu_batch.py tests/test_gpu_edges.py tests/test_gpu_configs.py -m gpu -q -x > $O/g3_pytest.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > $O/g3_bench.json 2>&1
for rb in 4 5 6 8 10; do PK_REBUILD_LOG2=$rb timeout 300 python tools/accuracy_rb.py 36 40 >> $O/g3_accuracy_rb.txt 2>&1; done
