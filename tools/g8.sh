O=gpurun_out; mkdir -p $O
timeout 120 python -m pytest tests/test_gpu_complex_pair.py -m gpu -q -x -k "not whole" > $O/g8_pytest_pair.txt 2>&1
timeout 100 python -m pytest tests/test_gpu_complex_pair.py -m gpu -q -x -k "whole" >> $O/g8_pytest_pair.txt 2>&1
for n in 28 32 36 40; do
  PK_C128_PAIR=1 timeout 60 python bench.py --workload haar --n $n --steps 3 --no-cpu-baseline > $O/g8_haar_pair_$n.json 2>/dev/null
done
for n in 44 48 63; do
  timeout 90 python bench.py --workload haar --n $n --steps 2 --warmup 3 --range-log2 38 --no-cpu-baseline > $O/g8_haar_pair_$n.json 2>/dev/null
done
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_complex.py tests/test_gpu_edges.py tests/test_gpu_sparse_complex.py tests/test_gpu_batch.py -m gpu -q > $O/g8_pytest.txt 2>&1
