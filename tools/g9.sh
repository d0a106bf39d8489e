O=gpurun_out; mkdir -p $O
for n in 24 28 32 36 40; do
  for v in 0 1 2; do
    PK_C128_VARIANT=$v timeout 100 python bench.py --workload haar --n $n --steps 3 --no-cpu-baseline > $O/g9_haar_v${v}_$n.json 2>/dev/null
  done
done
timeout 150 python bench.py --workload haar --n 63 --steps 2 --warmup 3 --range-log2 38 --no-cpu-baseline > $O/g9_haar_pair_63.json 2> $O/g9_haar_pair_63.err
timeout 120 python bench.py --workload haar --n 41 --steps 2 --warmup 3 --range-log2 38 --no-cpu-baseline > $O/g9_haar_pair_41.json 2> $O/g9_haar_pair_41.err
timeout 1200 python -m pytest tests/test_gpu_complex_pair.py tests/test_gpu_configs.py tests/test_gpu_complex.py tests/test_gpu_sparse_complex.py tests/test_gpu_batch.py tests/test_gpu_edges.py -m gpu -q > $O/g9_pytest.txt 2>&1
