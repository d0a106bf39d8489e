O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_complex_pair.py tests/test_gpu_configs.py tests/test_gpu_complex.py tests/test_gpu_edges.py -m gpu -q > $O/g7_pytest.txt 2>&1
for n in 24 28 32 36 40; do
  timeout 300 python bench.py --workload haar --n $n --steps 3 --no-cpu-baseline > $O/g7_haar_k3_$n.json 2>/dev/null
  PK_C128_PAIR=1 timeout 300 python bench.py --workload haar --n $n --steps 3 --no-cpu-baseline > $O/g7_haar_pair_$n.json 2>/dev/null
done
for n in 44 48 63; do
  timeout 300 python bench.py --workload haar --n $n --steps 2 --warmup 3 --range-log2 38 --no-cpu-baseline > $O/g7_haar_pair_$n.json 2>/dev/null
done
