O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi_device.py tests/test_gpu_configs.py tests/test_gpu_sparse_real.py tests/test_gpu_sparse_complex.py tests/test_gpu_complex.py tests/test_gpu_batch.py -m gpu -q > $O/g6_pytest.txt 2>&1
timeout 600 python bench.py > $O/g6_bench_dense40.json 2> $O/g6_bench_dense40.err
timeout 600 python bench.py --workload binary --no-cpu-baseline > $O/g6_bench_binary40.json 2>&1
timeout 600 python bench.py --workload haar --no-cpu-baseline > $O/g6_bench_haar32.json 2>&1
timeout 600 python bench.py --workload sparse --no-cpu-baseline > $O/g6_bench_sparse40.json 2>&1
timeout 600 python bench.py --n 36 --no-cpu-baseline > $O/g6_bench_dense36.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/g6_launches_dense40.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/g6_ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dense_f64_chunks -s 3 -c 1 -o $O/g6_k1 python bench.py --steps 1 --warmup 3 --range-log2 36 --no-cpu-baseline > $O/g6_ncu_k1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spa_f64 -s 3 -c 1 -o $O/g6_spa python bench.py --workload sparse --steps 1 --warmup 3 --range-log2 36 --no-cpu-baseline > $O/g6_ncu_spa.log 2>&1
