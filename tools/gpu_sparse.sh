O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse_real.py -q -x --durations=10 > $O/pytest_sparse.txt 2>&1
timeout 600 python bench.py --workload sparse --no-cpu-baseline > $O/bench_sparse40.json 2> $O/bench_sparse40.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:spa_f64 -s 3 -c 1 -o $O/spa_f64_full python bench.py --workload sparse --steps 1 --warmup 3 --range-log2 36 --no-cpu-baseline > $O/ncu_spa.log 2>&1
