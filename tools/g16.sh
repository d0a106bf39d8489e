O=gpurun_out; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_configs.py -m gpu -q -k "n48" > $O/g16_pytest_n48.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/g16_launches_dense40.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > $O/g16_ncu_launch.log 2>&1
timeout 300 python bench.py --no-extra --workload binary --no-cpu-baseline > $O/g16_bench_binary40.json 2>/dev/null
timeout 300 python bench.py --no-extra --workload sparse --no-cpu-baseline > $O/g16_bench_sparse40.json 2>/dev/null
