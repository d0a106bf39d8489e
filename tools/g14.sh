O=gpurun_out; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dense_c128_chunks -s 3 -c 1 -o $O/g14_k3 python bench.py --workload haar --steps 1 --warmup 3 --no-cpu-baseline > $O/g14_ncu_k3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dense_c128_pair -s 3 -c 1 -o $O/g14_k3p python bench.py --workload haar --n 44 --steps 1 --warmup 3 --range-log2 34 --no-cpu-baseline > $O/g14_ncu_k3p.log 2>&1
timeout 300 python bench.py --workload haar --no-cpu-baseline > $O/g14_bench_haar32.json 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/g14_pytest_gpu.txt 2>&1
