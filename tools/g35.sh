O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > $O/g35_pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py > $O/g35_smoke.txt 2>&1
timeout 400 python bench.py > $O/g35_bench.json 2> $O/g35_bench.err
timeout 400 python bench.py --impl reference > $O/g35_bench_ref.json 2> $O/g35_bench_ref.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dense_c128_pair -s 3 -c 1 -o $O/g35_k3p python bench.py --no-extra --workload haar --n 44 --steps 1 --warmup 3 --range-log2 34 --no-cpu-baseline > $O/g35_ncu_k3p.log 2>&1
