O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > $O/g38_pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py > $O/g38_smoke.txt 2>&1
timeout 400 python bench.py > $O/g38_bench.json 2> $O/g38_bench.err
