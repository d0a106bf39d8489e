O=gpurun_out; mkdir -p $O
timeout 600 python tools/accuracy_precise.py 32 36 40 > $O/g45_precise.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/g45_pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py > $O/g45_smoke.txt 2>&1
timeout 400 python bench.py > $O/g45_bench.json 2> $O/g45_bench.err
