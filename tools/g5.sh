O=gpurun_out; mkdir -p $O
timeout 900 python tools/accuracy_precise.py 32 36 40 > $O/g5_precise.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > $O/g5_bench.json 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $O/g5_pytest.txt 2>&1
