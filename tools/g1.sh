O=gpurun_out; mkdir -p $O
nvidia-smi > $O/g1_smi.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > $O/g1_pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py > $O/g1_smoke.txt 2>&1
timeout 600 python bench.py > $O/g1_bench.json 2> $O/g1_bench.err
timeout 600 python bench.py --impl reference > $O/g1_bench_ref.json 2> $O/g1_bench_ref.err
