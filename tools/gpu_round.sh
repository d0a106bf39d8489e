#!/bin/bash
# One GPU evidence pass (run under gpurun from the repo root):
# tests, smoke, bench lines for every workload, reference arm, launch list,
# one ncu --set full of K1.
set -x
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench_dense40.json 2> $O/bench_dense40.err
timeout 600 python bench.py --workload binary --no-cpu-baseline > $O/bench_binary40.json 2> $O/bench_binary40.err
timeout 600 python bench.py --workload haar --no-cpu-baseline > $O/bench_haar32.json 2> $O/bench_haar32.err
timeout 600 python bench.py --workload sparse --no-cpu-baseline > $O/bench_sparse40.json 2> $O/bench_sparse40.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_dense40.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_bench.log 2>&1
