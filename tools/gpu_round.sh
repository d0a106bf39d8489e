#!/bin/bash
# One GPU evidence pass (run under gpurun from the repo root):
# tests, smoke, bench lines for the three workloads, launch list, one ncu --set full.
set -x
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench_dense40.json 2> $O/bench_dense40.err
timeout 600 python bench.py --workload binary --no-cpu-baseline > $O/bench_binary40.json 2> $O/bench_binary40.err
timeout 600 python bench.py --workload haar --no-cpu-baseline > $O/bench_haar32.json 2> $O/bench_haar32.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_dense40.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dense_f64_chunks -s 3 -c 1 \
    -o $O/k1_full python bench.py --steps 1 --warmup 3 --range-log2 36 --no-cpu-baseline > $O/ncu_full.log 2>&1
