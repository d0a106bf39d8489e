O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > $O/g23_pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py > $O/g23_smoke.txt 2>&1
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/memcheck_paths.py > $O/g23_memcheck.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/racecheck_paths.py > $O/g23_racecheck.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python tools/racecheck_paths.py > $O/g23_synccheck.txt 2>&1
timeout 400 python bench.py > $O/g23_bench.json 2> $O/g23_bench.err
