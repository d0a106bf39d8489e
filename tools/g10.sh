O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > $O/g10_pytest_gpu.txt 2>&1
timeout 300 python __graft_entry__.py > $O/g10_smoke.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/memcheck_paths.py > $O/g10_memcheck.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/racecheck_paths.py > $O/g10_racecheck.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python tools/racecheck_paths.py > $O/g10_synccheck.txt 2>&1
