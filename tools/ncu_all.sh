# ncu --set full of each workload's dominant kernel (one launch each)
O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dense_f64_chunks -s 3 -c 1 -o $O/k1_final python bench.py --steps 1 --warmup 3 --range-log2 36 --no-cpu-baseline > $O/ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dense_c128_chunks -s 3 -c 1 -o $O/k3_final python bench.py --workload haar --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:spa_f64 -s 3 -c 1 -o $O/spa_final python bench.py --workload sparse --steps 1 --warmup 3 --range-log2 36 --no-cpu-baseline > $O/ncu2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:spa_int -s 3 -c 1 -o $O/k6_final python bench.py --workload binary --steps 1 --warmup 3 --range-log2 36 --no-cpu-baseline > $O/ncu6.log 2>&1
