# A/B of the generated SpaRyser integer kernels (config 3 workload)
O=gpurun_out
for mode in 0 2; do
  PK_SPA_INT_FLOAT=$mode timeout 300 python bench.py --workload binary --no-cpu-baseline --steps 3 > $O/bin_m${mode}.json 2> $O/bin_m${mode}.err
done
PK_SPA_INT_FLOAT=2 timeout 600 python -m pytest tests/test_gpu_integer.py tests/test_preprocess.py -q -x -m gpu > $O/pytest_int.txt 2>&1
PK_SPA_INT_FLOAT=2 timeout 600 ncu --set full --import-source on --clock-control none -k regex:spa_int -s 3 -c 1 -o $O/k6m2_full python bench.py --workload binary --steps 1 --warmup 3 --range-log2 36 --no-cpu-baseline > $O/ncu_k6m2.log 2>&1
