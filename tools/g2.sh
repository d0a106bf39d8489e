O=gpurun_out; mkdir -p $O
./tools/proto_cvt > $O/g2_cvt.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -rA --durations=10 > $O/g2_pytest_configs.txt 2>&1
for rb in 4 6 8 10; do PK_REBUILD_LOG2=$rb timeout 300 python tools/accuracy_rb.py 36 40 >> $O/g2_accuracy_rb.txt 2>&1; done
