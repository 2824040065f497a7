bash tools/ab_so.sh 3
cp paper_1008_0502_b200/libgc_B.so paper_1008_0502_b200/libgc.so
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
