mkdir -p gpurun_out/s2
o=gpurun_out/s2/ab.log; : > $o
for v in head new head new; do cp scripts/ablib/libcpddg_$v.so paper_1909_08734_b200/lib/libcpddg.so; echo "== $v" >> $o; timeout 60 python scripts/pc_time.py 0 >> $o 2>&1; done
cp scripts/ablib/libcpddg_new.so paper_1909_08734_b200/lib/libcpddg.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s2/parity_ab.log 2>&1
