for r in 1 2; do
for L in libcpddg.so libcpddg_prev.so; do
  CPDDG_LIB=$PWD/paper_1909_08734_b200/lib/$L python scripts/pc_time.py 0 | sed "s/^/$L /"
done; done
python scripts/spec_compare.py 2>&1 | head -2
