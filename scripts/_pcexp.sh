for r in 1 2; do for L in libcpddg.so libcpddg_cs.so libcpddg_nc.so; do
  CPDDG_LIB=$PWD/paper_1909_08734_b200/lib/$L python scripts/pc_time.py 0 | sed "s/^/$L /"
done; done
for L in libcpddg.so libcpddg_cs.so libcpddg_nc.so; do
  CPDDG_LIB=$PWD/paper_1909_08734_b200/lib/$L ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_solve -s 2 -c 1 --csv python scripts/profile_pc_mode.py 0 2>/dev/null | grep k_solve | awk -F'","' '{print "'$L'", $(NF-2), $NF}'
done
