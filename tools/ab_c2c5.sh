O=gpurun_out/ab; mkdir -p $O
for v in base r14 r16; do
  L=$PWD/paper_2507_11794_b200/_lib/var_$v.so
  CLOTHSIM_LIB=$L timeout 120 python tools/prof_kernels.py C2 50 > $O/c2_$v.txt 2>&1
  CLOTHSIM_LIB=$L timeout 200 python tools/prof_kernels.py C5 20 > $O/c5_$v.txt 2>&1
  for h in 4 5 6 8; do CS_STRIP_ROWS=$h CLOTHSIM_LIB=$L timeout 120 python tools/prof_kernels.py C2 50 > $O/c2_${v}_h$h.txt 2>&1; done
done
