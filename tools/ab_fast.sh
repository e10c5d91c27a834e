# fast mode C2 / C5 A/B over build variants (tools/ab_build.py)
O=gpurun_out/abf; mkdir -p $O
for v in "$@"; do
  L=$PWD/paper_2507_11794_b200/_lib/var_$v.so
  [ "$v" = base ] && L=$PWD/paper_2507_11794_b200/_lib/libclothsim_b200.so
  CLOTHSIM_LIB=$L CS_MODES=fast timeout 200 python tools/modes_bench.py C2 100 > $O/c2_$v.txt 2>&1
  CLOTHSIM_LIB=$L CS_MODES=fast timeout 200 python tools/modes_bench.py C5 20 > $O/c5_$v.txt 2>&1
  CLOTHSIM_LIB=$L timeout 200 python tools/prof_kernels.py C2 30 > $O/p2_$v.txt 2>&1
done
