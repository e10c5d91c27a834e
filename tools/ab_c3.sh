# C3/C4 collision frame A/B over narrow-phase build variants (tools/ab_build.py)
O=gpurun_out/ab3; mkdir -p $O
for v in "$@"; do
  L=$PWD/paper_2507_11794_b200/_lib/var_$v.so
  [ "$v" = base ] && L=$PWD/paper_2507_11794_b200/_lib/libclothsim_b200.so
  CLOTHSIM_LIB=$L timeout 200 python tools/prof_c3.py C3 50 > $O/c3_$v.txt 2>&1
  CLOTHSIM_LIB=$L timeout 200 python tools/prof_c3.py C4 50 > $O/c4_$v.txt 2>&1
done
