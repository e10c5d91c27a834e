# A/B of library build variants (tools/ab_build.py; VARS="prev base ...",
# base = the in-tree library): C2 fast + fixed frames, C5 fast frame and the
# 8-way band of C5 (plain / stream / in-kernel seam)
for v in ${VARS:-prev base}; do
  L=$PWD/paper_2507_11794_b200/_lib/var_$v.so; [ $v = base ] && L=$PWD/paper_2507_11794_b200/_lib/libclothsim_b200.so
  echo "== $v"
  CLOTHSIM_LIB=$L CS_MODES=fast,fixed timeout 120 python tools/modes_bench.py C2 50
  CLOTHSIM_LIB=$L CS_MODES=fast timeout 200 python tools/modes_bench.py C5 20
  CLOTHSIM_LIB=$L timeout 300 python tools/band_overhead.py 100 8 | tail -3
done
