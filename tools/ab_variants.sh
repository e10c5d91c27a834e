# A/B of library build variants (tools/ab_build.py; VARS="base v1 v2 ...",
# base = the in-tree library): C2 / C5 fast frames and the 8-way / 4-way
# bands of C5 (plain, stream and in-kernel seam)
for v in ${VARS:-base}; do
  L=$PWD/paper_2507_11794_b200/_lib/var_$v.so; [ $v = base ] && L=$PWD/paper_2507_11794_b200/_lib/libclothsim_b200.so
  echo "== $v"
  CLOTHSIM_LIB=$L CS_MODES=fast timeout 60 python tools/modes_bench.py C2 200 2>/dev/null | head -1
  CLOTHSIM_LIB=$L CS_MODES=fast timeout 90 python tools/modes_bench.py C5 48 2>/dev/null | head -1
  CLOTHSIM_LIB=$L timeout 150 python tools/band_overhead.py 200 8,4 | cut -c1-140
done
