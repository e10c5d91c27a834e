# exact (fixed) mode A/B over build variants (tools/ab_build.py): fused and split normals
O=gpurun_out/abx; mkdir -p $O
for v in "$@"; do
  L=$PWD/paper_2507_11794_b200/_lib/var_$v.so
  [ "$v" = base ] && L=$PWD/paper_2507_11794_b200/_lib/libclothsim_b200.so
  for nm in auto split; do
    CLOTHSIM_LIB=$L CS_MODES=fixed CS_NORMALS=$nm timeout 200 python tools/modes_bench.py C2 > $O/c2_${v}_$nm.txt 2>&1
  done
done
