# exact normals kernel (fixed mode, split) over forced strip heights, C2 and C5
O=gpurun_out/abn; mkdir -p $O
for h in "$@"; do
  CS_NRMX_ROWS=$h CS_MODES=fixed timeout 200 python tools/modes_bench.py C2 50 > $O/c2_h$h.txt 2>&1
  CS_NRMX_ROWS=$h CS_MODES=fixed timeout 300 python tools/modes_bench.py C5 10 > $O/c5_h$h.txt 2>&1
done
