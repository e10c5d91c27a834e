# exact (fixed) mode at C2 over forced strip heights (CS_STRIP_ROWS)
O=gpurun_out/abr; mkdir -p $O
for h in "$@"; do
  CS_STRIP_ROWS=$h CS_MODES=fixed CS_NORMALS=split timeout 200 python tools/modes_bench.py C2 > $O/c2_h$h.txt 2>&1
done
CS_MODES=fixed CS_NORMALS=split timeout 200 python tools/modes_bench.py C2 > $O/c2_model.txt 2>&1
