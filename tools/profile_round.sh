#!/bin/bash
# Round profiling bundle (run on the GPU box from the repo root):
#   bench line, the bench command's ncu launch list, and one `ncu --set full`
#   capture per dominant kernel (C2 frame, C5 frame / force / normals, C3
#   detect + respond).  Everything lands in gpurun_out/.
set -u
O=gpurun_out
mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
NCU="ncu --set full --import-source on --clock-control none"
$NCU -k regex:k_pair3 -c 3 -o $O/c2_frame python tools/prof_kernels.py C2 1 > $O/ncu_c2.log 2>&1
$NCU -k regex:k_pair -c 3 -o $O/c5_passes python tools/prof_kernels.py C5 1 > $O/ncu_c5.log 2>&1
# C3: skip the 200 draping frames (one detect + one respond launch each) so the
# captured pair is a frame with the cloth on the sphere
$NCU -k regex:"k_detect|k_respond" --launch-skip 400 -c 2 -o $O/c3_draped python tools/prof_c3.py C3 1 > $O/ncu_c3.log 2>&1
ls -la $O
