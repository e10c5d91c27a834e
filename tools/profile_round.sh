#!/bin/bash
# Round profiling bundle (run on the GPU box from the repo root):
#   the bench line, the bench command's ncu launch list, and one
#   `ncu --set full` capture per dominant kernel:
#     c2_frame   C2 frame (k_pair3<NORMALS=1>)
#     c5_frame   C5 fused frame (k_pair3<NORMALS=1>)
#     c5_split   C5 stand-alone normals + force pass (k_pair_normals, k_pair3<0>)
#     c3_draped  C3 narrow phase + respond of a draped frame (after 200 frames)
#     c2_fixed   C2 exact pair: k_pair_normals_x + guarded exact k_pair3<0,0,0,1>
#     band8      8-way band of C5, self-linked: BAND k_pair3 with the in-kernel seam
#   Everything lands in gpurun_out/; tools/update_profiles.py copies it.
set -u
O=gpurun_out
mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_launches.log 2>&1
NCU="ncu --set full --import-source on --clock-control none"
$NCU -k regex:k_pair3 -c 1 -o $O/c2_frame python tools/prof_kernels.py C2 1 > $O/ncu_c2.log 2>&1
$NCU -k regex:k_pair3 -c 1 -o $O/c5_frame python tools/prof_kernels.py C5 1 > $O/ncu_c5.log 2>&1
# after 5 fused frames the first force pass refreshes the stale normals
# (k_pair_normals) and then runs k_pair3<0>
$NCU -k regex:k_pair -s 5 -c 2 -o $O/c5_split python tools/prof_kernels.py C5 1 > $O/ncu_c5s.log 2>&1
$NCU -k regex:"k_detect|k_respond" -s 400 -c 2 -o $O/c3_draped python tools/prof_c3.py C3 1 > $O/ncu_c3.log 2>&1
# prof_fixed: 3 graph frames (force + forked normals), then the force pass
# (which first refreshes the lagged normals) -- skip 6, capture normals + force
$NCU -k regex:k_pair -s 6 -c 2 -o $O/c2_fixed python tools/prof_fixed.py C2 2 > $O/ncu_fixed.log 2>&1
$NCU -k regex:k_pair3 -s 2 -c 1 -o $O/band8 python tools/prof_band.py 8 4 > $O/ncu_band.log 2>&1
ls -la $O
