# frames per graph (CS_GRAPH_FRAMES) x programmatic dependent launch (CS_PDL):
# C2 / C5 fast frames and the 8-way / 4-way bands of C5 (plain, in-kernel seam)
for cfg in "1 0" "4 0" "4 1" "8 1" "2 1"; do
  set -- $cfg
  echo "== frames/graph $1 pdl $2"
  CS_GRAPH_FRAMES=$1 CS_PDL=$2 CS_MODES=fast timeout 60 python tools/modes_bench.py C2 200 2>/dev/null | head -1
  CS_GRAPH_FRAMES=$1 CS_PDL=$2 CS_MODES=fast timeout 90 python tools/modes_bench.py C5 40 2>/dev/null | head -1
  CS_GRAPH_FRAMES=$1 CS_PDL=$2 timeout 120 python tools/band_overhead.py 200 8,4 | cut -c1-140
done
