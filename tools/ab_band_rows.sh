# 8-way band of C5 (plain band engine) over forced strip heights
for h in "$@"; do
  echo "h=$h $(CS_STRIP_ROWS=$h timeout 120 python tools/band_sweep.py 8 100)"
done
echo "model $(timeout 120 python tools/band_sweep.py 8 100)"
