# slicers without the last slice's residual update (w -= x is dead after slice k): A/B of the
# row split (cluster kernel) and the two-pass column split at C3 and C2, alternating builds
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
for round in 1 2; do
for v in base lastslice; do
  cp tools/_alt/$v.so $L
  echo "== $v (round $round)"
  python tools/cols_probe.py 2>&1 | grep -iE "row|two|default|GB/s"
  python tools/cols_probe.py --n 8192 --p 8192 2>&1 | grep -iE "row|two|default|GB/s"
done
done
cp /tmp/rel.so $L
