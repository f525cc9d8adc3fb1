# same-box A/B of the device GEMM: current build vs another libozmm_b200.so ($1), probe_r2 configs ($2)
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/cur.so
for v in cur alt cur alt; do
  if [ $v = alt ]; then cp $1 $L; else cp /tmp/cur.so $L; fi
  echo "== $v"; python tools/probe_r2.py --cfg $2 --rounds 1 --reps 3 2>&1 | grep TOPS
done
cp /tmp/cur.so $L
