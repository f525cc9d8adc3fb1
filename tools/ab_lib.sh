# same-call A/B of the current build against another libozmm_b200.so ($1), several configs
set -u
ALT=$1
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2))"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 4 --warmup 2"
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/cur.so
for shape in "" "--m 8192 --n 8192 --p 8192" "--k 12 --phi 4" "--m 8192 --n 65536 --p 8192"; do
  line="shape [$shape]:"
  for v in cur alt cur alt; do
    if [ $v = alt ]; then cp $ALT $L; else cp /tmp/cur.so $L; fi
    line="$line $v $($B $shape 2>/dev/null | j)"
  done
  echo "$line"
done
cp /tmp/cur.so $L
