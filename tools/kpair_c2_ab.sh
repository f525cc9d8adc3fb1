# size heuristic: K pairs on for C blocks <= 8192^2 (default) vs OZMM_KPAIR=0, C2 k=8 and C3
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2))"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 4 --warmup 2"
for shape in "--m 8192 --n 8192 --p 8192" "--m 8192 --n 8192 --p 8192 --k 6" ""; do
  line="default-vs-off [$shape]:"
  for v in d 0 d 0; do if [ $v = d ]; then r=$($B $shape 2>/dev/null | j); else r=$(OZMM_KPAIR=0 $B $shape 2>/dev/null | j); fi; line="$line $v $r"; done
  echo "$line"
done
