# same-call A/B: old issue (one A group per round, 4-stage ring) vs new defaults (2 per round, 5)
set -u
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2))"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 4 --warmup 2"
for shape in "" "--m 8192 --n 8192 --p 8192" "--m 8192 --n 8192 --p 8192 --k 12" "--k 12 --phi 4" "--m 8192 --n 65536 --p 8192"; do
  o1=$(OZMM_GROUP_PAIRS=1 OZMM_STAGES=4 $B $shape 2>/dev/null | j); n1=$($B $shape 2>/dev/null | j)
  o2=$(OZMM_GROUP_PAIRS=1 OZMM_STAGES=4 $B $shape 2>/dev/null | j); n2=$($B $shape 2>/dev/null | j)
  echo "shape [$shape]: old $o1 $o2 | new $n1 $n2"
done
