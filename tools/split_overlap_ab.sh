# device entry: B column split on the side stream beside A row split (OZMM_SPLIT_OVERLAP=2) vs only the column maxima (1)
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['ms_per_step'],3))"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 6 --warmup 2"
for shape in "" "--m 8192 --n 8192 --p 8192 --k 6"; do
  line="shape [$shape]:"
  for v in 1 2 1 2 1 2; do line="$line ov$v $(OZMM_SPLIT_OVERLAP=$v $B $shape 2>/dev/null | j)"; done
  echo "$line"
done
