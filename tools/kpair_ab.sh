# thin passes in K-block pairs (OZMM_KPAIR=1: runs of 8 MMAs per accumulator) vs 0
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2))"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 4 --warmup 2"
for shape in "" "--m 8192 --n 8192 --p 8192" "--k 12 --phi 4" "--m 8192 --n 65536 --p 8192"; do
  line="shape [$shape]:"
  for v in 0 1 0 1; do line="$line kpair$v $(OZMM_KPAIR=$v $B $shape 2>/dev/null | j)"; done
  echo "$line"
done
for v in 0 1; do echo "kpair=$v"; OZMM_KPAIR=$v OZMM_TILE_TRACE=1 python bench.py --no-cpu --no-cublas --no-e2e --steps 2 --warmup 1 2>&1 | grep "tile trace" | tail -1; done
