# K blocks per B buffer for thin passes (OZMM_B_KPB=2) against one (1): value TFLOPS, ms/step
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2))"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 4 --warmup 2"
for shape in "" "--m 8192 --n 8192 --p 8192" "--k 12 --phi 4" "--m 8192 --n 65536 --p 8192"; do
  line="shape [$shape]:"
  for v in 1 2 1 2; do line="$line kpb$v $(OZMM_B_KPB=$v $B $shape 2>/dev/null | j)"; done
  echo "$line"
done
for v in 1 2; do echo "kpb=$v"; OZMM_B_KPB=$v OZMM_TILE_TRACE=1 python bench.py --no-cpu --no-cublas --no-e2e --steps 2 --warmup 1 2>&1 | grep "tile trace" | tail -1; done
