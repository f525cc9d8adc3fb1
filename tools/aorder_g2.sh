# A-group order under two-group issue rounds: default (interleaved for k <= 8) vs forced sorted
set -u
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2))"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 4 --warmup 2"
for shape in "" "--m 8192 --n 8192 --p 8192" "--m 8192 --n 8192 --p 8192 --k 6" "--k 10 --phi 4"; do
  echo "shape [$shape]: default $($B $shape 2>/dev/null | j) $($B $shape 2>/dev/null | j) | sorted $(OZMM_AORDER=sorted $B $shape 2>/dev/null | j) $(OZMM_AORDER=sorted $B $shape 2>/dev/null | j)"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "chunk_sums or random or large" 2>&1 | tail -1
