# issue order: back-to-back products into one accumulator avoided (OZMM_AVOID_RAW) or not
set -u
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['roofline']['kernel_ms'],2))"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 3 --warmup 2"
for r in 0 1 0 1; do echo "batch0 avoid_raw=$r: $(OZMM_ONLY_BATCH=0 OZMM_AVOID_RAW=$r $B 2>/dev/null | j)"; done
for r in 0 1 0 1; do echo "C3 avoid_raw=$r: $(OZMM_AVOID_RAW=$r $B 2>/dev/null | j)"; done
for r in 0 1; do echo "C5k12 avoid_raw=$r: $(OZMM_AVOID_RAW=$r $B --k 12 --phi 4 2>/dev/null | j)"; done
OZMM_AVOID_RAW=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "chunk_sums or random" 2>&1 | tail -1
