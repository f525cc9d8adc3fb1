# MMA execution vs issue overhead: each product's 4 MMAs issued 1x / 2x / 3x (timing only)
set -u
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['roofline']['kernel_ms'],2), d['clocks']['sm_mhz'])"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 3 --warmup 2"
for b in 0 1; do for d in 0 1 2; do echo "batch $b dup=$d: $(OZMM_ONLY_BATCH=$b OZMM_DUP_MMA=$d $B 2>/dev/null | j)"; done; done
