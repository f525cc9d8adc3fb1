# per-tile fixed cost: same tiles (m = p = 16384), same schedule (k = 8, r >= 8), inner dimension n varied
set -u
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['roofline']['kernel_ms'],2), d['clocks']['sm_mhz'])"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 3 --warmup 2"
for n in 2048 4096 8192 16384; do echo "n=$n: $($B --n $n 2>/dev/null | j)"; done
for n in 2048 4096 8192 16384; do echo "batch0 n=$n: $(OZMM_ONLY_BATCH=0 $B --n $n 2>/dev/null | j)"; done
