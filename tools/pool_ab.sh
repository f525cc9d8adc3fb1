# pool build (per-pass B buffers / A ring) vs the committed build ($1), same call; batch 0 probe
set -u
bash tools/ab_lib.sh $1
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['roofline']['kernel_ms'],2), d['clocks']['sm_mhz'])"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 3 --warmup 2"
for cfg in "3 8" "3 7" "2 8" "3 6"; do set -- $cfg
  echo "batch0 nb=$1 na=$2: $(OZMM_ONLY_BATCH=0 OZMM_THIN_BBUFS=$1 OZMM_THIN_STAGES=$2 $B 2>/dev/null | j)"; done
echo "batch1: $(OZMM_ONLY_BATCH=1 $B 2>/dev/null | j)"
