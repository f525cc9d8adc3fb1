# G=2 issue rounds x A-ring depth, C3 (+ ncu DRAM / tensor), C4 depth
set -u
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['roofline']['kernel_ms'],2), d['clocks']['sm_mhz'])"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 5 --warmup 3"
for cfg in "2 4" "2 5" "2 6" "2 5" "2 4" "1 4"; do set -- $cfg
  echo "C3 G=$1 stages=$2: $(OZMM_GROUP_PAIRS=$1 OZMM_STAGES=$2 $B 2>/dev/null | j)"; done
for st in 5 6; do
echo "ncu G=2 stages=$st"; OZMM_GROUP_PAIRS=2 OZMM_STAGES=$st ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:ozimmu -c 1 $B --steps 1 --warmup 0 2>&1 | grep -E "^\s+(gpu__|sm__|lts__|dram__)"
done
for st in 6 8; do echo "C4 G=2 stages=$st: $(OZMM_GROUP_PAIRS=2 OZMM_STAGES=$st $B --m 8192 --n 65536 --p 8192 2>/dev/null | j)"; done
