# A-group issue order (interleaved vs sorted) x A-ring depth, C3 (bench value, GEMM ms, MHz)
set -u
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['roofline']['kernel_ms'],2), d['clocks']['sm_mhz'])"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 5 --warmup 3 ${SHAPE:-}"
for cfg in "interleave 4" "sorted 4" "interleave 3" "interleave 5" "interleave 4" "sorted 4"; do
  set -- $cfg
  echo "$1 stages=$2: $(OZMM_AORDER=$1 OZMM_STAGES=$2 $B 2>/dev/null | j)"
done
for o in interleave sorted; do
echo "ncu $o"; OZMM_AORDER=$o ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:ozimmu -c 1 $B --steps 1 --warmup 0 2>&1 | grep -E "^\s+(gpu__|sm__|lts__|dram__)"
done
