set -u
OZMM_QUAD=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for g in 2 4; do
  v=$(OZMM_QUAD=1 OZMM_GROUP_M=$g timeout 300 python bench.py --no-cpu --no-cublas --no-e2e --steps 8 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])")
  echo "quadA group=$g: $v"
  OZMM_QUAD=1 OZMM_GROUP_M=$g ncu --metrics dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum --clock-control none -k regex:ozimmu -c 1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-cublas 2>&1 | grep -E "dram__|tensor|duration"
done
v=$(timeout 300 python bench.py --no-cpu --no-cublas --no-e2e --steps 8 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])")
echo "pair (default): $v"
