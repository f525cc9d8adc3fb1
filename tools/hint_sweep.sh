# L2 policy hints of the slice loads (0 normal, 1 evict_first, 2 evict_last) at the default raster;
# bench value / GEMM ms / MHz, then ncu DRAM read per launch
set -u
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['roofline']['kernel_ms'],2), d['clocks']['sm_mhz'])"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 5 --warmup 3 ${SHAPE:-}"
for cfg in ${CFGS:-"2,0" "0,0" "0,1" "2,1" "1,0"}; do
  IFS=',' read -r ha hb <<< "$cfg"
  d=$(OZMM_HINT_A=$ha OZMM_HINT_B=$hb ncu --metrics dram__bytes_read.sum --clock-control none -k regex:ozimmu -c 1 $B --steps 1 --warmup 0 2>&1 | grep dram__ | awk '{print $3}')
  echo "hintA=$ha hintB=$hb: $(OZMM_HINT_A=$ha OZMM_HINT_B=$hb $B 2>/dev/null | j) dramGB $d"
done
