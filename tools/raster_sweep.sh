# raster group / L2 hint / A-ring depth sweep of the CTA-pair GEMM (bench value, GEMM ms, MHz)
set -u
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['roofline']['kernel_ms'],2), d['clocks']['sm_mhz'])"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 5 --warmup 3 ${SHAPE:-}"
IFS=';' read -ra LIST <<< "${CFGS:-4 2 2;4 1 2;4 3 2;4 4 2;4 2 0;4 1 0;3 2 2;4 2 2}"
for cfg in "${LIST[@]}"; do
  IFS=' ' read -r st g ha <<< "$cfg"
  echo "stages=$st group=$g hintA=$ha: $(OZMM_STAGES=$st OZMM_GROUP_M=$g OZMM_HINT_A=$ha $B 2>/dev/null | j)"
done
