# A-ring depth of the CTA-pair GEMM: bench value / GEMM ms / SM MHz per depth (C3, k=8)
set -u
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['roofline']['kernel_ms'],2), d['clocks']['sm_mhz'])"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 5 --warmup 3 ${SHAPE:-}"
for st in ${STAGES:-6 5 4 6 5}; do echo "stages=$st: $(OZMM_STAGES=$st $B 2>/dev/null | j)"; done
