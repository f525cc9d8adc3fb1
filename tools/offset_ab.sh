# A/B of the offset-binary (u8 x u8) slice planes against the signed planes (bench value, GEMM ms, MHz)
set -u
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['roofline']['kernel_ms'],2), d['clocks']['sm_mhz'], 'e2e', round(d['e2e']['value'],2) if d.get('e2e') else None)"; }
B="python bench.py --no-cpu --no-cublas --steps 5 --warmup 3 --e2e-steps 2 ${SHAPE:-}"
for sg in ${ORDER:-0 1 0 1}; do echo "signed=$sg: $(OZMM_SIGNED=$sg $B 2>/dev/null | j)"; done
