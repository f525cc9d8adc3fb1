# per-batch time of the fused GEMM at C3 (OZMM_ONLY_BATCH: timing only, wrong results) + ncu
set -u
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['roofline']['kernel_ms'],2), d['clocks']['sm_mhz'])"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 5 --warmup 3 ${SHAPE:-}"
echo "all: $($B 2>/dev/null | j)"
for b in 0 1; do echo "batch $b only: $(OZMM_ONLY_BATCH=$b $B 2>/dev/null | j)"; done
echo "all: $($B 2>/dev/null | j)"
for b in 0 1; do
echo "ncu batch $b"; OZMM_ONLY_BATCH=$b ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,lts__cycles_elapsed.avg.per_second --clock-control none -k regex:ozimmu -c 1 $B --steps 1 --warmup 0 2>&1 | grep -E "^\s+(gpu__|sm__|lts__|dram__)"
done
