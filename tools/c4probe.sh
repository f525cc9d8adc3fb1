set -u
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 3 --warmup 3 --m 8192 --n 65536 --p 8192"
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['roofline']['kernel_ms'],2), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"; }
echo "C4 default: $($B 2>/dev/null | j)"
echo "C4 quad: $(OZMM_QUAD=1 $B 2>/dev/null | j)"
for g in 1 4 8; do echo "C4 group=$g: $(OZMM_GROUP_M=$g $B 2>/dev/null | j)"; done
echo "C4 quad group4: $(OZMM_QUAD=1 OZMM_GROUP_M=4 $B 2>/dev/null | j)"
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes.sum --clock-control none -k regex:ozimmu -c 1 $B --steps 1 --warmup 0 2>&1 | grep -E "^\s+(gpu__|sm__|lts__|dram__|l1tex__)"
