# 4-CTA (A-multicast) kernel vs the pair kernel (bench value, GEMM ms, MHz), plus ncu L2/tensor
set -u
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['roofline']['kernel_ms'],2), d['clocks']['sm_mhz'])"; }
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 5 --warmup 3 ${SHAPE:-}"
for cfg in "pair" "quad" "quad_g2" "quad_s6" "pair" "quad"; do
  case $cfg in
    pair) E="";; quad) E="OZMM_QUAD=1";; quad_g2) E="OZMM_QUAD=1 OZMM_GROUP_M=2";; quad_s6) E="OZMM_QUAD=1 OZMM_STAGES=6";;
  esac
  echo "$cfg: $(env $E $B 2>/dev/null | j)"
done
OZMM_QUAD=1 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:ozimmu -c 1 $B --steps 1 --warmup 0 2>&1 | grep -E "^\s+(gpu__|sm__|lts__|dram__)"
