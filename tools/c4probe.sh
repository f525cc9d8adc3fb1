# C4 (m=p=8192, n=65536, k=8: r=2, 20 chunks) raster / L2-hint sweep on one B200.
# Each line: group_m hint_a hint_b -> emulated TFLOPS, GEMM ms, INT8 TOPS, SM MHz (bench.py,
# CUDA events), then ncu DRAM read GB and L2 read sectors for one launch.
set -u
SHAPE=${SHAPE:-"--m 8192 --n 65536 --p 8192"}
B="python bench.py --no-cpu --no-cublas --no-e2e --steps 3 --warmup 3 $SHAPE"
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['roofline']['kernel_ms'],2), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"; }
# CFGS: ';'-separated "group_m hint_a hint_b" triples
IFS=';' read -ra LIST <<< "${CFGS:-2 2 0;2 0 0;4 0 0;6 0 0;4 2 0;8 0 0;6 0 2}"
for cfg in "${LIST[@]}"; do
  IFS=' ' read -r g ha hb <<< "$cfg"; set -- $g $ha $hb
  v=$(OZMM_GROUP_M=$1 OZMM_HINT_A=$2 OZMM_HINT_B=$3 $B 2>/dev/null | j)
  d=$(OZMM_GROUP_M=$1 OZMM_HINT_A=$2 OZMM_HINT_B=$3 ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:ozimmu -c 1 $B --steps 1 --warmup 0 2>&1 | grep -E "dram__|lts__" | awk '{printf "%s=%s ", $1, $3}')
  echo "group=$1 hintA=$2 hintB=$3 -> $v | $d"
done
