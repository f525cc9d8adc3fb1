for cfg in "4 0 0" "2 2 0" "2 2 1" "3 2 0" "4 2 0" "1 2 0" "2 0 0"; do
  set -- $cfg
  v=$(OZMM_GROUP_M=$1 OZMM_HINT_A=$2 OZMM_HINT_B=$3 timeout 300 python bench.py --no-cpu --no-cublas --no-e2e --steps 8 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.2f %.1f %s' % (d['value'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz']))")
  d=$(OZMM_GROUP_M=$1 OZMM_HINT_A=$2 OZMM_HINT_B=$3 ncu --metrics dram__bytes_read.sum --clock-control none -k regex:ozimmu -c 1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-cublas 2>&1 | grep dram__ | awk '{print $3}')
  echo "group=$1 hintA=$2 hintB=$3 -> TFLOPS/kernel_ms/MHz: $v  dramGB: $d"
done
