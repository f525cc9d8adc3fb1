# ncu DRAM / L2 / clock of the pair GEMM per raster group (C3, k=8; one launch), then bench values
for g in ${GS:-2 4 8}; do
  echo "group=$g"
  OZMM_GROUP_M=$g ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:ozimmu -c 1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-cublas 2>&1 | grep -E "^\s+(gpu__|sm__|lts__|dram__)"
done
j() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['roofline']['kernel_ms'],2), d['clocks']['sm_mhz'])"; }
for g in ${GS:-2 4 8} ${GS:-2 4 8}; do echo "bench group=$g: $(OZMM_GROUP_M=$g python bench.py --no-cpu --no-cublas --no-e2e --steps 5 --warmup 3 2>/dev/null | j)"; done
