# ncu DRAM / L2 / tensor-pipe metrics of the CTA-pair GEMM per A-ring depth (C3, k=8; one launch)
for st in ${STAGES:-6 4}; do
  echo "stages=$st"
  OZMM_STAGES=$st ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct --clock-control none -k regex:ozimmu -c 1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-cublas ${SHAPE:-} 2>&1 | grep -E "^\s+(gpu__|sm__|lts__|dram__)"
done
