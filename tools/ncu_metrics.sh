# key ncu metrics of the fused GEMM at C2 k=8, C3 k=8, C4 (one launch each)
set -u
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes.sum
B="python bench.py --no-cpu --no-cublas --no-e2e --no-parity --steps 1 --warmup 0"
for args in "--m 8192 --n 8192 --p 8192 --k 8" "--k 8" "--m 8192 --n 65536 --p 8192 --k 8"; do
  echo "== $args"
  ncu --metrics $M --clock-control none -k regex:ozimmu_gemm_pair -c 1 $B $args 2>&1 | grep -E "^\s+(gpu__|sm__|lts__|dram__|l1tex__)"
done
