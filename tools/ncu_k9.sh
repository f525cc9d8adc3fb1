# key ncu metrics of the fused GEMM at k >= 9 next to k = 8 (C3, C2), one launch each,
# plus a --set full capture of C3 k = 9
set -u
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes.sum
B="python bench.py --no-cpu --no-cublas --no-e2e --no-parity --steps 1 --warmup 0"
for args in "--k 8" "--k 9" "--k 10" "--m 8192 --n 8192 --p 8192 --k 8" "--m 8192 --n 8192 --p 8192 --k 9" "--m 8192 --n 8192 --p 8192 --k 12"; do
  echo "== $args"
  ncu --metrics $M --clock-control none -k regex:ozimmu_gemm_pair -c 1 $B $args 2>&1 | grep -E "^\s+(gpu__|sm__|lts__|dram__|l1tex__)"
done
ncu --set full --clock-control none --import-source on -k regex:ozimmu_gemm_pair -c 1 -f -o gpurun_out/c3_k9_full $B --k 9 > /dev/null 2>&1
ncu -i gpurun_out/c3_k9_full.ncu-rep --page raw --csv > gpurun_out/c3_k9_full_raw.csv 2>&1
