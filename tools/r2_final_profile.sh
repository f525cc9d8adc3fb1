# round-2 evidence: launch list of the bench step and ncu --set full of the GEMM and the slicers (C3)
set -u
B="python bench.py --no-cpu --no-cublas --no-e2e --no-parity --int8-seconds 0"
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_r2.csv $B --steps 2 --warmup 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ozimmu_gemm_pair|slice_rows|slice_cols|colmax" -c 4 \
  -o gpurun_out/c3_r2 $B --steps 1 --warmup 0 > gpurun_out/c3_r2_ncu.log 2>&1
