# ncu metrics of one C4 GEMM launch (release build): parked schedule vs flush-order batches (diag env)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second
ncu --metrics $M --clock-control none -k regex:ozimmu_gemm_pair -c 1 python tools/probe_r2.py --cfg C4 --opt "rel:" --rounds 1 --reps 1 2>&1 | grep -E "gpu__|dram__|l1tex__|pipe_tensor|cycles_elapsed"
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
echo "== flush-order batches (OZMM_SCHED_FREE=0)"
ncu --metrics $M --clock-control none -k regex:ozimmu_gemm_pair -c 1 python tools/probe_r2.py --cfg C4 --opt "std:env.OZMM_SCHED_FREE=0" --rounds 1 --reps 1 2>&1 | grep -E "gpu__|dram__|l1tex__|pipe_tensor|cycles_elapsed"
cp /tmp/rel.so $L
