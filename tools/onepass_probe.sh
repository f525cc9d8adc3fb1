# one-pass TMA cluster column split vs the two-pass path (diag OZMM_COLS_TWO_PASS=1), rows per CTA 512*U (OZMM_COLS_UNITS)
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
V="two:OZMM_COLS_TWO_PASS=1,u2:OZMM_COLS_TWO_PASS=0+OZMM_COLS_UNITS=2,db:OZMM_COLS_TWO_PASS=0+OZMM_COLS_UNITS=2+OZMM_COLS_DB=1"
timeout 300 python tools/cols_probe.py --variants "$V"
timeout 300 python tools/cols_probe.py --n 8192 --p 8192 --variants "$V"
timeout 300 python tools/cols_probe.py --n 1000 --p 777 --k 12 --variants "two:OZMM_COLS_TWO_PASS=1,one:OZMM_COLS_TWO_PASS=0"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:"slice_cols|colmax|slice_rows" -c 4 python tools/cols_probe.py --reps 1 --variants "one:OZMM_COLS_TWO_PASS=0" 2>&1 | grep -E "^  [a-z]|dram__|gpu__time|issue_active|warps_active" | head -24
cp /tmp/rel.so $L
