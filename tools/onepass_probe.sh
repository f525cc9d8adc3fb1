# one-pass TMA cluster column split vs the two-pass path (diag OZMM_COLS_TWO_PASS=1): timing, bitwise check, ncu DRAM bytes
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
V="two:OZMM_COLS_TWO_PASS=1,one:OZMM_COLS_TWO_PASS=0,one_u3:OZMM_COLS_UNITS=3"
timeout 300 python tools/cols_probe.py --variants "$V" --row-variants "c128:OZMM_ROW_CTA=128"
timeout 300 python tools/cols_probe.py --n 8192 --p 8192 --variants "$V" --row-variants "c128:OZMM_ROW_CTA=128"
timeout 300 python tools/cols_probe.py --n 1000 --p 777 --k 12 --variants "two:OZMM_COLS_TWO_PASS=1,one:OZMM_COLS_TWO_PASS=0"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:"slice_cols|colmax" -c 3 python tools/cols_probe.py --reps 1 --variants "one:OZMM_COLS_TWO_PASS=0" 2>&1 | grep -E "slice_cols|colmax|dram__|gpu__time|issue_active|warps_active" | head -20
cp /tmp/rel.so $L
