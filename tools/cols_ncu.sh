# ncu of the column split: two-pass (colmax + slice_cols) vs the one-pass panel walk (diag build)
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
ncu --set full --clock-control none --import-source on -k regex:"colmax|slice_cols|slice_rows" -c 6 \
  -o gpurun_out/cols_ncu python tools/cols_probe.py --reps 1 --variants "two:OZMM_COLS_TWO_PASS=1,one:OZMM_COLS_TWO_PASS=0+OZMM_PANEL_MB=32" > gpurun_out/cols_ncu.log 2>&1
cp /tmp/rel.so $L
