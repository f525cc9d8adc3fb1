# B-window width (resident B slices per K block) on multi-window schedules (diag build)
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
python tools/probe_r2.py --cfg C2:9,C2:10,C2:12,C2:14,C3:9,C5:12 --opt "bw8:" --opt "bw9:env.OZMM_BWIN=9" --opt "bw10:env.OZMM_BWIN=10" --opt "bw11:env.OZMM_BWIN=11" --rounds 2 --reps 2
cp /tmp/rel.so $L
