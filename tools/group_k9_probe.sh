# raster group / ring depth at k >= 9 (diag): the schedule's `dense` test puts k = 9 / 10 at
# group 2 / 6 stages (20 A loads per K block for 45 products < 1 / 2.5)
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
python tools/probe_r2.py --cfg C3:9,C3:10,C2:9,C2:10,C5:12 --opt "default:" \
  --opt "g4:env.OZMM_GROUP_M=4" --opt "g4s5:env.OZMM_GROUP_M=4+env.OZMM_STAGES=5" \
  --opt "g3:env.OZMM_GROUP_M=3" --rounds 3 --reps 2
cp /tmp/rel.so $L
