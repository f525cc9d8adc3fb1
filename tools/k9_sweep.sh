# k >= 9 schedule knobs (diag build): issue-round size, ring depth, cost-model fill scale, A-group order
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
python tools/probe_r2.py --cfg C3:9,C2:9,C2:10,C2:12,C5:12,C5:14 --opt "default:" \
  --opt "gp3:env.OZMM_GROUP_PAIRS=3" --opt "s6:env.OZMM_STAGES=6" \
  --opt "gp3s6:env.OZMM_GROUP_PAIRS=3+env.OZMM_STAGES=6" \
  --opt "fill08:env.OZMM_SCHED_FILL=0.8" --opt "fill13:env.OZMM_SCHED_FILL=1.3" \
  --opt "il:env.OZMM_AORDER=interleave" --rounds 2 --reps 2
cp /tmp/rel.so $L
