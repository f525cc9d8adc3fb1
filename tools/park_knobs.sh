# knobs on the parked (free) schedules: raster group, ring depth, issue-round size (diag build)
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
python tools/probe_r2.py --cfg C4,C5:12 --opt "default:" --opt "g2:env.OZMM_GROUP_M=2" --opt "g8:env.OZMM_GROUP_M=8" \
  --opt "s4:env.OZMM_STAGES=4" --opt "s6:env.OZMM_STAGES=6" --opt "gp3:env.OZMM_GROUP_PAIRS=3" --opt "fwd:env.OZMM_KSNAKE=0" --rounds 2 --reps 2
cp /tmp/rel.so $L
