# C4 (thin A groups, ~1.4 products each): A groups per issue round and ring depth (diag), each option bounded
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
for o in "gp2:" "gp3:env.OZMM_GROUP_PAIRS=3" "gp4:env.OZMM_GROUP_PAIRS=4" "s8:env.OZMM_STAGES=8" "gp4s8:env.OZMM_GROUP_PAIRS=4+env.OZMM_STAGES=8"; do
  timeout 120 python tools/probe_r2.py --cfg C4 --opt "$o" --rounds 1 --reps 2 2>&1 | grep TOPS || echo "$o: timed out / failed"
done
cp /tmp/rel.so $L
