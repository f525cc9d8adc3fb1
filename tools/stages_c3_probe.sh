# A-ring depth at the headline C3 k=8 on the HEAD build (diag OZMM_STAGES): 4 / 5 (default) / 6
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
python tools/probe_r2.py --cfg C3:8 --opt "default:" --opt "s4:env.OZMM_STAGES=4" --opt "s6:env.OZMM_STAGES=6" --rounds 4 --reps 2
python tools/probe_r2.py --cfg C2:8,C4 --opt "default:" --opt "s4:env.OZMM_STAGES=4" --rounds 2 --reps 2
cp /tmp/rel.so $L
