# odd passes sweep K in reverse (P.ksnake, default on) vs every pass forward (diag build)
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
python tools/probe_r2.py --cfg ${CFGS:-C3:8,C2:8,C3:9,C4,C5:12,C2:12} --opt "snake:" --opt "fwd:env.OZMM_KSNAKE=0" --rounds ${ROUNDS:-3} --reps 2
cp /tmp/rel.so $L
