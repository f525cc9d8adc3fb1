# C3 k=8 after the K-snake pass order: K-pair thin passes and raster group re-checked (diag build)
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
python tools/probe_r2.py --cfg ${CFGS:-C3:8,C2:8} --opt "default:" --opt "kpair1:env.OZMM_KPAIR=1" ${MORE:---opt "g2:env.OZMM_GROUP_M=2" --opt "g8:env.OZMM_GROUP_M=8" --opt "s4:env.OZMM_STAGES=4"} --rounds ${ROUNDS:-3} --reps 2
cp /tmp/rel.so $L
