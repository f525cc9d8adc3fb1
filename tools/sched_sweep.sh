# schedule cost-model knobs (diag): fill-term scale (OZMM_SCHED_FILL) and per-batch cost (OZMM_SCHED_BATCH)
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
python tools/probe_r2.py --cfg C2:9,C2:10,C2:12,C2:14,C3:9,C4,C5:12 --opt "default:" --opt "fill0.5:env.OZMM_SCHED_FILL=0.5" --opt "fill1.6:env.OZMM_SCHED_FILL=1.6" --opt "fill2.5:env.OZMM_SCHED_FILL=2.5" --opt "batch300:env.OZMM_SCHED_BATCH=300" --rounds 2 --reps 2
cp /tmp/rel.so $L
