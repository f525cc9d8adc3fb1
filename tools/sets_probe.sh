# k = 9 / 10 explicit batch sets (diag OZMM_SCHED_SETS): does the batch cut the
# schedule model prefers match the measured one?
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
# C3 k=9, r=8: chunks 0..7 = g2..g9, 8 = g10 s1..8, 9 = g10 s9
python tools/probe_r2.py --cfg C3:9 --opt "default:" \
  --opt "a:env.OZMM_SCHED_SETS=0.1.2.3/4.5.6.7/8.9" --opt "b:env.OZMM_SCHED_SETS=0.1.2/3.4.5.6/7.8.9" \
  --opt "c:env.OZMM_SCHED_SETS=0.1.2.9/3.4.5/6.7.8" --opt "d:env.OZMM_SCHED_SETS=0.1.2.3/4.5.6.9/7.8" \
  --opt "e:env.OZMM_SCHED_SETS=0.1/2.3.4.5/6.7.8.9" --rounds 2 --reps 2
# C2 k=9, r=16: chunks 0..8 = g2..g10;  k=10: 0..9 = g2..g11
python tools/probe_r2.py --cfg C2:9 --opt "default:" \
  --opt "a:env.OZMM_SCHED_SETS=0.1.2.3/4.5.6.7/8" --opt "b:env.OZMM_SCHED_SETS=0.1.2/3.4.5.6/7.8" \
  --opt "c:env.OZMM_SCHED_SETS=0.1/2.3.4.5/6.7.8" --opt "d:env.OZMM_SCHED_SETS=0.1.2.3/4.5.6/7.8" \
  --opt "e:env.OZMM_SCHED_SETS=0.1.2.8/3.4.5/6.7" --rounds 2 --reps 3
python tools/probe_r2.py --cfg C2:10 --opt "default:" \
  --opt "a:env.OZMM_SCHED_SETS=0.1.2.3/4.5.6/7.8.9" --opt "b:env.OZMM_SCHED_SETS=0.1.2/3.4.5.6/7.8.9" \
  --opt "c:env.OZMM_SCHED_SETS=0.1.2.3/4.5.6.7/8.9" --opt "d:env.OZMM_SCHED_SETS=0.1/2.3.4/5.6.7/8.9" \
  --rounds 2 --reps 3
python tools/sets_check.py
cp /tmp/rel.so $L
