# chunk pieces (a chunk's products split over batches, partial INT32 sums added in the
# epilogue) so that no batch needs more than 8 resident B slices: k = 9 / 10 cuts (diag
# OZMM_SCHED_SETS) vs the default schedule
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/pieces_diag.so $L
python tools/pieces_check.py
python tools/probe_r2.py --cfg C3:9 --opt "default:" \
  --opt "p1:env.OZMM_SCHED_SETS=0.1.2.8:1-1/3.4.5/6.7.8:2-8.9" --opt "p2:env.OZMM_SCHED_SETS=0.1.8:1-1/2.3.4.5/6.7.8:2-8.9" \
  --opt "e:env.OZMM_SCHED_SETS=0.1/2.3.4.5/6.7.8.9" --rounds 3 --reps 2
python tools/probe_r2.py --cfg C2:9 --opt "default:" \
  --opt "p1:env.OZMM_SCHED_SETS=0.1.2.8:1-1/3.4.5/6.7.8:2-9" --opt "p2:env.OZMM_SCHED_SETS=0.1.8:1-1/2.3.4.5/6.7.8:2-9" \
  --rounds 3 --reps 3
python tools/probe_r2.py --cfg C2:10 --opt "default:" \
  --opt "p1:env.OZMM_SCHED_SETS=0.1.2.9:1-2/3.4.5.8:1-1/6.7.8:2-9.9:3-10" --rounds 3 --reps 3
cp /tmp/rel.so $L
