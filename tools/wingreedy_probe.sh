# (the OZMM_WIN_GREEDY knob was removed after this probe) multi-window batches: B windows cut every 8 slices from the lowest (one wide pass plus a
# thin remainder, diag OZMM_WIN_GREEDY) vs the modelled cut (two balanced passes)
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
python tools/probe_r2.py --cfg C3:9,C2:9,C2:10,C2:12,C5:12 --opt "default:" --opt "wg:env.OZMM_WIN_GREEDY=1" --rounds 3 --reps 2
OZMM_WIN_GREEDY=1 python tools/sets_check.py 2>&1 | tail -4
cp /tmp/rel.so $L
