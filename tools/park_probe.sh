# chunks batched by shared A slices with early ones parked (default auto) vs flush-order
# batches (OZMM_SCHED_FREE=0), diag build
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
python tools/probe_r2.py --cfg ${CFGS:-C4,C5:12,C5:14,C5:10,C3:8} --opt "park:" --opt "flush_order:env.OZMM_SCHED_FREE=0" ${MORE:-} --rounds ${ROUNDS:-3} --reps 2
cp /tmp/rel.so $L
