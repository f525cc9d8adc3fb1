# one traced pinned and one traced pageable host-entry call at C3 (diag build, OZMM_TRACE timeline)
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
OZMM_TRACE=1 python tools/e2e_jitter.py --calls 2 2>&1 | tail -52
OZMM_TRACE=1 python tools/e2e_jitter.py --calls 2 --pageable 2>&1 | tail -52
cp /tmp/rel.so $L
