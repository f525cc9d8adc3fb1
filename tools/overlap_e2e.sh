# pageable e2e at C3 with the overlapped D2H driver (pinned for comparison) + one traced call (diag)
for rep in 1 2; do
  echo "pinned   $(python tools/e2e_jitter.py --calls 4 2>/dev/null)"
  echo "pageable $(python tools/e2e_jitter.py --calls 4 --pageable 2>/dev/null)"
done
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
OZMM_TRACE=1 python tools/e2e_jitter.py --calls 2 --pageable 2>&1 | grep -E "gate|strip (0|1|2|2[0-9]|30) |step 1[45]|ms" | tail -14
cp /tmp/rel.so $L
