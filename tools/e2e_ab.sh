# e2e A/B of host-entry builds on one box: per-call ms of ozmm_dgemm_host at C3
# (pinned, then pageable) for tools/_alt/{new,old}.so, alternating; then one
# traced call of the diag build (OZMM_TRACE timeline on stderr).
set -u
L=paper_2409_13313_b200/libozmm_b200.so
for v in new old new old; do
  cp tools/_alt/$v.so $L
  echo "$v pinned   $(python tools/e2e_jitter.py --calls 5 2>/dev/null)"
  echo "$v pageable $(python tools/e2e_jitter.py --calls 3 --pageable 2>/dev/null)"
done
cp tools/_alt/new_diag.so $L
OZMM_TRACE=1 python tools/e2e_jitter.py --calls 2 2>&1 | tail -60
OZMM_TRACE=1 python tools/e2e_jitter.py --calls 2 --pageable 2>&1 | tail -60
cp tools/_alt/new.so $L
