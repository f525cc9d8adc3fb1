# pageable C3 call: non-finite-C patch fused into the D2H copy (default) vs C scanned
# up front by scanner threads and copied out with streaming / plain stores (diag build)
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
for round in 1 2 3; do
  echo "patch      $(python tools/e2e_jitter.py --calls 3 --pageable 2>/dev/null)"
  echo "scan+nt    $(OZMM_C_SCAN=1 python tools/e2e_jitter.py --calls 3 --pageable 2>/dev/null)"
  echo "scan+plain $(OZMM_C_SCAN=1 OZMM_D2H_NT=0 python tools/e2e_jitter.py --calls 3 --pageable 2>/dev/null)"
  echo "scan4+nt   $(OZMM_C_SCAN=1 OZMM_SCAN_THREADS=4 python tools/e2e_jitter.py --calls 3 --pageable 2>/dev/null)"
done
cp /tmp/rel.so $L
