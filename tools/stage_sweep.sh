# pageable e2e at C3 over staging team size / slot size / slot count (diag build), then one trace
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
for cfg in "8 8 2" "12 8 2" "16 8 2" "12 16 2" "12 4 3"; do
  set -- $cfg
  echo "threads=$1 slot_mb=$2 slots=$3 $(OZMM_STAGE_THREADS=$1 OZMM_STAGE_SLOT_MB=$2 OZMM_STAGE_SLOTS=$3 python tools/e2e_jitter.py --calls 4 --pageable 2>/dev/null)"
done
OZMM_TRACE=1 python tools/e2e_jitter.py --calls 2 --pageable 2>&1 | tail -52
cp /tmp/rel.so $L
