# pageable e2e at C3: staging slot size / slots per thread with the 16-thread team (diag build), two rounds
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket|NUMA node\(s\)"
for round in 1 2; do
for cfg in ${CFGS:-"16 8 2" "16 4 2" "16 4 3" "16 2 4" "16 8 3" "16 16 2"}; do
  set -- $cfg
  echo "threads=$1 slot_mb=$2 slots=$3 $(OZMM_STAGE_THREADS=$1 OZMM_STAGE_SLOT_MB=$2 OZMM_STAGE_SLOTS=$3 python tools/e2e_jitter.py --calls 3 --pageable 2>/dev/null)"
done
done
cp /tmp/rel.so $L
