# host entry, pageable result: strip results DMA'd into a pinned mirror of C before the
# range gate, copied to C by the team after it (diag OZMM_MIRROR=1, the default) vs the
# slot rings after the gate (OZMM_MIRROR=0): per-call ms at C3, alternating; traced calls
set -u
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/mirror_diag.so $L
for round in 1 2 3; do
for mv in 1 0; do
  echo "mirror=$mv pageable $(OZMM_MIRROR=$mv python tools/e2e_jitter.py --calls 4 --pageable 2>/dev/null)"
done
done
echo "pinned   $(python tools/e2e_jitter.py --calls 5 2>/dev/null)"
for mv in 1 0; do
  echo "== trace mirror=$mv"
  OZMM_MIRROR=$mv OZMM_TRACE=1 python tools/e2e_jitter.py --calls 2 --pageable 2>&1 | grep -E "strip (2[6-9]|3[0-9])|gate|scan|ms"
done
cp /tmp/rel.so $L
python -m pytest tests/test_gpu_semantics.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "host" 2>&1 | tail -3
