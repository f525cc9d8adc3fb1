# host entry: the last arrival's strip cut into column pieces whose D2H runs under the
# later pieces' GEMM (diag OZMM_TAIL_PIECES), per-call ms at C3, pinned and pageable,
# alternating; then traced calls of 1 and 4 pieces
set -u
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/tail_diag.so $L
for round in 1 2; do
for tp in 1 2 4 8; do
  echo "tail=$tp pinned   $(OZMM_TAIL_PIECES=$tp python tools/e2e_jitter.py --calls 6 2>/dev/null)"
  echo "tail=$tp pageable $(OZMM_TAIL_PIECES=$tp python tools/e2e_jitter.py --calls 3 --pageable 2>/dev/null)"
done
done
for tp in 1 4; do
  echo "== trace tail=$tp"
  OZMM_TAIL_PIECES=$tp OZMM_TRACE=1 python tools/e2e_jitter.py --calls 2 2>&1 | grep -E "strip (2[6-9]|3[0-9])|gate|ms"
done
python - <<'PY'
import os, sys, numpy as np
sys.path.insert(0, '.')
from oracle import oracle
from paper_2409_13313_b200 import ozmm
m, n, p = 3000, 1500, 4100
A = ozmm.gen_phi_matrix(m, n, 1.0, 7); B = ozmm.gen_phi_matrix(n, p, 1.0, 8); C = ozmm.gen_phi_matrix(m, p, 1.0, 9)
want = oracle.best().gemm(1.5, A, B, 0.5, C, k=8)
for tp in ("1", "3", "4", "8"):
    os.environ["OZMM_TAIL_PIECES"] = tp
    for panels in (4, 16):
        got = ozmm.ozaki_gemm(1.5, A, B, 0.5, C, ozmm.config_for("ozIMMU_H", 8), host_panels=panels)
        print("tail", tp, "panels", panels, "differ:", int((got.view(np.uint64) != want.view(np.uint64)).sum()))
PY
cp /tmp/rel.so $L
