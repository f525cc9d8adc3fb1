# 4-CTA A-multicast variant (cta_pair=3) on the L2-bound C4: ring depth and raster (diag)
L=paper_2409_13313_b200/libozmm_b200.so
cp $L /tmp/rel.so
cp tools/_alt/new_diag.so $L
python tools/probe_r2.py --cfg C4,C2:12 --opt "pair:" --opt "quad:cta_pair=3" --opt "quad_s8:cta_pair=3,env.OZMM_STAGES=8" --opt "quad_s4:cta_pair=3,env.OZMM_STAGES=4" --opt "quad_g4:cta_pair=3,env.OZMM_GROUP_M=4" --opt "quad_g1:cta_pair=3,env.OZMM_GROUP_M=1" --rounds 2 --reps 2
for cp in 2 3; do
  echo "== tile trace cta_pair=$cp"
  OZMM_TILE_TRACE=1 python -c "
import torch, sys
sys.path.insert(0, '.')
from paper_2409_13313_b200 import ozmm as oz
g = torch.Generator(device='cuda').manual_seed(1)
A = (torch.rand(8192, 65536, device='cuda', dtype=torch.float64, generator=g) - 0.5)
B = (torch.rand(65536, 8192, device='cuda', dtype=torch.float64, generator=g) - 0.5)
C = torch.zeros(8192, 8192, device='cuda', dtype=torch.float64)
oz.ozaki_gemm_ex(1.0, A, B, 0.0, C, oz.config_for('ozIMMU_H', 8), out=C, timings=False, cta_pair=$cp)
torch.cuda.synchronize()
" 2>&1 | grep "tile trace" | tail -2
done
cp /tmp/rel.so $L
