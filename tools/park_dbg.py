import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2409_13313_b200 import ozmm as oz
m, n, p, k, r = 300, 1500, 260, 8, 2
A = oz.gen_phi_matrix(m, n, 1.0, 131); B = oz.gen_phi_matrix(n, p, 1.0, 132); C = oz.gen_phi_matrix(m, p, 1.0, 133)
cfg = oz.config_for("ozIMMU_H", k); cfg.force_r = r; cfg.overflow = oz.OverflowMode.Wrapping
dev = lambda x: torch.tensor(x, dtype=torch.float64, device="cuda")
got = oz.ozaki_gemm(1.5, dev(A), dev(B), 0.5, dev(C), cfg).cpu().numpy()
print("ok", got[0, :3])
