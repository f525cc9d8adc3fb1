"""GPU: the 2-D partition's CUDA backend (grid2d.Backend) through
torch.distributed/NCCL with world size 1 (the pod exposes one GPU), checked
bit-exactly against the single-call path.  Multi-rank gather logic is covered
on CPU by tests/test_grid2d_gloo.py."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_grid2d_cuda_world1():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist
    from paper_2409_13313_b200 import ozmm
    from paper_2409_13313_b200.grid2d import Backend, Grid2DGemm
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        m, n, p, k = 512, 3000, 384, 8
        A = torch.tensor(ozmm.gen_phi_matrix(m, n, 1.0, 1), device="cuda")
        B = torch.tensor(ozmm.gen_phi_matrix(n, p, 1.0, 2), device="cuda")
        C = torch.tensor(ozmm.gen_phi_matrix(m, p, 1.0, 3), device="cuda")
        G = Grid2DGemm(m, n, p, k, backend=Backend(0))
        got = C.clone()
        G.step(A, B, got, 1.5, 0.5)
        want = ozmm.ozaki_gemm(1.5, A, B, 0.5, C, ozmm.config_for("ozIMMU_H", k))
        assert torch.equal(got.view(torch.int64), want.view(torch.int64))
    finally:
        dist.destroy_process_group()
