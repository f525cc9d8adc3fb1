"""D2H / H2D throughput of cudaMemcpy2DAsync (pinned host) by row-segment width:
the host entry's strip copies.  Uses cuda-python's runtime bindings."""
import time

import torch
from cuda.bindings import runtime as rt

n = 16384
h = torch.empty((n, n), dtype=torch.float64).pin_memory()
d = torch.empty((n, n), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
_, s = rt.cudaStreamCreate()
for cols in (1024,):
    for name, kind, dst, src in (("D2H", rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, h, d),
                                 ("H2D", rt.cudaMemcpyKind.cudaMemcpyHostToDevice, d, h)):
        def fn():
            err, = rt.cudaMemcpy2DAsync(dst.data_ptr(), n * 8, src.data_ptr(), n * 8, cols * 8, n,
                                        kind, s)
            assert err == rt.cudaError_t.cudaSuccess, err
        fn()
        rt.cudaStreamSynchronize(s)
        reps = max(2, 16384 // cols)
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        rt.cudaStreamSynchronize(s)
        dt = (time.perf_counter() - t) / reps
        print(f"{name} {n} x {cols:5d} (segment {cols * 8 // 1024:4d} KB): {n * cols * 8 / dt / 1e9:6.1f} GB/s",
              flush=True)

# the same D2H while the fused GEMM runs on another stream (C3 shape, k=8)
import sys, os  # noqa: E401
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_13313_b200 import ozmm  # noqa: E402
A = torch.from_numpy(ozmm.gen_phi_block(n, n, 0.5, 1)).cuda()
B = torch.from_numpy(ozmm.gen_phi_block(n, n, 0.5, 2)).cuda()
C = torch.zeros((n, n), dtype=torch.float64, device="cuda")
hnd = ozmm.Handle(0)
gs = torch.cuda.Stream()
hnd.set_stream(gs.cuda_stream)
cfg = ozmm.config_for(ozmm.Method.ozIMMU_H, 8)
for cols in (1024, 2048, 4096, 8192, 16384):
    ozmm.ozaki_gemm_ex(1.0, A, B, 0.0, C, cfg, handle=hnd, out=C, timings=False)
    torch.cuda.synchronize()
    hnd.set_stream(gs.cuda_stream)
    ozmm.lib.ozmm_dgemm_ex(hnd.h, b"N", b"N", n, n, n, 1.0, A.data_ptr(), n, B.data_ptr(), n, 0.0,
                           C.data_ptr(), n, 8, None, None, None)
    time.sleep(0.01)
    t = time.perf_counter()
    reps = 16384 // cols
    for _ in range(reps):
        err, = rt.cudaMemcpy2DAsync(h.data_ptr(), n * 8, d.data_ptr(), n * 8, cols * 8, n,
                                    rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s)
    rt.cudaStreamSynchronize(s)
    dt = (time.perf_counter() - t) / reps
    print(f"D2H during GEMM {n} x {cols:5d}: {n * cols * 8 / dt / 1e9:6.1f} GB/s", flush=True)
    # packed device source (pitch = width), strided host destination
    t = time.perf_counter()
    for _ in range(reps):
        err, = rt.cudaMemcpy2DAsync(h.data_ptr(), n * 8, d.data_ptr(), cols * 8, cols * 8, n,
                                    rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s)
    rt.cudaStreamSynchronize(s)
    dt = (time.perf_counter() - t) / reps
    print(f"D2H during GEMM, packed device side {n} x {cols:5d}: {n * cols * 8 / dt / 1e9:6.1f} GB/s", flush=True)
    # packed host destination, strided device source
    t = time.perf_counter()
    for _ in range(reps):
        err, = rt.cudaMemcpy2DAsync(h.data_ptr(), cols * 8, d.data_ptr(), n * 8, cols * 8, n,
                                    rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s)
    rt.cudaStreamSynchronize(s)
    dt = (time.perf_counter() - t) / reps
    print(f"D2H during GEMM, packed host side {n} x {cols:5d}: {n * cols * 8 / dt / 1e9:6.1f} GB/s", flush=True)
    torch.cuda.synchronize()
