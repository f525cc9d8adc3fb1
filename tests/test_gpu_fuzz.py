"""Seeded random shapes and options against the reference build: every
combination of the knobs a caller can turn (shape including 1-element edges,
k in 1..32, phi, alpha/beta including zeros and negatives, transposes, method,
device vs host entry, pinned-free host buffers, column-split path, signed
planes, forced small r -- which selects the parked schedules, schedule.hpp
make_schedule_free) must give the reference's bits."""
import numpy as np
import pytest

from tests.helpers import assert_bitwise

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

METHODS = ["ozIMMU_H"] * 5 + ["ozIMMU_EF", "ozIMMU", "ozIMMU_RN"]


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle
    from paper_2409_13313_b200 import ozmm
    if not oracle.have_ref():
        pytest.skip("reference build absent")
    return ozmm, oracle.RefLib()


def _case(seed):
    rng = np.random.default_rng(seed)
    dim = lambda: int(rng.choice([1, 2, 3, 17, 64, 127, 129, 255, 256, 300, 513, 700, 1025, 2100]))  # noqa: E731
    m, n, p = dim(), dim(), dim()
    k = int(rng.integers(1, 33)) if rng.random() < 0.3 else int(rng.integers(4, 15))
    return dict(m=m, n=n, p=p, k=k, phi=float(rng.choice([0.0, 0.5, 1.0, 2.0, 4.0])),
                alpha=float(rng.choice([1.0, -1.5, 0.0, 2.0 ** -3])),
                beta=float(rng.choice([0.0, 0.5, -1.0, 0.0])),
                ta=bool(rng.random() < 0.3), tb=bool(rng.random() < 0.3),
                method=str(rng.choice(METHODS)), host=bool(rng.random() < 0.4),
                col_split=int(rng.choice([0, 1, 2])), signed=bool(rng.random() < 0.2),
                force_r=int(rng.choice([0, 0, 0, 1, 2, 3, 4])))


@pytest.mark.parametrize("seed", range(200))
def test_random_configuration(env, seed):
    ozmm, ref = env
    c = _case(seed)
    m, n, p, k = c["m"], c["n"], c["p"], c["k"]
    A = ozmm.gen_phi_matrix(m, n, c["phi"], 1000 + seed)
    B = ozmm.gen_phi_matrix(n, p, c["phi"], 2000 + seed)
    C = ozmm.gen_phi_matrix(m, p, c["phi"], 3000 + seed)
    r_nat = ozmm.compute_r(n, ozmm.compute_beta(n))
    force_r = c["force_r"] if 0 < c["force_r"] <= r_nat else 0  # never past the natural r
    want = ref.gemm(c["alpha"], A, B, c["beta"], C, k=k, method=c["method"], force_r=force_r)
    As = np.ascontiguousarray(A.T) if c["ta"] else A
    Bs = np.ascontiguousarray(B.T) if c["tb"] else B
    cfg = ozmm.config_for(c["method"], k)
    cfg.force_r = force_r
    kw = dict(transa=c["ta"], transb=c["tb"], col_split=c["col_split"])
    if c["host"]:
        got = ozmm.ozaki_gemm(c["alpha"], As, Bs, c["beta"], C, cfg, **kw)
    else:
        dev = lambda x: torch.tensor(x, dtype=torch.float64, device="cuda")  # noqa: E731
        got = ozmm.ozaki_gemm(c["alpha"], dev(As), dev(Bs), c["beta"], dev(C), cfg,
                              signed_slices=c["signed"] and c["method"] == "ozIMMU_H",
                              **kw).cpu().numpy()
    assert_bitwise(got, want, str(c))
