import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def b200lib():
    """The product library; built in-tree if missing (build() is the driver's job)."""
    from paper_2307_12119_b200 import api, build
    if not api.library_path().exists():
        build.build()
    return api.lib()


@pytest.fixture(scope="session")
def oracle():
    from oracle import refpy
    if not refpy.build_if_possible():
        pytest.skip("CPU oracle not built (no /root/reference and no prebuilt oracle/_ref)")
    return refpy


@pytest.fixture(scope="session")
def greens64():
    from paper_2307_12119_b200.api import GreensArrays
    return GreensArrays.from_npz(GOLDEN / "greens_n64.npz")


@pytest.fixture(scope="session")
def greens256():
    import numpy as np
    from paper_2307_12119_b200.api import GreensArrays
    z = np.load(GOLDEN / "greens_n256.npz")
    f = z["f_sp0"]
    n = int(z["n"])
    c = n // 2
    g_sp0 = f + (f[c, c] - float(z["kappa_inf"]))  # make_g_shift, reference greens.cpp:170-175
    return GreensArrays(n=n, pitch=float(z["pitch"]), f_sp0=f, g_sp0=g_sp0, phi=float(z["phi"]),
                        kappa_inf=float(z["kappa_inf"]), alpha=float(z["alpha"]), beta=float(z["beta"]),
                        mu=float(z["mu"]), capacitance=float(z["capacitance"]), rand_scale=float(z["rand_scale"]))
