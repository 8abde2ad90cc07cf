import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")


def golden_cases():
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and f != "reference_goldens.npz")


def load_golden(name):
    import numpy as np
    from paper_2005_05386_b200.config import parse_config
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    cfg = parse_config(str(z["config"]))
    cam_cfg = parse_config(str(z["camera_config"]))
    return cfg, cam_cfg, z


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference_lib():
    from oracle import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


def outcomes_identical(a, b) -> bool:
    """Field-wise bitwise equality of PixelOutcome arrays (padding ignored:
    the reference leaves it uninitialised), test_simd.cpp:62-74."""
    import numpy as np
    return (np.array_equal(a["status"], b["status"]) and np.array_equal(a["prim"], b["prim"])
            and np.array_equal(a["steps"], b["steps"])
            and np.array_equal(np.ascontiguousarray(a["point"]).view(np.uint64),
                               np.ascontiguousarray(b["point"]).view(np.uint64))
            and np.array_equal(np.ascontiguousarray(a["t"]).view(np.uint64),
                               np.ascontiguousarray(b["t"]).view(np.uint64)))
