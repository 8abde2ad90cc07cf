"""GPU: the reference-side binding (integration/kernel_cuda.cpp) works as a
drop-in inside the reference's own code: a MarchFn called row by row exactly
like render.cpp:72-76, and render() routed as whole frames, both compared
with the reference's Scalar kernel under the parity contract."""
import ctypes
import json
import os

import numpy as np
import pytest

from conftest import ROOT, load_golden

pytestmark = pytest.mark.gpu
SHIM = os.path.join(ROOT, "oracle", "_ref", "libkernel_cuda_shim.so")


@pytest.fixture(scope="module")
def shim():
    if not os.path.exists(SHIM):
        pytest.skip("integration shim not built (make -C oracle ref)")
    lib = ctypes.CDLL(SHIM)
    lib.shim_last_error.restype = ctypes.c_char_p
    lib.shim_march_both.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                    ctypes.c_void_p]
    lib.shim_render_both.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.POINTER(ctypes.c_longlong),
                                     ctypes.POINTER(ctypes.c_longlong)]
    return lib


@pytest.mark.parametrize("name", ["c1_gauss1_512", "c3_bumps16_1080p", "ref_twist",
                                  "diffeo_nested_chain", "graph_nested_mix"])
def test_marchfn_shim_matches_reference_kernel(shim, name):
    from paper_2005_05386_b200 import abi
    from oracle.parity import compare_outcomes
    cfg, _, z = load_golden(name)
    w, h = int(z["w"]), int(z["h"])
    ref = np.zeros(w * h, abi.OUTCOME_DTYPE)
    cuda = np.zeros(w * h, abi.OUTCOME_DTYPE)
    rc = shim.shim_march_both(str(z["config"]).encode(), w, h, ref.ctypes.data, cuda.ctypes.data)
    assert rc == 0, shim.shim_last_error()
    rep = compare_outcomes(cuda, ref, z["flags"])
    assert rep.ok, rep.summary()


@pytest.mark.parametrize("name", ["c1_gauss1_512", "ref_quadric_graph", "ref_grid_euclid"])
def test_render_shim_matches_reference_render(shim, name):
    from oracle.parity import compare_rgb
    cfg, _, z = load_golden(name)
    w, h = int(z["w"]), int(z["h"])
    ref = np.zeros((h, w, 3), np.uint8)
    cuda = np.zeros((h, w, 3), np.uint8)
    rs, cs = ctypes.c_longlong(), ctypes.c_longlong()
    rc = shim.shim_render_both(str(z["config"]).encode(), ref.ctypes.data, cuda.ctypes.data,
                               ctypes.byref(rs), ctypes.byref(cs))
    assert rc == 0, shim.shim_last_error()
    assert np.array_equal(ref, z["rgb"])           # the reference itself, as dumped
    assert compare_rgb(cuda, ref, z["flags"]).ok
    assert abs(cs.value - rs.value) <= max(2, 0.01 * rs.value)


def test_marchfn_row_pattern_threads(shim):
    """render()'s frame loop (render.cpp:57-104) with the CUDA MarchFn from 1
    and 16 worker threads, each on its own context: images byte-identical
    across worker counts (acceptance.cpp:243-253) and within parity of the
    FP64 oracle; the row-pattern wall time is logged (RR_PARITY_LOG)."""
    import time
    from oracle import Oracle
    from oracle.parity import compare_rgb
    from paper_2005_05386_b200.config import load_config
    cfg = load_config(os.path.join(ROOT, "configs", "c3_bumps16_1080p.json"))
    cfg.output.width, cfg.output.height = 320, 180
    from paper_2005_05386_b200.config import reference_json
    doc = reference_json(cfg).encode()
    shim.shim_render_rows_cuda.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_void_p,
                                           ctypes.POINTER(ctypes.c_double),
                                           ctypes.POINTER(ctypes.c_longlong)]
    imgs, times = {}, {}
    for workers in (1, 16, 16):
        img = np.zeros((180, 320, 3), np.uint8)
        sec, steps = ctypes.c_double(), ctypes.c_longlong()
        rc = shim.shim_render_rows_cuda(doc, workers, img.ctypes.data, ctypes.byref(sec), ctypes.byref(steps))
        assert rc == 0, shim.shim_last_error()
        imgs[workers], times[workers] = img, sec.value
    assert np.array_equal(imgs[1], imgs[16])
    ref_rgb, _, _, flags = Oracle().render(cfg, 320, 180, with_flags=True)
    assert compare_rgb(imgs[16], ref_rgb, flags).ok
    path = os.environ.get("RR_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"case": "MarchFn row pattern 320x180 (C3)", "seconds_1_worker": times[1],
                                "seconds_16_workers": times[16]}) + "\n")
