"""CPU: the reference-API mirror's host logic (no device calls):
KernelKind / RRAY_KERNEL parsing (kernel_dispatch.cpp:28-31, 40-54, 66-76),
unavailable-kernel errors, and PPM image I/O (image.cpp:11-46)."""
import numpy as np
import pytest

from paper_2005_05386_b200 import render as R
from paper_2005_05386_b200.errors import IoError, ValidationError


@pytest.mark.parametrize("value,kind", [(None, R.KernelKind.Auto), ("", R.KernelKind.Auto),
                                        ("auto", R.KernelKind.Auto), ("scalar", R.KernelKind.Scalar),
                                        ("generic", R.KernelKind.Generic), ("avx2", R.KernelKind.Avx2),
                                        ("cuda", R.KernelKind.Cuda)])
def test_kernel_from_env(monkeypatch, value, kind):
    if value is None:
        monkeypatch.delenv("RRAY_KERNEL", raising=False)
    else:
        monkeypatch.setenv("RRAY_KERNEL", value)
    assert R.kernel_from_env() == kind


def test_kernel_from_env_rejects_unknown(monkeypatch):
    monkeypatch.setenv("RRAY_KERNEL", "sse2")
    with pytest.raises(ValidationError):
        R.kernel_from_env()


def test_only_the_cuda_kernel_is_available():
    assert R.resolve_kernel(R.KernelKind.Auto) == R.KernelKind.Cuda
    assert R.kernel_name(R.KernelKind.Cuda) == "cuda"
    for kind in (R.KernelKind.Scalar, R.KernelKind.Generic, R.KernelKind.Avx2):
        with pytest.raises(ValidationError):        # kernel_dispatch.cpp:50
            R.march_fn(kind)
        with pytest.raises(ValidationError):
            R.render(None, None, None, None, 4, 4, R.RenderOptions(kernel=kind))


def test_ppm_round_trip(tmp_path):
    rng = np.random.default_rng(7)
    img = R.Image(5, 3, rng.integers(0, 256, (3, 5, 3), dtype=np.uint8))
    path = tmp_path / "a.ppm"
    R.write_ppm(img, str(path))
    blob = path.read_bytes()
    assert blob.startswith(b"P6\n5 3\n255\n") and len(blob) == 11 + 45
    back = R.read_ppm(str(path))
    assert (back.width, back.height) == (5, 3)
    assert np.array_equal(back.data, img.data)
    assert back.get(4, 2) == tuple(int(x) for x in img.data[2, 4])


def test_ppm_errors(tmp_path):
    with pytest.raises(IoError):
        R.read_ppm(str(tmp_path / "missing.ppm"))
    bad = tmp_path / "bad.ppm"
    bad.write_bytes(b"P3\n1 1\n255\n000")
    with pytest.raises(IoError):
        R.read_ppm(str(bad))
    short = tmp_path / "short.ppm"
    short.write_bytes(b"P6\n2 2\n255\n" + bytes(5))
    with pytest.raises(IoError):
        R.read_ppm(str(short))
    with pytest.raises(IoError):
        R.write_ppm(R.Image(1, 1, np.zeros((1, 1, 3), np.uint8)), str(tmp_path / "no" / "dir.ppm"))


def test_animation_driver_grid():
    """`animate` rebuilds the culling grid every frame and selects the grid
    that rebuilds fast (192^3) instead of the static default (256^3)."""
    from paper_2005_05386_b200 import cli
    assert cli.ANIMATION_CULL_GRID == 192
