"""pytest plugin (-p svsim_cuda_default): make the staged reference's default
kernel backend the B200 one, so the reference's own engine tests drive
libsvb.so through the seam (engine.py:356, 443, 450 pass kernel_backend=None,
which resolves svsim.kernel.BACKEND at call time, kernel/__init__.py:66-68)."""


def pytest_configure(config):
    import svsim.kernel as k

    assert "cuda" in k.available_backends(), "cuda backend not registered in the staged svsim"
    k.BACKEND = "cuda"
