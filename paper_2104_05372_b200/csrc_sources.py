"""Device sources shipped with the package (for compile-only checks and tools)."""
import os

_CSRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc")


def _read(name: str) -> str:
    with open(os.path.join(_CSRC, name)) as f:
        return f.read()


def gmm_module_source() -> str:
    """The NVRTC source of the GMM module as gmm.cpp builds it (the device
    runtime dx_device.cuh is prepended by the compiler wrapper)."""
    return _read("dx_gemm.cuh") + "\n" + _read("dx_gmm.cuh")
