"""CPU tests of the C-ABI boundary: the library loads, exports every symbol include/glsgpu.h declares,
and fails loudly (no CPU fallback) when there is no CUDA device."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2510_14471_b200 import _lib, api, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "glsgpu.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(glsgpu_[a-z_0-9]+)\s*\(", txt)))


def test_header_and_binding_agree():
    assert sorted(_lib.EXPORTS) == declared_symbols()


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.glsgpu_version()


def _c_layout(struct, fields):
    """sizeof / offsetof as the C compiler lays out include/glsgpu.h."""
    import subprocess
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    body = "".join(f'printf("%zu\\n", offsetof({struct}, {f}));' for f in fields)
    src = ("#include <stdio.h>\n#include <stddef.h>\n#include \"glsgpu.h\"\n"
           f'int main(void){{printf("%zu\\n", sizeof({struct}));{body}return 0;}}\n')
    with tempfile.TemporaryDirectory() as d:
        open(os.path.join(d, "l.c"), "w").write(src)
        subprocess.run(["gcc", "-I", os.path.join(root, "include"), "-o", os.path.join(d, "l"),
                        os.path.join(d, "l.c")], check=True)
        out = subprocess.run([os.path.join(d, "l")], check=True, capture_output=True, text=True).stdout.split()
    return [int(x) for x in out]


def test_config_struct_layout_matches_header():
    # glsgpu_pcg_config: the ctypes mirror matches the C compiler's layout field by field
    names = [f for f, _ in _lib.PcgConfigC._fields_]
    lay = _c_layout("glsgpu_pcg_config", names)
    assert ctypes.sizeof(_lib.PcgConfigC) == lay[0]
    assert [getattr(_lib.PcgConfigC, f).offset for f in names] == lay[1:]
    assert ctypes.sizeof(_lib.TraceRowC) == 48
    assert ctypes.sizeof(_lib.ResultC) == 8 + 4 + 4 + 8 + 8 + 8 + 8 + 8
    c = _lib.PcgConfigC()
    _lib.load().glsgpu_default_config(ctypes.byref(c))
    assert (c.tol_rel, c.max_iter, c.breakdown_tol, c.stagnation_window, c.growth_tol, c.growth_window,
            c.record_z_every) == (1e-10, 0, 1e-14, 5, 1e4, 10, 1)  # gls::PcgConfig defaults (pcg.hpp:12-30)


def test_make_sur_validation_mirrors_reference():
    y = np.zeros((5, 2))
    with pytest.raises(api.DimensionMismatch, match="need at least one block"):
        api.make_sur([], y, np.eye(2))
    with pytest.raises(api.DimensionMismatch, match="Y/blocks mismatch"):
        api.make_sur([np.ones((5, 1))], y, np.eye(2))
    with pytest.raises(api.DimensionMismatch, match="block row mismatch"):
        api.make_sur([np.ones((5, 1)), np.ones((4, 1))], y, np.eye(2))
    with pytest.raises(api.DimensionMismatch, match="Sigma0 must be G x G"):
        api.make_sur([np.ones((5, 1)), np.ones((5, 1))], y, np.eye(3))


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES") is None and api.device_count() > 0,
                    reason="a CUDA device is present")
def test_no_device_fails_loudly():
    if api.device_count() > 0:
        pytest.skip("CUDA device present")
    p = synth.random_sur(2, 6, [2, 2], seed=1)
    with pytest.raises(api.DeviceError, match="no CPU fallback"):
        api.sur_preconditioner(api.sur_from_problem(p))
